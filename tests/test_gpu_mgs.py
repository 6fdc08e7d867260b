"""The Arnoldi step's modified Gram-Schmidt kernel (csrc/blas.cu, through the tpdg_gpu_mgs_step test hook) against
the reference's loop (solve/gmres.hpp:112-121: h_j = <w, v_j>, w -= h_j v_j for j = 0..k, then h_{k+1} = ||w||,
w /= h_{k+1}) in float64 with torch on the same device data. The kernel sums in its own fixed order,
so the gate is 1e-12 relative, not bitwise; the sizes cover every launch shape of the streaming kernel (4 register
rows + ring depth 8; 10 + 8; 10 register rows + shared rows + ring depth 4 with rows parked past tensor-memory
capacity), odd lengths and partial last rows, and the global-memory fallback for slices too large for the chip."""
import numpy as np
import pytest
import torch

import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return T.Context(0)


def reference_mgs(V, k, n):
    w = V[k + 1, :n].clone()
    h = []
    for j in range(k + 1):
        hj = torch.dot(w, V[j, :n])
        w -= hj * V[j, :n]
        h.append(float(hj))
    nrm = float(torch.linalg.vector_norm(w))
    h.append(nrm)
    return np.array(h), w / nrm


CASES = [  # (n, k)
    (37, 2),            # one partial row, most threads idle
    (5184, 5),          # cfg1
    (1048576, 7),       # cfg2 p = 15: 4 rows, registers only
    (1048575, 3),       # odd length: a half pair at the end
    (1806336, 4),       # cfg2 p = 20: 6 rows
    (3936256, 3),       # cfg2 p = 30: 13 rows, three of them in shared memory
    (5451776, 6),       # cfg4: 18 rows, rows 16-17 parked in shared memory
    (5451775, 0),       # k = 0: first dot and the norm only
    (6000001, 2),       # slices beyond the on-chip budget: global-memory kernel
]


@pytest.mark.parametrize("n,k", CASES)
def test_mgs_step_matches_reference_loop(ctx, n, k):
    g = torch.Generator(device="cuda").manual_seed(1234 + n % 1000 + k)
    ldv = (n + 31) // 32 * 32
    V = torch.zeros((k + 2, ldv), dtype=torch.float64, device="cuda")
    V[:, :n] = torch.rand((k + 2, n), generator=g, dtype=torch.float64, device="cuda") - 0.5
    V[: k + 1, :n] /= torch.linalg.vector_norm(V[: k + 1, :n], dim=1, keepdim=True)
    V[k + 1, n:] = 7.0  # padding of w must be neither read into the sums nor written
    h_ref, w_ref = reference_mgs(V, k, n)
    basis = V[: k + 1].clone()
    torch.cuda.synchronize()
    h = T.mgs_step(ctx, V, k, n)
    scale = np.abs(h_ref).max()
    assert np.abs(h - h_ref).max() <= 1e-12 * scale, (h, h_ref)
    err = float(torch.linalg.vector_norm(V[k + 1, :n] - w_ref))
    assert err <= 1e-12, err
    assert torch.equal(V[: k + 1], basis)              # the basis is read-only
    assert bool((V[k + 1, n:] == 7.0).all())           # nothing written past n


def test_mgs_step_is_deterministic(ctx):
    n, k = 3936256, 5
    g = torch.Generator(device="cuda").manual_seed(7)
    V0 = torch.rand((k + 2, n), generator=g, dtype=torch.float64, device="cuda") - 0.5  # not normalized: any
    outs = []                                                                           # last-bit change is amplified
    for _ in range(2):
        V = V0.clone()
        torch.cuda.synchronize()  # the library runs on its own stream
        h = T.mgs_step(ctx, V, k, n)
        outs.append((h, V[k + 1].clone()))
    assert np.array_equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
