"""Numerics study: the 3D KSVD apply with explicit inverses (A1^-1 along the outer axis, L = Q1^T B2^-1,
R = C1^-T Q2 folded into the rotations, per-T2-block inverses G_b for the Sylvester solve) vs the
oracle's apply (bit-exact to the reference) on the first 64 elements of cfg4."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import paper_1704_04549_b200 as T
import _oracle as O
from test_gpu_full_pc_parity import slice_system_3d  # noqa

sub, osys, K3 = slice_system_3d()
opc = osys.form()
q = 11
x = T.uniform_vector(7, sub.N, 1.0)
ref = opc.apply(x)
out = np.zeros_like(x)
for b in range(K3):
    f = opc.factors(b)
    a1, b1, c1, b2, c2 = (f[i * q * q:(i + 1) * q * q].reshape(q, q) for i in range(5))
    rec, piv = opc.record(b)
    o = q * q * 3
    Q1 = rec[o:o + q * q].reshape(q, q); T1 = rec[o + q * q:o + 2 * q * q].reshape(q, q)
    Q2 = rec[o + 2 * q * q:o + 3 * q * q].reshape(q, q); T2 = rec[o + 3 * q * q:o + 4 * q * q].reshape(q, q)
    X = x[b * q ** 3:(b + 1) * q ** 3].reshape(q, q, q)
    X = np.einsum('as,srj->arj', np.linalg.inv(a1), X)
    L = Q1.T @ np.linalg.inv(b2)
    R = np.linalg.inv(c1).T @ Q2
    M = np.einsum('br,arj,jc->abc', L, X, R)
    # Sylvester T1 Y + Y T2^T = M_s, blocks of T2 right to left, G_b explicit
    blocks, k = [], 0
    while k < q:
        sz = 2 if k + 1 < q and T2[k + 1, k] != 0.0 else 1
        blocks.append((k, sz)); k += sz
    Y = np.zeros_like(M)
    for (k0, sz) in reversed(blocks):
        cols = slice(k0, k0 + sz)
        rhs = M[:, :, cols] - np.einsum('sil,kl->sik', Y[:, :, k0 + sz:], T2[cols, k0 + sz:])
        Kb = np.kron(np.eye(sz), T1) + np.kron(T2[cols, cols], np.eye(q))  # column-major vec of Y_b
        G = np.linalg.inv(Kb)
        v = rhs.transpose(0, 2, 1).reshape(q, sz * q)  # per slice: vec col-major = [col0; col1]
        Y[:, :, cols] = (v @ G.T).reshape(q, sz, q).transpose(0, 2, 1)
    Z = np.einsum('br,arj,cj->abc', Q1, Y, Q2)
    out[b * q ** 3:(b + 1) * q ** 3] = Z.ravel()
print("explicit-inverse apply vs oracle: rel-L2", O.rel_l2(out, ref), " max rel", np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
