"""Multi-rank decomposition on CPU (gloo, world_size 2): the element partition and face-neighbour halo
plan the CUDA library uses for nranks > 1 (paper_1704_04549_b200/csrc/halo.cpp, exported through
the C ABI), driven with the oracle as the per-rank compute:

  * distributed Jv = halo exchange (torch.distributed send/recv of the planned face node layers,
    n_c q^(d-1) doubles per cut face; the rest of each halo block is NaN) + local operator apply;
    must equal the single-rank reference Jv bit for bit;
  * distributed right-preconditioned MGS-GMRES with every dot product all-reduced (the structure of
    the multi-rank path in capi.cu: halo before each Jv, element-local KSVD apply, allreduce per
    MGS dot); must take the reference's iteration count.

The GPU build runs the same plan with NCCL (ncclSend/ncclRecv halo, ncclAllReduce) on the device.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle as O
import paper_1704_04549_b200 as T


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def local_system(z, plan):
    """Oracle system of one rank: its elements, neighbours remapped to local ids / halo slots."""
    m = z["meta"]
    dim, nc, p, mu = int(m[0]), int(m[1]), int(m[2]), int(m[3])
    e0, e1 = plan["e_begin"], plan["e_end"]
    nl = e1 - e0
    nqv, nqf = mu ** dim, mu ** (dim - 1)
    arrays = dict(z)
    arrays["meta"] = np.array(m, dtype=np.float64).copy()
    arrays["meta"][4] = nl
    arrays["jdet"] = z["jdet"][e0 * nqv:e1 * nqv]
    arrays["face_w"] = z["face_w"][e0 * 2 * dim * nqf:e1 * 2 * dim * nqf]
    arrays["dft"] = z["dft"][e0 * dim * nqv * nc * nc:e1 * dim * nqv * nc * nc]
    arrays["dfm"] = z["dfm"][e0 * 2 * dim * nqf * nc * nc:e1 * 2 * dim * nqf * nc * nc]
    arrays["dfp"] = z["dfp"][e0 * 2 * dim * nqf * nc * nc:e1 * 2 * dim * nqf * nc * nc]
    arrays["conn"] = plan["conn"].astype(np.int64)
    return O.System(arrays)


def exchange(plan, v_local, nc, npe, dim, q):
    """Halo of one rank per the plan (capi.cu's exchange_halo over gloo): the face node layers the
    peers need cross ranks, n_c q^(d-1) values per cut face; everything else in the halo blocks is
    NaN, so an operator that read beyond the layers would not reproduce the reference."""
    L = q ** (dim - 1)
    idx = [T.face_layer_nodes(dim, q, f) for f in range(2 * dim)]
    halo = np.full(plan["n_halo"] * nc * npe, np.nan)
    reqs, bufs = [], []
    for p in plan["peers"]:
        if len(p["send_pairs"]):
            send = torch.from_numpy(np.concatenate([v_local[(e * nc + c) * npe + idx[f]]
                                                    for e, f in p["send_pairs"] for c in range(nc)]))
            reqs.append(dist.isend(send, p["rank"]))
            bufs.append(send)
        if len(p["recv_pairs"]):
            recv = torch.zeros(len(p["recv_pairs"]) * nc * L, dtype=torch.float64)
            reqs.append(dist.irecv(recv, p["rank"]))
            bufs.append((p, recv))
    for r in reqs:
        r.wait()
    for b in bufs:
        if isinstance(b, tuple):
            p, recv = b
            r = recv.numpy()
            for k, (slot, f) in enumerate(p["recv_pairs"]):
                for c in range(nc):
                    halo[(slot * nc + c) * npe + idx[f]] = r[(k * nc + c) * L:(k * nc + c + 1) * L]
    return halo


def allreduce(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


def dist_gmres(jv, pc, b, tol=1e-10, m=30, max_it=2000):
    """Right-preconditioned restarted MGS-GMRES (solve/gmres.hpp:52-179), dots all-reduced."""
    n = b.size
    nrm = lambda v: np.sqrt(allreduce(float(v @ v)))
    target = tol * nrm(b)
    x = np.zeros(n)
    its = 0
    while its < max_it:
        r = b - jv(x)
        beta = nrm(r)
        if beta <= target:
            return x, its, True
        V = [r / beta]
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        k = 0
        while k < m and its < max_it:
            its += 1
            w = jv(pc(V[k]))
            for j in range(k + 1):
                H[j, k] = allreduce(float(V[j] @ w))
                w = w - H[j, k] * V[j]
            H[k + 1, k] = nrm(w)
            V.append(w / H[k + 1, k] if H[k + 1, k] > 0 else w)
            for j in range(k):
                t1, t2 = H[j, k], H[j + 1, k]
                H[j, k] = cs[j] * t1 + sn[j] * t2
                H[j + 1, k] = -sn[j] * t1 + cs[j] * t2
            d = np.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = (1.0, 0.0) if d == 0 else (H[k, k] / d, H[k + 1, k] / d)
            H[k, k], H[k + 1, k] = d, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            k += 1
            if abs(g[k]) <= target:
                break
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + pc(sum(y[j] * V[j] for j in range(k)))
        if abs(g[k]) <= target:
            return x, its, True
    return x, its, False


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = O.load_raw(case)
        sysg = T.System.from_golden(z)
        plan = T.halo_plan(sysg, rank, world)
        loc = local_system(z, plan)
        blk = loc.n_c * loc.npe
        e0, e1 = plan["e_begin"], plan["e_end"]
        a, b = loc.coeffs

        def jv(v_local):
            ext = np.concatenate([v_local, exchange(plan, v_local, loc.n_c, loc.npe, loc.dim, loc.q)])
            out = np.zeros(v_local.size)
            O.lib().or_jv(O.C.byref(loc._or), O.C.c_double(a), O.C.c_double(b), loc.small, O.ptr(ext), O.ptr(out))
            return out

        v = z["jv_in"][e0 * blk:e1 * blk]
        jv_ok = np.array_equal(jv(v), z["jv_out"][e0 * blk:e1 * blk])
        pc = loc.form()
        rhs = z["rhs"][e0 * blk:e1 * blk]
        pc_ok = np.array_equal(pc.apply(rhs), z["pc_out"][e0 * blk:e1 * blk])
        _, its, conv = dist_gmres(jv, pc.apply, rhs)
        q.put((rank, jv_ok, pc_ok, its, conv, plan["n_halo"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cfg1", "adv3d_p4", "euler2d"])
def test_two_rank_jv_pc_gmres(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    z = O.load_raw(case)
    ref_its = int(z["gmres_meta"][0])
    for rank, jv_ok, pc_ok, its, conv, n_halo in res:
        assert jv_ok, f"rank {rank}: distributed Jv differs from the reference"
        assert pc_ok, f"rank {rank}: element-local PC apply differs"
        assert conv and its == ref_its, (rank, its, ref_its)
        assert n_halo > 0


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_halo_plan_is_consistent(nranks):
    """Every rank's received layers (halo element, face) are what its peers send, in the same order,
    and they are exactly the faces the rank's elements see across the cut."""
    for case in ["cfg1", "adv3d_p4"]:
        z = O.load_raw(case)
        s = T.System.from_golden(z)
        dim = s.dim
        plans = [T.halo_plan(s, r, nranks) for r in range(nranks)]
        E = int(z["meta"][4])
        gconn = np.asarray(z["conn"]).reshape(E, 2 * dim, 3)
        assert plans[0]["e_begin"] == 0 and plans[-1]["e_end"] == E
        for r, p in enumerate(plans):
            nl = p["e_end"] - p["e_begin"]
            need = set()
            for le in range(nl):
                for f in range(2 * dim):
                    nb, nf = int(gconn[p["e_begin"] + le, f, 0]), int(gconn[p["e_begin"] + le, f, 1])
                    if nb >= 0 and not (p["e_begin"] <= nb < p["e_end"]):
                        need.add((nb, nf))
            got = set()
            for peer in p["peers"]:
                other = plans[peer["rank"]]
                back = [q for q in other["peers"] if q["rank"] == r]
                recv = [(int(p["halo_gid"][slot]), int(f)) for slot, f in peer["recv_pairs"]]
                sent = [(int(e) + other["e_begin"], int(f)) for e, f in back[0]["send_pairs"]] if back else []
                assert recv == sent
                got |= set(recv)
            assert got == need
            conn = p["conn"].reshape(-1, 3)
            nl = p["e_end"] - p["e_begin"]
            assert conn[:, 0].max() < nl + p["n_halo"]
