"""Multi-process (gloo, CPU) execution of libeqc's direct-send and binary-swap
plans: world_size 2 and 4 processes each hold a contiguous block of sources,
exchange real bytes over torch.distributed (gloo, 127.0.0.1), composite with
the CPU oracle at every step and must reproduce the oracle over ALL sources
bit-exactly (schedule soundness; tie rule R-C5).  This pins the host
logic of the N > 1 path (plans, tie preference, band bookkeeping) without a
GPU; the GPU/NCCL path executes the same plans (tests/test_gpu_multi.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1902_08755_b200 import eqc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _send(arr, dst):
    dist.send(torch.from_numpy(np.ascontiguousarray(arr).view(np.int32)), dst)


def _recv(shape, src):
    t = torch.empty(shape, dtype=torch.int32)
    dist.recv(t, src)
    return t.numpy().view(np.uint32)


def _exchange(sends, recvs):
    """Post all sends and receives of one step (non-blocking), then wait."""
    reqs = []
    for arr, dst in sends:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr).view(np.int32)), dst))
    outs = []
    for shape, src in recvs:
        t = torch.empty(shape, dtype=torch.int32)
        reqs.append(dist.irecv(t, src))
        outs.append(t)
    for r in reqs:
        r.wait()
    return [o.numpy().view(np.uint32) for o in outs]


def _worker(rank, world, port, algo, n_local, w, h, dest, tie_alphabet, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = world * n_local
        if tie_alphabet:
            c, d = synth.random_frames(77, n, w, h, depth_alphabet=[0, 3, 0xFFFFFFFF])
        else:
            c, d = synth.depth_sources(20190213 + 3, n, w, h)
        mine_c = c[rank * n_local:(rank + 1) * n_local]
        mine_d = d[rank * n_local:(rank + 1) * n_local]
        pc, pd = oracle.depth_composite(mine_c, mine_d)  # local pre-composite
        msgs = 0
        if algo == "ds":
            row0 = eqc.eqc_plan_bands(h, world)
            y0, y1 = row0[rank], row0[rank + 1]
            sends, recvs = [], []
            for j in range(world):
                if j != rank and row0[j + 1] > row0[j]:
                    sends += [(pc[row0[j]:row0[j + 1]], j), (pd[row0[j]:row0[j + 1]], j)]
                    msgs += 1
            srcs = [q for q in range(world) if q != rank and y1 > y0]
            for q in srcs:
                recvs += [((y1 - y0, w), q), ((y1 - y0, w), q)]
            got = _exchange(sends, recvs)
            bands_c, bands_d = [], []
            it = iter(got)
            recv_map = {q: (next(it), next(it)) for q in srcs}
            for q in range(world):
                if q == rank:
                    bands_c.append(pc[y0:y1])
                    bands_d.append(pd[y0:y1])
                elif y1 > y0:
                    bands_c.append(recv_map[q][0])
                    bands_d.append(recv_map[q][1])
            fin = oracle.depth_composite(bands_c, bands_d)[0] if y1 > y0 else np.zeros((0, w), np.uint32)
            regions = [(row0[q], row0[q + 1]) for q in range(world)]
        elif algo == "s23":
            # 2-3 swap (R-C21): fold pairs, then mixed-radix groups of 2 / 3
            plan = eqc.eqc_plan_swap23(h, world, rank)
            cur_c, cur_d = pc.copy(), pd.copy()
            if plan["fold_role"] == 2:
                _exchange([(cur_c, plan["fold_partner"]), (cur_d, plan["fold_partner"])], [])
                msgs += 1
            elif plan["fold_role"] == 1:
                tc, td = _exchange([], [((h, w), plan["fold_partner"])] * 2)
                cur_c, cur_d = oracle.depth_composite([cur_c, tc], [cur_d, td])  # lower rank first
            for rd in plan["rounds"]:
                k, t, mem, bnd = rd["k"], rd["t"], rd["members"], rd["bounds"]
                ky0, ky1 = bnd[t], bnd[t + 1]
                sends, recvs, others = [], [], []
                for u in range(k):
                    if u == t:
                        continue
                    if bnd[u + 1] > bnd[u]:
                        sends += [(cur_c[bnd[u]:bnd[u + 1]], mem[u]), (cur_d[bnd[u]:bnd[u + 1]], mem[u])]
                        msgs += 1
                    if ky1 > ky0:
                        recvs += [((ky1 - ky0, w), mem[u])] * 2
                        others.append(u)
                got = _exchange(sends, recvs)
                if ky1 > ky0:
                    parts = {t: (cur_c[ky0:ky1].copy(), cur_d[ky0:ky1].copy())}
                    for i, u in enumerate(others):
                        parts[u] = (got[2 * i], got[2 * i + 1])
                    oc, od = oracle.depth_composite([parts[u][0] for u in range(k)], [parts[u][1] for u in range(k)])
                    cur_c[ky0:ky1] = oc
                    cur_d[ky0:ky1] = od
            regions = [eqc.eqc_plan_swap23(h, world, q)["final"] for q in range(world)]
            y0, y1 = regions[rank]
            fin = cur_c[y0:y1]
        else:
            plan = eqc.eqc_plan_binary_swap(h, world, rank)
            cur_c, cur_d = pc.copy(), pd.copy()
            for partner, low, ky0, ky1, sy0, sy1 in plan:
                sends = [(cur_c[sy0:sy1], partner), (cur_d[sy0:sy1], partner)] if sy1 > sy0 else []
                recvs = [((ky1 - ky0, w), partner)] * 2 if ky1 > ky0 else []
                msgs += 1 if sy1 > sy0 else 0
                got = _exchange(sends, recvs)
                if ky1 > ky0:
                    mc, md = cur_c[ky0:ky1], cur_d[ky0:ky1]
                    tc, td = got
                    cs = [mc, tc] if low else [tc, mc]  # ties -> group whose bit r is 0
                    ds = [md, td] if low else [td, md]
                    oc, od = oracle.depth_composite(cs, ds)
                    cur_c[ky0:ky1] = oc
                    cur_d[ky0:ky1] = od
            regions = []
            for q in range(world):
                pq = eqc.eqc_plan_binary_swap(h, world, q)
                regions.append((pq[-1][2], pq[-1][3]) if pq else (0, h))
            y0, y1 = regions[rank]
            fin = cur_c[y0:y1]
        # gather colour to dest
        if rank != dest:
            if y1 > y0:
                _send(fin, dest)
            result_q.put((rank, msgs, None))
        else:
            out = np.zeros((h, w), np.uint32)
            out[y0:y1] = fin
            for q in range(world):
                qy0, qy1 = regions[q]
                if q != dest and qy1 > qy0:
                    out[qy0:qy1] = _recv((qy1 - qy0, w), q)
            want, _ = oracle.depth_composite(c, d)
            result_q.put((rank, msgs, bool((out == want).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo,world,n_local,w,h,dest,ties", [
    ("ds", 2, 2, 64, 41, 0, False),
    ("ds", 3, 1, 50, 31, 2, True),
    ("ds", 4, 2, 33, 9, 1, True),
    ("bs", 2, 3, 40, 33, 1, True),
    ("bs", 4, 1, 64, 37, 0, False),
    ("bs", 4, 2, 16, 5, 3, True),
    ("s23", 3, 2, 40, 31, 1, True),
    ("s23", 5, 1, 24, 17, 4, True),
    ("s23", 6, 1, 33, 12, 0, False),
])
def test_schedule_equals_oracle_over_all_sources(algo, world, n_local, w, h, dest, ties):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, algo, n_local, w, h, dest, ties, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ok = [r[2] for r in res if r[0] == dest]
    assert ok == [True]
    msgs = sum(r[1] for r in res)
    if algo == "ds":
        assert msgs == world * (world - 1)  # n(n-1) band messages
    elif algo == "bs":
        assert msgs == world * (world.bit_length() - 1)  # n log2 n swaps


# ---- ordered blending through the schedules ---------
# The schedule must merge partials in rank (= draw) order: "over" is not
# commutative.  Partials are exact float64 premultiplied (rgb, a) planes here
# (test-side arithmetic: the plain definition x = s + x (1 - a_s)); the final
# band is rounded once and compared with O2 over all layers.
def _over(back, front):
    return front + back * (1.0 - front[..., 3:4])


def _partial(layers):
    acc = np.zeros(layers[0].shape + (4,))
    for l in layers:
        acc = _over(acc, l.view(np.uint8).reshape(l.shape + (4,)).astype(np.float64) / 255.0)
    return acc


def _blend_worker(rank, world, port, algo, n_local, w, h, dest, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def xchg(sends, recvs):
        reqs, outs = [], []
        for arr, dst in sends:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr)), dst))
        for shape, src in recvs:
            t = torch.empty(shape, dtype=torch.float64)
            reqs.append(dist.irecv(t, src))
            outs.append(t)
        for r in reqs:
            r.wait()
        return [o.numpy() for o in outs]

    try:
        n = world * n_local
        layers = synth.premultiplied_noise(900 + n, n, w, h)
        part = _partial(layers[rank * n_local:(rank + 1) * n_local])
        if algo == "ds":
            row0 = eqc.eqc_plan_bands(h, world)
            y0, y1 = row0[rank], row0[rank + 1]
            sends = [(part[row0[j]:row0[j + 1]], j) for j in range(world) if j != rank and row0[j + 1] > row0[j]]
            srcs = [q for q in range(world) if q != rank and y1 > y0]
            got = dict(zip(srcs, xchg(sends, [((y1 - y0, w, 4), q) for q in srcs])))
            band = np.zeros((y1 - y0, w, 4))
            for q in range(world):  # rank order = draw order
                band = _over(band, part[y0:y1] if q == rank else got[q]) if y1 > y0 else band
            regions = [(row0[q], row0[q + 1]) for q in range(world)]
            fin = band
        else:  # 2-3 swap
            plan = eqc.eqc_plan_swap23(h, world, rank)
            cur = part.copy()
            if plan["fold_role"] == 2:
                xchg([(cur, plan["fold_partner"])], [])
            elif plan["fold_role"] == 1:
                (their,) = xchg([], [((h, w, 4), plan["fold_partner"])])
                cur = _over(cur, their)  # the partner holds the next (front) layers
            for rd in plan["rounds"]:
                k, t, mem, bnd = rd["k"], rd["t"], rd["members"], rd["bounds"]
                ky0, ky1 = bnd[t], bnd[t + 1]
                sends = [(cur[bnd[u]:bnd[u + 1]], mem[u]) for u in range(k) if u != t and bnd[u + 1] > bnd[u]]
                others = [u for u in range(k) if u != t] if ky1 > ky0 else []
                got = xchg(sends, [((ky1 - ky0, w, 4), mem[u]) for u in others])
                if ky1 > ky0:
                    parts = {t: cur[ky0:ky1].copy(), **{u: g for u, g in zip(others, got)}}
                    acc = np.zeros((ky1 - ky0, w, 4))
                    for u in range(k):
                        acc = _over(acc, parts[u])
                    cur[ky0:ky1] = acc
            regions = [eqc.eqc_plan_swap23(h, world, q)["final"] for q in range(world)]
            y0, y1 = regions[rank]
            fin = cur[y0:y1]
        if rank != dest:
            if y1 > y0:
                xchg([(fin, dest)], [])
            result_q.put((rank, None))
        else:
            out = np.zeros((h, w, 4))
            out[y0:y1] = fin
            for q in range(world):
                qy0, qy1 = regions[q]
                if q != dest and qy1 > qy0:
                    (out[qy0:qy1],) = xchg([], [((qy1 - qy0, w, 4), q)])
            got8 = np.clip(np.floor(255.0 * out + 0.5), 0, 255).astype(np.uint8)
            want = oracle.blend_ordered(layers).view(np.uint8).reshape(h, w, 4)
            result_q.put((rank, int(np.abs(got8.astype(int) - want.astype(int)).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo,world,n_local,w,h,dest", [
    ("ds", 2, 3, 40, 21, 0), ("ds", 3, 2, 33, 17, 2), ("s23", 3, 2, 24, 19, 1), ("s23", 5, 1, 20, 11, 4),
])
def test_blend_schedule_keeps_draw_order(algo, world, n_local, w, h, dest):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blend_worker, args=(r, world, port, algo, n_local, w, h, dest, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    err = [r[1] for r in res if r[0] == dest]
    assert err[0] <= 1  # float64 partials: the exact chain, rounded once (R-C4)
