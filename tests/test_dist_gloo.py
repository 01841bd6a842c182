"""CPU, world_size 2 over gloo: the multi-GPU partition (2D output tiling x
k-split) and the reduce-scatter combine of paper_1911_05328_b200.distributed.
The local product is the CPU oracle (injected), so this exercises exactly the
host-side logic that the NCCL path runs on the 8xB200 box."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_05328_b200.distributed import (DistributedMM, block_bounds, choose_grid,
                                               ks_groups)


def test_choose_grid():
    assert choose_grid(1) .__dict__ == {"pr": 1, "pc": 1, "ks": 1}
    g = choose_grid(2)
    assert (g.pr, g.pc, g.ks) == (1, 2, 1)
    g = choose_grid(8)
    assert (g.pr, g.pc, g.ks) == (2, 4, 1)
    g = choose_grid(8, ks=2)
    assert (g.pr, g.pc, g.ks) == (2, 2, 2)
    assert [g.coords(r) for r in range(4)] == [(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1)]


def test_block_bounds_cover_exactly():
    for n, parts in [(49152, 2), (16384, 4), (1000, 3), (130, 2)]:
        edges = [block_bounds(n, parts, i) for i in range(parts)]
        assert edges[0][0] == 0 and edges[-1][1] == n
        assert all(edges[i][1] == edges[i + 1][0] for i in range(parts - 1))


def _oracle_local(sr):
    from oracle import oracle as O

    def local(C, A, B, init_identity):
        Cn = C.numpy()
        if init_identity:
            Cn[...] = O.matmul(sr, np.ascontiguousarray(A.numpy()), np.ascontiguousarray(B.numpy()))
        else:
            O.gemm_fold(sr, Cn, np.ascontiguousarray(A.numpy()), np.ascontiguousarray(B.numpy()))
    return local


def _worker(rank, world, port, sid, ks, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1911_05328_b200 as sm
        from oracle import oracle as O
        s = sm.get_semiring(sid)
        sr = O.SR_BY_NAME[sid]
        rng = np.random.default_rng(42)
        if sid == "int":
            A = rng.integers(-9, 10, (n, n)).astype(np.int64)
            B = rng.integers(-9, 10, (n, n)).astype(np.int64)
            C0 = rng.integers(-9, 10, (n, n)).astype(np.int64)
        else:
            A = rng.integers(1, 50, (n, n)).astype(s.dtype)
            B = rng.integers(1, 50, (n, n)).astype(s.dtype)
            C0 = rng.integers(1, 90, (n, n)).astype(s.dtype)
        grid = choose_grid(world, ks)
        group = ks_groups(grid)
        dmm = DistributedMM(n, s, grid, rank, group_ks=group, local_mm=_oracle_local(sr))
        Ct = torch.from_numpy(C0[dmm.r0:dmm.r1, dmm.c0:dmm.c1].copy())
        if dmm.init_identity:
            Ct.fill_(s.zero.item())
        At = torch.from_numpy(np.ascontiguousarray(dmm.a_panel(A)))
        Bt = torch.from_numpy(np.ascontiguousarray(dmm.b_panel(B)))
        out = dmm.step(Ct, At, Bt)
        want = C0.copy()
        O.gemm_fold(sr, want, A, B)
        lo, hi = dmm.owned_rows()
        ok = np.array_equal(out.numpy(), want[lo:hi, dmm.c0:dmm.c1])
        q.put((rank, ok, (lo, hi, dmm.c0, dmm.c1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sid,ks", [("int", 1), ("int", 2), ("tropical_i32", 2),
                                    ("tropical_f32", 1)])
def test_two_rank_partition_and_combine(sid, ks):
    world, n = 2, 256
    port = 29500 + (hash((sid, ks)) % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sid, ks, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    # the owned pieces tile C exactly once
    cover = np.zeros((n, n), int)
    for _, _, (lo, hi, c0, c1) in res:
        cover[lo:hi, c0:c1] += 1
    assert np.all(cover == 1)


def test_decide_combine_falls_back_without_peer_access():
    from paper_1911_05328_b200.distributed import decide_combine
    assert decide_combine("fused", [True, True]) == "fused"
    assert decide_combine("fused", [True, False]) == "nccl"
    assert decide_combine("nccl", [True, True]) == "nccl"
    assert decide_combine("fused", None) == "fused"


def _gen_worker(rank, world, port, cid, ks, n, q):
    """Each rank generates ONLY its own panels (counter-based, global coordinates) and
    gathers the peer-access verdicts; the distributed product must equal the product of
    the full matrices generated in one piece."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1911_05328_b200 as sm
        from bench_configs import CONFIGS, device_gen_spec
        from oracle import oracle as O
        from paper_1911_05328_b200.distributed import decide_combine, gather_peer_access
        cfg = CONFIGS[cid]
        s = sm.get_semiring(cfg["semiring"])
        sr = O.SR_BY_NAME[cfg["semiring"]]

        def panel(what, rows, cols, r0, c0):
            spec = device_gen_spec(cid, what)
            if spec == "zeros":
                return np.zeros((rows, cols), dtype=O.DTYPES[sr])
            spec = dict(spec)
            spec["stream"] = spec.pop("stream_id")
            return O.generate(sr, rows=rows, cols=cols, row0=r0, col0=c0, **spec)

        grid = choose_grid(world, ks)
        group = ks_groups(grid)
        verdicts = gather_peer_access(0, group) if ks > 1 else [True]
        dmm = DistributedMM(n, s, grid, rank, group_ks=group, local_mm=_oracle_local(sr))
        At = torch.from_numpy(panel("A", dmm.m, dmm.k, dmm.r0, dmm.k0))
        Bt = torch.from_numpy(panel("B", dmm.k, dmm.nn, dmm.k0, dmm.c0))
        Ct = torch.from_numpy(panel("C", dmm.m, dmm.nn, dmm.r0, dmm.c0))
        if dmm.init_identity:
            Ct.fill_(s.zero.item())
        out = dmm.step(Ct, At, Bt)
        A, B, C = panel("A", n, n, 0, 0), panel("B", n, n, 0, 0), panel("C", n, n, 0, 0)
        O.gemm_fold(sr, C, A, B)
        lo, hi = dmm.owned_rows()
        ok = np.array_equal(out.numpy(), C[lo:hi, dmm.c0:dmm.c1])
        q.put((rank, ok, verdicts, decide_combine("fused", verdicts)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cid,ks", [(3, 2), (5, 1), (2, 2)])
def test_two_rank_generated_panels_need_no_distribution(cid, ks):
    world, n = 2, 256
    port = 31500 + (hash((cid, ks)) % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gen_worker, args=(r, world, port, cid, ks, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    assert all(v == [True] * len(v) and c == "fused" for _, _, v, c in res)
