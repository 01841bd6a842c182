"""Multi-GPU partitioning of C <- C (+) A (x) B: 2D output tiling x optional k-split.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
path shards naturally:

  G = pr * pc * ks ranks; rank -> (I, J, K) with K fastest, so each k-split
  group is ks consecutive ranks.  Rank (I, J, K) computes the partial block
      P_IJ^K = A[rows_I, kslice_K] (x) B[kslice_K, cols_J]
  with the K = 0 rank folding C0 into it exactly once and every other rank
  starting from the additive identity (STARMM_F_INIT_IDENTITY).  With ks > 1
  the partials are combined by ONE collective, a reduce-scatter within the
  (I, J) group with op = SUM (fp64, int64 two's-complement wrap) or MIN
  (the (min,+) semirings); rank K keeps row-chunk K of the reduced block.
  Min and integer sums are order-independent, so the combine is bit-exact.

Two combines for ks > 1:
  combine="fused" (default on GPUs) -- the reduce-scatter disappears into the
      tile epilogue: each owner exposes its row chunk to the k-split group over
      CUDA IPC (NVLink peer memory), pre-loads C0 there, and every rank's tile
      kernel folds its partial tiles straight into the owners' rows with the
      semiring's atomic-madd (starmm_plan_set_peers) -- TAR's accumulate_region
      (ops.py:76-101) across GPUs, overlapped tile by tile with the math;
  combine="nccl" -- partial blocks + one NCCL reduce-scatter (the baseline).

The local product is pluggable (``local_mm``) so that the partition and
combine logic can be exercised on CPU with the gloo backend (tests/), while
the GPU path calls the C ABI.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import _lib
from .errors import ContractViolation

__all__ = ["Grid", "choose_grid", "block_bounds", "DistributedMM", "reduce_op_for"]


@dataclass(frozen=True)
class Grid:
    pr: int
    pc: int
    ks: int

    @property
    def size(self):
        return self.pr * self.pc * self.ks

    def coords(self, rank: int):
        k = rank % self.ks
        ij = rank // self.ks
        return ij // self.pc, ij % self.pc, k


def choose_grid(world: int, ks: int = 1) -> Grid:
    """pr x pc x ks = world with pr <= pc as square as possible (1x2, 2x2, 2x4 ...)."""
    if world % ks:
        raise ContractViolation(f"k-split {ks} does not divide world size {world}")
    rest = world // ks
    pr = int(rest ** 0.5)
    while rest % pr:
        pr -= 1
    return Grid(pr, rest // pr, ks)


def block_bounds(n: int, parts: int, idx: int, align: int = 128):
    """[lo, hi) of part idx when n is split into `parts` nearly equal aligned chunks."""
    units = (n + align - 1) // align
    lo_u = units * idx // parts
    hi_u = units * (idx + 1) // parts
    return min(n, lo_u * align), min(n, hi_u * align)


def reduce_op_for(sid: str):
    return dist.ReduceOp.SUM if sid in ("int", "float") else dist.ReduceOp.MIN


class DistributedMM:
    """One rank's share of a distributed semiring MM.

    ``local_mm(C, A, B, init_identity)`` computes C <- (C or identity) (+) A (x) B
    on this rank's panels; the default is the native plan (GPU)."""

    def __init__(self, n: int, semiring, grid: Grid, rank: int, algo: str = "star",
                 base_dim: int = 64, workers: int = 1, group_ks=None,
                 local_mm: Optional[Callable] = None, device: Optional[int] = None,
                 time_kernel: bool = False, combine: str = "nccl", int_tensor: bool = False,
                 fp64_emu: bool = False, fastpath: bool = True, async_exec: bool = False):
        self.n, self.s, self.grid, self.rank = n, semiring, grid, rank
        self.I, self.J, self.K = grid.coords(rank)
        self.r0, self.r1 = block_bounds(n, grid.pr, self.I)
        self.c0, self.c1 = block_bounds(n, grid.pc, self.J)
        self.k0, self.k1 = block_bounds(n, grid.ks, self.K)
        self.m, self.nn, self.k = self.r1 - self.r0, self.c1 - self.c0, self.k1 - self.k0
        self.group_ks = group_ks
        self.init_identity = self.K > 0
        self.local_mm = local_mm
        self.plan = None
        self.combine_requested = combine
        self.peer_verdicts = None
        if local_mm is None and combine == "fused" and grid.ks > 1:
            # the fused combine writes into the owners' rows over NVLink peer memory: every
            # member of the k-split group must reach every other member's device, else the
            # group falls back to the NCCL reduce-scatter (all members decide alike)
            dev = device if device is not None else torch.cuda.current_device()
            self.peer_verdicts = gather_peer_access(dev, group_ks)
            combine = decide_combine(combine, self.peer_verdicts)
        if local_mm is None:
            fused = combine == "fused" and grid.ks > 1
            # the fused combine folds every partial into the owners' rows, so no rank
            # needs an identity-initialised local block
            flags = _lib.F_ALLOW_NONPOW2 | (_lib.F_INIT_IDENTITY
                                            if (self.init_identity and not fused) else 0)
            if time_kernel:
                flags |= _lib.F_TIME_MAIN
            if int_tensor:
                flags |= _lib.F_INT_TENSOR
            if fp64_emu:
                flags |= _lib.F_FP64_EMU
            if not fastpath:
                flags |= _lib.F_NO_FASTPATH
            if async_exec:            # stream-ordered, the caller synchronises (bench loops)
                flags |= _lib.F_ASYNC
            self.plan = _lib.Plan(semiring.sr_id, algo, "pooled", self.m, self.nn, self.k,
                                  base_dim, workers, -1,
                                  device if device is not None else torch.cuda.current_device(),
                                  flags)
        # rows of the (I, J) block each k-split member keeps after the reduce-scatter
        self.chunk_rows = -(-self.m // grid.ks)
        self.combine_mode = combine if (grid.ks > 1 and local_mm is None) else "nccl"
        self.owned = None
        self._peer_tensors = []
        if self.combine_mode == "fused":
            self._setup_fused(device if device is not None else torch.cuda.current_device())

    # -- fused combine: owners' rows shared over CUDA IPC ----------------------
    def _setup_fused(self, device):
        from torch.multiprocessing.reductions import reduce_tensor
        self.owned = torch.empty((self.chunk_rows, self.nn), dtype=self.s.torch_dtype,
                                 device=torch.device("cuda", device))
        mine = reduce_tensor(self.owned)
        shared = [None] * self.grid.ks
        dist.all_gather_object(shared, mine, group=self.group_ks)
        peers = []
        for j, (rebuild, args) in enumerate(shared):
            t = self.owned if j == self.K else rebuild(*args)
            peers.append(t)
        self._peer_tensors = peers            # keep the mappings alive
        self.plan.set_peers([t.data_ptr() for t in peers], self.nn, self.chunk_rows)

    # -- panels -----------------------------------------------------------
    def a_panel(self, A_full):
        return A_full[self.r0:self.r1, self.k0:self.k1]

    def b_panel(self, B_full):
        return B_full[self.k0:self.k1, self.c0:self.c1]

    def c_block(self, C_full):
        return C_full[self.r0:self.r1, self.c0:self.c1]

    def owned_rows(self):
        """Global row range of the reduced block this rank owns after combine()."""
        lo = self.r0 + self.K * self.chunk_rows
        return min(lo, self.r1), min(lo + self.chunk_rows, self.r1)

    # -- compute ----------------------------------------------------------
    def local(self, C_blk: torch.Tensor, A_pan: torch.Tensor, B_pan: torch.Tensor) -> None:
        if self.local_mm is not None:
            self.local_mm(C_blk, A_pan, B_pan, self.init_identity)
            return
        stream = torch.cuda.current_stream(C_blk.device).cuda_stream
        self.plan.execute(C_blk.data_ptr(), C_blk.stride(0), A_pan.data_ptr(), A_pan.stride(0),
                          B_pan.data_ptr(), B_pan.stride(0), stream)

    def combine(self, C_blk: torch.Tensor) -> torch.Tensor:
        """Reduce-scatter the ks partial blocks; returns this rank's reduced row chunk."""
        if self.grid.ks == 1:
            return C_blk
        pad_rows = self.chunk_rows * self.grid.ks
        if pad_rows != self.m:
            buf = torch.full((pad_rows, self.nn), self.s.zero.item(), dtype=C_blk.dtype,
                             device=C_blk.device)
            buf[: self.m].copy_(C_blk)
        else:
            buf = C_blk.contiguous()
        out = torch.empty((self.chunk_rows, self.nn), dtype=C_blk.dtype, device=C_blk.device)
        dist.reduce_scatter_tensor(out, buf, op=reduce_op_for(self.s.id), group=self.group_ks)
        lo, hi = self.owned_rows()
        return out[: hi - lo]

    def step(self, C_blk, A_pan, B_pan) -> torch.Tensor:
        if self.combine_mode == "fused":
            return self.step_fused(C_blk, A_pan, B_pan)
        self.local(C_blk, A_pan, B_pan)
        return self.combine(C_blk)

    def step_fused(self, C_blk, A_pan, B_pan) -> torch.Tensor:
        """Owner pre-loads C0 into its shared rows; after a group barrier every rank's
        tile kernel atomically folds its partial tiles into the owners' rows; a second
        barrier closes the step.  Returns this rank's reduced rows."""
        lo, hi = self.owned_rows()
        r = hi - lo
        # C0 is folded exactly once: by the owner of each row chunk (C_blk holds C0 of
        # the (I, J) block on every member; only the owner's rows are loaded)
        self.owned[:r].copy_(C_blk[lo - self.r0:hi - self.r0])
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group_ks)
        self.local(C_blk, A_pan, B_pan)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group_ks)
        return self.owned[:r]

    def step_host(self, C_h: torch.Tensor, A_h: torch.Tensor, B_h: torch.Tensor,
                  out_h: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The step with this rank's panels in HOST memory (pinned CPU tensors or strided
        views of pinned full matrices); returns this rank's reduced rows on the host.

        Without a k-split the rank's sub-problem is independent, so it runs through
        starmm_execute_host: uploads, tile kernels and downloads overlap,
        and C_h is updated in place.  With a k-split the panels are uploaded, the
        combine runs on the device, and the owned rows are copied into ``out_h``."""
        if self.combine_mode == "fused":
            return self._step_host_fused(C_h, A_h, B_h, out_h)
        if self.grid.ks == 1 and self.plan is not None:
            for t in (C_h, A_h, B_h):
                if t.device.type != "cpu" or (t.shape[1] > 1 and t.stride(1) != 1):
                    raise ContractViolation("step_host needs row-major CPU panels")
            stream = torch.cuda.current_stream().cuda_stream
            self.plan.execute_host(C_h.data_ptr(), max(1, C_h.stride(0)), A_h.data_ptr(),
                                   max(1, A_h.stride(0)), B_h.data_ptr(), max(1, B_h.stride(0)),
                                   stream)
            return C_h
        dev = torch.device("cuda", torch.cuda.current_device())
        Ad = A_h.to(dev, non_blocking=True)
        Bd = Ad if B_h is A_h else B_h.to(dev, non_blocking=True)
        Cd = C_h.to(dev, non_blocking=True)
        r = self.step(Cd, Ad, Bd)
        if out_h is None:
            out_h = torch.empty(r.shape, dtype=r.dtype).pin_memory()
        out_h.copy_(r, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out_h

    def _step_host_fused(self, C_h, A_h, B_h, out_h):
        """k-split rank with the fused combine, host panels: the owner uploads its C0 rows
        into the shared owner buffer, then starmm_execute_host streams A and B in k-chunks
        and every chunk's tile kernels fold into the owners' rows over peer memory (the
        uploads overlap the math); the owner reads its rows back."""
        for t in (C_h, A_h, B_h):
            if t.device.type != "cpu" or (t.shape[1] > 1 and t.stride(1) != 1):
                raise ContractViolation("step_host needs row-major CPU panels")
        lo, hi = self.owned_rows()
        r = hi - lo
        self.owned[:r].copy_(C_h[lo - self.r0:hi - self.r0], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group_ks)
        stream = torch.cuda.current_stream().cuda_stream
        self.plan.execute_host(C_h.data_ptr(), max(1, C_h.stride(0)), A_h.data_ptr(),
                               max(1, A_h.stride(0)), B_h.data_ptr(), max(1, B_h.stride(0)), stream)
        dist.barrier(group=self.group_ks)
        if out_h is None:
            out_h = torch.empty((r, self.nn), dtype=self.owned.dtype).pin_memory()
        out_h.copy_(self.owned[:r], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out_h

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None


def peer_access_local(device: int, peer_devices) -> bool:
    """Can `device` map every peer's memory (CUDA IPC + peer access over NVLink)?  The
    same device (ranks sharing a GPU) always can."""
    return all(d == device or torch.cuda.can_device_access_peer(device, d) for d in peer_devices)


def gather_peer_access(device: int, group=None):
    """Every group member's peer-access verdict towards all the others."""
    devs = [None] * dist.get_world_size(group)
    dist.all_gather_object(devs, int(device), group=group)
    ok = peer_access_local(device, devs)
    verdicts = [None] * len(devs)
    dist.all_gather_object(verdicts, bool(ok), group=group)
    return verdicts


def decide_combine(requested: str, verdicts) -> str:
    """The k-split combine a group runs: the fused peer-memory one only if every member
    can reach every other; otherwise the NCCL reduce-scatter."""
    if requested == "fused" and verdicts is not None and not all(verdicts):
        return "nccl"
    return requested


def ks_groups(grid: Grid):
    """Create the (I, J) k-split process groups (every rank must call this)."""
    groups = []
    mine = None
    rank = dist.get_rank()
    for ij in range(grid.pr * grid.pc):
        ranks = [ij * grid.ks + k for k in range(grid.ks)]
        g = dist.new_group(ranks) if grid.ks > 1 else None
        groups.append(g)
        if rank in ranks:
            mine = g
    return mine
