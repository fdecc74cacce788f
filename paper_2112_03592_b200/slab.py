"""z-slab decomposition of APR-native convolution over several GPUs
(DESIGN.md §6).

One process (rank) per GPU; every rank holds the WHOLE access structure (it
is static and small next to 180 GB: ~2 GB at C4) and full-size value arrays
in the global particle / node numbering, but owns only its slab:

* the finest-level pixel planes [z_lo, z_hi) are cut into blocks of
  2^c planes; rank r owns a contiguous run of blocks.  Level l >= lc =
  l_max - c is PARTITIONED (a level-l cell never straddles two slabs); levels
  < lc are REPLICATED (tiny: coarse cells);
* rows at a level are z-major in the CSR, so "rows [za, zb) of level l" is
  ONE contiguous particle range -- every exchange below is a contiguous slice.

A convolution on slabs (SlabConvolver.convolve) is:

1. halo exchange of leaf values: for every partitioned level, the `halo`
   level-l rows next to each slab boundary go to the neighbour (grouped
   point-to-point send/recv);
2. the tree fill: fp64 sums of the partitioned interior levels over the
   slab's own rows (every child of such a node lies in the slab); an
   all-gather of the cut level (level-lc leaf values and tree-level-lc sums)
   so that every rank then computes the replicated levels < lc itself, in the
   reference's order (no partial-sum combining: bit-exact); finalize;
3. halo exchange of tree values;
4. the convolution restricted to the slab's tiles/rows (aprgpu_convolve_slab)
   plus every replicated level.

Owned outputs are bit-identical to the single-domain result (EXACT mode) by
construction: each output reads only cells within the stencil half-width of
its own cell, and the halo carries exactly those rows at every partitioned
level; coarse covering leaves of a level-l halo row lie at most one row
beyond the boundary at their own level.

The algorithm is written once over a list of RankState objects and a
communicator: TorchComm (torch.distributed, NCCL between GPUs or gloo on CPU;
one state per process) or LocalComm (several virtual ranks in one process,
used to prove slab results bit-identical on a single GPU).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .aprkit import LinearAccess
from .errors import RangeError

Range = Tuple[int, int]


def _row_particles(a: LinearAccess, l: int, za: int, zb: int) -> Range:
    """Particle range of rows z in [za, zb) of level l (contiguous, z-major)."""
    if l < a.l_min or l > a.l_max or a.row_count() == 0:
        return (0, 0)
    za = max(0, min(za, int(a.z_dim[l])))
    zb = max(za, min(zb, int(a.z_dim[l])))
    xd = int(a.x_dim[l])
    r0 = int(a.level_offset[l]) + za * xd
    r1 = int(a.level_offset[l]) + zb * xd
    begin = lambda r: 0 if r == 0 else int(a.xz_end[r - 1])  # noqa: E731
    return (begin(r0), begin(r1))


@dataclass
class SlabPlan:
    """Who owns what, and which contiguous ranges move between which ranks."""
    world: int
    rank: int
    l_max: int            # geometric finest level (cells are pixels)
    c: int                # slab block = 2^c finest planes
    lc: int               # cut level: levels >= lc partitioned, < lc replicated
    bounds: List[Range]   # per rank: finest-level planes [z_lo, z_hi)
    halo: int             # rows exchanged per side at every partitioned level
    leaf: LinearAccess
    tree: Optional[LinearAccess]

    @staticmethod
    def make(leaf: LinearAccess, tree: Optional[LinearAccess], dims: Sequence[int], world: int, rank: int,
             halo: int = 2) -> "SlabPlan":
        nz = int(dims[0])
        l_max = leaf.l_max
        if world < 1 or rank < 0 or rank >= world:
            raise ValueError("bad world/rank")
        # the largest block 2^c such that every rank gets >= halo blocks (a
        # level-lc row is one block, so a halo never reaches past a neighbour)
        c = None
        for cc in range(l_max, -1, -1):
            nb = -(-nz // (1 << cc))
            if nb // world >= max(halo, 1):
                c = cc
                break
        if c is None:
            raise ValueError(f"volume of {nz} planes is too thin for {world} slabs with a {halo}-row halo")
        nb = -(-nz // (1 << c))
        bounds = []
        for r in range(world):
            b0, b1 = r * nb // world, (r + 1) * nb // world
            bounds.append((min(b0 << c, nz), min(b1 << c, nz)))
        return SlabPlan(world, rank, l_max, c, l_max - c, bounds, halo, leaf, tree)

    # -- geometry ---------------------------------------------------------
    def rows(self, l: int, r: Optional[int] = None) -> Range:
        """Level-l rows of rank r's slab (levels >= lc)."""
        z_lo, z_hi = self.bounds[self.rank if r is None else r]
        sh = self.l_max - l
        return (z_lo >> sh, (z_hi + (1 << sh) - 1) >> sh)

    def _levels(self, a: Optional[LinearAccess]):
        if a is None or a.row_count() == 0:
            return range(0)
        return range(max(self.lc, a.l_min), a.l_max + 1)

    def owned(self, which: str, r: Optional[int] = None) -> List[Range]:
        """Particle/node ranges rank r owns at the partitioned levels."""
        a = self.leaf if which == "leaf" else self.tree
        return [_row_particles(a, l, *self.rows(l, r)) for l in self._levels(a)]

    def replicated(self, which: str) -> Range:
        """Ranges of the replicated levels < lc (one contiguous prefix)."""
        a = self.leaf if which == "leaf" else self.tree
        if a is None or a.row_count() == 0 or self.lc <= a.l_min:
            return (0, 0)
        return (0, _row_particles(a, min(self.lc, a.l_max + 1) - 1, 0, 1 << 30)[1])

    def halo_transfers(self, which: str) -> List[Tuple[int, int, Range]]:
        """(src rank, dst rank, range) for every partitioned level and boundary."""
        a = self.leaf if which == "leaf" else self.tree
        out = []
        for l in self._levels(a):
            for r in range(self.world - 1):
                za, zb = self.rows(l, r)
                na, nb_ = self.rows(l, r + 1)
                # rank r's top rows -> r+1 ; rank r+1's bottom rows -> r
                rng = _row_particles(a, l, max(za, zb - self.halo), zb)
                if rng[1] > rng[0]:
                    out.append((r, r + 1, rng))
                rng = _row_particles(a, l, na, min(nb_, na + self.halo))
                if rng[1] > rng[0]:
                    out.append((r + 1, r, rng))
        return out

    def bands(self, r: Optional[int] = None):
        """(interior, [boundary bands]) of rank r's slab, in finest planes: the
        interior lies at least halo level-lc rows (= halo * 2^c planes, which
        covers every partitioned level's halo) from each cut, so its outputs
        read no halo; the bands are the rest of the slab."""
        r = self.rank if r is None else r
        z0, z1 = self.bounds[r]
        m = self.halo << self.c
        lo = z0 + (m if r > 0 else 0)
        hi = z1 - (m if r + 1 < self.world else 0)
        edges = []
        if r > 0:
            edges.append((z0, min(z0 + m, z1)))
        if r + 1 < self.world:
            edges.append((max(hi, lo, z0), z1))
        return (lo, hi), [(a, b) for a, b in edges if b > a]

    def cut_ranges(self, which: str) -> List[Range]:
        """Per rank, its rows of the cut level lc (leaf level lc / tree level lc)."""
        a = self.leaf if which == "leaf" else self.tree
        if a is None or a.row_count() == 0 or self.lc < a.l_min or self.lc > a.l_max:
            return [(0, 0)] * self.world
        return [_row_particles(a, self.lc, *self.rows(self.lc, r)) for r in range(self.world)]


# --------------------------------------------------------------- comms -------
class LocalComm:
    """Virtual ranks in one process: exchanges are tensor copies."""

    def exchange(self, states, attr: str, transfers):
        for src, dst, (b, e) in transfers:
            getattr(states[dst], attr)[b:e].copy_(getattr(states[src], attr)[b:e])

    def exchange_async(self, states, attr: str, transfers):
        self.exchange(states, attr, transfers)
        return []

    def wait(self, works):
        pass

    def allgather_ranges(self, states, attr: str, ranges):
        for s in states:
            for r, (b, e) in enumerate(ranges):
                if e > b and s.rank != r:
                    getattr(s, attr)[b:e].copy_(getattr(states[r], attr)[b:e])


class TorchComm:
    """One state per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def exchange(self, states, attr: str, transfers):
        self.wait(self.exchange_async(states, attr, transfers))

    def exchange_async(self, states, attr: str, transfers):
        """Grouped point-to-point sends/receives, returned in flight (NCCL runs
        them on its own stream, after the work already queued on ours)."""
        (s,) = states
        arr = getattr(s, attr)
        ops = []
        for src, dst, (b, e) in transfers:
            if s.rank == src:
                ops.append(self.dist.P2POp(self.dist.isend, arr[b:e], dst, self.group))
            elif s.rank == dst:
                ops.append(self.dist.P2POp(self.dist.irecv, arr[b:e], src, self.group))
        return self.dist.batch_isend_irecv(ops) if ops else []

    def wait(self, works):
        for req in works:
            req.wait()  # (NCCL: the current stream waits; the host does not)

    def allgather_ranges(self, states, attr: str, ranges):
        import torch
        (s,) = states
        arr = getattr(s, attr)
        m = max(e - b for b, e in ranges)
        if m == 0:
            return
        b, e = ranges[s.rank]
        mine = torch.zeros(m, dtype=arr.dtype, device=arr.device)
        mine[:e - b].copy_(arr[b:e])
        parts = [torch.empty_like(mine) for _ in ranges]
        self.dist.all_gather(parts, mine, group=self.group)
        for r, (rb, re_) in enumerate(ranges):
            if r != s.rank and re_ > rb:
                arr[rb:re_].copy_(parts[r][:re_ - rb])


# ------------------------------------------------------------ GPU state ------
class _CudaArray:
    """__cuda_array_interface__ view of a device pointer owned by libaprgpu."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class GpuRankState:
    """One rank's device state: the full structure on its GPU, full-size value
    arrays (only owned + replicated + halo entries are meaningful)."""

    def __init__(self, plan: SlabPlan, dev, device: int = 0, stream=None):
        import torch
        self.plan, self.rank, self.dev = plan, plan.rank, dev
        self.device = torch.device("cuda", device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        if self.stream.cuda_stream == 0:
            # the legacy default stream would not order the C-ABI calls (handle 0
            # means "the context's own stream") against torch's copies
            raise RuntimeError("GpuRankState needs a non-default current CUDA stream (torch.cuda.set_stream)")
        n_p, n_t = dev.n_particles, dev.n_tree
        self.values = torch.zeros(max(n_p, 1), dtype=torch.float32, device=self.device)
        self.tree = torch.zeros(max(n_t, 1), dtype=torch.float32, device=self.device)
        self.out = torch.zeros(max(n_p, 1), dtype=torch.float32, device=self.device)
        # the APR's per-tile convolution state only for this rank's slab (before its first convolution;
        # a handle that has already convolved keeps its whole-volume state)
        try:
            z_lo, z_hi = plan.bounds[plan.rank]
            dev.restrict(plan.lc, z_lo, z_hi)
        except RangeError:
            pass
        vs, ws = C.c_void_p(), C.c_void_p()
        L.check(L.lib().aprgpu_tree_scratch(dev.handle, C.byref(vs), C.byref(ws)))
        self.vsum = torch.as_tensor(_CudaArray(vs.value, max(n_t, 1), "<f8"), device=self.device)
        self.wsum = torch.as_tensor(_CudaArray(ws.value, max(n_t, 1), "<f8"), device=self.device)

    def _s(self):
        return self.stream.cuda_stream or None

    def tree_sums(self, lt_lo: int, lt_hi: int, slab: bool):
        z_lo, z_hi = self.plan.bounds[self.rank] if slab else (0, -1)
        L.check(L.lib().aprgpu_fill_tree_sums(self.dev.handle, self.values.data_ptr(), lt_lo, lt_hi, z_lo, z_hi,
                                              self._s()))

    def finalize(self):
        L.check(L.lib().aprgpu_fill_tree_finalize(self.dev.handle, self.tree.data_ptr(), self._s()))

    def convolve_slab(self, pyr, pad: int, accum: int):
        z_lo, z_hi = self.plan.bounds[self.rank]
        L.check(L.lib().aprgpu_convolve_slab(self.dev.handle, self.values.data_ptr(), self.tree.data_ptr(),
                                             pyr.handle, int(pad), int(accum), self.plan.lc, z_lo, z_hi,
                                             self.out.data_ptr(), self._s()))

    def convolve_band(self, pyr, pad: int, accum: int, z_lo: int, z_hi: int, replicated: bool):
        if z_hi <= z_lo and not replicated:
            return
        L.check(L.lib().aprgpu_convolve_slab_band(self.dev.handle, self.values.data_ptr(), self.tree.data_ptr(),
                                                  pyr.handle, int(pad), int(accum), self.plan.lc, z_lo,
                                                  max(z_lo, z_hi), int(replicated), self.out.data_ptr(), self._s()))


# ------------------------------------------------------------ algorithm ------
class SlabConvolver:
    """fill_tree / convolve_apr over slabs (see the module docstring)."""

    def __init__(self, states, comm):
        self.states, self.comm = list(states), comm
        self.plan = self.states[0].plan

    def fill_tree(self):
        p = self.plan
        t = p.tree
        if t is None or t.row_count() == 0:
            return
        for s in self.states:  # partitioned interior levels, own rows only
            s.tree_sums(max(p.lc, t.l_min), t.l_max, slab=True)
        # the cut: level-lc leaves and tree-level-lc sums, so that every rank
        # computes the replicated levels < lc in the reference order
        self.comm.allgather_ranges(self.states, "values", p.cut_ranges("leaf"))
        tr = p.cut_ranges("tree")
        self.comm.allgather_ranges(self.states, "vsum", tr)
        self.comm.allgather_ranges(self.states, "wsum", tr)
        if p.lc - 1 >= t.l_min:
            for s in self.states:
                s.tree_sums(t.l_min, p.lc - 1, slab=False)
        for s in self.states:
            s.finalize()

    def exchange_and_convolve(self, pyr, pad: int = L.PAD_REFLECT, accum: int = L.ACCUM_EXACT):
        """The conv-only step with the tree values already filled: the leaf and
        tree halo exchanges in flight while every rank convolves its interior,
        then the boundary bands once the halos have landed."""
        p = self.plan
        works = self.comm.exchange_async(self.states, "values", p.halo_transfers("leaf"))
        if p.tree is not None:
            works += self.comm.exchange_async(self.states, "tree", p.halo_transfers("tree"))
        for s in self.states:
            (lo, hi), _ = p.bands(s.rank)
            s.convolve_band(pyr, pad, accum, lo, hi, True)
        self.comm.wait(works)
        for s in self.states:
            for lo, hi in p.bands(s.rank)[1]:
                s.convolve_band(pyr, pad, accum, lo, hi, False)

    def convolve(self, pyr, pad: int = L.PAD_REFLECT, accum: int = L.ACCUM_EXACT):
        p = self.plan
        hw = pyr.half_width(p.lc, p.l_max) if hasattr(pyr, "half_width") else None
        if hw is not None and hw > p.halo:
            raise ValueError(f"stencil half-width {hw} at the partitioned levels exceeds the plan's halo "
                             f"of {p.halo} rows: make the SlabPlan with halo >= {hw}")
        self.comm.exchange(self.states, "values", p.halo_transfers("leaf"))
        self.fill_tree()
        if p.tree is not None:
            self.comm.exchange(self.states, "tree", p.halo_transfers("tree"))
        for s in self.states:
            s.convolve_slab(pyr, pad, accum)
