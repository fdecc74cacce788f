"""CPU rank state for the z-slab algorithm (TEST INFRASTRUCTURE).

Lets paper_2112_03592_b200.slab run over torch.distributed/gloo on CPU in
world_size > 1 tests: interior-level fp64 sums in the reference's exact
per-parent order (numpy, vectorised per child class; pinned against the
reference's fill_tree in tests/test_slab.py) and the convolution from the C
oracle.  Entries a rank neither owns nor receives are NaN-poisoned by the
tests, so any missing halo row shows up in the owned outputs.
"""
from __future__ import annotations

import numpy as np
import torch

from pyoracle import Oracle


def _keys(a):
    """Sorted key (row << 16 | y) of every particle of an access structure."""
    n = a.row_count()
    ends = np.asarray(a.xz_end, np.int64)
    counts = np.diff(np.concatenate([[0], ends]))
    rows = np.repeat(np.arange(n, dtype=np.int64), counts)
    return (rows << 16) | np.asarray(a.y_idx, np.int64)


def tree_sums(leaf, tree, dims, values, vsum, wsum, lt_lo, lt_hi, z_range=None):
    """tree.hpp:110-143 for interior levels lt_hi .. lt_lo (finest first),
    parents with z in z_range (finest-level planes [z_lo, z_hi)) only.
    Accumulation order per parent: for (cz, cx) lexicographic, leaf children
    y = 2py, 2py+1, then interior children y = 2py, 2py+1 -- as
    synchronized_parent_pass visits them."""
    glm = leaf.l_max
    lkeys, tkeys = _keys(leaf), _keys(tree)
    vals = np.asarray(values, np.float32).astype(np.float64)
    nz, nx, ny = (int(d) for d in dims)
    for lt in range(min(lt_hi, tree.l_max), max(lt_lo, tree.l_min) - 1, -1):
        c = lt + 1
        zd, xd = int(tree.z_dim[lt]), int(tree.x_dim[lt])
        r0 = int(tree.level_offset[lt])
        b = 0 if r0 == 0 else int(tree.xz_end[r0 - 1])
        e = int(tree.xz_end[r0 + zd * xd - 1]) if zd * xd else b
        if e <= b:
            continue
        j = np.arange(b, e, dtype=np.int64)
        rows = (tkeys[b:e] >> 16) - r0
        pz, px, py = rows // xd, rows % xd, tkeys[b:e] & 0xffff
        if z_range is not None:
            sh = glm - lt
            keep = (pz >= (z_range[0] >> sh)) & (pz < ((z_range[1] + (1 << sh) - 1) >> sh))
            j, pz, px, py = j[keep], pz[keep], px[keep], py[keep]
        vsum[j] = 0.0
        wsum[j] = 0.0
        s = 1 << (glm - c)
        czd = -(-nz // s)
        cxd = -(-nx // s)
        for dz in (0, 1):
            for dx in (0, 1):
                cz, cx = 2 * pz + dz, 2 * px + dx
                ok = (cz < czd) & (cx < cxd)
                if leaf.l_min <= c <= leaf.l_max:
                    row = int(leaf.level_offset[c]) + cz * int(leaf.x_dim[c]) + cx
                    for dy in (0, 1):
                        cy = 2 * py + dy
                        q = (row << 16) | cy
                        i = np.searchsorted(lkeys, q)
                        hit = ok & (i < lkeys.size)
                        hit[hit] = lkeys[i[hit]] == q[hit]
                        fz = np.minimum((cz + 1) * s, nz) - cz * s
                        fx = np.minimum((cx + 1) * s, nx) - cx * s
                        fy = np.minimum((cy + 1) * s, ny) - cy * s
                        w = fz.astype(np.float64) * fx.astype(np.float64) * fy.astype(np.float64)
                        jj, ii, ww = j[hit], i[hit], w[hit]
                        vsum[jj] += ww * vals[ii]
                        wsum[jj] += ww
                if c <= tree.l_max:
                    row = int(tree.level_offset[c]) + cz * int(tree.x_dim[c]) + cx
                    for dy in (0, 1):
                        cy = 2 * py + dy
                        q = (row << 16) | cy
                        i = np.searchsorted(tkeys, q)
                        hit = ok & (i < tkeys.size)
                        hit[hit] = tkeys[i[hit]] == q[hit]
                        jj, ii = j[hit], i[hit]
                        vsum[jj] += vsum[ii]
                        wsum[jj] += wsum[ii]


def finalize(vsum, wsum):
    out = np.zeros(vsum.size, np.float32)
    nz = wsum > 0
    out[nz] = (vsum[nz] / wsum[nz]).astype(np.float32)
    return out


class CpuRankState:
    """RankState interface of paper_2112_03592_b200.slab on CPU tensors."""

    def __init__(self, plan, dims, levels, level_min):
        self.plan, self.rank, self.dims = plan, plan.rank, dims
        self.levels, self.level_min = levels, level_min
        n_p = plan.leaf.particle_count()
        n_t = plan.tree.particle_count() if plan.tree is not None else 0
        self.values = torch.zeros(n_p, dtype=torch.float32)
        self.tree = torch.zeros(max(n_t, 1), dtype=torch.float32)
        self.out = torch.zeros(n_p, dtype=torch.float32)
        self.vsum = torch.zeros(max(n_t, 1), dtype=torch.float64)
        self.wsum = torch.zeros(max(n_t, 1), dtype=torch.float64)

    def tree_sums(self, lt_lo, lt_hi, slab):
        z = self.plan.bounds[self.rank] if slab else None
        tree_sums(self.plan.leaf, self.plan.tree, self.dims, self.values.numpy(), self.vsum.numpy(),
                  self.wsum.numpy(), lt_lo, lt_hi, z)

    def finalize(self):
        self.tree.copy_(torch.from_numpy(finalize(self.vsum.numpy(), self.wsum.numpy())))

    def convolve_slab(self, pyr, pad, accum):
        full = Oracle().convolve(self.plan.leaf, self.plan.tree, self.values.numpy(), self.tree.numpy(),
                                 self.levels, self.level_min, int(pad))
        self.out.copy_(torch.from_numpy(full))

    def convolve_band(self, pyr, pad, accum, z_lo, z_hi, replicated):
        """aprgpu_convolve_slab_band restated: only the outputs of the band's
        rows at the partitioned levels (and the replicated levels if asked)."""
        from paper_2112_03592_b200.slab import _row_particles
        full = torch.from_numpy(Oracle().convolve(self.plan.leaf, self.plan.tree, self.values.numpy(),
                                                  self.tree.numpy(), self.levels, self.level_min, int(pad)))
        p = self.plan
        if replicated:
            b, e = p.replicated("leaf")
            self.out[b:e] = full[b:e]
        for l in p._levels(p.leaf):
            sh = p.l_max - l
            b, e = _row_particles(p.leaf, l, z_lo >> sh, (z_hi + (1 << sh) - 1) >> sh)
            self.out[b:e] = full[b:e]
