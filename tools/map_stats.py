"""Gather-map record statistics on C3 (3^3, reflect): how many of a tile's box
cells its active blocks read, and how compressible the 16-bit code rows are
(a design study for cutting the map's bytes; prints one line per level and a
total).  Needs a GPU:  python tools/map_stats.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
dapr = apr.device()
a = apr.access
pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device()
v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
tv = torch.empty(max(dapr.n_tree, 1), dtype=torch.float32, device="cuda")
out = torch.empty_like(v)
s = torch.cuda.current_stream().cuda_stream
dapr.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
dapr.convolve_ptr(v.data_ptr(), tv.data_ptr(), pyr, 1, L.ACCUM_EXACT, out.data_ptr(), s)
torch.cuda.synchronize()

BZ = BX = 10
BY = 36  # (MapBox rows: kTY + 4 cells)
NC = BZ * BX * BY
CW = NC // 2
BM = np.zeros((256, BZ, BX, BY), np.float32)  # cells each 2x2x2 block's 4x4x4 neighbourhood reads
for b in range(256):
    qz, qx, qy = b // 64, (b // 16) & 3, b & 15
    BM[b, 2 * qz:2 * qz + 4, 2 * qx:2 * qx + 4, 2 * qy:2 * qy + 4] = 1.0
BM = torch.from_numpy(BM.reshape(256, -1)).cuda()
allch = []
tot = dict(ivl=0, tiles=0, cells=0, read=0, pairs_read=0, breaks=0, rows=0, rows_read=0, rowdup=0, nblk=0)
for l in range(a.l_min, a.l_max + 1):
    nw, t0, nt = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.check(L.lib().aprgpu_map_records(dapr.handle, 1, 1, l, None, 0, None, C.byref(nw), C.byref(t0), C.byref(nt)))
    if nt.value == 0:
        continue
    buf = np.empty(nw.value, np.uint32)
    L.check(L.lib().aprgpu_map_records(dapr.handle, 1, 1, l, buf.ctypes.data, buf.size, None, C.byref(nw),
                                       C.byref(t0), C.byref(nt)))
    rec = buf.reshape(nt.value, -1)  # (fixed-length records: codes, then masks, first indices, counts, blocks)
    codes = rec[:, :CW].view(np.uint16).reshape(-1, BZ, BX, BY).astype(np.int32)
    nblk = rec[:, CW + 129].astype(np.int64)
    nch = rec[:, CW + 128].astype(np.int64)  # 16-byte source chunks of the tile (the staged F: 4 floats each)
    allch.append(nch)
    blist = rec[:, CW + 132:CW + 132 + 64].view(np.uint8)
    # cells the active blocks read (union of 4x4x4 neighbourhoods)
    act = np.zeros((nt.value, 256), np.float32)
    k = np.arange(256)[None, :] < nblk[:, None]
    act[np.nonzero(k)[0], blist[k]] = 1.0
    read = (torch.from_numpy(act).cuda() @ BM).cpu().numpy().reshape(-1, BZ, BX, BY) > 0
    pairs = read.reshape(nt.value, -1, 2).any(-1)
    # per box row: the read words as an interval [first, last] (no popc to index)
    pw = pairs.reshape(nt.value, BZ * BX, BY // 2)
    anyw = pw.any(-1)
    first = np.argmax(pw, -1)
    last = BY // 2 - 1 - np.argmax(pw[..., ::-1], -1)
    ivl = int(np.where(anyw, last - first + 1, 0).sum())
    # code-row breaks: a cell whose code is neither its left neighbour's nor +4
    d = np.diff(codes, axis=-1)
    brk = (d != 0) & (d != 4)
    rows_read = read.any(-1)
    # a box row identical to the previous row along x (common under coarse cells)
    dup = np.all(codes[:, :, 1:, :] == codes[:, :, :-1, :], axis=-1)
    st = dict(ivl=ivl, tiles=nt.value, cells=NC * nt.value, read=int(read.sum()), pairs_read=int(pairs.sum()),
              breaks=int(brk.sum()), rows=BZ * BX * nt.value, rows_read=int(rows_read.sum()), rowdup=int(dup.sum()),
              nblk=int(nblk.sum()))
    for k in tot:
        tot[k] += st[k]
    print(f"level {l}: tiles {nt.value}, blocks/tile {st['nblk'] / nt.value:.1f}, cells read "
          f"{st['read'] / st['cells']:.3f}, pairs read {st['pairs_read'] / (CW * nt.value):.3f}, rows read "
          f"{st['rows_read'] / st['rows']:.3f}, breaks/row {st['breaks'] / st['rows']:.2f}, x-dup rows "
          f"{st['rowdup'] / st['rows']:.3f}", flush=True)
T = tot
print(f"TOTAL tiles {T['tiles']}, code MB {T['cells'] * 2 / 1e6:.1f}, blocks/tile {T['nblk'] / T['tiles']:.1f}, "
      f"cells read {T['read'] / T['cells']:.3f}, pairs read {T['pairs_read'] / (T['cells'] / 2):.3f}, rows read "
      f"{T['rows_read'] / T['rows']:.3f}, breaks/row {T['breaks'] / T['rows']:.2f}, x-dup rows "
      f"{T['rowdup'] / T['rows']:.3f}, interval words {T['ivl'] / (T['cells'] / 2):.3f}")
ch = np.concatenate(allch)
print("chunks per tile: p50 %d p90 %d p99 %d max %d; tiles with <= 256 / 384 / 512 chunks: %.3f / %.3f / %.3f" % (
    np.percentile(ch, 50), np.percentile(ch, 90), np.percentile(ch, 99), ch.max(), (ch <= 256).mean(), (ch <= 384).mean(),
    (ch <= 512).mean()))
print("active blocks per tile: p50 %d p90 %d max %d; <= 96: %.3f" % (0, 0, 0, 0) if False else "")
