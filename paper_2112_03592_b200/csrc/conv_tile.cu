// Box-tile convolution for isotropic 3^3 / 5^3 levels (the hot path).
//
// Work item: one (level l, 8z x 8x x kTY y) output tile holding at least one
// particle (tile lists are built once per APR at upload, from the non-empty
// rows).  All levels that use the same isotropic extent run in ONE launch
// (coarse levels first, so their few tiles overlap the finest level's bulk).
// One 128-thread CTA per tile:
//
//   rows    every source row that can reach the tile's (8+2H)x(8+2H)x(kTY+2H)
//           box -- the level-l leaf rows and interior rows of the halo plane,
//           and the level l-d leaf rows covering it for d = 1..D -- is
//           resolved by one thread: its particle range inside the box's
//           y-extent (two lower_bounds) and its box geometry, packed.
//   flatten a block-wide scan of the ranges numbers every source particle of
//           the tile; each particle gets its row id in shared memory.
//   fill    one thread per source PARTICLE (warp-uniform work: no per-row
//           loops): level-l leaves / interior nodes write their cell and the
//           output map, a coarse leaf at depth d writes its 2^d-aligned group
//           of cells (constant upsampling, fill_level_row semantics,
//           reconstruct.hpp:41-69) as vector stores (the box's y origin is
//           y0 - 4, so pairs and quads are aligned); leaves >= 3 levels
//           coarser are queued and filled by the whole CTA.  In a valid APR
//           every in-domain cell is covered by exactly one source, so all
//           particles scatter in one unordered pass.
//   pad     out-of-domain cells within H of the domain: reflect_index / 0.
//   apply   the tile is cut into 2x2x2 cell blocks (an APR refines cells into
//           sibling octets, so finest-level particles come in complete
//           blocks); blocks holding particles are compacted and each is
//           evaluated by one thread from a (2+2H)^3 neighbourhood streamed
//           plane by plane through registers.  Every output's taps accumulate
//           in the reference's exact (az, ax, ay) order (LevelSlab::apply,
//           convolve.hpp:154-169): fp64 FMA of exact products in EXACT mode
//           (bit-identical), fp32 FMA (packed fp32x2 over the block's y pair)
//           in FAST mode.
//
// A probe kernel (k_tile_probe) runs once per APR and stores one byte per
// tile: D (deepest coarse depth whose leaves reach into the 5^3 box, so no
// coverage counting is needed), OVERLAP (malformed APR: some cell covered
// twice -> the tile is filled in the reference's order, level l, l-1, ...,
// then interior nodes, last writer wins) and HOLES (some cell uncovered -> the
// box is zeroed first).  The probe uses the 5^3 box, a superset of the 3^3
// box, so one byte serves both stencil sizes.
#include <algorithm>
#include <cstdlib>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"

#ifndef APRGPU_TILE_Y
#define APRGPU_TILE_Y 32
#endif

namespace aprgpu {

constexpr int kTZ = 8, kTX = 8, kTY = APRGPU_TILE_Y, kTileThreads = 128;
constexpr int kBlocks = (kTZ / 2) * (kTX / 2) * (kTY / 2);  // 2x2x2 output blocks per tile
static_assert(kBlocks <= 256, "block ids are bytes");
constexpr int kProbeH = 2;
constexpr int kMaxSrcRows = 512;   // >= 2*(8+2*2)^2 + coarse rows of a 5^3 box
constexpr int kMaxFlat = 960;      // source particles per flattened chunk (fits 8 CTAs/SM)
constexpr int kPadY = 4;           // box y origin = y0 - kPadY (>= H, multiple of 4)
enum : uint8_t { kMetaDepth = 0x1f, kMetaOverlap = 0x20, kMetaHoles = 0x40 };

namespace {

struct TileLaunch {
    AccessView leaf, tree;
    const float* val;
    const float* tval;
    const uint32_t* tiles;   // tile ids of all levels (absolute indexing)
    const uint8_t* meta;     // one byte per tile
    const uint2* runs;       // per-tile source runs (see k_tile_runs)
    const uint32_t* run_off; // n_tiles + 1
    uint32_t tile_base;      // first tile of the launch (blocks map to consecutive tiles)
    int n_levels;                   // level segments in this launch
    int lvl[kMaxLevels];            // level of each segment
    uint32_t seg_end[kMaxLevels];   // exclusive end (in blocks) of each level segment
    // per segment: tiles skipped before its first block (a slab's launch covers only the z-range of
    // tiles it computes), so block b of segment s is tile tile_base + b + seg_shift[s]
    uint32_t seg_shift[kMaxLevels];
    int tdim[kMaxLevels][3];        // tile grid dims of each segment's level
    uint64_t woff[kMaxLevels];      // weight offset of each segment's level
    const float* wf;
    const double* wd;
    const float* sep[kMaxLevels];   // per segment: rank-1 factors fz, fx, fy of its stencil, or null
    int tree_lmin, tree_lmax;       // interior levels present (tree_lmax < tree_lmin: none)
    int pad;
    float* out;
    EpiArgs epi;
    int slab_lc, slab_zlo, slab_zhi;  // z-slab restriction (Slab, internal.cuh)
    uint32_t* map[kMaxLevels];        // per segment: gather-map records (k_conv_map), or the build target
    uint32_t map_base[kMaxLevels];    // per segment: the tile whose record is map[s][0]
    uint32_t* flat;                   // per H flattened source lists (DevAccess::tile_flat)
    const uint32_t* flat_off;         // n_tiles + 1 exact offsets (chunk counts; the lists sit at tix * flat_cap)
    uint32_t flat_cap;                // entries per tile in flat (the largest tile's chunk count)
    int place_drop;                   // k_map_place: drop the chunks no active block reads (3^3)
    int* map_overflow;                // set by the build when a tile has > MapBox::NC sources
    int* map_maxg;                    // the build's largest per-tile chunk count (atomicMax)
    uint32_t n_leaf, n_tree;          // value-array lengths (a tail chunk copies only valid elements)
    int map_ng;                       // k_conv_map: largest chunk count of the launch's tiles
    int aligned16;                    // both value arrays 16-byte aligned (else 4-byte copies)
    int list_in_f;                    // k_conv_map 3^3: the chunk list staged in F's tail (launch_map)
    int l2hint;                       // k_conv_map: records and lists copied evict-first in L2
};

struct Geo {
    int l;
    int z0, x0, y0;                    // tile origin (level-l cells)
    int bz0, bx0, by0;                 // box origin
    int zlo, zhi, xlo, xhi, ylo, yhi;  // in-domain part of the box
};

// Box layout: (8+2H) x (8+2H) rows of kTY + 2*kPadY cells, y origin y0 - 4,
// so a coarse leaf's 2^d cells start at an index aligned to min(2^d, 4).
template <int H>
struct Box {
    static constexpr int BZ = kTZ + 2 * H, BX = kTX + 2 * H, BY = kTY + 2 * kPadY;
    static constexpr int NR = BZ * BX, NC = BZ * BX * BY;
};

// Gather-map record of a tile (k_conv_map): the box as (8+2H) x (8+2H) rows
// of kTY + 2H cells (y origin y0 - H: exactly the cells the stencil reads),
// one 16-bit code per cell -- the byte offset in F (the staged values) of its
// source, 4 * (kFlat0 + its index in the tile's flattened source list, the
// concatenation of its source runs, k_tile_runs), ZERO = F[0] = 0 for a zero
// cell; byte offsets spare the apply an address multiply -- then per inner row an output mask over
// y0 .. y0+kTY-1 and the index of its first output particle, then the number
// of leaf sources (the list holds the leaf runs' particles, then the interior
// runs' nodes, so each part copies from one base pointer).  The flattened
// source list itself (particle or node index per entry, padded to 4) lives
// in DevAccess::tile_flat, shared by both pad modes.  In a valid APR every box
// cell has one source, so a tile has at most NC sources (the build checks; a
// malformed APR's overlapping sources can exceed it, and its levels then
// reconstruct).
constexpr int kFlat0 = 4;  // F[0 .. 3]: the zero (and 16-byte alignment of the staged values)
// The staged source list is stored in aligned 16-byte CHUNKS: every source run
// of the tile (a contiguous particle or node range starting at particle b) is
// placed in F at a fresh 4-slot boundary plus b mod 4 and covers whole chunks,
// so each chunk is ONE 16-byte copy whose source (4 particles from b - b mod 4
// on) is 16-byte aligned too; the few extra particles it brings land in
// padding slots no code points at.  One u32 per chunk: its first particle
// (bit 31: interior node, bit 30: the array's tail chunk -- only its valid
// elements are copied).  A tile's chunk count is padded to 4 (16-byte bulk
// copies of the list).
constexpr uint32_t kChunkTree = 1u << 31, kChunkTail = 1u << 30, kChunkIdx = kChunkTail - 1;
constexpr uint32_t kListHead = 512;  // 3^3 chunk-list entries copied with the record (k_conv_map)
constexpr int kMaxChunks = 4000;  // 16-bit byte offsets into F: 4 * (kFlat0 + 4 * chunks) < 65536
template <int H>
struct MapBox {
    // rows of kTY + 4 cells for both extents (3^3: two padding cells -- an
    // even word stride of 18 spreads the apply's code-word banks: blocks in
    // different z planes no longer share a bank pattern)
    static constexpr int BZ = kTZ + 2 * H, BX = kTX + 2 * H, BY = kTY + 4;
    static constexpr int NC = BZ * BX * BY;
    // 5^3's expanded box: planes padded by one float4 (a plane stride of 218
    // float2 instead of 216 -- blocks that differ only in z no longer read the
    // same banks: offline 2.84 -> 2.43 wavefronts per pair load)
    static constexpr int PL = BX * BY + (H == 2 ? 4 : 0), SN = BZ * PL;
    // codes in cell order, two per word: the apply reads a cell pair (c, c+1),
    // c even, with one 32-bit load
    static constexpr int CW = NC / 2;                   // code words
    // + per inner row mask and first index, nleaf, the active-block count, pad,
    // and the active blocks' order (bytes; see k_conv_tile's map mode).  H = 1:
    // codes first; H = 2: this header first, then the codes (the 5^3 box is
    // expanded in place over the codes, so the header must lie before them)
    static constexpr int HDR = 2 * kTZ * kTX + 4 + kBlocks / 4;  // header words
    static constexpr int CODE0 = H == 2 ? HDR : 0;               // first code word
    static constexpr int MASK0 = H == 2 ? 0 : CW;                // masks, then first indices
    static constexpr int W_NLEAF = MASK0 + 2 * kTZ * kTX, W_NBLK = W_NLEAF + 1, W_BLK = W_NLEAF + 4;
    static constexpr int REC = CW + HDR;                // 32-bit words per record
    // bank key of an apply block: its first pair's word (H = 1: code words,
    // 32 banks; H = 2: float2 box pairs, 16 double banks) modulo the bank count
    static constexpr int NK = H == 1 ? 32 : 16;
    static_assert((CW * 4) % 16 == 0 && (REC * 4) % 16 == 0 && (HDR * 4) % 16 == 0, "16-byte bulk copies");
    static constexpr uint32_t ZERO = 0;
    static constexpr int NF = kFlat0 + ((NC + 3) & ~3);  // F entries
};
static_assert(kTY == 32, "one 32-bit output mask per inner row");

template <int H>
__device__ __forceinline__ Geo make_geo(int l, uint32_t id, int txd, int tyd, const LevelG& g) {
    Geo G;
    G.l = l;
    const int ty = static_cast<int>(id % tyd);
    const uint32_t t2 = id / tyd;
    const int tx = static_cast<int>(t2 % txd), tz = static_cast<int>(t2 / txd);
    G.z0 = tz * kTZ;
    G.x0 = tx * kTX;
    G.y0 = ty * kTY;
    G.bz0 = G.z0 - H;
    G.bx0 = G.x0 - H;
    G.by0 = G.y0 - kPadY;
    G.zlo = max(G.bz0, 0);
    G.zhi = min(G.z0 + kTZ + H, g.zd);
    G.xlo = max(G.bx0, 0);
    G.xhi = min(G.x0 + kTX + H, g.xd);
    G.ylo = max(G.y0 - H, 0);
    G.yhi = min(G.y0 + kTY + H, g.yd);
    return G;
}

// Level segment of launch block b.  Searched from the last segment: levels run
// coarse to fine, so most blocks (the finest level's) resolve at once.
__device__ __forceinline__ int seg_of(const uint32_t* seg_end, int n, uint32_t b) {
    int s = n - 1;
    while (s > 0 && b < seg_end[s - 1]) --s;
    return s;
}

// Number of level l-d rows covering the in-domain box (d >= 1).
__device__ __forceinline__ int coarse_rows(const Geo& G, int d, int& czlo, int& cxlo, int& nxc) {
    czlo = G.zlo >> d;
    cxlo = G.xlo >> d;
    const int nzc = ((G.zhi - 1) >> d) - czlo + 1;
    nxc = ((G.xhi - 1) >> d) - cxlo + 1;
    return nzc * nxc;
}

// Source rows of a box, in the reference's fill order: [0, NR) level-l leaf
// rows, then for d = 1..D the level l-d leaf rows covering it, then [.., +NR)
// the level-l interior rows (when the level has interior nodes).  Depends on
// the box's z/x extent only, so one table serves every tile of a segment.
struct SrcTable {
    int D, tree, n;
    int base[kMetaDepth + 3];
};

template <int H>
__device__ __forceinline__ void make_src_table(const Geo& G, int D, int tree, SrcTable& T) {
    T.D = D;
    T.tree = tree;
    int n = Box<H>::NR;
    T.base[0] = 0;
    for (int d = 1; d <= D; ++d) {
        T.base[d] = n;
        int czlo, cxlo, nxc;
        n += coarse_rows(G, d, czlo, cxlo, nxc);
    }
    T.base[D + 1] = n;
    if (tree) n += Box<H>::NR;
    T.n = n;
}

// One source row, resolved: particles [b, e) of the row; d = coarse depth
// (0: level-l leaf or interior row); (zA, zB) x (xA, xB) = the clipped level-l
// rows its cells cover; r00 = box offset of cell (zA, xA, y = 0); obase =
// output-map offset of y = 0 when the row is an inner level-l leaf row.
struct RowJob {
    uint32_t b, e;
    int d, is_tree, inner;
    int zA, zB, xA, xB;
    int r00, obase;
};

template <int H, bool LOAD = true>
__device__ __forceinline__ bool resolve_row(const TileLaunch& a, const Geo& G, const SrcTable& T, int t, RowJob& J) {
    using B = Box<H>;
    int d = 0;
    int r = t;
    J.is_tree = 0;
    if (t >= T.base[T.D + 1]) {
        J.is_tree = 1;
        r = t - T.base[T.D + 1];
    } else {
        while (d < T.D && t >= T.base[d + 1]) ++d;
        r = t - T.base[d];
    }
    J.d = d;
    uint32_t row;
    const AccessView& av = J.is_tree ? a.tree : a.leaf;
    if (d == 0) {
        const int bz = r / B::BX, bx = r - (r / B::BX) * B::BX;
        const int zz = G.bz0 + bz, xx = G.bx0 + bx;
        if (zz < G.zlo || zz >= G.zhi || xx < G.xlo || xx >= G.xhi) return false;
        const LevelG g = av.g[G.l];
        row = g.row0 + static_cast<uint32_t>(zz) * g.xd + xx;
        J.zA = zz;
        J.zB = zz + 1;
        J.xA = xx;
        J.xB = xx + 1;
        J.inner = !J.is_tree && bz >= H && bz < H + kTZ && bx >= H && bx < H + kTX;
        J.obase = (bz - H) * kTX + (bx - H);  // inner row id (when inner)
    } else {
        int czlo, cxlo, nxc;
        coarse_rows(G, d, czlo, cxlo, nxc);
        const int cz = czlo + r / nxc, cx = cxlo + r % nxc;
        const LevelG gc = a.leaf.g[G.l - d];
        if (cz >= gc.zd || cx >= gc.xd) return false;
        row = gc.row0 + static_cast<uint32_t>(cz) * gc.xd + cx;
        J.zA = max(cz << d, G.zlo);
        J.zB = min((cz + 1) << d, G.zhi);
        J.xA = max(cx << d, G.xlo);
        J.xB = min((cx + 1) << d, G.xhi);
        J.inner = 0;
        J.obase = 0;
    }
    J.r00 = ((J.zA - G.bz0) * B::BX + (J.xA - G.bx0)) * B::BY - G.by0;
    if (!LOAD) return true;
    J.b = __ldg(av.rb + row);
    J.e = __ldg(av.rb + row + 1);
    return J.e > J.b;
}

// ---------------------------------------------------------------- probe ----
// Per tile: deepest coarse depth reaching into the (5^3) box and whether the
// sources overlap or leave holes there.  Scans every depth down to l_min, so D
// is exact even for malformed APRs.
__global__ void __launch_bounds__(kTileThreads) k_tile_probe(const __grid_constant__ TileLaunch a) {
    using B = Box<kProbeH>;
    __shared__ uint8_t cnt[B::NC];
    __shared__ int hit[kMetaDepth + 2];
    __shared__ int flags;
    __shared__ SrcTable T;
    const int tid = threadIdx.x;
    const int s = seg_of(a.seg_end, a.n_levels, blockIdx.x);
    const int l = a.lvl[s];
    const LevelG g = a.leaf.g[l];
    const uint32_t tile = a.tile_base + blockIdx.x + a.seg_shift[s];
    const Geo G = make_geo<kProbeH>(l, a.tiles[tile], a.tdim[s][1], a.tdim[s][2], g);
    for (int i = tid; i < B::NC; i += kTileThreads) cnt[i] = 0;
    if (tid < kMetaDepth + 2) hit[tid] = 0;
    const int tree = (l >= a.tree_lmin && l <= a.tree_lmax) ? 1 : 0;
    const int Dall = min(l - a.leaf.l_min, static_cast<int>(kMetaDepth));
    if (tid == 0) {
        flags = 0;
        make_src_table<kProbeH>(G, Dall, tree, T);
    }
    __syncthreads();
    for (int t = tid; t < T.n; t += kTileThreads) {
        RowJob J;
        if (!resolve_row<kProbeH>(a, G, T, t, J)) continue;
        const uint16_t* ys = J.is_tree ? a.tree.y : a.leaf.y;
        const int d = J.d;
        bool any = false;
        for (uint32_t i = lower_bound_u16(ys, J.b, J.e, G.ylo >> d); i < J.e; ++i) {
            const int yy = __ldg(ys + i);
            if ((yy << d) >= G.yhi) break;
            const int yA = max(yy << d, G.ylo), yB = min((yy + 1) << d, G.yhi);
            for (int z = J.zA; z < J.zB; ++z)
                for (int x = J.xA; x < J.xB; ++x)
                    for (int y = yA; y < yB; ++y) {
                        const int c = ((z - G.bz0) * B::BX + (x - G.bx0)) * B::BY + (y - G.by0);
                        // byte counters packed in words (a cell sees at most one source per depth + 1)
                        atomicAdd(reinterpret_cast<uint32_t*>(cnt + (c & ~3)), 1u << (8 * (c & 3)));
                        any = true;
                    }
        }
        if (any) hit[d] = 1;
    }
    __syncthreads();
    int f = 0;
    for (int c = tid; c < B::NC; c += kTileThreads) {
        const int bz = c / (B::BX * B::BY);
        const int rem = c - bz * (B::BX * B::BY);
        const int bx = rem / B::BY, by = rem - bx * B::BY;
        const int zz = G.bz0 + bz, xx = G.bx0 + bx, yy = G.by0 + by;
        if (zz < G.zlo || zz >= G.zhi || xx < G.xlo || xx >= G.xhi || yy < G.ylo || yy >= G.yhi) continue;
        const int v = cnt[c];
        if (v == 0) f |= kMetaHoles;
        if (v > 1) f |= kMetaOverlap;
    }
    if (f) atomicOr(&flags, f);
    __syncthreads();
    if (tid == 0) {
        int D = 0;
        for (int d = 1; d <= Dall; ++d)
            if (hit[d]) D = d;
        const_cast<uint8_t*>(a.meta)[tile] = static_cast<uint8_t>(D | flags);
    }
}

// --------------------------------------------------------------- tile runs --
// Once per APR and stencil half-width: for every tile, the non-empty source
// rows of its box and their particle ranges inside the box's y-extent --
// {first particle, row slot | count << 16}, in row-slot (= reference fill)
// order.  This is the structure-only part of the convolution's row phase
// (row lookups + dependent searches), hoisted out of every call.
template <int H>
__global__ void __launch_bounds__(kTileThreads) k_tile_runs(const __grid_constant__ TileLaunch a, int mode,
                                                           uint32_t* __restrict__ counts, uint2* __restrict__ runs) {
    __shared__ SrcTable T;
    __shared__ int cnt[kMaxSrcRows];
    __shared__ int wsum[kTileThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = seg_of(a.seg_end, a.n_levels, blockIdx.x);
    const int l = a.lvl[s];
    const uint32_t tix = a.tile_base + blockIdx.x + a.seg_shift[s];
    const Geo G = make_geo<H>(l, a.tiles[tix], a.tdim[s][1], a.tdim[s][2], a.leaf.g[l]);
    const int tree = (l >= a.tree_lmin && l <= a.tree_lmax) ? 1 : 0;
    if (tid == 0) make_src_table<H>(G, a.meta[tix] & kMetaDepth, tree, T);
    __syncthreads();
    uint32_t s0v[kMaxSrcRows / kTileThreads];
#pragma unroll
    for (int k = 0; k < kMaxSrcRows / kTileThreads; ++k) {
        const int t = tid + k * kTileThreads;
        RowJob J;
        int n = 0;
        uint32_t s0 = 0;
        if (t < T.n && resolve_row<H>(a, G, T, t, J)) {
            const uint16_t* ys = J.is_tree ? a.tree.y : a.leaf.y;
            uint32_t s1;
            lower_bound2_kary(ys, J.b, J.e, G.ylo >> J.d, (G.yhi + (1 << J.d) - 1) >> J.d, s0, s1);
            n = static_cast<int>(s1 - s0);
        }
        s0v[k] = s0;
        // mode 0: non-empty flag; mode 1: flag in bit 0, count above it
        cnt[t] = mode == 0 ? (n > 0) : (n > 0 ? (n << 1) | 1 : 0);
    }
    __syncthreads();
    if (mode == 0) {
        int c = 0;
        for (int t = tid; t < kMaxSrcRows; t += kTileThreads) c += cnt[t];
        c = warp_sum(c);
        if (lane == 0) wsum[warp] = c;
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < kTileThreads / 32; ++w) tot += wsum[w];
            counts[tix] = static_cast<uint32_t>(tot);
        }
        return;
    }
    // mode 1: ordered compaction (rows 4*tid .. 4*tid+3 per thread for the scan)
    int f[4], fsum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f[k] = cnt[4 * tid + k] & 1;
        fsum += f[k];
    }
    const int incl = warp_incl_scan(fsum, lane);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int base = incl - fsum;
    for (int w = 0; w < warp; ++w) base += wsum[w];
    int pos[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        pos[k] = base;
        base += f[k];
    }
    __syncthreads();
    // publish positions through cnt (flag bit 0 | n << 1 stays in the high bits)
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (f[k]) cnt[4 * tid + k] = (cnt[4 * tid + k] >> 1) | (pos[k] << 16);
    __syncthreads();
    const uint32_t o = a.run_off[tix];
#pragma unroll
    for (int k = 0; k < kMaxSrcRows / kTileThreads; ++k) {
        const int t = tid + k * kTileThreads;
        if (t >= T.n) continue;
        const int c = cnt[t];
        const int n = c & 0xffff;
        if (!n) continue;
        runs[o + (c >> 16)] = make_uint2(s0v[k], static_cast<uint32_t>(t) | (static_cast<uint32_t>(n) << 16));
    }
}

// ------------------------------------------------------------ convolution --
template <typename Acc>
__device__ __forceinline__ Acc fma_t(Acc w, Acc u, Acc acc);
template <>
__device__ __forceinline__ double fma_t<double>(double w, double u, double acc) { return __fma_rn(w, u, acc); }
template <>
__device__ __forceinline__ float fma_t<float>(float w, float u, float acc) { return __fmaf_rn(w, u, acc); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {  // fma.rn.f32x2 (sm_100)
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float to_f(double v) { return __double2float_rn(v); }
__device__ __forceinline__ float to_f(float v) { return v; }

constexpr int kMaxRegions = 32;

// A leaf >= 3 levels coarser than the tile's level: the box offset of its
// first clipped row (z, x at y = by0), nz x nx clipped rows, and nq quads of 4
// box cells from quad q0, filled cooperatively.
template <typename Acc>
struct Region {
    int rbase, nz, nx, q0, nq;
    Acc v;
};

template <typename Acc> struct Vec;
template <> struct Vec<float> {
    using T2 = float2;
    __device__ static void st2(float* p, float v) { *reinterpret_cast<float2*>(p) = make_float2(v, v); }
    __device__ static void st4(float* p, float v) { *reinterpret_cast<float4*>(p) = make_float4(v, v, v, v); }
};
template <> struct Vec<double> {
    using T2 = double2;
    __device__ static void st2(double* p, double v) { *reinterpret_cast<double2*>(p) = make_double2(v, v); }
    __device__ static void st4(double* p, double v) {
        reinterpret_cast<double2*>(p)[0] = make_double2(v, v);
        reinterpret_cast<double2*>(p)[1] = make_double2(v, v);
    }
};

// One 2x2x2 output block (qz, qx, qy) of a box with rows of BY cells whose y
// origin is PADY cells below the tile's: all 8 outputs, taps accumulated in
// the reference's (az, ax, ay) order (convolve.hpp:154-169).  The
// neighbourhood's y window (box index 2qy + PADY - H .. +N) is loaded as
// aligned pairs from the even index at or below it.
// pair(c): the values of box cells c, c + 1 (c even) -- from the box itself
// (k_conv_tile) or through the cells' codes (k_conv_map)
template <typename Acc, int H, int BX, int BY, int PADY, int PL = BX * BY, typename Pair>
__device__ __forceinline__ void apply_block_pairs(Pair pair, const Acc* W, int qz, int qx, int qy, Acc (&acc)[8]) {
    constexpr int K = 2 * H + 1, N = 2 + 2 * H;
    constexpr int Y0 = PADY - H;
    constexpr int YA = Y0 & ~1, SH = Y0 - YA, NP = (SH + N + 1) / 2;
    const int base = (2 * qz) * PL + (2 * qx) * BY + 2 * qy + YA;  // (PL: the plane stride)
    if constexpr (sizeof(Acc) == 4) {
        // FAST: the block's two y-outputs share every tap's weight -> packed
        // fp32x2 FMA (same per-element rounding as two FFMAs)
        float2 acc2[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc2[i] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int nz = N - 1; nz >= 0; --nz) {
            float v[N][N];
#pragma unroll
            for (int nx = 0; nx < N; ++nx) {
                float r[2 * NP];
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) {
                    const float2 t2 = pair(base + nz * PL + nx * BY + 2 * pp);
                    r[2 * pp] = t2.x;
                    r[2 * pp + 1] = t2.y;
                }
#pragma unroll
                for (int ny = 0; ny < N; ++ny) v[nx][ny] = r[SH + ny];
            }
#pragma unroll
            for (int oz = 0; oz < 2; ++oz) {
                const int az = oz + 2 * H - nz;
                if (az < 0 || az > 2 * H) continue;
#pragma unroll
                for (int ox = 0; ox < 2; ++ox)
#pragma unroll
                    for (int ax = 0; ax < K; ++ax)
#pragma unroll
                        for (int ay = 0; ay < K; ++ay) {
                            const float w = W[(az * K + ax) * K + ay];
                            const int vx = ox + 2 * H - ax, vy = 2 * H - ay;
                            acc2[oz * 2 + ox] =
                                ffma2(make_float2(w, w), make_float2(v[vx][vy], v[vx][vy + 1]), acc2[oz * 2 + ox]);
                        }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc[2 * i] = acc2[i].x;
            acc[2 * i + 1] = acc2[i].y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = Acc(0);
        // output (oz, ox, oy) reads neighbourhood cell (oz + 2H - az, ox + 2H - ax, oy + 2H - ay).
        // Rows stream from the top plane and, within a plane, from the last
        // row: each output then sees (az, ax) ascending and ay ascending within
        // a row -- the reference's (az, ax, ay) order -- while only ONE row of
        // doubles is live (a plane of them would cost (2+2H)^2 more registers)
#pragma unroll
        for (int nz = N - 1; nz >= 0; --nz)
#pragma unroll
            for (int nx = N - 1; nx >= 0; --nx) {
                Acc r[2 * NP];
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) {  // exact: every float is a double
                    const float2 t2 = pair(base + nz * PL + nx * BY + 2 * pp);
                    r[2 * pp] = static_cast<Acc>(t2.x);
                    r[2 * pp + 1] = static_cast<Acc>(t2.y);
                }
                // ay outermost: the row's (up to 8) accumulator chains interleave
                // (each still sees ay ascending -- the same order, bit-identical)
#pragma unroll
                for (int ay = 0; ay < K; ++ay)
#pragma unroll
                    for (int oz = 0; oz < 2; ++oz) {
                        const int az = oz + 2 * H - nz;
                        if (az < 0 || az > 2 * H) continue;
#pragma unroll
                        for (int ox = 0; ox < 2; ++ox) {
                            const int ax = ox + 2 * H - nx;
                            if (ax < 0 || ax > 2 * H) continue;
#pragma unroll
                            for (int oy = 0; oy < 2; ++oy)
                                acc[(oz * 2 + ox) * 2 + oy] = fma_t<Acc>(W[(az * K + ax) * K + ay],
                                                                         r[SH + oy + 2 * H - ay],
                                                                         acc[(oz * 2 + ox) * 2 + oy]);
                        }
                    }
            }
    }
}

template <typename Acc, int H, int BX, int BY, int PADY, int PL = BX * BY>
__device__ __forceinline__ void apply_block(const float* S, const Acc* W, int qz, int qx, int qy, Acc (&acc)[8]) {
    apply_block_pairs<Acc, H, BX, BY, PADY, PL>(
        [S](int c) { return *reinterpret_cast<const float2*>(S + c); }, W, qz, qx, qy, acc);
}

// FAST, rank-1 stencil (w = fz (x) fx (x) fy): the same 8 outputs in three
// passes -- y per neighbourhood row, then x, then z -- 2x fewer FMAs than the
// dense 5^3 taps.  Tolerance-matched like every FAST path (the sums are
// reassociated), never used for EXACT.
template <int H, int BX, int BY, int PADY, int PL = BX * BY>
__device__ __forceinline__ void apply_block_sep(const float* S, const float* f, int qz, int qx, int qy,
                                                float (&acc)[8]) {
    constexpr int K = 2 * H + 1, N = 2 + 2 * H, NP = N / 2;
    static_assert((PADY - H) % 2 == 0, "aligned pair loads");
    const float* fz = f;
    const float* fx = f + K;
    const float* fy = f + 2 * K;
    const int base = (2 * qz) * PL + (2 * qx) * BY + 2 * qy + PADY - H;
    float2 o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int nz = 0; nz < N; ++nz) {
        float2 u[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
        for (int nx = 0; nx < N; ++nx) {
            float r[N];
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                const float2 t2 = *reinterpret_cast<const float2*>(S + base + nz * PL + nx * BY + 2 * pp);
                r[2 * pp] = t2.x;
                r[2 * pp + 1] = t2.y;
            }
            float2 t = make_float2(0.0f, 0.0f);  // (oy = 0, 1) reads r[oy + 2H - ay]
#pragma unroll
            for (int ay = 0; ay < K; ++ay)
                t = ffma2(make_float2(fy[ay], fy[ay]), make_float2(r[2 * H - ay], r[2 * H + 1 - ay]), t);
#pragma unroll
            for (int ox = 0; ox < 2; ++ox) {
                const int ax = ox + 2 * H - nx;
                if (ax >= 0 && ax < K) u[ox] = ffma2(make_float2(fx[ax], fx[ax]), t, u[ox]);
            }
        }
#pragma unroll
        for (int oz = 0; oz < 2; ++oz) {
            const int az = oz + 2 * H - nz;
            if (az < 0 || az >= K) continue;
#pragma unroll
            for (int ox = 0; ox < 2; ++ox) o[oz * 2 + ox] = ffma2(make_float2(fz[az], fz[az]), u[ox], o[oz * 2 + ox]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        acc[2 * i] = o[i].x;
        acc[2 * i + 1] = o[i].y;
    }
}

// The block's (up to 8) outputs through the epilogue, batched: all indices
// first, then the epilogue's own loads, then the stores -- so RL's fp64
// divisions (and their operand loads) overlap instead of running one output
// at a time.  Output (oz, ox, oy) of block (qz, qx, qy) is inner row
// r = (2qz + oz) * 8 + 2qx + ox at y = 2qy + oy; its particle is
// ofirst[r] + popc(omask[r] below y).
// Tile-local output rows [lo, hi) a slab-restricted launch may write (a tile
// can straddle two slabs: its other rows belong to the neighbour, whose inputs
// were never exchanged); every row otherwise.
struct RowRange {
    int lo, hi;
};
__device__ __forceinline__ RowRange slab_rows(const TileLaunch& a, int l, int z0) {
    if (l < a.slab_lc) return RowRange{0, kTZ};
    const int sh = a.leaf.l_max - l;
    const int zlo = a.slab_zlo >> sh, zhi = (a.slab_zhi + (1 << sh) - 1) >> sh;
    return RowRange{max(zlo - z0, 0), min(zhi - z0, kTZ)};
}

template <typename Acc>
__device__ __forceinline__ void store_block(const TileLaunch& a, const uint32_t* omask, const uint32_t* ofirst, int qz,
                                            int qx, int qy, const Acc (&acc)[8], RowRange rr) {
    uint32_t idx[8];
    bool ok[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int oz = j >> 2, ox = (j >> 1) & 1, oy = j & 1;
        const int r = (2 * qz + oz) * kTX + 2 * qx + ox, y = 2 * qy + oy;
        const uint32_t m = (2 * qz + oz >= rr.lo && 2 * qz + oz < rr.hi) ? omask[r] : 0u;
        ok[j] = (m >> y) & 1u;
        idx[j] = ofirst[r] + __popc(m & ((1u << y) - 1u));
    }
    if (a.epi.mode == EPI_STORE) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (ok[j]) a.out[idx[j]] = to_f(acc[j]);
    } else if (a.epi.mode == EPI_RL_RATIO) {
        float u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = ok[j] ? __ldg(a.epi.u + idx[j]) : 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (ok[j]) a.out[idx[j]] = rl_ratio(u[j], to_f(acc[j]), a.epi.eps);
    } else {
        float e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = ok[j] ? a.epi.est[idx[j]] : 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (ok[j]) a.epi.est[idx[j]] = __fmul_rn(e[j], to_f(acc[j]));  // deconv.hpp:102
    }
}

// Output i of the launch's epilogue (EpiArgs, internal.cuh).
__device__ __forceinline__ void store_out(const TileLaunch& a, uint32_t i, float r) {
    if (a.epi.mode == EPI_STORE) {
        a.out[i] = r;
    } else if (a.epi.mode == EPI_RL_RATIO) {
        a.out[i] = rl_ratio(__ldg(a.epi.u + i), r, a.epi.eps);
    } else {
        a.epi.est[i] = __fmul_rn(a.epi.est[i], r);  // deconv.hpp:102
    }
}

// (async-copy helpers: common.cuh)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {  // (16-byte aligned both sides)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Ordered compaction of the tile's 2x2x2 output blocks (block-id order, so a
// warp's blocks are mostly y-neighbours: conflict-free pair loads in apply).
template <typename Pred>
__device__ __forceinline__ int compact_blocks(Pred active, uint8_t* blist, int* wcnt) {
    static_assert(kBlocks == 2 * kTileThreads, "two blocks per thread");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kTileThreads / 32;
    bool f[2];
    unsigned bal[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        f[k] = active(k * kTileThreads + tid);
        bal[k] = __ballot_sync(~0u, f[k]);
        if (lane == 0) wcnt[k * NW + warp] = __popc(bal[k]);
    }
    __syncthreads();
    // k = 0 blocks come first: this warp's k = 0 blocks follow the lower warps'
    // k = 0 blocks; its k = 1 blocks follow all k = 0 blocks and the lower warps' k = 1
    int pre = 0, all0 = 0, pre1 = 0, all1 = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        pre += i < warp ? wcnt[i] : 0;
        all0 += wcnt[i];
        pre1 += i < warp ? wcnt[NW + i] : 0;
        all1 += wcnt[NW + i];
    }
    pre1 += all0;
    const int total = all0 + all1;
    const unsigned below = (1u << lane) - 1u;
    if (f[0]) blist[pre + __popc(bal[0] & below)] = static_cast<uint8_t>(tid);
    if (f[1]) blist[pre1 + __popc(bal[1] & below)] = static_cast<uint8_t>(kTileThreads + tid);
    return total;
}

// MAP: instead of convolving, write the tile's gather-map record (k_conv_map):
// the fill runs unchanged on particle CODES (leaf i -> i + 1, interior node
// j -> 2^31 | j, 0 = zero) in place of values, so the map reproduces every
// fill rule -- overlap order, holes, reflect / zero pad -- by construction.
template <typename Acc, int H, bool MAP = false>
__global__ void __launch_bounds__(kTileThreads, sizeof(Acc) == 8 ? (H == 2 ? 3 : 6) : (H == 2 ? 5 : 8))
    k_conv_tile(const __grid_constant__ TileLaunch a) {
    using B = Box<H>;
    using VT = Vec<float>;  // the box holds the particle values themselves (floats) in both modes
    constexpr int K = 2 * H + 1, N = 2 + 2 * H, KW = K * K * K;
    // runs of a tile <= its source rows: 2*(8+2H)^2 level-l leaf + interior rows
    // plus <= 61 + 4 per extra depth coarse rows (<= 325 for H = 1, <= 493 for H = 2)
    constexpr int kRuns = H == 1 ? 384 : 512;
    extern __shared__ __align__(16) unsigned char box_smem[];
    float* S = reinterpret_cast<float*>(box_smem);  // B::NC cells
    // output map: per inner cell the particle's offset from its row's first
    // particle in the box (0xff: no output particle); per inner row that index
    __shared__ __align__(16) uint8_t omap[kTZ * kTX * kTY];
    __shared__ uint32_t orow[kTZ * kTX];
    __shared__ Acc W[KW];
    __shared__ float SF[3 * K];  // FAST 5^3, rank-1 stencil: its factors (as k_conv_map)
    __shared__ uint8_t blist[kBlocks];
    __shared__ int nreg;
    __shared__ Region<float> reg[kMaxRegions];
    __shared__ int rpre[kMaxRegions + 1];
    __shared__ SrcTable T;
    __shared__ uint32_t rinfo[kRuns];  // packed row geometry
    __shared__ uint32_t rsrc[kRuns];   // global index of the row's first particle in the box
    __shared__ uint16_t rslot[kRuns];  // run -> source-row slot
    __shared__ int8_t rorid[kRuns];    // run -> inner output row of the tile (-1: none)
    __shared__ int roff[kRuns + 1];    // flattened offsets; roff[kRuns] = total
    __shared__ uint16_t rpad[MAP ? kRuns + 1 : 1];  // MAP: each run's first F slot (whole 16-byte chunks)
    __shared__ int wsum[kTileThreads / 32];
    __shared__ int wcnt[2 * kTileThreads / 32];
    __shared__ __align__(16) uint16_t rid[kMaxFlat];  // run of each flattened particle (current chunk)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = seg_of(a.seg_end, a.n_levels, blockIdx.x);
    const int l = a.lvl[s];
    const LevelG g = a.leaf.g[l];
    const uint32_t tix = a.tile_base + blockIdx.x + a.seg_shift[s];
    const Geo G = make_geo<H>(l, a.tiles[tix], a.tdim[s][1], a.tdim[s][2], g);
    if (l >= a.slab_lc) {  // slab decomposition: only tiles touching this slab's planes
        const int sh = a.leaf.l_max - l;
        if ((G.z0 + kTZ) << sh <= a.slab_zlo || G.z0 << sh >= a.slab_zhi) return;
    }
    const int meta = a.meta[tix];
    const int tree = (l >= a.tree_lmin && l <= a.tree_lmax) ? 1 : 0;

    // ---- init: weights, output map, (holes only) zeroed box, source table
    constexpr bool kSepOk = H == 2 && sizeof(Acc) == 4 && !MAP;
    const bool sep = kSepOk && a.sep[s] != nullptr;
    if (kSepOk && sep && tid < 3 * K) SF[tid] = a.sep[s][tid];
    for (int i = tid; i < KW; i += kTileThreads)
        W[i] = sizeof(Acc) == 8 ? static_cast<Acc>(a.wd[a.woff[s] + i]) : static_cast<Acc>(a.wf[a.woff[s] + i]);
    {
        uint4* om = reinterpret_cast<uint4*>(omap);
        for (int i = tid; i < kTZ * kTX * kTY / 16; i += kTileThreads) om[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    if (MAP || (meta & kMetaHoles))  // (a map record must hold no stale codes)
        for (int i = tid; i < B::NC; i += kTileThreads) S[i] = MAP ? __uint_as_float(MapBox<H>::ZERO) : 0.0f;
    if (tid == 0) {
        nreg = 0;
        make_src_table<H>(G, meta & kMetaDepth, tree, T);
    }
    __syncthreads();

    // ---- rows: the tile's precomputed non-empty source runs (k_tile_runs) and
    // their packed box geometry, one thread per run:
    //   rinfo = d | is_tree << 5 | inner << 6 | (nz-1) << 7 | (nx-1) << 11 | rbase << 15
    //   rbase = box offset of the row's first clipped (z, x) at y = by0
    const uint32_t run0 = a.run_off[tix];
    const int nruns = min(static_cast<int>(a.run_off[tix + 1] - run0), kRuns);
    {
#pragma unroll
        for (int k = 0; k < kRuns / kTileThreads; ++k) {
            const int j = tid + k * kTileThreads;
            int n = 0;
            if (j < nruns) {
                const uint2 e = __ldg(a.runs + run0 + j);
                const int t = static_cast<int>(e.y & 0xffff);
                n = static_cast<int>(e.y >> 16);
                if (MAP) n |= static_cast<int>(((e.x & 3u) + n + 3) & ~3u) << 16;  // (and its F slots, one scan)
                RowJob J;
                resolve_row<H, false>(a, G, T, t, J);  // geometry only
                const uint32_t rbase = static_cast<uint32_t>(J.r00 + G.by0);
                rinfo[j] = static_cast<uint32_t>(J.d) | (J.is_tree << 5) | (J.inner << 6) |
                           (static_cast<uint32_t>(J.zB - J.zA - 1) << 7) |
                           (static_cast<uint32_t>(J.xB - J.xA - 1) << 11) | (rbase << 15);
                rsrc[j] = e.x;
                rslot[j] = static_cast<uint16_t>(t);
                rorid[j] = static_cast<int8_t>(J.inner ? J.obase : -1);
                if (J.inner) orow[J.obase] = e.x;
            }
            roff[j] = n;
        }
        __syncthreads();
        // exclusive scan over runs (thread tid owns runs 4*tid .. 4*tid+3)
        int cnt[kRuns / kTileThreads];
#pragma unroll
        for (int k = 0; k < kRuns / kTileThreads; ++k) cnt[k] = roff[kRuns / kTileThreads * tid + k];
        __syncthreads();
        int sum = 0;
#pragma unroll
        for (int k = 0; k < kRuns / kTileThreads; ++k) sum += cnt[k];
        const int incl = warp_incl_scan(sum, lane);
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int base = incl - sum;
        for (int w = 0; w < warp; ++w) base += wsum[w];
#pragma unroll
        for (int k = 0; k < kRuns / kTileThreads; ++k) {
            const int j = kRuns / kTileThreads * tid + k;
            roff[j] = MAP ? base & 0xffff : base;
            if (MAP) rpad[j] = static_cast<uint16_t>(base >> 16);
            base += cnt[k];
        }
        if (tid == kTileThreads - 1) {
            roff[kRuns] = MAP ? base & 0xffff : base;
            if (MAP) rpad[kRuns] = static_cast<uint16_t>(base >> 16);
        }
    }
    __syncthreads();

    // ---- fill: one thread per source particle
    const uint32_t flat0 = MAP ? tix * a.flat_cap : 0;
    int chunk0 = 0;  // first flattened index of the current rid chunk
    auto put = [&](int p) {
        const int t = rid[p - chunk0];
        const uint32_t info = rinfo[t];
        const int d = info & 31;
        const bool is_tree = (info >> 5) & 1;
        const int rbase = static_cast<int>(info >> 15);
        const uint32_t gi = rsrc[t] + static_cast<uint32_t>(p - roff[t]);
        const int yy = __ldg((is_tree ? a.tree.y : a.leaf.y) + gi);
        float v;
        if constexpr (MAP) {  // byte offset into F of the source's slot (its run's chunks, phase b mod 4)
            v = __uint_as_float(static_cast<uint32_t>(4 * (kFlat0 + rpad[t] + (rsrc[t] & 3u) + (p - roff[t]))));
        } else {
            v = __ldg((is_tree ? a.tval : a.val) + gi);
        }
        if (d == 0) {
            S[rbase - G.by0 + yy] = v;
            const int orid = rorid[t];  // inner output row of the tile, or -1
            if (orid >= 0 && static_cast<unsigned>(yy - G.y0) < static_cast<unsigned>(kTY))
                omap[orid * kTY + yy - G.y0] = static_cast<uint8_t>(p - roff[t]);  // orow[orid] = rsrc[t]
            return;
        }
        const int nzr = ((info >> 7) & 15) + 1, nxr = ((info >> 11) & 15) + 1;
        float* p0 = S + rbase - G.by0 + (yy << d);
        if (d == 1) {
            VT::st2(p0, v);
            if (nxr == 2) VT::st2(p0 + B::BY, v);
            if (nzr == 2) {
                VT::st2(p0 + B::BX * B::BY, v);
                if (nxr == 2) VT::st2(p0 + B::BX * B::BY + B::BY, v);
            }
        } else if (d == 2) {
#pragma unroll
            for (int z = 0; z < 4; ++z)
#pragma unroll
                for (int x = 0; x < 4; ++x)
                    if (z < nzr && x < nxr) VT::st4(p0 + (z * B::BX + x) * B::BY, v);
        } else {
            const int c0 = max((yy << d) - G.by0, 0), c1 = min(((yy + 1) << d) - G.by0, B::BY);
            const int slot = atomicAdd(&nreg, 1);
            if (slot < kMaxRegions) {
                reg[slot] = Region<float>{rbase, nzr, nxr, c0 >> 2, (c1 - c0) >> 2, v};
            } else {
                for (int z = 0; z < nzr; ++z)
                    for (int x = 0; x < nxr; ++x)
                        for (int c = c0; c < c1; c += 4) VT::st4(S + rbase + (z * B::BX + x) * B::BY + c, v);
            }
        }
    };
    // cooperative fill of the queued regions (leaves >= 3 levels coarser)
    auto fill_regions = [&]() {
        __syncthreads();
        const int n = min(nreg, kMaxRegions);
        if (n == 0) return;
        if (warp == 0) {
            static_assert(kMaxRegions == 32, "one region per lane");
            const int c0 = lane < n ? reg[lane].nz * reg[lane].nx * reg[lane].nq : 0;
            const int incl = warp_incl_scan(c0, lane);
            rpre[lane] = incl - c0;
            if (lane == 31) rpre[kMaxRegions] = incl;
        }
        __syncthreads();
        const int total = rpre[kMaxRegions];
        for (int c = tid; c < total; c += kTileThreads) {
            int lo = 0, hi = n - 1;  // region of quad c
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (rpre[mid] <= c) lo = mid; else hi = mid - 1;
            }
            const Region<float> R = reg[lo];
            const int j = c - rpre[lo];
            // small-integer quotients through fast float division: the 0.5 margin
            // dwarfs its 2-ulp error for j < 2^12, divisors <= 16
            const int row = __float2int_rz(__fdividef(j + 0.5f, static_cast<float>(R.nq))), qd = j - row * R.nq;
            const int zz = __float2int_rz(__fdividef(row + 0.5f, static_cast<float>(R.nx))), xx = row - zz * R.nx;
            VT::st4(S + R.rbase + (zz * B::BX + xx) * B::BY + 4 * (R.q0 + qd), R.v);
        }
        __syncthreads();
        if (tid == 0) nreg = 0;
    };
    // particles [q0, q1) of the flattened numbering, in chunks of kMaxFlat
    auto scatter_range = [&](int r0, int r1) {
        const int q0 = roff[r0], q1 = roff[r1];
        for (int c0 = q0; c0 < q1; c0 += kMaxFlat) {
            const int c1 = min(c0 + kMaxFlat, q1);
            for (int t = r0 + tid; t < r1; t += kTileThreads) {
                const int lo = max(roff[t], c0), hi = min(roff[t + 1], c1);
                for (int q = lo; q < hi; ++q) rid[q - c0] = static_cast<uint16_t>(t);
            }
            __syncthreads();
            chunk0 = c0;
            for (int q = c0 + tid; q < c1; q += kTileThreads) put(q);
            __syncthreads();
        }
    };
    if (!(meta & kMetaOverlap)) {
        scatter_range(0, nruns);
        fill_regions();
    } else {
        // reference order: level l, l-1, ..., l-D, then interior nodes (last writer
        // wins); runs are in row-slot order, so each phase is a run range
        int j0 = 0;
        for (int ph = 0; ph <= T.D + 1; ++ph) {
            const int t1 = ph <= T.D ? T.base[ph + 1] : T.n;
            int j1 = j0;
            while (j1 < nruns && rslot[j1] < t1) ++j1;
            scatter_range(j0, j1);
            fill_regions();
            j0 = j1;
        }
    }
    __syncthreads();

    // ---- pad: out-of-domain box cells within H of the domain
    if (G.z0 - H < 0 || G.x0 - H < 0 || G.y0 - H < 0 || G.z0 + kTZ + H > g.zd || G.x0 + kTX + H > g.xd ||
        G.y0 + kTY + H > g.yd) {
        for (int r = tid; r < B::NR; r += kTileThreads) {
            const int bz = r / B::BX, bx = r - bz * B::BX;
            const int zz = G.bz0 + bz, xx = G.bx0 + bx;
            if (zz >= g.zd + H || xx >= g.xd + H) continue;  // read by no output
            const bool row_out = zz < 0 || zz >= g.zd || xx < 0 || xx >= g.xd;
            const int rz = reflect_dev(zz, g.zd) - G.bz0, rx = reflect_dev(xx, g.xd) - G.bx0;
            float* dst = S + r * B::BY - G.by0;
            const float* src = S + (rz * B::BX + rx) * B::BY - G.by0;
            for (int yy = G.y0 - H; yy < min(G.y0 + kTY + H, g.yd + H); ++yy) {
                const bool out = row_out || yy < 0 || yy >= g.yd;
                if (!out) continue;
                dst[yy] = a.pad == APRGPU_PAD_ZERO ? (MAP ? __uint_as_float(MapBox<H>::ZERO) : 0.0f)
                                                   : src[reflect_dev(yy, g.yd)];
            }
        }
        __syncthreads();
    }

    if constexpr (MAP) {
        using M = MapBox<H>;
        uint32_t* rec = a.map[s] + static_cast<size_t>(tix - a.map_base[s]) * M::REC;
        const int nchunks = ((rpad[nruns] >> 2) + 3) & ~3;  // (== k_tile_nflat)
        if (tid == 0) {
            if (roff[nruns] > M::NC || nchunks > kMaxChunks) atomicOr(a.map_overflow, 1);
            atomicMax(a.map_maxg, nchunks);
        }
        if (nchunks <= kMaxChunks)  // the chunk list: one u32 per 16-byte chunk of every run
            for (int t = tid; t < nruns; t += kTileThreads) {
                const bool tr = (rinfo[t] >> 5) & 1u;
                const uint32_t b0 = rsrc[t] & ~3u, lim = tr ? a.n_tree : a.n_leaf;
                for (int c = rpad[t] >> 2; c < rpad[t + 1] >> 2; ++c) {
                    const uint32_t first = b0 + 4u * (c - (rpad[t] >> 2));
                    a.flat[flat0 + c] = first | (tr ? kChunkTree : 0u) | (first + 4 > lim ? kChunkTail : 0u);
                }
            }
        auto code = [&](int c) -> uint32_t {
            const int r = c / M::BY;
            return __float_as_uint(S[r * B::BY + (c - r * M::BY) + (kPadY - H)]);
        };
        for (int u = tid; u < M::CW; u += kTileThreads) rec[M::CODE0 + u] = code(2 * u) | code(2 * u + 1) << 16;
        if (tid < kTZ * kTX) {  // per inner row: output mask over y0 .. y0+31 and the first output's index
            uint32_t m = 0;
            int first = -1;
            for (int y = 0; y < kTY; ++y) {
                const int o = omap[tid * kTY + y];
                if (o == 0xff) continue;
                m |= 1u << y;
                if (first < 0) first = o;
            }
            rec[M::MASK0 + tid] = m;
            rec[M::MASK0 + kTZ * kTX + tid] = m ? orow[tid] + first : 0u;
        }
        if (tid == 0) {
            rec[M::W_NLEAF] = static_cast<uint32_t>(nchunks);
            // the active 2x2x2 blocks, dealt round-robin over their bank keys so
            // that a warp's 32 blocks start on as many distinct banks as possible
            // (every tap load of the apply shifts all lanes alike)
            uint8_t keyed[kBlocks], bkey[kBlocks];  // active blocks and their keys, then sorted by key
            int nbk[M::NK] = {}, start[M::NK];
            int total = 0;
            for (int b = 0; b < kBlocks; ++b) {
                const int qz = b / (kBlocks / 4), qx = (b / (kTY / 2)) & 3, qy = b & (kTY / 2 - 1);
                const uint8_t* o = omap + ((2 * qz) * kTX + 2 * qx) * kTY + 2 * qy;
                const unsigned m = *reinterpret_cast<const uint16_t*>(o) & *reinterpret_cast<const uint16_t*>(o + kTY) &
                                   *reinterpret_cast<const uint16_t*>(o + kTX * kTY) &
                                   *reinterpret_cast<const uint16_t*>(o + kTX * kTY + kTY);
                if (m == 0xffffu) continue;
                const int key = H == 1 ? (((2 * qz) * M::BX + 2 * qx) * (M::BY / 2) + qy) % M::NK
                                       : ((2 * qz) * (M::PL / 2) + qx * M::BY + qy) % M::NK;
                keyed[total] = static_cast<uint8_t>(b);
                bkey[total++] = static_cast<uint8_t>(key);
                ++nbk[key];
            }
            for (int k = 0, acc = 0; k < M::NK; ++k) {
                start[k] = acc;
                acc += nbk[k];
            }
            uint8_t sorted[kBlocks];
            int fill[M::NK];
            for (int k = 0; k < M::NK; ++k) fill[k] = start[k];
            for (int i = 0; i < total; ++i) sorted[fill[bkey[i]]++] = keyed[i];
            uint8_t* lst = reinterpret_cast<uint8_t*>(rec + M::W_BLK);
            int n = 0;
            for (int r = 0; n < total; ++r)
                for (int k = 0; k < M::NK; ++k)
                    if (r < nbk[k]) lst[n++] = sorted[start[k] + r];
            for (int i = n; i < kBlocks; ++i) lst[i] = 0;
            rec[M::W_NBLK] = static_cast<uint32_t>(total);
            rec[M::W_NBLK + 1] = rec[M::W_NBLK + 2] = 0u;
        }
        return;
    }

    // ---- compact the 2x2x2 blocks that hold output particles
    const int nb = compact_blocks(
        [&](int b) {
            const int qz = b / (kBlocks / 4), qx = (b / (kTY / 2)) & 3, qy = b & (kTY / 2 - 1);
            const uint8_t* o = omap + ((2 * qz) * kTX + 2 * qx) * kTY + 2 * qy;
            const unsigned m = *reinterpret_cast<const uint16_t*>(o) & *reinterpret_cast<const uint16_t*>(o + kTY) &
                               *reinterpret_cast<const uint16_t*>(o + kTX * kTY) &
                               *reinterpret_cast<const uint16_t*>(o + kTX * kTY + kTY);
            return m != 0xffffu;
        },
        blist, wcnt);
    __syncthreads();

    // ---- apply: one thread per active block, 8 outputs
    const RowRange rr = slab_rows(a, l, G.z0);
    for (int q = tid; q < nb; q += kTileThreads) {
        const int bidx = blist[q];
        const int qz = bidx / (kBlocks / 4), qx = (bidx / (kTY / 2)) & 3, qy = bidx & (kTY / 2 - 1);
        Acc acc[8];
        if constexpr (kSepOk) {
            if (sep)
                apply_block_sep<H, B::BX, B::BY, kPadY>(S, SF, qz, qx, qy, acc);
            else
                apply_block<Acc, H, B::BX, B::BY, kPadY>(S, W, qz, qx, qy, acc);
        } else {
            apply_block<Acc, H, B::BX, B::BY, kPadY>(S, W, qz, qx, qy, acc);
        }
        const uint8_t* o = omap + ((2 * qz) * kTX + 2 * qx) * kTY + 2 * qy;
#pragma unroll
        for (int oz = 0; oz < 2; ++oz)
#pragma unroll
            for (int ox = 0; ox < 2; ++ox)
#pragma unroll
                for (int oy = 0; oy < 2; ++oy) {
                    const int off = o[(oz * kTX + ox) * kTY + oy];
                    if (off == 0xff || 2 * qz + oz < rr.lo || 2 * qz + oz >= rr.hi) continue;
                    store_out(a, orow[(2 * qz + oz) * kTX + 2 * qx + ox] + off, to_f(acc[(oz * 2 + ox) * 2 + oy]));
                }
    }
}

// Convolution of one tile through its resident gather map: the box is one
// streamed pass over the record (4 codes per 16-byte load) with a gather of
// each code's value, then the same block-compacted apply as k_conv_tile.
// Results are bit-identical to k_conv_tile's (same box contents, same taps).
template <typename Acc, int H, int NT = kTileThreads>
__global__ void __launch_bounds__(NT, (sizeof(Acc) == 8 ? (H == 2 ? 4 : 8) : (H == 2 ? 5 : 8)) * 128 / NT)
    k_conv_map(const __grid_constant__ TileLaunch a) {
    using M = MapBox<H>;
    constexpr int K = 2 * H + 1, KW = K * K * K;
    // dynamic: the tile's map record, then the zero + its flattened source values
    extern __shared__ __align__(16) unsigned char map_smem[];
    uint32_t* Mb = reinterpret_cast<uint32_t*>(map_smem);
    // F: the staged source values.  FAST 5^3 keeps the box S between the
    // header and F (the codes arrive at S's start and are expanded over in
    // place: shared memory bounds its occupancy); EXACT 5^3 (register-bound)
    // puts S after F and expands in one pass
    constexpr bool kInPlace = H == 2 && sizeof(Acc) == 4;
    float* F = reinterpret_cast<float*>(Mb + (kInPlace ? M::HDR + M::SN : M::REC));
    __shared__ __align__(8) uint64_t mbar;
    __shared__ Acc W[KW];
    __shared__ float SF[3 * K];  // FAST 5^3, rank-1 stencil: its factors
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = seg_of(a.seg_end, a.n_levels, blockIdx.x);
    constexpr bool kSepOk = H == 2 && sizeof(Acc) == 4;
    const bool sep = kSepOk && a.sep[s] != nullptr;
    if (kSepOk && sep && tid < 3 * K) SF[tid] = a.sep[s][tid];
    const int l = a.lvl[s];
    const uint32_t tix = a.tile_base + blockIdx.x + a.seg_shift[s];
    const uint32_t* rec = a.map[s] + static_cast<size_t>(tix - a.map_base[s]) * M::REC;
    // a slab launch's tiles straddling the slab: the row range needs the tile's
    // z (a load); other launches decide nothing from it
    RowRange rr{0, kTZ};
    if (l >= a.slab_lc) {
        const int z0 = static_cast<int>(a.tiles[tix] / (static_cast<uint32_t>(a.tdim[s][1]) * a.tdim[s][2])) * kTZ;
        rr = slab_rows(a, l, z0);
        if (rr.lo >= rr.hi) return;  // slab decomposition: no row of this tile is in the slab
    }
    // the record and the tile's chunk list stream in by two bulk copies, both
    // issued before the CTA loads anything: the lists sit at a fixed stride
    // (tix * flat_cap) and are copied at the launch's largest extent (map_ng
    // entries; the tile's own count arrives with the record)
    const int nf = kFlat0 + 4 * a.map_ng;  // F floats of this launch
    // the staged chunk list: after F -- or, for EXACT 5^3, inside the box S it
    // precedes (S is written only after the gather).  3^3 and FAST 5^3: in the
    // tail of F's region, which the gather then fills from the front -- a
    // chunk's copy can only land on list entries at or below its own, read in
    // its round or before (rounds below): 4 bytes per chunk of shared memory
    // less per CTA
    constexpr bool kListInBox = H == 2 && !kInPlace;
    const bool list_in_f = (H == 1 || kInPlace) && a.list_in_f;
    uint32_t* Gs = reinterpret_cast<uint32_t*>(F + nf) - (list_in_f ? a.map_ng : 0);
    // the list's head (most tiles' whole list) comes with the record; a longer
    // list's rest follows once the record has brought its count
    const uint32_t* lst = a.flat + static_cast<size_t>(tix) * a.flat_cap;
    // (5^3 lists are longer: most would need the second copy, so they come whole)
    const uint32_t head = H == 1 ? min(static_cast<uint32_t>(a.map_ng), kListHead) : static_cast<uint32_t>(a.map_ng);
    if (tid == 0) {
        mbar_init(&mbar, 1);
        mbar_expect(&mbar, (M::REC + head) * 4);  // (arrive.expect_tx)
        // (records and lists are read once per pass: evict-first, leaving L2 to
        // the source values neighbouring tiles re-read)
        if (a.l2hint) {
            const uint64_t pol = l2_evict_first();
            bulk_copy_hint(Mb, rec, M::REC * 4, &mbar, pol);
            if (head) bulk_copy_hint(Gs, lst, head * 4, &mbar, pol);
        } else {
            bulk_copy(Mb, rec, M::REC * 4, &mbar);
            if (head) bulk_copy(Gs, lst, head * 4, &mbar);
        }
    }
    if (tid < kFlat0) F[tid] = 0.0f;
    for (int i = tid; i < KW; i += NT)
        W[i] = sizeof(Acc) == 8 ? static_cast<Acc>(a.wd[a.woff[s] + i]) : static_cast<Acc>(a.wf[a.woff[s] + i]);
    __syncthreads();  // (the barrier's init is visible)
    mbar_wait(&mbar, 0);
    // the chunks to gather: the record's count (3^3: the placement pass drops
    // chunks no active block reads, so it can be below the list's extent)
    const uint32_t ng = Mb[M::W_NLEAF];
    if (ng > head) {  // (uniform) the list's rest, in whole 16-byte units (the entries past ng are zeros)
        if (tid == 0) {
            const uint32_t n4 = (ng + 3u) & ~3u;
            mbar_expect(&mbar, (n4 - head) * 4);
            if (a.l2hint) bulk_copy_hint(Gs + head, lst + head, (n4 - head) * 4, &mbar, l2_evict_first());
            else bulk_copy(Gs + head, lst + head, (n4 - head) * 4, &mbar);
        }
        mbar_wait(&mbar, 1);
    }
    // every source value copied once: one 16-byte copy per chunk (a warp's
    // chunks are mostly consecutive 16-byte pieces of one run: coalesced);
    // the array's tail chunk copies only its valid elements
    auto gather = [&](uint32_t c, uint32_t e) {
        const float* src = ((e & kChunkTree) ? a.tval : a.val) + (e & kChunkIdx);
        float* dst = F + kFlat0 + 4 * c;
        if (!(e & kChunkTail) && a.aligned16) {
            cp_async16(dst, src);
        } else {
            const uint32_t lim = (e & kChunkTree) ? a.n_tree : a.n_leaf;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                if ((e & kChunkIdx) + k < lim) cp_async4(dst + k, src + k);
        }
    };
    if (list_in_f) {
        // rounds of 4 * NT chunks: every entry a round's copies may overwrite
        // (at or below their own) is read before its barrier
        constexpr int KR = 4;
        for (uint32_t c0 = 0; c0 < ng; c0 += KR * NT) {  // (uniform trip count)
            uint32_t e[KR];
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const uint32_t c = c0 + k * NT + tid;
                e[k] = c < ng ? Gs[c] : 0u;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const uint32_t c = c0 + k * NT + tid;
                if (c < ng) gather(c, e[k]);
            }
        }
    } else {
        for (uint32_t c = tid; c < ng; c += NT) gather(c, Gs[c]);
    }
    cp_async_wait_all();
    __syncthreads();
    // 5^3 (H = 2): each box cell is read by ~3x more taps than at 3^3, so the
    // box is expanded once (8 cells per thread) and the apply reads it; 3^3
    // reads cells straight through their codes.  The expansion writes S over
    // the codes it reads (S[c] lands on code word c, which holds cells 2c and
    // 2c+1): descending chunks of one 8-cell group per thread, each chunk's
    // codes and values read before its writes, never clobber a code still to
    // be read -- so the box needs no storage of its own beyond the codes'.
    constexpr bool kBox = H == 2;
    float* S = kInPlace ? reinterpret_cast<float*>(Mb + M::HDR) : F + nf + (kListInBox ? 0 : a.map_ng);  // (SN floats)
    if constexpr (kBox) {
        const uint4* C4 = reinterpret_cast<const uint4*>(Mb + M::CODE0);
        float4* S4 = reinterpret_cast<float4*>(S);
        const char* Fb = reinterpret_cast<const char*>(F);
        auto at = [Fb](uint32_t off) { return *reinterpret_cast<const float*>(Fb + off); };
        constexpr int NG = M::NC / 8;
        static_assert(M::NC % 8 == 0, "8-cell groups");
        constexpr int kGPlane = M::BX * M::BY / 8;  // 8-cell groups per plane
        static_assert(M::BX * M::BY % 8 == 0 && M::PL == M::BX * M::BY + 4, "float4-padded planes");
        auto group = [&](int g, float4& v0, float4& v1) {
            const uint4 c = C4[g];
            v0 = make_float4(at(c.x & 0xffffu), at(c.x >> 16), at(c.y & 0xffffu), at(c.y >> 16));
            v1 = make_float4(at(c.z & 0xffffu), at(c.z >> 16), at(c.w & 0xffffu), at(c.w >> 16));
        };
        if constexpr (kInPlace) {
#pragma unroll 1
            for (int j = (NG - 1) / NT; j >= 0; --j) {
                const int g = j * NT + tid;
                float4 v0, v1;
                if (g < NG) group(g, v0, v1);
                __syncthreads();
                if (g < NG) {  // (one float4 of padding per plane)
                    S4[2 * g + g / kGPlane] = v0;
                    S4[2 * g + 1 + g / kGPlane] = v1;
                }
            }
        } else {
            for (int g = tid; g < NG; g += NT) {
                float4 v0, v1;
                group(g, v0, v1);
                S4[2 * g + g / kGPlane] = v0;
                S4[2 * g + 1 + g / kGPlane] = v1;
            }
        }
        __syncthreads();
    }
    const uint32_t* omask = Mb + M::MASK0;
    const uint32_t* ofirst = omask + kTZ * kTX;
    // the active blocks in their bank-interleaved order (map build)
    const int nb = static_cast<int>(Mb[M::W_NBLK]);
    const uint8_t* blist = reinterpret_cast<const uint8_t*>(Mb + M::W_BLK);
    for (int q = tid; q < nb; q += NT) {
        const int bidx = blist[q];
        const int qz = bidx / (kBlocks / 4), qx = (bidx / (kTY / 2)) & 3, qy = bidx & (kTY / 2 - 1);
        Acc acc[8];
        if constexpr (kBox) {
            if constexpr (kSepOk) {
                if (sep)
                    apply_block_sep<H, M::BX, M::BY, H, M::PL>(S, SF, qz, qx, qy, acc);
                else
                    apply_block<Acc, H, M::BX, M::BY, H, M::PL>(S, W, qz, qx, qy, acc);
            } else {
                apply_block<Acc, H, M::BX, M::BY, H, M::PL>(S, W, qz, qx, qy, acc);
            }
        } else {  // box cells straight from their codes: no box is materialised
            apply_block_pairs<Acc, H, M::BX, M::BY, H>(
                [Mb](int c) {  // codes are byte offsets into F, which sits at a fixed offset
                    const uint32_t w = Mb[c >> 1];
                    const char* Fb = reinterpret_cast<const char*>(Mb + M::REC);
                    return make_float2(*reinterpret_cast<const float*>(Fb + (w & 0xffffu)),
                                       *reinterpret_cast<const float*>(Fb + (w >> 16)));
                },
                W, qz, qx, qy, acc);
        }
        store_block(a, omask, ofirst, qz, qx, qy, acc, rr);
    }
}

// Bank-aware placement of a 3^3 tile's staged chunks in F (run once per map
// build, after it).  The apply's source loads (k_conv_map: one warp-load per
// neighbourhood cell of its 32 blocks) gather from F through the codes, and a
// warp-load costs as many shared-memory wavefronts as the most-requested bank
// holds distinct words; the build's F order leaves those banks as good as
// random.  A chunk's bank is fixed by its F position mod 8 (its colour), and
// permuting the chunks WITHIN each aligned group of 32 list entries changes
// nothing else: a warp's gather copies the same 32 chunks (same cache lines,
// lanes reordered) and the list-in-F rounds keep their invariant.  So every
// value-load instruction of the tile's apply is enumerated, and the chunks
// take colours greedily -- in steps: the r-th most-referenced chunk of each
// group of one half of the groups picks, against the histogram as it stood at
// the step's start, the colour (within its group's remaining capacity) that
// raises those instructions' bank maxima least; then the step's picks are
// added.  The list and the codes
// are rewritten to the chosen positions.  Only interior tiles (no padding
// cells) are permuted: their codes and blocks, and so this deterministic
// placement, are the same under both pad modes, which share one chunk list.
// Results are bit-identical (the same values, elsewhere in F).
// 5^3 (H = 2): the same for the loads of the box expansion (every box cell, 8
// consecutive cells per lane; the apply then reads the expanded box).
constexpr int kPlaceMaxRounds = 8;                        // kBlocks / 32 warp-rounds of apply blocks
constexpr int kPlaceMaxI = 64 * kPlaceMaxRounds;          // 3^3: 64 value loads per warp-round (5^3: 8 per round, 21 rounds)
constexpr int kPlaceWarps = 16;
template <int H>
__host__ __device__ constexpr int place_smem(int nch) {  // (per-chunk arrays after the fixed ones)
    return 2 * MapBox<H>::NC + kBlocks + kPlaceMaxI * 32 + 4 * kPlaceMaxI + 2 * kPlaceMaxI * 32 + 4 * (nch + 1) +
           4 * nch + 2 * nch + 2 * nch + 2 * nch + 2 * nch + 11 * (nch / 32 + 1) + 32;
}

template <int H>
__global__ void __launch_bounds__(32 * kPlaceWarps) k_map_place(const __grid_constant__ TileLaunch a,
                                                                const uint32_t* __restrict__ list_in) {
    using M = MapBox<H>;
    static_assert(H == 1 || (M::NC / 8 + 31) / 32 * 8 <= kPlaceMaxI, "5^3 expansion loads");
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char psm[];
    uint16_t* C = reinterpret_cast<uint16_t*>(psm);                       // the codes (byte offsets into F)
    uint8_t* BL = psm + 2 * M::NC;                                        // active blocks
    uint32_t* Hh = reinterpret_cast<uint32_t*>(BL + kBlocks);             // [I][32] u8: distinct words per bank
    uint32_t* cur = Hh + kPlaceMaxI * 8;                                  // [I] bank maximum
    uint16_t* refs = reinterpret_cast<uint16_t*>(cur + kPlaceMaxI);        // per chunk: (instruction << 2 | word)
    uint32_t* roff = reinterpret_cast<uint32_t*>(refs + kPlaceMaxI * 32);  // [nch + 1]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int s = seg_of(a.seg_end, a.n_levels, blockIdx.x);
    const int l = a.lvl[s];
    const uint32_t tix = a.tile_base + blockIdx.x + a.seg_shift[s];
    uint32_t* rec = a.map[s] + static_cast<size_t>(tix - a.map_base[s]) * M::REC;
    const uint32_t f0 = tix * a.flat_cap;
    const int nch = static_cast<int>(a.flat_off[tix + 1] - a.flat_off[tix]);
    const int nb = static_cast<int>(rec[M::W_NBLK]);
    const LevelG g = a.leaf.g[l];
    const Geo G = make_geo<H>(l, a.tiles[tix], a.tdim[s][1], a.tdim[s][2], g);
    const bool interior = G.z0 - H >= 0 && G.x0 - H >= 0 && G.y0 - H >= 0 && G.z0 + kTZ + H <= g.zd &&
                          G.x0 + kTX + H <= g.xd && G.y0 + kTY + H <= g.yd;
    if (!interior || nb == 0 || nch <= 8) {  // the build's order
        for (int c = threadIdx.x; c < nch; c += blockDim.x) a.flat[f0 + c] = list_in[f0 + c];
        return;
    }
    uint32_t* cnt = roff + nch + 1;
    uint16_t* order = reinterpret_cast<uint16_t*>(cnt + nch);  // per group: its chunks, most-referenced first
    uint16_t* npos = order + nch;
    uint16_t* kidx = npos + nch;  // 3^3: a chunk's position among the kept ones (0xffff: dropped)
    uint16_t* kc = kidx + nch;    // the kept chunks in order
    uint16_t* pick = kc + nch;    // per group: this round's chunk and colour
    uint8_t* cap = reinterpret_cast<uint8_t*>(pick + ((nch + 31) >> 5));  // [group][colour] positions left
    uint8_t* pk = cap + 8 * ((nch + 31) >> 5);
    __shared__ int nkeep_s;
    constexpr int NG8 = M::NC / 8;                           // 5^3: the expansion's 8-cell groups
    const int nwr = H == 1 ? (nb + 31) >> 5 : (NG8 + 31) >> 5, ni = (H == 1 ? 64 : 8) * nwr;
    for (int w = threadIdx.x; w < M::CW; w += blockDim.x) reinterpret_cast<uint32_t*>(C)[w] = rec[M::CODE0 + w];
    for (int q = threadIdx.x; q < nb; q += blockDim.x) BL[q] = reinterpret_cast<const uint8_t*>(rec + M::W_BLK)[q];
    for (int i = threadIdx.x; i < ni * 8; i += blockDim.x) Hh[i] = 0;
    for (int c = threadIdx.x; c < nch; c += blockDim.x) cnt[c] = 0;
    __syncthreads();
    auto hinc = [&](int i, uint32_t b) {  // one more distinct word in bank b of load i; returns the new count
        const uint32_t sh = 8 * (b & 3);
        return ((atomicAdd(&Hh[i * 8 + (b >> 2)], 1u << sh) >> sh) & 0xffu) + 1u;
    };
    auto hget = [&](int i, uint32_t b) { return (Hh[i * 8 + (b >> 2)] >> (8 * (b & 3))) & 0xffu; };
    // the loads: 3^3 warp-round j = apply blocks [32j, 32j + 32) (k_conv_map's q loop), load t = (row
    // nz, nx; pair pp; half h); 5^3 round j = expansion groups [32j, 32j + 32), load t = cell 8g + t.
    // Each lane's slot (F word); distinct words counted once.  Warp w takes rounds w, w + nw, ...
    auto each_load = [&](auto&& f) {
        for (int j = warp; j < nwr; j += nw) {
            if constexpr (H == 2) {
                const int gq = 32 * j + lane;
                for (int t = 0; t < 8; ++t) {
                    const uint32_t slot = gq < NG8 ? C[8 * gq + t] >> 2 : 0xffffu;
                    const unsigned m = __match_any_sync(FULL, slot);
                    if (slot != 0xffffu && lane == __ffs(m) - 1) f(8 * j + t, slot);
                }
            } else {
                const int q = 32 * j + lane;
                int base = -1;
                if (q < nb) {
                    const int b = BL[q];
                    base = ((2 * (b / (kBlocks / 4))) * M::BX + 2 * ((b / (kTY / 2)) & 3)) * M::BY +
                           2 * (b & (kTY / 2 - 1));
                }
                for (int t = 0; t < 64; ++t) {
                    const int nz = t >> 4, nx = (t >> 2) & 3, pp = (t >> 1) & 1, h = t & 1;
                    const uint32_t slot = base >= 0 ? C[base + (nz * M::BX + nx) * M::BY + 2 * pp + h] >> 2 : 0xffffu;
                    const unsigned m = __match_any_sync(FULL, slot);
                    if (slot != 0xffffu && lane == __ffs(m) - 1) f(64 * j + t, slot);
                }
            }
        }
    };
    each_load([&](int i, uint32_t slot) {
        if (slot < kFlat0) hinc(i, (M::REC + slot) & 31);  // (the zero's 4 words: 4 banks)
        else atomicAdd(&cnt[(slot - kFlat0) >> 2], 1u);
    });
    __syncthreads();
    for (int i = warp; i < ni; i += nw) {
        const unsigned v = __reduce_max_sync(FULL, hget(i, lane));
        if (lane == 0) cur[i] = v;
    }
    // 3^3: chunks no load references (sources only inactive regions read) are
    // dropped -- kidx = their rank among the kept ones; groups, colours and
    // positions below are over the kept chunks (5^3's expansion reads every
    // box cell: every chunk is kept)
    if (warp == 1 || nw == 1) {
        int carry = 0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
            const int c = c0 + lane;
            const bool keep = c < nch && (H == 2 || !a.place_drop || cnt[c] > 0);
            const unsigned b = __ballot_sync(FULL, keep);
            const int p = carry + __popc(b & ((1u << lane) - 1u));
            if (c < nch) kidx[c] = static_cast<uint16_t>(keep ? p : 0xffff);
            if (keep) kc[p] = static_cast<uint16_t>(c);
            carry += __popc(b);
        }
        if (lane == 0) nkeep_s = carry;
    }
    if (warp == 0) {  // roff = exclusive scan of cnt
        uint32_t carry = 0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
            const int c = c0 + lane;
            const uint32_t v = c < nch ? cnt[c] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, x, d);
                if (lane >= d) x += y;
            }
            if (c < nch) roff[c] = carry + x - v;
            carry += __shfl_sync(FULL, x, 31);
        }
        if (lane == 0) roff[nch] = carry;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nch; c += blockDim.x) cnt[c] = roff[c];  // (the fill cursors)
    __syncthreads();
    each_load([&](int i, uint32_t slot) {
        if (slot >= kFlat0) {
            const uint32_t c = (slot - kFlat0) >> 2;
            refs[atomicAdd(&cnt[c], 1u)] = static_cast<uint16_t>(i << 2 | (slot & 3u));
        }
    });
    const int nk = nkeep_s, ngk = (nk + 31) >> 5;  // kept chunks, their groups of 32
    for (int i = threadIdx.x; i < 8 * ngk; i += blockDim.x) {
        const int gi = i >> 3, k = i & 7, n_g = min(32, nk - 32 * gi);
        cap[i] = static_cast<uint8_t>(k < n_g ? (n_g - k + 7) / 8 : 0);
    }
    // per group: its chunks by reference count, descending (ties: chunk order)
    for (int gi = warp; gi < ngk; gi += nw) {
        const int p = 32 * gi + lane;
        const int c = p < nk ? kc[p] : 0;
        const uint32_t nr = p < nk ? roff[c + 1] - roff[c] : 0u;
        int rank = 0;
        for (int j = 0; j < 32; ++j) {
            const uint32_t o = __shfl_sync(FULL, nr, j);
            rank += (o > nr || (o == nr && j < lane)) ? 1 : 0;
        }
        if (p < nk) order[32 * gi + rank] = static_cast<uint16_t>(c);
    }
    __syncthreads();
    // greedy colours in rounds: lane = (colour k = lane & 7, a quarter of the chunk's references)
    const int k = lane & 7;
    // (half of the groups per step: picks made together do not see each other,
    // and fewer of them keep the greedy close to one-at-a-time)
    for (int rr = 0; rr < 2 * 32; ++rr) {
        const int r = rr >> 1, part = rr & 1;
        for (int gi = 2 * warp + part; gi < ngk; gi += 2 * nw) {
            if (32 * gi + r >= nk) continue;
            const int c = order[32 * gi + r];
            const uint32_t r0 = roff[c], r1 = roff[c + 1];
            uint32_t cost = 0;
            for (uint32_t e0 = r0 + (lane >> 3); e0 < r1; e0 += 4) {
                const uint32_t e = refs[e0], i = e >> 2;
                const uint32_t h = hget(i, (M::REC + kFlat0 + (e & 3u) + 4u * k) & 31u), cu = cur[i];
                cost += max(cu, h + 1u) - cu;
            }
            cost += __shfl_xor_sync(FULL, cost, 8);
            cost += __shfl_xor_sync(FULL, cost, 16);
            const uint32_t key = cap[8 * gi + k] ? (cost << 3 | static_cast<uint32_t>(k)) : 0xffffffffu;
            const int kb = static_cast<int>(__reduce_min_sync(FULL, key) & 7u);
            if (lane == 0) {
                pick[gi] = static_cast<uint16_t>(c);
                pk[gi] = static_cast<uint8_t>(kb);
            }
        }
        __syncthreads();  // (every pick of the step made against the same histogram)
        for (int gi = 2 * warp + part; gi < ngk; gi += 2 * nw) {
            if (32 * gi + r >= nk) continue;
            const int c = pick[gi], kb = pk[gi];
            if (lane == 0) {
                --cap[8 * gi + kb];
                npos[c] = static_cast<uint16_t>(kb);  // (the colour; positions below)
            }
            for (uint32_t e0 = roff[c] + lane; e0 < roff[c + 1]; e0 += 32) {
                const uint32_t e = refs[e0], i = e >> 2;
                atomicMax(&cur[i], hinc(i, (M::REC + kFlat0 + (e & 3u) + 4u * kb) & 31u));
            }
        }
        __syncthreads();
    }
    // positions: a group's chunks of colour k take its positions k, k + 8, ... in chunk order
    for (int gi = warp; gi < ngk; gi += nw) {
        const int p = 32 * gi + lane;
        const int c = p < nk ? kc[p] : 0;
        const int kk = p < nk ? npos[c] : 8 + lane;
        const unsigned m = __match_any_sync(FULL, kk);
        if (p < nk) npos[c] = static_cast<uint16_t>(32 * gi + kk + 8 * __popc(m & ((1u << lane) - 1u)));
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nch; c += blockDim.x)
        if (kidx[c] != 0xffff) a.flat[f0 + npos[c]] = list_in[f0 + c];
    for (int p = nk + threadIdx.x; p < nch; p += blockDim.x) a.flat[f0 + p] = 0u;  // (the dropped tail: particle 0)
    auto moved = [&](uint32_t code) -> uint32_t {
        const uint32_t slot = code >> 2;
        if (slot < kFlat0) return code;
        const uint32_t c = (slot - kFlat0) >> 2;
        if (kidx[c] == 0xffff) return 0u;  // (a cell no active block reads: the zero)
        return (kFlat0 + 4u * npos[c] + (slot & 3u)) << 2;
    };
    for (int w = threadIdx.x; w < M::CW; w += blockDim.x)
        rec[M::CODE0 + w] = moved(C[2 * w]) | moved(C[2 * w + 1]) << 16;
    if (threadIdx.x == 0) rec[M::W_NLEAF] = static_cast<uint32_t>(nk);  // (the chunks k_conv_map gathers)
}

// tile occupancy: mark (z/8, x/8, y/16) of every particle of the level
__global__ void k_mark_tiles(const uint32_t* __restrict__ work, uint64_t n_work, LevelG g, const uint32_t* __restrict__ rb,
                             const uint16_t* __restrict__ y, int txd, int tyd, uint8_t* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = warp; w < n_work; w += nw) {
        const uint32_t row = work[w];
        const uint32_t loc = row - g.row0;
        const int z = static_cast<int>(loc / g.xd), x = static_cast<int>(loc % g.xd);
        const uint64_t base = (static_cast<uint64_t>(z / kTZ) * txd + x / kTX) * tyd;
        const uint32_t b = rb[row], e = rb[row + 1];
        for (uint32_t i = b + lane; i < e; i += 32) {  // (one store per distinct tile of the ascending row)
            const uint32_t t = y[i] / kTY;
            if (i == b || y[i - 1] / kTY != t) flags[base + t] = 1;
        }
    }
}

TileLaunch base_launch(const aprgpu_apr* apr) {
    const DevAccess& L = apr->leaf;
    const DevAccess& Tr = apr->tree;
    TileLaunch a{};
    a.leaf = L.view();
    a.tree = Tr.view();
    a.tree_lmin = Tr.n_particles ? Tr.l_min : 1;
    a.tree_lmax = Tr.n_particles ? Tr.l_max : 0;
    a.n_leaf = static_cast<uint32_t>(L.n_particles);
    a.n_tree = static_cast<uint32_t>(Tr.n_particles);
    return a;
}

void set_level(TileLaunch& a, const DevAccess& L, int l, uint32_t end) {
    const int s = a.n_levels++;
    a.lvl[s] = l;
    a.tdim[s][0] = L.tile_dims[3 * l];
    a.tdim[s][1] = L.tile_dims[3 * l + 1];
    a.tdim[s][2] = L.tile_dims[3 * l + 2];
    a.seg_end[s] = end;
}

// The tiles of level l a launch for slab sl computes, as absolute tile
// indices [first, second): the whole level below the cut, else the tile z-rows
// that meet the slab's planes (the kernels' own slab test, k_conv_tile)
std::pair<uint64_t, uint64_t> tile_range(const DevAccess& L, int l, const Slab& sl) {
    const uint64_t b = L.tile_off[l], e = L.tile_off[l + 1];
    if (l < sl.lc || e == b) return {b, e};
    const int sh = L.l_max - l, tzd = L.tile_dims[3 * l];
    const int64_t zlo = static_cast<int64_t>(sl.z_lo) >> sh;
    const int64_t zhi = (static_cast<int64_t>(sl.z_hi) + (int64_t(1) << sh) - 1) >> sh;
    const int t0 = static_cast<int>(std::clamp<int64_t>(zlo / kTZ, 0, tzd));
    const int t1 = static_cast<int>(std::clamp<int64_t>((zhi + kTZ - 1) / kTZ, t0, tzd));
    const uint32_t* zf = L.tile_zfirst.data() + L.tile_zfirst_off[l];
    return {b + zf[t0], b + zf[t1]};
}

// The per-tile state (probe, source runs, staged-source lists, gather maps)
// is built for the tiles an APR's convolutions can touch: every tile, or --
// once aprgpu_apr_restrict gave the APR a z-slab -- the tiles meeting the
// slab's planes (levels below its cut whole).  Fills launch a with one segment
// per level over those tiles; returns their count.
uint32_t restricted_segments(const aprgpu_apr* apr, TileLaunch& a) {
    const DevAccess& L = apr->leaf;
    uint32_t total = 0;
    uint64_t first = 0;
    for (int l = L.l_min; l <= L.l_max; ++l) {
        const auto r = tile_range(L, l, apr->tile_slab);
        const uint32_t c = static_cast<uint32_t>(r.second - r.first);
        if (!c) continue;
        if (!a.n_levels) first = r.first;
        a.seg_shift[a.n_levels] = static_cast<uint32_t>(r.first - first - total);
        total += c;
        set_level(a, L, l, total);
    }
    a.tile_base = static_cast<uint32_t>(first);
    return total;
}

// First use of an APR by the tile path: probe every tile once.
void ensure_tile_meta(aprgpu_apr* apr, cudaStream_t s) {
    DevAccess& L = apr->leaf;
    if (acquire_ptr(L.tile_meta) || !L.tiles) return;
    std::lock_guard<std::mutex> lk(apr->ctx->mu);
    if (L.tile_meta) return;
    const uint64_t n = L.tile_off[L.l_max + 1];
    uint8_t* meta = nullptr;
    APR_CUDA(cudaMalloc(&meta, n + 16));
    APR_CUDA(cudaMemsetAsync(meta, 0, n + 16, s));
    TileLaunch a = base_launch(apr);
    const uint32_t total = restricted_segments(apr, a);
    if (total) {
        a.tiles = L.tiles;
        a.meta = meta;
        k_tile_probe<<<total, kTileThreads, 0, s>>>(a);
        count_launch(apr->ctx);
        APR_CUDA(cudaGetLastError());
        APR_CUDA(cudaStreamSynchronize(s));
    }
    publish_ptr(L.tile_meta, meta);
}

// First use of an APR with stencil half-width H: the per-tile source runs.
template <int H>
void ensure_tile_runs(aprgpu_apr* apr, cudaStream_t s) {
    DevAccess& L = apr->leaf;
    if (acquire_ptr(L.tile_runs[H - 1]) || !L.tiles) return;
    std::lock_guard<std::mutex> lk(apr->ctx->mu);
    if (L.tile_runs[H - 1]) return;
    const uint64_t n = L.tile_off[L.l_max + 1];
    TileLaunch a = base_launch(apr);
    const uint32_t total = restricted_segments(apr, a);
    uint32_t* off = nullptr;
    APR_CUDA(cudaMalloc(&off, 4 * (n + 1)));
    APR_CUDA(cudaMemsetAsync(off, 0, 4 * (n + 1), s));
    uint2* runs = nullptr;
    uint32_t nruns = 0;
    if (total) {
        a.tiles = L.tiles;
        a.meta = L.tile_meta;
        GpuBuf counts, temp;
        counts.ensure(4 * (n + 1));
        APR_CUDA(cudaMemsetAsync(counts.p, 0, 4 * (n + 1), s));
        k_tile_runs<H><<<total, kTileThreads, 0, s>>>(a, 0, counts.as<uint32_t>(), nullptr);
        count_launch(apr->ctx);
        APR_CUDA(cudaGetLastError());
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.as<uint32_t>(), off, static_cast<int64_t>(n + 1), s);
        temp.ensure(tb + 16);
        tb = temp.bytes;
        APR_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, counts.as<uint32_t>(), off, static_cast<int64_t>(n + 1), s));
        count_launch(apr->ctx);
        APR_CUDA(cudaMemcpyAsync(&nruns, off + n, 4, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
        APR_CUDA(cudaMalloc(&runs, 8ull * nruns + 8));
        a.run_off = off;
        k_tile_runs<H><<<total, kTileThreads, 0, s>>>(a, 1, nullptr, runs);
        count_launch(apr->ctx);
        APR_CUDA(cudaGetLastError());
        APR_CUDA(cudaStreamSynchronize(s));
    } else {
        APR_CUDA(cudaMalloc(&runs, 8));
    }
    L.tile_run_off[H - 1] = off;
    publish_ptr(L.tile_runs[H - 1], runs);  // (tile_run_off is read only after tile_runs)
}

// per tile: its chunk count (k_conv_tile's map mode writes the chunks)
__global__ void k_tile_nflat(const uint32_t* __restrict__ run_off, const uint2* __restrict__ runs, uint64_t n,
                             uint32_t* __restrict__ counts) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t c = 0;  // F slots: every run covers whole 16-byte chunks from its first particle's phase
        for (uint32_t j = run_off[t]; j < run_off[t + 1]; ++j) c += ((runs[j].x & 3u) + (runs[j].y >> 16) + 3) & ~3u;
        counts[t] = ((c >> 2) + 3) & ~3u;  // chunks, padded to 4 (16-byte bulk copies of the list)
    }
}

// The flattened source lists' layout for half-width H (allocated zeroed; the
// map build writes them).
__global__ void k_max_u32(const uint32_t* __restrict__ v, uint64_t n, uint32_t* out) {
    uint32_t m = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, v[i]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

template <int H>
void ensure_tile_flat(aprgpu_apr* apr, cudaStream_t s) {
    DevAccess& L = apr->leaf;
    if (L.tile_flat[H - 1]) return;
    const uint64_t n = L.tile_off[L.l_max + 1];
    uint32_t* off = nullptr;
    APR_CUDA(cudaMalloc(&off, 4 * (n + 1)));
    GpuBuf counts, temp;
    counts.ensure(4 * (n + 1));
    APR_CUDA(cudaMemsetAsync(counts.p, 0, 4 * (n + 1), s));
    if (n) {
        k_tile_nflat<<<std::min<unsigned>(blocks_for(n, 256), apr->ctx->sm_count * 8), 256, 0, s>>>(
            L.tile_run_off[H - 1], L.tile_runs[H - 1], n, counts.as<uint32_t>());
        count_launch(apr->ctx);
        APR_CUDA(cudaGetLastError());
    }
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.as<uint32_t>(), off, static_cast<int64_t>(n + 1), s);
    temp.ensure(tb + 16);
    tb = temp.bytes;
    APR_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, counts.as<uint32_t>(), off, static_cast<int64_t>(n + 1), s));
    count_launch(apr->ctx);
    // the lists at a fixed stride: the largest tile's chunk count (a multiple of 4)
    uint32_t cap = 0;
    if (n) {
        GpuBuf mx;
        mx.ensure(16);
        APR_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
        k_max_u32<<<std::min<unsigned>(blocks_for(n, 256), apr->ctx->sm_count * 8), 256, 0, s>>>(counts.as<uint32_t>(), n,
                                                                                                 mx.as<uint32_t>());
        count_launch(apr->ctx);
        APR_CUDA(cudaGetLastError());
        APR_CUDA(cudaMemcpyAsync(&cap, mx.p, 4, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
    }
    cap = std::max<uint32_t>((cap + 3u) & ~3u, 4u);
    if (static_cast<uint64_t>(n) * cap >= (1ull << 32)) fail(APRGPU_ERR_CAPABILITY, "chunk lists exceed u32 offsets");
    uint32_t* flat = nullptr;
    APR_CUDA(cudaMalloc(&flat, 4ull * n * cap + 16));
    APR_CUDA(cudaMemsetAsync(flat, 0, 4ull * n * cap + 16, s));  // padding entries: particle 0
    L.tile_flat_off[H - 1] = off;
    L.tile_flat[H - 1] = flat;
    L.tile_flat_n[H - 1] = static_cast<uint64_t>(n) * cap;
    L.tile_flat_cap[H - 1] = cap;
}

// APRGPU_MAP_DROP=0: the placement pass keeps chunks no active block reads (A/B experiments)
bool map_drop_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("APRGPU_MAP_DROP");
        return !(e && e[0] == '0');
    }();
    return on;
}

// APRGPU_MAP_PLACE=0: keep the build's F order (A/B experiments)
bool map_place_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("APRGPU_MAP_PLACE");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename Acc, int H, bool MAP = false>
void launch_tiles(aprgpu_ctx* ctx, const TileLaunch& a, uint32_t n, cudaStream_t s) {
    constexpr int bytes = Box<H>::NC * static_cast<int>(sizeof(float));
    static OncePerDevice attr;
    attr([] {
        APR_CUDA(cudaFuncSetAttribute(k_conv_tile<Acc, H, MAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    });
    k_conv_tile<Acc, H, MAP><<<n, kTileThreads, bytes, s>>>(a);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
}

template <typename Acc, int H>
void launch_map(aprgpu_ctx* ctx, const TileLaunch& a, uint32_t n, cudaStream_t s) {
    // [record (FAST 5^3: header + box)][F: kFlat0 + 4 chunks][chunk list][EXACT 5^3: box]
    using M = MapBox<H>;
    const int fw = kFlat0 + 5 * a.map_ng;
    const int lf = a.list_in_f ? a.map_ng : 0;  // (the list in F's tail: no words of its own)
    const int bytes = (H == 2 && sizeof(Acc) == 4 ? M::HDR + M::SN + fw - lf
                       : H == 2                   ? M::REC + fw - a.map_ng + std::max(M::SN, a.map_ng)  // list in the box
                                                  : M::REC + fw - lf) * 4;
    if (bytes > 225 * 1024) fail(APRGPU_ERR_CAPABILITY, "gather map exceeds shared memory");
    // 3^3: 96-thread CTAs (a C3 tile has ~65 active blocks: the apply's one
    // round fits 3 warps; A/B EXACT 0.173 -> 0.167 ms, FAST unchanged);
    // APRGPU_MAP_THREADS=128 restores 4 warps (A/B experiments)
    static const int nt = [] {  // (5^3 on 96 threads measured slower: 0.364 -> 0.376 ms EXACT)
        const char* e = std::getenv("APRGPU_MAP_THREADS");
        return H == 1 && !(e && std::atoi(e) == 128) ? 96 : kTileThreads;
    }();
    static OncePerDevice attr;
    attr([] {
        APR_CUDA(cudaFuncSetAttribute(k_conv_map<Acc, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        APR_CUDA(cudaFuncSetAttribute(k_conv_map<Acc, H, (H == 1 ? 96 : kTileThreads)>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        // 3^3 EXACT: with 128-thread CTAs (8 CTAs/SM by registers, 7 by shared
        // memory) a 164 KB carveout left the gathers L1 (A/B on C3: 58 % 0.185,
        // 72 % 0.180, 86 % 0.184 ms); at 96 threads 86 and 100 % tie (0.1667)
        // and 72 % caps it at 6 CTAs/SM.  FAST and 5^3: the default
        int carve = sizeof(Acc) == 8 && H == 1 ? (nt == 96 ? 100 : 72) : -1;
        if (const char* e = std::getenv(sizeof(Acc) == 8 ? "APRGPU_CARVEOUT_EXACT" : "APRGPU_CARVEOUT_FAST"))
            carve = std::atoi(e);  // (A/B experiments)
        if (carve >= 0) {
            APR_CUDA(cudaFuncSetAttribute(k_conv_map<Acc, H>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            APR_CUDA(cudaFuncSetAttribute(k_conv_map<Acc, H, (H == 1 ? 96 : kTileThreads)>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
        }
    });
    if (nt == 96)
        k_conv_map<Acc, H, (H == 1 ? 96 : kTileThreads)><<<n, nt, bytes, s>>>(a);
    else
        k_conv_map<Acc, H><<<n, kTileThreads, bytes, s>>>(a);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
}

// APRGPU_TILE_MAP=0: no resident gather maps (every call reconstructs its boxes)
bool maps_enabled() {
    const char* e = std::getenv("APRGPU_TILE_MAP");
    return !(e && e[0] == '0');
}

// The gather maps of launch b's levels for half-width H and pad mode: built on
// first use (one map-mode launch of k_conv_tile), kept with the APR.  A map
// holds the records of the tiles [a0, a1) of its level: a slab launch (rng:
// each segment's absolute tile range) builds only the tiles it computes, and
// a later launch that needs more replaces the window by the hull of both (the
// old one is kept until the APR is freed: launches in flight may read it).
// Returns false -- the caller reconstructs -- when the missing maps would take
// more than half of the free device memory.
template <int H>
bool ensure_tile_maps(aprgpu_apr* apr, TileLaunch& b, const uint64_t (*rng)[2], int pad, cudaStream_t s) {
    using Win = DevAccess::MapWin;
    DevAccess& L = apr->leaf;
    const int pm = pad == APRGPU_PAD_ZERO ? 1 : 0;
    for (int i = 0; i < b.n_levels; ++i)
        if (__atomic_load_n(&L.tile_map_fail[H - 1][pm][b.lvl[i]], __ATOMIC_ACQUIRE)) return false;
    auto covers = [&](int i) {
        const Win* w = acquire_ptr(L.tile_map[H - 1][pm][b.lvl[i]]);
        return w && w->a0 <= rng[i][0] && w->a1 >= rng[i][1];
    };
    auto all_covered = [&] {
        for (int i = 0; i < b.n_levels; ++i)
            if (!covers(i)) return false;
        return true;
    };
    if (!all_covered()) {
        std::lock_guard<std::mutex> lk(apr->ctx->mu);
        // the build launch: one segment per level whose window is missing or too narrow
        TileLaunch m = b;
        m.n_levels = 0;
        uint64_t lo[kMaxLevels], hi[kMaxLevels];
        uint32_t total = 0;
        size_t need = 0;
        for (int i = 0; i < b.n_levels; ++i) {
            if (covers(i)) continue;
            const Win* w = L.tile_map[H - 1][pm][b.lvl[i]];
            const int j = m.n_levels;
            lo[j] = w ? std::min(w->a0, rng[i][0]) : rng[i][0];
            hi[j] = w ? std::max(w->a1, rng[i][1]) : rng[i][1];
            total += static_cast<uint32_t>(hi[j] - lo[j]);
            need += (hi[j] - lo[j]) * MapBox<H>::REC * sizeof(uint32_t);
            set_level(m, L, b.lvl[i], total);
            m.woff[j] = b.woff[i];
            m.sep[j] = b.sep[i];
        }
        if (m.n_levels) {
            size_t free_b = 0, total_b = 0;
            APR_CUDA(cudaMemGetInfo(&free_b, &total_b));
            if (need > free_b / 2) {
                for (int j = 0; j < m.n_levels; ++j)
                    __atomic_store_n(&L.tile_map_fail[H - 1][pm][m.lvl[j]], 1, __ATOMIC_RELEASE);
                return false;
            }
            NvtxRange nr(H == 1 ? "aprgpu: gather-map build (3^3)" : "aprgpu: gather-map build (5^3)");
            ensure_tile_flat<H>(apr, s);
            // built into local buffers, published only after the build kernel
            // has completed and passed the overflow check
            uint32_t* fresh[kMaxLevels] = {};
            m.tile_base = static_cast<uint32_t>(lo[0]);
            for (int j = 0; j < m.n_levels; ++j) {
                APR_CUDA(cudaMalloc(&fresh[j], (hi[j] - lo[j]) * MapBox<H>::REC * sizeof(uint32_t) + 16));
                m.map[j] = fresh[j];
                m.map_base[j] = static_cast<uint32_t>(lo[j]);
                m.seg_shift[j] = static_cast<uint32_t>(lo[j] - m.tile_base - (j ? m.seg_end[j - 1] : 0));
            }
            // the build writes its chunk lists to scratch, k_map_place then writes
            // them (and the codes) in their bank-aware order
            const bool place = map_place_enabled();
            GpuBuf list_scratch;
            if (place) {  // (the build leaves a tile's padding entries alone: particle 0, like tile_flat's)
                list_scratch.ensure(4 * L.tile_flat_n[H - 1] + 16);
                APR_CUDA(cudaMemsetAsync(list_scratch.p, 0, 4 * L.tile_flat_n[H - 1] + 16, s));
            }
            m.flat = place ? list_scratch.as<uint32_t>() : L.tile_flat[H - 1];
            m.flat_off = L.tile_flat_off[H - 1];
            m.flat_cap = L.tile_flat_cap[H - 1];
            m.slab_lc = 1 << 20;  // every tile of the windows
            GpuBuf flag;
            flag.ensure(16);
            APR_CUDA(cudaMemsetAsync(flag.p, 0, 8, s));
            m.map_overflow = flag.as<int>();
            m.map_maxg = flag.as<int>() + 1;
            launch_tiles<float, H, true>(apr->ctx, m, total, s);
            int fl[2] = {0, 0};
            APR_CUDA(cudaMemcpyAsync(fl, flag.p, 8, cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            if (fl[0]) {  // some tile has too many sources for k_conv_map: reconstruct these levels
                for (int j = 0; j < m.n_levels; ++j) {
                    cudaFree(fresh[j]);
                    __atomic_store_n(&L.tile_map_fail[H - 1][pm][m.lvl[j]], 1, __ATOMIC_RELEASE);
                }
                return false;
            }
            if (place) {
                TileLaunch pl = m;
                pl.flat = L.tile_flat[H - 1];
                pl.place_drop = map_drop_enabled();
                const int bytes = place_smem<H>(fl[1]);
                APR_CUDA(cudaFuncSetAttribute(k_map_place<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
                k_map_place<H><<<total, 32 * kPlaceWarps, bytes, s>>>(pl, list_scratch.as<uint32_t>());
                count_launch(apr->ctx);
                APR_CUDA(cudaGetLastError());
                APR_CUDA(cudaStreamSynchronize(s));
            }
            for (int j = 0; j < m.n_levels; ++j) {
                const int l = m.lvl[j];
                L.tile_map_ng[H - 1][l] = std::max(L.tile_map_ng[H - 1][l], fl[1]);
                Win* old = L.tile_map[H - 1][pm][l];
                publish_ptr(L.tile_map[H - 1][pm][l], new Win{fresh[j], lo[j], hi[j]});
                if (old) L.tile_map_retired.push_back(old);
            }
        }
    }
    b.map_ng = 0;
    for (int i = 0; i < b.n_levels; ++i) {
        const Win* w = acquire_ptr(L.tile_map[H - 1][pm][b.lvl[i]]);
        b.map[i] = w->rec;
        b.map_base[i] = static_cast<uint32_t>(w->a0);
        b.map_ng = std::max(b.map_ng, L.tile_map_ng[H - 1][b.lvl[i]]);
    }
    b.flat = L.tile_flat[H - 1];
    b.flat_off = L.tile_flat_off[H - 1];
    b.flat_cap = L.tile_flat_cap[H - 1];
    b.aligned16 = ((reinterpret_cast<uintptr_t>(b.val) | reinterpret_cast<uintptr_t>(b.tval)) & 15) == 0;
    static const bool lf = [] {  // APRGPU_MAP_LISTF=0: the list after F (A/B experiments)
        const char* e = std::getenv("APRGPU_MAP_LISTF");
        return !(e && e[0] == '0');
    }();
    b.list_in_f = lf;
    static const bool hint = [] {  // APRGPU_L2HINT=0: no L2 eviction hints (A/B experiments)
        const char* e = std::getenv("APRGPU_L2HINT");
        return !(e && e[0] == '0');
    }();
    b.l2hint = hint;  // (3^3 and FAST 5^3; EXACT 5^3 keeps its list inside the box)
    return true;
}

}  // namespace

void build_tile_lists(aprgpu_ctx* ctx, DevAccess& a) {
    a.tile_off.assign(a.l_max + 2, 0);
    a.tile_dims.assign(3 * (a.l_max + 1), 0);
    uint64_t total_flags = 0;
    for (int l = a.l_min; l <= a.l_max; ++l) {
        const uint64_t tzd = (a.zd[l] + kTZ - 1) / kTZ, txd = (a.xd[l] + kTX - 1) / kTX, tyd = (a.yd[l] + kTY - 1) / kTY;
        a.tile_dims[3 * l] = static_cast<int>(tzd);
        a.tile_dims[3 * l + 1] = static_cast<int>(txd);
        a.tile_dims[3 * l + 2] = static_cast<int>(tyd);
        total_flags = std::max<uint64_t>(total_flags, tzd * txd * tyd);
    }
    if (total_flags >= (1ull << 32)) fail(APRGPU_ERR_CAPABILITY, "tile grid exceeds u32 ids");
    GpuBuf flags, out, nsel, temp;
    flags.ensure(total_flags + 16);
    std::vector<std::vector<uint32_t>> per_level(a.l_max + 1);
    uint64_t off = 0;
    for (int l = a.l_min; l <= a.l_max; ++l) {
        a.tile_off[l] = off;
        const uint64_t n_work = a.work_off[l + 1] - a.work_off[l];
        if (!n_work) continue;
        const int txd = a.tile_dims[3 * l + 1], tyd = a.tile_dims[3 * l + 2];
        const uint64_t nflags = static_cast<uint64_t>(a.tile_dims[3 * l]) * txd * tyd;
        APR_CUDA(cudaMemsetAsync(flags.p, 0, nflags, ctx->stream));
        LevelG g{a.zd[l], a.xd[l], a.yd[l], static_cast<uint32_t>(a.level_offset[l])};
        k_mark_tiles<<<std::min<unsigned>(blocks_for(n_work * 32, 256), ctx->sm_count * 16), 256, 0, ctx->stream>>>(
            a.work + a.work_off[l], n_work, g, a.rb, a.y, txd, tyd, flags.as<uint8_t>());
        count_launch(ctx);
        APR_CUDA(cudaGetLastError());
        out.ensure(4 * nflags + 16);
        nsel.ensure(16);
        size_t tb = 0;
        thrust::counting_iterator<uint32_t> it(0);
        cub::DeviceSelect::Flagged(nullptr, tb, it, flags.as<uint8_t>(), out.as<uint32_t>(), nsel.as<uint64_t>(),
                                   static_cast<int64_t>(nflags), ctx->stream);
        temp.ensure(tb + 16);
        tb = temp.bytes;
        APR_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, it, flags.as<uint8_t>(), out.as<uint32_t>(),
                                            nsel.as<uint64_t>(), static_cast<int64_t>(nflags), ctx->stream));
        count_launch(ctx);
        uint64_t c = 0;
        APR_CUDA(cudaMemcpyAsync(&c, nsel.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        APR_CUDA(cudaStreamSynchronize(ctx->stream));
        per_level[l].resize(c);
        if (c) APR_CUDA(cudaMemcpy(per_level[l].data(), out.p, 4 * c, cudaMemcpyDeviceToHost));
        off += c;
    }
    a.tile_off[a.l_max + 1] = off;
    for (int l = 0; l < a.l_min; ++l) a.tile_off[l] = 0;
    a.tile_zfirst.clear();
    a.tile_zfirst_off.assign(a.l_max + 1, 0);
    for (int l = a.l_min; l <= a.l_max; ++l) {
        a.tile_zfirst_off[l] = a.tile_zfirst.size();
        const uint64_t plane = static_cast<uint64_t>(a.tile_dims[3 * l + 1]) * a.tile_dims[3 * l + 2];
        const std::vector<uint32_t>& t = per_level[l];
        for (int tz = 0, i = 0; tz <= a.tile_dims[3 * l]; ++tz) {  // (ids ascending: z-rows in order)
            while (i < static_cast<int>(t.size()) && t[i] / plane < static_cast<uint64_t>(tz)) ++i;
            a.tile_zfirst.push_back(static_cast<uint32_t>(i));
        }
    }
    APR_CUDA(cudaMalloc(&a.tiles, 4 * off + 4));
    for (int l = a.l_min; l <= a.l_max; ++l)
        if (!per_level[l].empty())
            APR_CUDA(cudaMemcpy(a.tiles + a.tile_off[l], per_level[l].data(), 4 * per_level[l].size(),
                                cudaMemcpyHostToDevice));
}

namespace {

struct RowNonEmpty {
    const uint32_t* rb;
    __host__ __device__ bool operator()(uint32_t r) const { return rb[r + 1] > rb[r]; }
};

struct LevelTiles {
    LevelG g[kMaxLevels];
    int txd[kMaxLevels], tyd[kMaxLevels];
    uint64_t fbase[kMaxLevels];  // first flag of each level in the combined flag space
    uint64_t col0[kMaxLevels];   // first (8 x 8 row) tile column of each level
    int l_min, l_max;
};

// every non-empty row of every level marks the (8z, 8x, 32y) tiles its
// particles fall in.  Four rows per warp (8 lanes each) keep four rows' loads
// in flight (a warp per row is latency-bound on its work -> rb -> y chain);
// a row's y are ascending, so a lane stores only where the tile changes from
// its left neighbour (a shuffle, not a reload)
template <int LPR>  // lanes per row (32 / LPR rows per warp)
__global__ void k_mark_tiles_all(const uint32_t* __restrict__ work, const uint64_t* __restrict__ n_work_p,
                                 const __grid_constant__ LevelTiles lt, const uint32_t* __restrict__ rb,
                                 const uint16_t* __restrict__ y, uint8_t* __restrict__ flags) {
    constexpr int RPW = 32 / LPR;
    const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
    const unsigned grp = static_cast<unsigned>((1ull << LPR) - 1) << (LPR * sub);
    const uint64_t n_work = *n_work_p;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w0 = warp * RPW; w0 < n_work; w0 += nw * RPW) {
        const uint64_t w = w0 + sub;
        if (w >= n_work) continue;  // (whole lane groups drop out together)
        const uint32_t row = work[w];
        int l = lt.l_max;
        while (l > lt.l_min && row < lt.g[l].row0) --l;
        const uint32_t loc = row - lt.g[l].row0;
        const int z = static_cast<int>(loc / lt.g[l].xd), x = static_cast<int>(loc % lt.g[l].xd);
        const uint64_t base = lt.fbase[l] + (static_cast<uint64_t>(z / kTZ) * lt.txd[l] + x / kTX) * lt.tyd[l];
        const uint32_t b = rb[row], e = rb[row + 1];
        // no value carried between chunks (the chunk's first lane reads its left
        // neighbour's y itself): the chunks' loads pipeline
#pragma unroll 4
        for (uint32_t i0 = b; i0 < e; i0 += LPR) {
            const uint32_t i = i0 + sl;
            const uint32_t t = i < e ? static_cast<uint32_t>(y[i]) / kTY : 0xffffffffu;
            const uint32_t up = __shfl_up_sync(grp, t, 1, LPR);
            const uint32_t left = sl ? up : (i > b && i < e ? static_cast<uint32_t>(y[i - 1]) / kTY : 0xfffffffeu);
            if (i < e && t != left) flags[base + t] = 1;
        }
    }
}

}  // namespace

// The per-call index step of the paper's GPU protocol ("row
// index + tree fill + convolution"): nonempty_row_index (convolve.hpp:32-44)
// over every level and the occupied-tile lists derived from it, recomputed on
// the device into APR-owned scratch, stream-ordered with no host round trip.
// (The convolution's own lists, built at upload, are identical; this step
// exists so the protocol's timing includes the work.)  Returns nothing; the
// counts land in scratch.
void rebuild_index_device(aprgpu_apr* apr, cudaStream_t s) {
    DevAccess& L = apr->leaf;
    if (L.n_rows == 0) return;
    LevelTiles lt{};
    lt.l_min = L.l_min;
    lt.l_max = L.l_max;
    uint64_t nflags = 0;
    for (int l = L.l_min; l <= L.l_max; ++l) {
        lt.g[l] = LevelG{L.zd[l], L.xd[l], L.yd[l], static_cast<uint32_t>(L.level_offset[l])};
        lt.txd[l] = L.tile_dims[3 * l + 1];
        lt.tyd[l] = L.tile_dims[3 * l + 2];
        lt.fbase[l] = nflags;
        nflags += static_cast<uint64_t>(L.tile_dims[3 * l]) * lt.txd[l] * lt.tyd[l];
    }
    thrust::counting_iterator<uint32_t> it(0);
    // scratch: [work list n_rows u32][2 counts u64][flags nflags][tile list nflags u32][cub temp]
    size_t t1 = 0, t2 = 0;
    cub::DeviceSelect::If(nullptr, t1, it, static_cast<uint32_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                          static_cast<int64_t>(L.n_rows), RowNonEmpty{L.rb}, s);
    cub::DeviceSelect::Flagged(nullptr, t2, it, static_cast<uint8_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                               static_cast<uint64_t*>(nullptr), static_cast<int64_t>(nflags), s);
    const size_t o_cnt = (4 * L.n_rows + 15) & ~size_t(15);
    const size_t o_flags = o_cnt + 16;
    const size_t o_tiles = (o_flags + nflags + 15) & ~size_t(15);
    const size_t o_temp = (o_tiles + 4 * nflags + 255) & ~size_t(255);
    apr->index_scratch.ensure(o_temp + std::max(t1, t2) + 256);
    char* base = apr->index_scratch.as<char>();
    uint32_t* work = reinterpret_cast<uint32_t*>(base);
    uint64_t* cnt = reinterpret_cast<uint64_t*>(base + o_cnt);
    uint8_t* flags = reinterpret_cast<uint8_t*>(base + o_flags);
    uint32_t* tiles = reinterpret_cast<uint32_t*>(base + o_tiles);
    void* temp = base + o_temp;
    size_t tb = std::max(t1, t2);
    APR_CUDA(cub::DeviceSelect::If(temp, tb, it, work, cnt, static_cast<int64_t>(L.n_rows), RowNonEmpty{L.rb}, s));
    APR_CUDA(cudaMemsetAsync(flags, 0, nflags, s));
    // 8 lanes per row (A/B at C3: 4 lanes 95 us, 8 lanes 89 us, 16 lanes 104 us for the whole index step)
    k_mark_tiles_all<8><<<apr->ctx->sm_count * 16, 256, 0, s>>>(work, cnt, lt, L.rb, L.y, flags);
    tb = std::max(t1, t2);
    APR_CUDA(cub::DeviceSelect::Flagged(temp, tb, it, flags, tiles, cnt + 1, static_cast<int64_t>(nflags), s));
    count_launch(apr->ctx, 3);
    APR_CUDA(cudaGetLastError());
    static const bool verify = [] {  // APRGPU_VERIFY_INDEX=1: check the rebuilt lists against the upload's
        const char* e = std::getenv("APRGPU_VERIFY_INDEX");
        return e && e[0] == '1';
    }();
    if (verify) {
        uint64_t c[2];
        APR_CUDA(cudaMemcpyAsync(c, cnt, 16, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
        const uint64_t nwork = L.work_off[L.l_max + 1], ntiles = L.tile_off[L.l_max + 1];
        bool ok = c[0] == nwork && c[1] == ntiles;
        if (ok) {
            std::vector<uint32_t> w0(nwork), w1(nwork), t0(ntiles), t1v(ntiles);
            APR_CUDA(cudaMemcpy(w0.data(), L.work, 4 * nwork, cudaMemcpyDeviceToHost));
            APR_CUDA(cudaMemcpy(w1.data(), work, 4 * nwork, cudaMemcpyDeviceToHost));
            APR_CUDA(cudaMemcpy(t0.data(), L.tiles, 4 * ntiles, cudaMemcpyDeviceToHost));
            APR_CUDA(cudaMemcpy(t1v.data(), tiles, 4 * ntiles, cudaMemcpyDeviceToHost));
            ok = w0 == w1;
            for (int l = L.l_min; l <= L.l_max && ok; ++l)  // combined flag ids -> per-level tile ids
                for (uint64_t i = L.tile_off[l]; i < L.tile_off[l + 1] && ok; ++i)
                    ok = t1v[i] - lt.fbase[l] == t0[i];
        }
        if (!ok) fail(APRGPU_ERR_INTEGRITY, "rebuild_index: the rebuilt row / tile lists differ from the upload's");
    }
}

// Runs every level whose stencil is an isotropic 3^3 or 5^3 through the tile
// kernel (one launch per extent and run of consecutive levels, coarse levels
// first); sets done[l] for them.
void conv_tile_levels(aprgpu_apr* apr, const aprgpu_pyramid* pyr, const float* values, const float* tree_values,
                      int pad, int accum, float* out, const EpiArgs& epi, const Slab& slab, cudaStream_t s,
                      bool* done) {
    const DevAccess& L = apr->leaf;
    if (!L.tiles) return;
    ensure_tile_meta(apr, s);
    // APRGPU_TILE_SPLIT=1: one launch per level (profiling aid)
    static const bool split = [] {
        const char* e = std::getenv("APRGPU_TILE_SPLIT");
        return e && e[0] == '1';
    }();
    const bool exact = accum == APRGPU_ACCUM_EXACT;
    for (int H = 1; H <= 2; ++H) {
        const int K = 2 * H + 1;
        auto ok = [&](int lv) {
            const int* k = &pyr->k3[3 * (lv - pyr->l_min)];
            return k[0] == K && k[1] == K && k[2] == K;
        };
        int l = L.l_min;
        while (l <= L.l_max) {
            if (!ok(l)) {
                ++l;
                continue;
            }
            TileLaunch b = base_launch(apr);
            b.val = values;
            b.tval = tree_values;
            b.wf = pyr->w_dev;
            b.wd = pyr->wd_dev;
            b.pad = pad;
            b.out = out;
            b.epi = epi;
            b.slab_lc = slab.lc;
            b.slab_zlo = slab.z_lo;
            b.slab_zhi = slab.z_hi;
            if (H == 1) ensure_tile_runs<1>(apr, s); else ensure_tile_runs<2>(apr, s);
            b.tiles = L.tiles;
            b.meta = L.tile_meta;
            b.runs = L.tile_runs[H - 1];
            b.run_off = L.tile_run_off[H - 1];
            uint64_t rng[kMaxLevels][2];  // each segment's tiles (absolute; a slab's z-range of them)
            uint32_t total = 0;
            for (; l <= L.l_max && ok(l); ++l) {
                done[l] = true;
                if (l < slab.lc && !slab.rep) continue;  // (a replicated level another pass computes)
                const auto r = tile_range(L, l, slab);
                const uint32_t c = static_cast<uint32_t>(r.second - r.first);
                if (!c) continue;
                const auto rr = tile_range(L, l, apr->tile_slab);
                if (r.first < rr.first || r.second > rr.second)
                    fail(APRGPU_ERR_CAPABILITY, "convolve: planes outside the APR's slab restriction (aprgpu_apr_restrict)");
                rng[b.n_levels][0] = r.first;
                rng[b.n_levels][1] = r.second;
                b.seg_shift[b.n_levels] = static_cast<uint32_t>(r.first - rng[0][0] - total);
                total += c;
                b.woff[b.n_levels] = pyr->off[l - pyr->l_min];
                b.sep[b.n_levels] = pyr->sep_off[l - pyr->l_min] >= 0 ? pyr->sep_dev + pyr->sep_off[l - pyr->l_min]
                                                                      : nullptr;
                set_level(b, L, l, total);
                if (split) {
                    ++l;
                    break;
                }
            }
            if (!total) continue;
            b.tile_base = static_cast<uint32_t>(rng[0][0]);
            const bool map = maps_enabled() && (H == 1 ? ensure_tile_maps<1>(apr, b, rng, pad, s)
                                                       : ensure_tile_maps<2>(apr, b, rng, pad, s));
            if (map) {
                if (H == 1) {
                    if (exact) launch_map<double, 1>(apr->ctx, b, total, s); else launch_map<float, 1>(apr->ctx, b, total, s);
                } else {
                    if (exact) launch_map<double, 2>(apr->ctx, b, total, s); else launch_map<float, 2>(apr->ctx, b, total, s);
                }
            } else if (H == 1) {
                if (exact) launch_tiles<double, 1>(apr->ctx, b, total, s); else launch_tiles<float, 1>(apr->ctx, b, total, s);
            } else {
                if (exact) launch_tiles<double, 2>(apr->ctx, b, total, s); else launch_tiles<float, 2>(apr->ctx, b, total, s);
            }
        }
    }
}

}  // namespace aprgpu

int aprgpu_map_records(const aprgpu_apr* apr, int half_width, int pad, int level, uint32_t* out,
                       uint64_t cap_words, uint32_t* offsets, uint64_t* n_words, uint64_t* first_tile,
                       uint64_t* n_tiles) {
    using namespace aprgpu;
    return guard([&] {
        need(apr && n_words && first_tile && n_tiles, "null argument");
        need(half_width == 1 || half_width == 2, "half_width must be 1 or 2");
        need(pad == APRGPU_PAD_REFLECT || pad == APRGPU_PAD_ZERO, "bad pad mode");
        const DevAccess& L = apr->leaf;
        need(level >= L.l_min && level <= L.l_max, "level out of range");
        DeviceGuard g(apr->ctx->device);
        std::lock_guard<std::mutex> lk(apr->ctx->mu);
        const DevAccess::MapWin* w = L.tile_map[half_width - 1][pad == APRGPU_PAD_ZERO ? 1 : 0][level];
        const uint32_t rw = half_width == 1 ? MapBox<1>::REC : MapBox<2>::REC;
        const uint64_t n = w ? w->a1 - w->a0 : 0;
        std::vector<uint32_t> off(n + 1);  // (records have a fixed length today)
        for (uint64_t i = 0; i <= n; ++i) off[i] = static_cast<uint32_t>(i * rw);
        *first_tile = w ? w->a0 - L.tile_off[level] : 0;
        *n_tiles = n;
        *n_words = off[n];
        if (offsets) std::copy(off.begin(), off.end(), offsets);
        if (out && n) {
            need(cap_words >= off[n], "output buffer too small");
            APR_CUDA(cudaDeviceSynchronize());
            APR_CUDA(cudaMemcpy(out, w->rec, 4ull * off[n], cudaMemcpyDeviceToHost));
        }
    });
}
