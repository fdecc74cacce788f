// Box-tile convolution for isotropic 3^3 / 5^3 levels (the hot path).
//
// Work item: one (level l, 8z x 8x x 16y) output tile that holds at least one
// particle (tile lists are built once per APR at upload, from the non-empty
// rows).  One CTA per tile reconstructs the level-l image over the tile plus
// its H halo -- a (8+2H) x (8+2H) x (16+2H) box -- into shared memory, once,
// and every output particle of the tile reads its k^3 neighbourhood from it.
// Measured on C3's finest level this box holds ~4.6 reconstructed cells per
// output particle, against ~20 for per-row windows (the v1 kernel in conv.cu):
// the halo rows are shared by the 64 output rows of the tile.
//
// Box fill (fill_level_row semantics, reconstruct.hpp:41-69):
//   phase 1  one thread per (halo row, source) finds, with an L1-resident
//            lower_bound, the particles of the level-l leaf row and of the
//            level-l interior row whose y falls in the box, and for the 64
//            inner rows the output particles of the tile;
//   phase 2  one warp per halo z-plane scatters those particles into the box
//            (the plane's rows flattened across the lanes) and flags the cells;
//   phase 3  for d = 1, 2, ... the few level l-d leaf rows covering the box
//            are searched once and each coarse particle is scattered ONCE into
//            a small coarse box of level l-d -- repeated only while the
//            coverage count says some in-domain box cell is still uncovered (a
//            valid APR covers every cell exactly once);
//   resolve  one cell-parallel pass fills every unflagged box cell from the
//            finest coarse box that holds its ancestor (constant upsampling);
//   phase 4  out-of-domain box cells: reflect_index copies or zeros.
// Outputs: one thread per particle, (az,ax,ay)-ordered FMA chain exactly as
// LevelSlab::apply (convolve.hpp:154-169): fp64 with exact products in EXACT
// mode (bit-identical), fp32 in FAST mode.  Weights travel in the kernel
// parameter block (constant bank operands).
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"

namespace aprgpu {

constexpr int kTZ = 8, kTX = 8, kTY = 16, kTileThreads = 128;

namespace {

struct TileArgs {
    AccessView leaf, tree;
    const float* val;
    const float* tval;
    const uint32_t* tiles;
    uint32_t n_tiles;
    int tzd, txd, tyd;
    int l, pad, tree_at_l;
    float* out;
    EpiArgs epi;
    double wd[125];
    float wf[125];
};

template <int H>
struct Box {
    static constexpr int BZ = kTZ + 2 * H, BX = kTX + 2 * H, BY = kTY + 2 * H;
    static constexpr int NR = BZ * BX, NC = BZ * BX * BY;
};

template <typename Acc>
__device__ __forceinline__ Acc wsel(const TileArgs& a, int i);
template <>
__device__ __forceinline__ double wsel<double>(const TileArgs& a, int i) { return a.wd[i]; }
template <>
__device__ __forceinline__ float wsel<float>(const TileArgs& a, int i) { return a.wf[i]; }

__device__ __forceinline__ double fma_t(double w, double u, double acc) { return __fma_rn(w, u, acc); }
__device__ __forceinline__ float fma_t(float w, float u, float acc) { return __fmaf_rn(w, u, acc); }
__device__ __forceinline__ float to_f(double v) { return __double2float_rn(v); }
__device__ __forceinline__ float to_f(float v) { return v; }

__device__ __forceinline__ int block_sum_add(int v, int* target) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(target, v);
    return v;
}

template <int H>
struct CoarseCap {  // sum over d >= 1 of the coarse-box sizes, rounded up
    static constexpr int value = H == 1 ? 640 : 1024;
};

template <typename Acc, int H>
__global__ void __launch_bounds__(kTileThreads) k_conv_tile(const __grid_constant__ TileArgs a) {
    using B = Box<H>;
    constexpr int K = 2 * H + 1;
    constexpr int CC = CoarseCap<H>::value;
    constexpr int kMaxD = 20;
    __shared__ Acc S[B::NC];                       // level-l box
    __shared__ Acc CV[CC];                         // coarse boxes, level by level
    __shared__ __align__(16) uint8_t F[(B::NC + 15) & ~15];  // box cell written by a level-l source
    __shared__ __align__(16) uint8_t CF[CC];       // coarse cell holds a leaf
    __shared__ int c_s[2 * B::NR], c_n[2 * B::NR];
    __shared__ int o_s[kTZ * kTX], o_n[kTZ * kTX], o_pre[kTZ * kTX + 1];
    __shared__ uint8_t o_row[kTZ * kTX * kTY];
    __shared__ int r_s[64], r_n[64];
    __shared__ int coff[kMaxD + 2];
    __shared__ int cov;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l = a.l;
    const LevelG g = a.leaf.g[l];
    const uint32_t id = a.tiles[blockIdx.x];
    const int ty = static_cast<int>(id % a.tyd);
    const uint32_t t2 = id / a.tyd;
    const int tx = static_cast<int>(t2 % a.txd), tz = static_cast<int>(t2 / a.txd);
    const int z0 = tz * kTZ, x0 = tx * kTX, y0 = ty * kTY;
    const int bz0 = z0 - H, bx0 = x0 - H, by0 = y0 - H;  // box origin (level-l cells)
    const int zlo = max(bz0, 0), zhi = min(z0 + kTZ + H, g.zd);
    const int xlo = max(bx0, 0), xhi = min(x0 + kTX + H, g.xd);
    const int ylo = max(by0, 0), yhi = min(y0 + kTY + H, g.yd);
    const int needed = (zhi - zlo) * (xhi - xlo) * (yhi - ylo);
    const int nsrc = 1 + a.tree_at_l;

    // ---- phase 0: clear coverage flags
    {
        uint32_t* f = reinterpret_cast<uint32_t*>(F);
        for (int i = tid; i < static_cast<int>(sizeof(F) / 4); i += kTileThreads) f[i] = 0u;
        uint32_t* cf = reinterpret_cast<uint32_t*>(CF);
        for (int i = tid; i < CC / 4; i += kTileThreads) cf[i] = 0u;
    }
    // ---- phase 1: candidate ranges of the halo rows, output ranges of the tile
    for (int t = tid; t < nsrc * B::NR; t += kTileThreads) {
        const int src = t >= B::NR;
        const int q = t - src * B::NR;
        const int bz = q / B::BX, bx = q - bz * B::BX;
        const int zz = bz0 + bz, xx = bx0 + bx;
        const bool inner = !src && bz >= H && bz < H + kTZ && bx >= H && bx < H + kTX;
        int s = 0, n = 0, os = 0, on = 0;
        if (zz >= 0 && zz < g.zd && xx >= 0 && xx < g.xd) {
            const uint16_t* ys = src ? a.tree.y : a.leaf.y;
            const uint32_t* rb = src ? a.tree.rb : a.leaf.rb;
            const LevelG gg = src ? a.tree.g[l] : g;
            const uint32_t row = gg.row0 + static_cast<uint32_t>(zz) * gg.xd + xx;
            const uint32_t b = __ldg(rb + row), e = __ldg(rb + row + 1);
            if (e > b) {
                const uint32_t s0 = lower_bound_u16(ys, b, e, ylo);
                s = static_cast<int>(s0);
                n = min(static_cast<int>(e - s0), yhi - ylo);
                if (inner) {
                    const uint32_t o0 = lower_bound_u16(ys, s0, s0 + n, y0);
                    const uint32_t o1 = lower_bound_u16(ys, o0, s0 + n, y0 + kTY);
                    os = static_cast<int>(o0);
                    on = static_cast<int>(o1 - o0);
                }
            }
        }
        c_s[t] = s;
        c_n[t] = n;
        if (inner) {
            const int k = (bz - H) * kTX + (bx - H);
            o_s[k] = os;
            o_n[k] = on;
        }
    }
    if (tid == 0) {
        cov = 0;
        coff[1] = 0;
    }
    __syncthreads();

    // ---- output map (inner row of every output) and level-l scatter
    if (warp == 0) {
        const int v0 = o_n[lane * 2], v1 = o_n[lane * 2 + 1];
        const int incl = warp_incl_scan(v0 + v1, lane);
        const int p0 = incl - v0 - v1, p1 = incl - v1;
        o_pre[lane * 2] = p0;
        o_pre[lane * 2 + 1] = p1;
        if (lane == 31) o_pre[64] = incl;
        for (int j = 0; j < v0; ++j) o_row[p0 + j] = static_cast<uint8_t>(lane * 2);
        for (int j = 0; j < v1; ++j) o_row[p1 + j] = static_cast<uint8_t>(lane * 2 + 1);
    }
    int mine = 0;
    // one warp per (source, z-plane of halo rows); the plane's BX rows are
    // flattened so all lanes scatter particles
    for (int p = warp; p < nsrc * B::BZ; p += kTileThreads / 32) {
        const int src = p >= B::BZ;
        const int bz = p - src * B::BZ;
        const int ebase = src * B::NR + bz * B::BX;
        const int n_l = lane < B::BX ? c_n[ebase + lane] : 0;
        const int s_l = lane < B::BX ? c_s[ebase + lane] : 0;
        const int incl = warp_incl_scan(n_l, lane);
        const int excl = incl - n_l;
        const int total = __shfl_sync(kFull, incl, B::BX - 1);
        const uint16_t* ys = src ? a.tree.y : a.leaf.y;
        const float* vs = src ? a.tval : a.val;
        for (int e0 = 0; e0 < total; e0 += 32) {
            const int e = e0 + lane;
            // owning row: last bx with excl[bx] <= e (binary search over lanes)
            int lo = 0, hi = B::BX - 1;
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                const int mid = (lo + hi + 1) >> 1;
                const int em = __shfl_sync(kFull, excl, mid);
                if (em <= e) lo = mid; else hi = mid - 1;
            }
            const int ex = __shfl_sync(kFull, excl, lo);
            const int sx = __shfl_sync(kFull, s_l, lo);
            if (e < total) {
                const int idx = sx + (e - ex);
                const int yy = __ldg(ys + idx);
                if (yy < yhi) {
                    const int c = (bz * B::BX + lo) * B::BY + (yy - by0);
                    S[c] = static_cast<Acc>(__ldg(vs + idx));
                    F[c] = 1;
                    ++mine;
                }
            }
        }
    }
    block_sum_add(mine, &cov);

    // ---- coarse levels: scatter each level-(l-d) leaf once into its coarse box
    int dmax = 0;
    for (int d = 1; d <= kMaxD; ++d) {
        __syncthreads();
        if (cov >= needed || l - d < a.leaf.l_min) break;
        const int czlo = zlo >> d, cxlo = xlo >> d, cylo = ylo >> d;
        const int nzc = ((zhi - 1) >> d) - czlo + 1, nxc = ((xhi - 1) >> d) - cxlo + 1;
        const int nyc = ((yhi - 1) >> d) - cylo + 1;
        const int base = coff[d];
        if (base + nzc * nxc * nyc > CC) break;  // cannot happen for H <= 2 (see CoarseCap)
        const int ncr = nzc * nxc;
        const LevelG gc = a.leaf.g[l - d];
        if (tid < ncr) {
            const int cz = czlo + tid / nxc, cx = cxlo + tid % nxc;
            int s = 0, n = 0;
            if (cz < gc.zd && cx < gc.xd) {
                const uint32_t row = gc.row0 + static_cast<uint32_t>(cz) * gc.xd + cx;
                const uint32_t b = __ldg(a.leaf.rb + row), e = __ldg(a.leaf.rb + row + 1);
                if (e > b) {
                    const uint32_t s0 = lower_bound_u16(a.leaf.y, b, e, cylo);
                    s = static_cast<int>(s0);
                    n = min(static_cast<int>(e - s0), nyc);
                }
            }
            r_s[tid] = s;
            r_n[tid] = n;
        }
        if (tid == 0) coff[d + 1] = base + nzc * nxc * nyc;
        dmax = d;
        __syncthreads();
        mine = 0;
        // (coarse row, candidate) pairs; nyc <= 11 candidates per row
        for (int t = tid; t < ncr * nyc; t += kTileThreads) {
            const int r = t / nyc, j = t - r * nyc;
            if (j >= r_n[r]) continue;
            const int idx = r_s[r] + j;
            const int yy = __ldg(a.leaf.y + idx);
            if (yy - cylo >= nyc) continue;
            const int rz = r / nxc, rx = r - rz * nxc;
            const int ci = base + (rz * nxc + rx) * nyc + (yy - cylo);
            CV[ci] = static_cast<Acc>(__ldg(a.val + idx));
            CF[ci] = 1;
            const int cz = czlo + rz, cx = cxlo + rx;
            const int zA = max(cz << d, zlo), zB = min((cz + 1) << d, zhi);
            const int xA = max(cx << d, xlo), xB = min((cx + 1) << d, xhi);
            const int yA = max(yy << d, ylo), yB = min((yy + 1) << d, yhi);
            mine += (zB - zA) * (xB - xA) * (yB - yA);
        }
        block_sum_add(mine, &cov);
    }
    __syncthreads();

    // ---- resolve every in-domain cell not written at level l through the
    // coarse boxes, finest first (uncovered cells of a malformed APR -> 0)
    if (dmax > 0 || cov < needed) {
        for (int c = tid; c < B::NC; c += kTileThreads) {
            if (F[c]) continue;
            const int bz = c / (B::BX * B::BY);
            const int rem = c - bz * (B::BX * B::BY);
            const int bx = rem / B::BY, by = rem - bx * B::BY;
            const int zz = bz0 + bz, xx = bx0 + bx, yy = by0 + by;
            if (zz < zlo || zz >= zhi || xx < xlo || xx >= xhi || yy < ylo || yy >= yhi) continue;
            Acc v = Acc(0);
            for (int d = 1; d <= dmax; ++d) {
                const int czlo = zlo >> d, cxlo = xlo >> d, cylo = ylo >> d;
                const int nxc = ((xhi - 1) >> d) - cxlo + 1, nyc = ((yhi - 1) >> d) - cylo + 1;
                const int ci = coff[d] + (((zz >> d) - czlo) * nxc + ((xx >> d) - cxlo)) * nyc + ((yy >> d) - cylo);
                if (CF[ci]) {
                    v = CV[ci];
                    break;
                }
            }
            S[c] = v;
        }
        __syncthreads();
    }

    // ---- out-of-domain box cells (reflect_index / zero padding)
    if (bz0 < 0 || bx0 < 0 || by0 < 0 || bz0 + B::BZ > g.zd || bx0 + B::BX > g.xd || by0 + B::BY > g.yd) {
        for (int c = tid; c < B::NC; c += kTileThreads) {
            const int bz = c / (B::BX * B::BY);
            const int rem = c - bz * (B::BX * B::BY);
            const int bx = rem / B::BY, by = rem - bx * B::BY;
            const int zz = bz0 + bz, xx = bx0 + bx, yy = by0 + by;
            if (zz >= 0 && zz < g.zd && xx >= 0 && xx < g.xd && yy >= 0 && yy < g.yd) continue;
            // cells more than H beyond the domain are read by no output (and
            // their reflection may fall outside the box)
            if (zz >= g.zd + H || xx >= g.xd + H || yy >= g.yd + H) continue;
            if (a.pad == APRGPU_PAD_ZERO) {
                S[c] = Acc(0);
            } else {
                const int rz = reflect_dev(zz, g.zd) - bz0, rx = reflect_dev(xx, g.xd) - bx0,
                          ry = reflect_dev(yy, g.yd) - by0;
                S[c] = S[(rz * B::BX + rx) * B::BY + ry];
            }
        }
        __syncthreads();
    }

    // ---- outputs: one thread per particle, taps in the reference's order
    const int NO = o_pre[64];
    for (int o = tid; o < NO; o += kTileThreads) {
        const int k = o_row[o];
        const int i = o_s[k] + (o - o_pre[k]);
        const int yy = __ldg(a.leaf.y + i);
        const int bz = H + (k >> 3), bx = H + (k & 7);
        // cell (z + H - az, x + H - ax, y + H - ay) for tap (az, ax, ay)
        const Acc* base = S + ((bz + H) * B::BX + (bx + H)) * B::BY + (yy - by0 + H);
        Acc acc = Acc(0);
#pragma unroll
        for (int az = 0; az < K; ++az)
#pragma unroll
            for (int ax = 0; ax < K; ++ax)
#pragma unroll
                for (int ay = 0; ay < K; ++ay)
                    acc = fma_t(wsel<Acc>(a, (az * K + ax) * K + ay), base[-(az * B::BX + ax) * B::BY - ay], acc);
        const float o_ = to_f(acc);
        if (a.epi.mode == EPI_STORE) {
            a.out[i] = o_;
        } else if (a.epi.mode == EPI_RL_RATIO) {
            const double bd = static_cast<double>(o_);
            const double den = bd < a.epi.eps ? a.epi.eps : bd;  // std::max<double>(blurred, eps)
            a.out[i] = __double2float_rn(__ddiv_rn(static_cast<double>(__ldg(a.epi.u + i)), den));
        } else {
            a.epi.est[i] = __fmul_rn(a.epi.est[i], o_);
        }
    }
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
        for (uint32_t i = b + lane; i < e; i += 32) flags[base + y[i] / kTY] = 1;
    }
}

template <typename Acc, int H>
void launch_tile(aprgpu_ctx* ctx, const TileArgs& a, cudaStream_t s) {
    if (!a.n_tiles) return;
    k_conv_tile<Acc, H><<<a.n_tiles, kTileThreads, 0, s>>>(a);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
}

}  // namespace

void build_tile_lists(aprgpu_ctx* ctx, DevAccess& a) {
    a.tile_off.assign(a.l_max + 2, 0);
    a.tile_dims.assign(3 * (a.l_max + 1), 0);
    std::vector<uint32_t> counts(a.l_max + 1, 0);
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
    std::vector<uint32_t> host_tiles;
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
    APR_CUDA(cudaMalloc(&a.tiles, 4 * off + 4));
    for (int l = a.l_min; l <= a.l_max; ++l)
        if (!per_level[l].empty())
            APR_CUDA(cudaMemcpy(a.tiles + a.tile_off[l], per_level[l].data(), 4 * per_level[l].size(),
                                cudaMemcpyHostToDevice));
}

bool conv_tile_level(aprgpu_apr* apr, int l, const float* values, const float* tree_values, const int* k3,
                     const float* w_host, int pad, int accum, float* out, const EpiArgs& epi, cudaStream_t s) {
    const DevAccess& L = apr->leaf;
    const DevAccess& T = apr->tree;
    if (!L.tiles) return false;
    if (!(k3[0] == k3[1] && k3[1] == k3[2] && (k3[0] == 3 || k3[0] == 5))) return false;
    TileArgs a{};
    a.leaf = L.view();
    a.tree = T.view();
    a.val = values;
    a.tval = tree_values;
    a.tiles = L.tiles + L.tile_off[l];
    a.n_tiles = static_cast<uint32_t>(L.tile_off[l + 1] - L.tile_off[l]);
    a.tzd = L.tile_dims[3 * l];
    a.txd = L.tile_dims[3 * l + 1];
    a.tyd = L.tile_dims[3 * l + 2];
    a.l = l;
    a.pad = pad;
    a.tree_at_l = (T.n_particles > 0 && l >= T.l_min && l <= T.l_max) ? 1 : 0;
    a.out = out;
    a.epi = epi;
    const int n = k3[0] * k3[1] * k3[2];
    for (int i = 0; i < n; ++i) {
        a.wf[i] = w_host[i];
        a.wd[i] = static_cast<double>(w_host[i]);
    }
    const bool exact = accum == APRGPU_ACCUM_EXACT;
    if (k3[0] == 3) {
        if (exact) launch_tile<double, 1>(apr->ctx, a, s); else launch_tile<float, 1>(apr->ctx, a, s);
    } else {
        if (exact) launch_tile<double, 2>(apr->ctx, a, s); else launch_tile<float, 2>(apr->ctx, a, s);
    }
    return true;
}

}  // namespace aprgpu
