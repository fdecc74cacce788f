// APR-native convolution on the device (convolve_apr, convolve.hpp:220-303).
//
// Work decomposition: per level, one warp per non-empty output row (l,z,x),
// walking the row's particles in chunks of <= 32 whose y-span is <= WIN cells.
// For a chunk with outputs in [y0, y1] the warp reconstructs, into a per-warp
// shared-memory tile S[kz*kx][W], the level-l image of the kz*kx neighbour
// rows over the window [y0-hy, y1+hy] -- the device analogue of LevelSlab's
// ring of padded planes (convolve.hpp:104-150) restricted to what the chunk
// reads.  The fill is fully warp-parallel:
//   round 0: the same-level leaf row and the level-l interior row of every
//            neighbour row (one lane per (row, source) task: row lookup +
//            lower_bound), then all lanes scatter the flattened candidate list;
//   round d: the level l-d leaf row covering each neighbour row, each particle
//            constant-upsampled to 2^d cells (fill_level_row,
//            reconstruct.hpp:45-58), repeated for d = 1, 2, ... only until
//            every in-domain cell of the tile is covered (a valid APR covers
//            each cell exactly once), so coarse depths that cannot contribute
//            are never scanned;
//   fixup:   out-of-domain y cells by reflect_index / zero, zero-pad rows.
// Each lane then evaluates one output particle in the reference's exact
// (az,ax,ay) order: fp64 FMA of exact products (bit-identical to
// LevelSlab::apply) in EXACT mode, fp32 FMA in FAST mode.  Optional RL
// epilogues fuse deconv.hpp:98-99 (ratio) and :102 (multiply).
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace aprgpu {
namespace {

struct ConvArgs {
    AccessView leaf, tree;
    const float* val;
    const float* tval;
    const uint32_t* work;
    uint64_t n_work;
    int l, kz, kx, ky;
    const float* wf;
    const double* wd;
    int pad;
    int tree_at_l;
    int win, wbuf;
    float* out;
    EpiArgs epi;
    int z_lo, z_hi;  // output rows processed: z in [z_lo, z_hi) (slab decomposition)
};

template <typename Acc>
__device__ __forceinline__ Acc fma_acc(Acc w, Acc u, Acc acc);
template <>
__device__ __forceinline__ double fma_acc<double>(double w, double u, double acc) {
    return __fma_rn(w, u, acc);
}
template <>
__device__ __forceinline__ float fma_acc<float>(float w, float u, float acc) {
    return __fmaf_rn(w, u, acc);
}

__device__ __forceinline__ float to_float(double v) { return __double2float_rn(v); }
__device__ __forceinline__ float to_float(float v) { return v; }

// Warp-parallel fill of one round of (row, source) tasks into S.
// round 0: tasks (q, src) for src in {leaf l, interior l}; round d>0: tasks q
// read the leaf row at level l-d.  Returns the number of cells written.
template <typename Acc>
__device__ int fill_round(const ConvArgs& a, int d, int z, int x, int wa, int ya, int yb, int KQ, int hz, int hx,
                          Acc* S, int* task, int lane) {
    const int l = a.l;
    const int nsrc = (d == 0) ? (1 + a.tree_at_l) : 1;
    const int T = KQ * nsrc;
    const LevelG gl = a.leaf.g[l];
    const int lo_key = ya >> d, hi_key = (yb - 1) >> d;
    int written = 0;
    for (int tb = 0; tb < T; tb += 32) {
        const int t = tb + lane;
        uint32_t s = 0;
        int cnt = 0, meta = 0;
        if (t < T) {
            const int q = t / nsrc;
            const int src = t - q * nsrc;  // 0 leaf, 1 interior (round 0 only)
            const int az = q / a.kx, ax = q - az * a.kx;
            int zs = z + hz - az, xs = x + hx - ax;
            const bool out_zx = zs < 0 || zs >= gl.zd || xs < 0 || xs >= gl.xd;
            if (!(out_zx && a.pad == APRGPU_PAD_ZERO)) {
                if (out_zx) {
                    zs = reflect_dev(zs, gl.zd);
                    xs = reflect_dev(xs, gl.xd);
                }
                const AccessView& av = src ? a.tree : a.leaf;
                const int ls = l - d;
                const LevelG g = av.g[ls];
                const int zr = zs >> d, xr = xs >> d;
                if (zr < g.zd && xr < g.xd) {
                    const uint32_t row = g.row0 + static_cast<uint32_t>(zr) * g.xd + xr;
                    const uint32_t b = __ldg(av.rb + row), e = __ldg(av.rb + row + 1);
                    if (e > b) {
                        s = lower_bound_u16(av.y, b, e, lo_key);
                        cnt = min(static_cast<int>(e - s), hi_key - lo_key + 1);
                        cnt = max(cnt, 0);
                    }
                }
            }
            meta = q | (src << 16);
        }
        const int incl = warp_incl_scan(cnt, lane);
        const int total = __shfl_sync(kFull, incl, 31);
        task[lane] = incl - cnt;  // exclusive offset
        task[32 + lane] = static_cast<int>(s);
        task[64 + lane] = meta;
        __syncwarp();
        for (int e = lane; e < total; e += 32) {
            // owning task: last t with off[t] <= e
            int lo = 0, hi = 31;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (task[mid] <= e) lo = mid; else hi = mid - 1;
            }
            const int m = task[64 + lo];
            const int q = m & 0xffff, src = m >> 16;
            const uint32_t idx = static_cast<uint32_t>(task[32 + lo]) + (e - task[lo]);
            const uint16_t* ys = src ? a.tree.y : a.leaf.y;
            const int yy = __ldg(ys + idx);
            if (yy > hi_key) continue;
            const float v = src ? __ldg(a.tval + idx) : __ldg(a.val + idx);
            const int c0 = max(yy << d, ya), c1 = min((yy + 1) << d, yb);
            Acc* dst = S + q * a.wbuf - wa;
            for (int c = c0; c < c1; ++c) dst[c] = static_cast<Acc>(v);
            written += max(c1 - c0, 0);
        }
        __syncwarp();
    }
    return warp_sum(written);
}

template <typename Acc, int KZ, int KX, int KY>
__global__ void __launch_bounds__(256) k_conv(ConvArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int kz = KZ ? KZ : a.kz, kx = KX ? KX : a.kx, ky = KY ? KY : a.ky;
    const int hz = kz >> 1, hx = kx >> 1, hy = ky >> 1;
    const int KQ = kz * kx, KW = KQ * ky;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nwb = blockDim.x >> 5;
    Acc* wsm = reinterpret_cast<Acc*>(smem);
    for (int i = threadIdx.x; i < KW; i += blockDim.x)
        wsm[i] = sizeof(Acc) == 8 ? static_cast<Acc>(a.wd[i]) : static_cast<Acc>(a.wf[i]);
    const size_t wbytes = (static_cast<size_t>(KW) * sizeof(Acc) + 15) & ~size_t(15);
    const size_t per_warp = ((128 * sizeof(int) + static_cast<size_t>(KQ) * a.wbuf * sizeof(Acc)) + 15) & ~size_t(15);
    int* task = reinterpret_cast<int*>(smem + wbytes + per_warp * wib);
    Acc* S = reinterpret_cast<Acc*>(task + 128);
    __syncthreads();

    const int l = a.l;
    const LevelG gl = a.leaf.g[l];
    const int yd = gl.yd;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * nwb;
    for (uint64_t wi = blockIdx.x * static_cast<uint64_t>(nwb) + wib; wi < a.n_work; wi += nwarps) {
        const uint32_t row = __ldg(a.work + wi);
        const uint32_t loc = row - gl.row0;
        const int z = static_cast<int>(loc / gl.xd), x = static_cast<int>(loc % gl.xd);
        if (z < a.z_lo || z >= a.z_hi) continue;  // another slab's rows
        const uint32_t rb = __ldg(a.leaf.rb + row), re = __ldg(a.leaf.rb + row + 1);
        // number of neighbour rows that are real (not zero-padded)
        int real_rows = 0;
        for (int q = lane; q < KQ; q += 32) {
            const int az = q / kx, ax = q - az * kx;
            const int zs = z + hz - az, xs = x + hx - ax;
            const bool out_zx = zs < 0 || zs >= gl.zd || xs < 0 || xs >= gl.xd;
            real_rows += (out_zx && a.pad == APRGPU_PAD_ZERO) ? 0 : 1;
        }
        real_rows = warp_sum(real_rows);
        const bool has_zero_rows = real_rows < KQ;
        for (uint32_t c0 = rb; c0 < re;) {
            const uint32_t i = c0 + lane;
            const int yv = i < re ? static_cast<int>(__ldg(a.leaf.y + i)) : (1 << 30);
            const int y0 = __shfl_sync(kFull, yv, 0);
            const bool mine = i < re && yv < y0 + a.win;
            const unsigned mask = __ballot_sync(kFull, mine);
            const int n = __popc(mask);
            const int y1 = __shfl_sync(kFull, yv, n - 1);
            const int wa = y0 - hy, wb = y1 + hy + 1;
            const int ya = max(wa, 0), yb = min(wb, yd);
            const int needed = real_rows * (yb - ya);
            int covered = fill_round<Acc>(a, 0, z, x, wa, ya, yb, KQ, hz, hx, S, task, lane);
            for (int d = 1; covered < needed && l - d >= a.leaf.l_min; ++d)
                covered += fill_round<Acc>(a, d, z, x, wa, ya, yb, KQ, hz, hx, S, task, lane);
            if (covered < needed) {
                // malformed APR with uncovered cells: make holes deterministic (0)
                for (int q = 0; q < KQ; ++q)
                    for (int c = ya + lane; c < yb; c += 32) S[q * a.wbuf + c - wa] = Acc(0);
                __syncwarp();
                for (int d = 0; l - d >= a.leaf.l_min; ++d)
                    fill_round<Acc>(a, d, z, x, wa, ya, yb, KQ, hz, hx, S, task, lane);
            }
            if (wa < 0 || wb > yd || has_zero_rows) {
                __syncwarp();
                const int W = wb - wa;
                for (int q = 0; q < KQ; ++q) {
                    const int az = q / kx, ax = q - az * kx;
                    const int zs = z + hz - az, xs = x + hx - ax;
                    const bool zero_row =
                        a.pad == APRGPU_PAD_ZERO && (zs < 0 || zs >= gl.zd || xs < 0 || xs >= gl.xd);
                    Acc* Sq = S + q * a.wbuf;
                    for (int c = lane; c < W; c += 32) {
                        const int yy = wa + c;
                        if (zero_row) {
                            Sq[c] = Acc(0);
                        } else if (yy < 0 || yy >= yd) {
                            Sq[c] = a.pad == APRGPU_PAD_ZERO ? Acc(0) : Sq[reflect_dev(yy, yd) - wa];
                        }
                    }
                }
            }
            __syncwarp();
            if (mine) {
                Acc acc = Acc(0);
                const Acc* base = S + (yv + hy - wa);
                if (KZ) {
#pragma unroll
                    for (int az = 0; az < KZ; ++az)
#pragma unroll
                        for (int ax = 0; ax < KX; ++ax) {
                            const Acc* r = base + (az * KX + ax) * a.wbuf;
                            const Acc* wr = wsm + (az * KX + ax) * KY;
#pragma unroll
                            for (int ay = 0; ay < KY; ++ay) acc = fma_acc<Acc>(wr[ay], r[-ay], acc);
                        }
                } else {
                    for (int az = 0; az < kz; ++az)
                        for (int ax = 0; ax < kx; ++ax) {
                            const Acc* r = base + (az * kx + ax) * a.wbuf;
                            const Acc* wr = wsm + (az * kx + ax) * ky;
                            for (int ay = 0; ay < ky; ++ay) acc = fma_acc<Acc>(wr[ay], r[-ay], acc);
                        }
                }
                const float o = to_float(acc);
                if (a.epi.mode == EPI_STORE) {
                    a.out[i] = o;
                } else if (a.epi.mode == EPI_RL_RATIO) {
                    a.out[i] = rl_ratio(__ldg(a.epi.u + i), o, a.epi.eps);  // deconv.hpp:98-99
                } else {
                    // deconv.hpp:102: estimate *= corr
                    a.epi.est[i] = __fmul_rn(a.epi.est[i], o);
                }
            }
            __syncwarp();
            c0 += static_cast<uint32_t>(n);
        }
    }
}

template <typename Acc, int KZ, int KX, int KY>
void launch_conv(aprgpu_ctx* ctx, ConvArgs& a, cudaStream_t s) {
    const int KQ = a.kz * a.kx, KW = KQ * a.ky;
    const int hy = a.ky / 2;
    a.win = (KQ <= 49) ? 64 : 32;
    a.wbuf = a.win + 2 * hy;
    const size_t wbytes = (static_cast<size_t>(KW) * sizeof(Acc) + 15) & ~size_t(15);
    const size_t per_warp = ((128 * sizeof(int) + static_cast<size_t>(KQ) * a.wbuf * sizeof(Acc)) + 15) & ~size_t(15);
    const size_t budget = 200 * 1024;
    int nw = 8;
    while (nw > 1 && wbytes + per_warp * nw > budget) --nw;
    const size_t smem = wbytes + per_warp * nw;
    if (smem > 227 * 1024) fail(APRGPU_ERR_CAPABILITY, "stencil too large for the shared-memory tile");
    static OncePerDevice attr;  // per instantiation and device
    attr([] {
        APR_CUDA(cudaFuncSetAttribute(k_conv<Acc, KZ, KX, KY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    });
    const uint64_t blocks64 = (a.n_work + nw - 1) / nw;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(blocks64, 1u << 30));
    k_conv<Acc, KZ, KX, KY><<<grid, nw * 32, smem, s>>>(a);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
}

template <typename Acc>
void dispatch(aprgpu_ctx* ctx, ConvArgs& a, cudaStream_t s) {
    if (a.kz == 3 && a.kx == 3 && a.ky == 3) return launch_conv<Acc, 3, 3, 3>(ctx, a, s);
    if (a.kz == 5 && a.kx == 5 && a.ky == 5) return launch_conv<Acc, 5, 5, 5>(ctx, a, s);
    if (a.kz == 1 && a.kx == 1 && a.ky == 1) return launch_conv<Acc, 1, 1, 1>(ctx, a, s);
    return launch_conv<Acc, 0, 0, 0>(ctx, a, s);
}

bool use_tiles() {
    static const bool on = [] {
        const char* e = std::getenv("APRGPU_CONV_KERNEL");
        return !(e && std::string(e) == "rows");
    }();
    return on;
}

}  // namespace

void check_pyramid(const aprgpu_apr* apr, const aprgpu_pyramid* pyr) {
    const DevAccess& L = apr->leaf;
    if (pyr->l_min > L.l_min || pyr->l_max < L.l_max)
        fail(APRGPU_ERR_RANGE, "convolve_apr: pyramid does not cover the APR levels");
    for (int l = L.l_min; l <= L.l_max; ++l) {
        const int* k = &pyr->k3[3 * (l - pyr->l_min)];
        if (k[0] > kMaxExtent || k[1] > kMaxExtent || k[2] > kMaxExtent)
            fail(APRGPU_ERR_CAPABILITY, "convolve_apr: stencil extent exceeds the supported maximum");
    }
}

void convolve_device(aprgpu_apr* apr, const float* values, const float* tree_values, const aprgpu_pyramid* pyr,
                     int pad, int accum, float* out, const EpiArgs& epi, cudaStream_t s, const Slab& slab) {
    check_pyramid(apr, pyr);
    const DevAccess& L = apr->leaf;
    const DevAccess& T = apr->tree;
    ConvArgs a{};
    a.leaf = L.view();
    a.tree = T.view();
    a.val = values;
    a.tval = tree_values;
    a.pad = pad;
    a.out = out;
    a.epi = epi;
    bool done[kMaxLevels] = {};
    if (use_tiles()) conv_tile_levels(apr, pyr, values, tree_values, pad, accum, out, epi, slab, s, done);
    for (int l = L.l_max; l >= L.l_min; --l) {
        if (done[l] || (l < slab.lc && !slab.rep)) continue;
        a.n_work = L.work_off[l + 1] - L.work_off[l];
        if (a.n_work == 0) continue;
        a.work = L.work + L.work_off[l];
        a.l = l;
        const int li = l - pyr->l_min;
        a.kz = pyr->k3[3 * li];
        a.kx = pyr->k3[3 * li + 1];
        a.ky = pyr->k3[3 * li + 2];
        a.wf = pyr->w_dev + pyr->off[li];
        a.wd = pyr->wd_dev + pyr->off[li];
        a.tree_at_l = (T.n_particles > 0 && l >= T.l_min && l <= T.l_max) ? 1 : 0;
        a.z_lo = 0;
        a.z_hi = 1 << 30;
        if (l >= slab.lc) {
            const int sh = L.l_max - l;
            a.z_lo = slab.z_lo >> sh;
            a.z_hi = (slab.z_hi + (1 << sh) - 1) >> sh;
        }
        if (accum == APRGPU_ACCUM_EXACT)
            dispatch<double>(apr->ctx, a, s);
        else
            dispatch<float>(apr->ctx, a, s);
    }
}

}  // namespace aprgpu
