// APR tree on the device: structure (init_tree_structure, tree.hpp:26-82),
// parent-link verification (synchronized_parent_pass, tree.hpp:88-103) and the
// footprint-weighted fill (fill_tree, tree.hpp:110-150).
//
// Structure: level by level from l_max-1 down, one warp per parent row merges
// the y/2 values of its <= 8 child rows (4 leaf rows + 4 interior rows of the
// level below) through a shared-memory bitmap; a count pass, an exclusive scan
// and a fill pass produce the CSR rows.  Sets are order-free, so the result is
// bit-identical to the reference's push/sort/unique.
//
// Fill: level by level from the finest interior level, one warp per non-empty
// parent row, one lane per parent node.  Each node gathers its children in the
// reference's exact accumulation order -- for (cz,cx) in lexicographic order:
// leaf children y=2py, 2py+1, then interior children y=2py, 2py+1 -- with
// explicit fp64 round-to-nearest multiplies/adds (no FMA contraction), so the
// fp64 sums and the final float(vsum/wsum) are bit-identical to the reference.
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace aprgpu {
namespace {

constexpr int kTreeWarps = 8;
constexpr int kBitmapWords = 1024;  // 32768 bits: every parent y (< 32768) fits

struct ChildSrc {
    AccessView leaf;
    int leaf_ok;                 // child level is a leaf level
    const uint32_t* trb;         // interior child level (level-local row begins), or null
    const uint16_t* ty;
    int czd, cxd;                // child grid dims (reference geometry, glm)
    int ctxd;                    // x dim of the interior child level
};

// mode 0: counts[r] = |row|; mode 1: out_y[prb[r] ...] = sorted row
__global__ void __launch_bounds__(kTreeWarps * 32) k_tree_level(int mode, ChildSrc cs, int child_l, int zd, int xd,
                                                                  uint32_t* __restrict__ counts,
                                                                  const uint32_t* __restrict__ prb,
                                                                  uint16_t* __restrict__ out_y) {
    __shared__ uint32_t bm_all[kTreeWarps][kBitmapWords];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint32_t* bm = bm_all[wib];
    const uint64_t n_rows = static_cast<uint64_t>(zd) * xd;
    for (uint64_t r = blockIdx.x * (uint64_t)kTreeWarps + wib; r < n_rows; r += (uint64_t)gridDim.x * kTreeWarps) {
        const int z = static_cast<int>(r / xd), x = static_cast<int>(r % xd);
        // lanes 0..7 describe the child lists: k<4 leaf rows, k>=4 interior rows
        uint32_t lb = 0, le = 0;
        int src = 0;
        if (lane < 8) {
            const int k = lane & 3;
            const int cz = 2 * z + (k >> 1), cx = 2 * x + (k & 1);
            if (cz < cs.czd && cx < cs.cxd) {
                if (lane < 4 && cs.leaf_ok) {
                    const uint32_t row = cs.leaf.g[child_l].row0 + static_cast<uint32_t>(cz) * cs.leaf.g[child_l].xd + cx;
                    lb = cs.leaf.rb[row];
                    le = cs.leaf.rb[row + 1];
                    src = 0;
                } else if (lane >= 4 && cs.trb) {
                    const uint32_t row = static_cast<uint32_t>(cz) * cs.ctxd + cx;
                    lb = cs.trb[row];
                    le = cs.trb[row + 1];
                    src = 1;
                }
            }
        }
        int mn = 1 << 30, mx = -1;
        if (le > lb) {
            const uint16_t* ys = src ? cs.ty : cs.leaf.y;
            mn = ys[lb] >> 1;
            mx = ys[le - 1] >> 1;
        }
        mn = warp_min(mn);
        mx = warp_max(mx);
        if (mx < 0) {
            if (mode == 0 && lane == 0) counts[r] = 0;
            continue;
        }
        const int nwords = ((mx - mn) >> 5) + 1;
        for (int w = lane; w < nwords; w += 32) bm[w] = 0;
        __syncwarp();
        for (int k = 0; k < 8; ++k) {
            const uint32_t b = __shfl_sync(kFull, lb, k), e = __shfl_sync(kFull, le, k);
            const int sk = __shfl_sync(kFull, src, k);
            const uint16_t* ys = sk ? cs.ty : cs.leaf.y;
            for (uint32_t i = b + lane; i < e; i += 32) {
                const int v = (ys[i] >> 1) - mn;
                atomicOr(&bm[v >> 5], 1u << (v & 31));
            }
        }
        __syncwarp();
        if (mode == 0) {
            int c = 0;
            for (int w = lane; w < nwords; w += 32) c += __popc(bm[w]);
            c = warp_sum(c);
            if (lane == 0) counts[r] = static_cast<uint32_t>(c);
        } else {
            uint32_t base = prb[r];
            for (int w0 = 0; w0 < nwords; w0 += 32) {
                const int w = w0 + lane;
                uint32_t word = w < nwords ? bm[w] : 0u;
                const int pc = __popc(word);
                const int incl = warp_incl_scan(pc, lane);
                uint32_t pos = base + incl - pc;
                while (word) {
                    const int bit = __ffs(word) - 1;
                    out_y[pos++] = static_cast<uint16_t>(mn + (w << 5) + bit);
                    word &= word - 1;
                }
                base += __shfl_sync(kFull, incl, 31);
            }
        }
        __syncwarp();
    }
}

__global__ void k_assemble_rb(const uint32_t* __restrict__ local, uint64_t rows, uint32_t row0, uint32_t poff,
                              uint32_t* __restrict__ rb) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x)
        rb[row0 + r + 1] = poff + local[r + 1];
}

// IntegrityError check of synchronized_parent_pass (tree.hpp:96-100): every
// child (leaf at level c, or interior node at level c) has its parent y/2 in
// interior row (c-1, z/2, x/2).
__global__ void k_verify_links(AccessView child, AccessView tree, int c, uint64_t n_rows, int* bad) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const LevelG g = child.g[c];
    const LevelG pg = tree.g[c - 1];
    for (uint64_t r = warp; r < n_rows; r += nwarps) {
        const int z = static_cast<int>(r / g.xd), x = static_cast<int>(r % g.xd);
        const uint32_t b = child.rb[g.row0 + r], e = child.rb[g.row0 + r + 1];
        if (b == e) continue;
        if ((z >> 1) >= pg.zd || (x >> 1) >= pg.xd) {
            if (lane == 0) atomicOr(bad, 1);
            continue;
        }
        const uint32_t prow = pg.row0 + static_cast<uint32_t>(z >> 1) * pg.xd + (x >> 1);
        const uint32_t pb = tree.rb[prow], pe = tree.rb[prow + 1];
        for (uint32_t i = b + lane; i < e; i += 32) {
            const int t = child.y[i] >> 1;
            const uint32_t j = lower_bound_u16(tree.y, pb, pe, t);
            if (j == pe || tree.y[j] != t) atomicOr(bad, 1);
        }
    }
}

__device__ __forceinline__ double footprint_dev(int l, int iz, int ix, int iy, int glm, int nz, int nx, int ny) {
    // cell_footprint_volume (tree.hpp:15-22)
    const int s = 1 << (glm - l);
    if ((iz + 1) * s <= nz && (ix + 1) * s <= nx && (iy + 1) * s <= ny)  // unclipped: s^3, exactly (< 2^53)
        return static_cast<double>(s) * static_cast<double>(s) * static_cast<double>(s);
    const double dz = min((iz + 1) * s, nz) - iz * s;
    const double dx = min((ix + 1) * s, nx) - ix * s;
    const double dy = min((iy + 1) * s, ny) - iy * s;
    return __dmul_rn(__dmul_rn(dz, dx), dy);
}

// Child links of an interior node, one word per child row k (k = 0..3: leaf
// rows (2pz + k/2, 2px + k%2); k = 4..7: the interior rows): b | f0 << 30 |
// f1 << 31, b = lower_bound of 2py in the child row, f0 / f1 = children
// y = 2py / 2py + 1 present (at b and b + f0).  Structure only: built once per
// APR (the searches of synchronized_parent_pass, tree.hpp:88-103), then every
// fill is a gather.
struct Links {
    uint4 leaf, tree;
};
__device__ __forceinline__ uint32_t link_of(const uint16_t* y, uint32_t b, uint32_t e, int y0) {
    if (e <= b) return 0;
    const uint32_t i = lower_bound_u16(y, b, e, y0);
    const uint32_t f0 = (i < e && y[i] == y0) ? 1u : 0u;
    const uint32_t f1 = (i + f0 < e && y[i + f0] == y0 + 1) ? 1u : 0u;
    return i | f0 << 30 | f1 << 31;
}

struct FillArgs {
    AccessView leaf, tree;
    const float* leaf_v;
    double* vsum;
    double* wsum;
    const uint32_t* work;  // non-empty interior rows at level lt
    uint64_t n_work;
    int lt, c, leaf_ok, tree_ok;  // c = lt+1; children are leaves / interior nodes
    int czd, cxd, glm, nz, nx, ny;
    int pz_lo, pz_hi;  // parent rows processed: z in [pz_lo, pz_hi) (slab decomposition)
    Links* links;  // per interior node (written by the BUILD pass)
    float* tree_out;  // the fill's float result, written with the sums (nullptr: sums only, slab path)
};

template <bool BUILD>
__global__ void __launch_bounds__(256) k_fill_tree_level(FillArgs a) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const LevelG pg = a.tree.g[a.lt];
    for (uint64_t wi = warp; wi < a.n_work; wi += nwarps) {
        const uint32_t prow = a.work[wi];
        const uint32_t loc = prow - pg.row0;
        const int pz = static_cast<int>(loc / pg.xd), px = static_cast<int>(loc % pg.xd);
        if (pz < a.pz_lo || pz >= a.pz_hi) continue;  // another slab's rows
        const uint32_t pb = a.tree.rb[prow], pe = a.tree.rb[prow + 1];
        // child row ranges (4 leaf + 4 interior), held by lanes 0..7 and broadcast
        // (the BUILD pass only: the fill reads the links)
        uint32_t cb = 0, ce = 0;
        if (BUILD && lane < 8) {
            const int k = lane & 3;
            const int cz = 2 * pz + (k >> 1), cx = 2 * px + (k & 1);
            if (cz < a.czd && cx < a.cxd) {
                if (lane < 4 && a.leaf_ok) {
                    const LevelG g = a.leaf.g[a.c];
                    const uint32_t row = g.row0 + static_cast<uint32_t>(cz) * g.xd + cx;
                    cb = a.leaf.rb[row];
                    ce = a.leaf.rb[row + 1];
                } else if (lane >= 4 && a.tree_ok) {
                    const LevelG g = a.tree.g[a.c];
                    const uint32_t row = g.row0 + static_cast<uint32_t>(cz) * g.xd + cx;
                    cb = a.tree.rb[row];
                    ce = a.tree.rb[row + 1];
                }
            }
        }
        uint32_t rbk[8], rek[8];
        if (BUILD) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                rbk[k] = __shfl_sync(kFull, cb, k);
                rek[k] = __shfl_sync(kFull, ce, k);
            }
        }
        for (uint32_t j = pb + lane; j < pe; j += 32) {
            const int py = a.tree.y[j];
            const int y0 = 2 * py;
            if (BUILD) {
                uint32_t w[8];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    w[k] = link_of(a.leaf.y, rbk[k], rek[k], y0);
                    w[k + 4] = link_of(a.tree.y, rbk[k + 4], rek[k + 4], y0);
                }
                a.links[j] = Links{make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7])};
                continue;
            }
            const Links lk = a.links[j];
            const uint32_t wl[4] = {lk.leaf.x, lk.leaf.y, lk.leaf.z, lk.leaf.w};
            const uint32_t wt[4] = {lk.tree.x, lk.tree.y, lk.tree.z, lk.tree.w};
            double vs = 0.0, ws = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int cz = 2 * pz + (k >> 1), cx = 2 * px + (k & 1);
                // leaf children (tree.hpp:124-132): w * value, w = clipped footprint
                {
                    const uint32_t b = wl[k] & 0x3fffffffu, f0 = (wl[k] >> 30) & 1u, f1 = wl[k] >> 31;
                    if (f0) {
                        const double w = footprint_dev(a.c, cz, cx, y0, a.glm, a.nz, a.nx, a.ny);
                        vs = __dadd_rn(vs, __dmul_rn(w, static_cast<double>(a.leaf_v[b])));
                        ws = __dadd_rn(ws, w);
                    }
                    if (f1) {
                        const double w = footprint_dev(a.c, cz, cx, y0 + 1, a.glm, a.nz, a.nx, a.ny);
                        vs = __dadd_rn(vs, __dmul_rn(w, static_cast<double>(a.leaf_v[b + f0])));
                        ws = __dadd_rn(ws, w);
                    }
                }
                // interior children (tree.hpp:133-139): their own fp64 sums
                {
                    const uint32_t b = wt[k] & 0x3fffffffu, f0 = (wt[k] >> 30) & 1u, f1 = wt[k] >> 31;
                    if (f0) {
                        vs = __dadd_rn(vs, a.vsum[b]);
                        ws = __dadd_rn(ws, a.wsum[b]);
                    }
                    if (f1) {
                        vs = __dadd_rn(vs, a.vsum[b + f0]);
                        ws = __dadd_rn(ws, a.wsum[b + f0]);
                    }
                }
            }
            a.vsum[j] = vs;
            a.wsum[j] = ws;
            if (a.tree_out) a.tree_out[j] = ws > 0.0 ? __double2float_rn(__ddiv_rn(vs, ws)) : 0.0f;  // tree.hpp:146-148
        }
    }
}

// The fill of a level whose child cells are never clipped by the image edge
// (every dim a multiple of the child cell size -- C3, C4): every leaf child
// weighs s^3, so a node needs only its links -- one thread per node over the
// level's contiguous node range, no row walk.  Same per-node order and
// operations as k_fill_tree_level (bit-identical).
__device__ __forceinline__ void fill_node_flat(const FillArgs& a, uint32_t j, double w) {
    const Links lk = a.links[j];
    const uint32_t wl[4] = {lk.leaf.x, lk.leaf.y, lk.leaf.z, lk.leaf.w};
    const uint32_t wt[4] = {lk.tree.x, lk.tree.y, lk.tree.z, lk.tree.w};
    double vs = 0.0, ws = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        {
            const uint32_t b = wl[k] & 0x3fffffffu, f0 = (wl[k] >> 30) & 1u, f1 = wl[k] >> 31;
            if (f0) {
                vs = __dadd_rn(vs, __dmul_rn(w, static_cast<double>(a.leaf_v[b])));
                ws = __dadd_rn(ws, w);
            }
            if (f1) {
                vs = __dadd_rn(vs, __dmul_rn(w, static_cast<double>(a.leaf_v[b + f0])));
                ws = __dadd_rn(ws, w);
            }
        }
        {
            const uint32_t b = wt[k] & 0x3fffffffu, f0 = (wt[k] >> 30) & 1u, f1 = wt[k] >> 31;
            if (f0) {
                vs = __dadd_rn(vs, a.vsum[b]);
                ws = __dadd_rn(ws, a.wsum[b]);
            }
            if (f1) {
                vs = __dadd_rn(vs, a.vsum[b + f0]);
                ws = __dadd_rn(ws, a.wsum[b + f0]);
            }
        }
    }
    a.vsum[j] = vs;
    a.wsum[j] = ws;
    if (a.tree_out) a.tree_out[j] = ws > 0.0 ? __double2float_rn(__ddiv_rn(vs, ws)) : 0.0f;  // tree.hpp:146-148
}

__global__ void __launch_bounds__(256) k_fill_tree_flat(FillArgs a, uint32_t n0, uint32_t n1, double w) {
    for (uint32_t j = n0 + blockIdx.x * blockDim.x + threadIdx.x; j < n1; j += gridDim.x * blockDim.x)
        fill_node_flat(a, j, w);
}

// The small coarse levels (flat-eligible) in ONE block, level after level with
// a block barrier between them, instead of a launch each.
struct CoarseLevels {
    int n;
    uint32_t n0[kMaxLevels], n1[kMaxLevels];
    double w[kMaxLevels];
};
__global__ void __launch_bounds__(1024) k_fill_tree_coarse(FillArgs a, CoarseLevels c) {
    for (int i = 0; i < c.n; ++i) {
        for (uint32_t j = c.n0[i] + threadIdx.x; j < c.n1[i]; j += blockDim.x) fill_node_flat(a, j, c.w[i]);
        __syncthreads();
    }
}

__global__ void k_tree_finalize(const double* __restrict__ vsum, const double* __restrict__ wsum, uint64_t n,
                                float* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double w = wsum[i];
        out[i] = w > 0.0 ? __double2float_rn(__ddiv_rn(vsum[i], w)) : 0.0f;  // tree.hpp:146-148
    }
}

int compute_l_max_host(int nz, int nx, int ny) {
    const int m = std::max(nz, std::max(nx, ny));
    int l = 0;
    while ((1 << l) < m) ++l;
    return l;
}

}  // namespace

void build_tree_structure(aprgpu_ctx* ctx, aprgpu_apr* apr) {
    cudaStream_t s = ctx->stream;
    const DevAccess& L = apr->leaf;
    DevAccess& T = apr->tree;
    const int glm = L.l_max;
    const int* d = apr->dims;
    const int tmax = L.l_max - 1;
    const int tmin = std::max(L.l_min - 1, 0);
    if (tmax < tmin) {  // tree.hpp:31-42: single-cell domain, no interior nodes
        T.l_min = T.l_max = 0;
        T.zd = {grid_dim_dev(d[0], glm, 0)};
        T.xd = {grid_dim_dev(d[1], glm, 0)};
        T.yd = {grid_dim_dev(d[2], glm, 0)};
        T.level_offset = {0};
        T.n_rows = static_cast<uint64_t>(T.zd[0]) * T.xd[0];
        T.n_particles = 0;
        APR_CUDA(cudaMalloc(&T.y, 2));
        APR_CUDA(cudaMalloc(&T.rb, sizeof(uint32_t) * (T.n_rows + 1)));
        APR_CUDA(cudaMemsetAsync(T.rb, 0, sizeof(uint32_t) * (T.n_rows + 1), s));
        build_work_lists(ctx, T);
        return;
    }
    const int geom = std::max(tmax, compute_l_max_host(d[0], d[1], d[2]));  // assemble_access, linear_access.hpp:110
    // per-level temporaries (level-local row begins + y)
    std::vector<GpuBuf> lrb(tmax + 1), ly(tmax + 1);
    std::vector<uint64_t> lcount(tmax + 1, 0);
    GpuBuf counts, scan_tmp;
    const AccessView lv = L.view();
    for (int lt = tmax; lt >= tmin; --lt) {
        const int zd = grid_dim_dev(d[0], glm, lt), xd = grid_dim_dev(d[1], glm, lt);
        if (grid_dim_dev(d[0], geom, lt) != zd || grid_dim_dev(d[1], geom, lt) != xd)
            fail(APRGPU_ERR_RANGE, "assemble_access: row list does not match level grids");
        const int c = lt + 1;
        const uint64_t rows = static_cast<uint64_t>(zd) * xd;
        ChildSrc cs{};
        cs.leaf = lv;
        cs.leaf_ok = (c >= L.l_min && c <= L.l_max) ? 1 : 0;
        cs.czd = grid_dim_dev(d[0], glm, c);
        cs.cxd = grid_dim_dev(d[1], glm, c);
        if (c <= tmax) {
            cs.trb = lrb[c].as<uint32_t>();
            cs.ty = ly[c].as<uint16_t>();
            cs.ctxd = grid_dim_dev(d[1], glm, c);
        }
        counts.ensure(sizeof(uint32_t) * (rows + 1));
        lrb[lt].ensure(sizeof(uint32_t) * (rows + 1));
        APR_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * (rows + 1), s));
        const unsigned grid = std::min<unsigned>(blocks_for(rows, kTreeWarps), ctx->sm_count * 8);
        k_tree_level<<<grid, kTreeWarps * 32, 0, s>>>(0, cs, c, zd, xd, counts.as<uint32_t>(), nullptr, nullptr);
        APR_CUDA(cudaGetLastError());
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.as<uint32_t>(), lrb[lt].as<uint32_t>(),
                                      static_cast<int64_t>(rows + 1), s);
        scan_tmp.ensure(tb + 16);
        tb = scan_tmp.bytes;
        APR_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp.p, tb, counts.as<uint32_t>(), lrb[lt].as<uint32_t>(),
                                               static_cast<int64_t>(rows + 1), s));
        uint32_t total = 0;
        APR_CUDA(cudaMemcpyAsync(&total, lrb[lt].as<uint32_t>() + rows, 4, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
        lcount[lt] = total;
        ly[lt].ensure(2ull * total + 2);
        k_tree_level<<<grid, kTreeWarps * 32, 0, s>>>(1, cs, c, zd, xd, nullptr, lrb[lt].as<uint32_t>(),
                                                      ly[lt].as<uint16_t>());
        APR_CUDA(cudaGetLastError());
        count_launch(ctx, 3);
    }
    // assemble levels tmin..tmax (assemble_access, linear_access.hpp:101-130)
    T.l_min = tmin;
    T.l_max = tmax;
    T.zd.assign(tmax + 1, 0);
    T.xd.assign(tmax + 1, 0);
    T.yd.assign(tmax + 1, 0);
    T.level_offset.assign(tmax + 1, 0);
    uint64_t nrow = 0, np = 0;
    for (int lt = tmin; lt <= tmax; ++lt) {
        T.zd[lt] = grid_dim_dev(d[0], geom, lt);
        T.xd[lt] = grid_dim_dev(d[1], geom, lt);
        T.yd[lt] = grid_dim_dev(d[2], geom, lt);
        T.level_offset[lt] = nrow;
        nrow += static_cast<uint64_t>(T.zd[lt]) * T.xd[lt];
        np += lcount[lt];
    }
    if (np >= (1ull << 32)) fail(APRGPU_ERR_CAPABILITY, "interior node count exceeds u32");
    T.n_rows = nrow;
    T.n_particles = np;
    APR_CUDA(cudaMalloc(&T.y, 2 * np + 2));
    APR_CUDA(cudaMalloc(&T.rb, sizeof(uint32_t) * (nrow + 1)));
    APR_CUDA(cudaMemsetAsync(T.rb, 0, sizeof(uint32_t), s));
    uint64_t poff = 0;
    for (int lt = tmin; lt <= tmax; ++lt) {
        const uint64_t rows = static_cast<uint64_t>(T.zd[lt]) * T.xd[lt];
        if (lcount[lt])
            APR_CUDA(cudaMemcpyAsync(T.y + poff, ly[lt].p, 2 * lcount[lt], cudaMemcpyDeviceToDevice, s));
        k_assemble_rb<<<std::min<unsigned>(blocks_for(rows, 256), ctx->sm_count * 8), 256, 0, s>>>(
            lrb[lt].as<uint32_t>(), rows, static_cast<uint32_t>(T.level_offset[lt]), static_cast<uint32_t>(poff), T.rb);
        APR_CUDA(cudaGetLastError());
        count_launch(ctx);
        poff += lcount[lt];
    }
    APR_CUDA(cudaStreamSynchronize(s));
    for (auto& b : lrb) b.release();
    for (auto& b : ly) b.release();
    build_work_lists(ctx, T);
}

void verify_tree_links(aprgpu_ctx* ctx, aprgpu_apr* apr) {
    cudaStream_t s = ctx->stream;
    const DevAccess& L = apr->leaf;
    const DevAccess& T = apr->tree;
    GpuBuf flag;
    flag.ensure(sizeof(int));
    APR_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    const AccessView lv = L.view(), tv = T.view();
    for (int c = std::max(L.l_min, T.l_min + 1); c <= std::min(L.l_max, T.l_max + 1); ++c) {
        const uint64_t rows = static_cast<uint64_t>(L.zd[c]) * L.xd[c];
        k_verify_links<<<std::min<unsigned>(blocks_for(rows * 32, 256), ctx->sm_count * 8), 256, 0, s>>>(
            lv, tv, c, rows, flag.as<int>());
        count_launch(ctx);
    }
    for (int c = T.l_min + 1; c <= T.l_max; ++c) {
        const uint64_t rows = static_cast<uint64_t>(T.zd[c]) * T.xd[c];
        k_verify_links<<<std::min<unsigned>(blocks_for(rows * 32, 256), ctx->sm_count * 8), 256, 0, s>>>(
            tv, tv, c, rows, flag.as<int>());
        count_launch(ctx);
    }
    APR_CUDA(cudaGetLastError());
    int bad = 0;
    APR_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    APR_CUDA(cudaStreamSynchronize(s));
    if (bad) fail(APRGPU_ERR_INTEGRITY, "synchronized_parent_pass: missing parent for a child node");
}

namespace {

// Per-level launch parameters of the parent-row kernels (k_fill_tree_level,
// k_partition_check) for interior level lt.
void set_fill_level(FillArgs& a, const DevAccess& L, const DevAccess& T, int lt) {
    a.lt = lt;
    a.c = lt + 1;
    a.leaf_ok = (a.c >= L.l_min && a.c <= L.l_max) ? 1 : 0;
    a.tree_ok = (a.c <= T.l_max) ? 1 : 0;
    a.czd = grid_dim_dev(a.nz, a.glm, a.c);
    a.cxd = grid_dim_dev(a.nx, a.glm, a.c);
    a.pz_lo = 0;
    a.pz_hi = 1 << 30;
    a.work = T.work + T.work_off[lt];
    a.n_work = T.work_off[lt + 1] - T.work_off[lt];
}

FillArgs base_fill_args(aprgpu_apr* apr) {
    FillArgs a{};
    a.leaf = apr->leaf.view();
    a.tree = apr->tree.view();
    a.glm = apr->leaf.l_max;
    a.nz = apr->dims[0];
    a.nx = apr->dims[1];
    a.ny = apr->dims[2];
    return a;
}

// Domain-partition check of validate (apr.hpp:103-131) without pixels: one lane
// per interior node; every child cell whose origin lies in the image must be a
// leaf or an interior node, and not both.  (Leaves never have a leaf ancestor
// then: the ancestor would be an interior node too.)  min_unc = smallest
// uncovered pixel's flat index (a cell's smallest pixel is its origin).
__global__ void __launch_bounds__(256) k_partition_check(FillArgs a, int* dbl, unsigned long long* min_unc) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const LevelG pg = a.tree.g[a.lt];
    const int s = 1 << (a.glm - a.c);  // child cell size
    for (uint64_t wi = warp; wi < a.n_work; wi += nwarps) {
        const uint32_t prow = a.work[wi];
        const uint32_t loc = prow - pg.row0;
        const int pz = static_cast<int>(loc / pg.xd), px = static_cast<int>(loc % pg.xd);
        const uint32_t pb = a.tree.rb[prow], pe = a.tree.rb[prow + 1];
        for (uint32_t j = pb + lane; j < pe; j += 32) {
            const int py = a.tree.y[j];
            const Links lk = a.links[j];
            const uint32_t wl[4] = {lk.leaf.x, lk.leaf.y, lk.leaf.z, lk.leaf.w};
            const uint32_t wt[4] = {lk.tree.x, lk.tree.y, lk.tree.z, lk.tree.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int cz = 2 * pz + (k >> 1), cx = 2 * px + (k & 1);
                if (static_cast<int64_t>(cz) * s >= a.nz || static_cast<int64_t>(cx) * s >= a.nx) continue;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int cy = 2 * py + t;
                    if (static_cast<int64_t>(cy) * s >= a.ny) continue;
                    const uint32_t fl = a.leaf_ok ? (wl[k] >> (30 + t)) & 1u : 0u;
                    const uint32_t ft = a.tree_ok ? (wt[k] >> (30 + t)) & 1u : 0u;
                    if (fl && ft) atomicOr(dbl, 1);
                    if (!fl && !ft) {
                        const unsigned long long px0 =
                            (static_cast<unsigned long long>(cz) * s * a.nx + static_cast<unsigned long long>(cx) * s) *
                                a.ny +
                            static_cast<unsigned long long>(cy) * s;
                        atomicMin(min_unc, px0);
                    }
                }
            }
        }
    }
}

}  // namespace

// Child links of every interior node (structure only; built on first use).
void ensure_tree_links(aprgpu_apr* apr, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(apr->init_mu);
    if (apr->tree_links.p) return;
    const DevAccess& L = apr->leaf;
    const DevAccess& T = apr->tree;
    if (T.n_particles == 0) return;
    if (L.n_particles >= (1ull << 30) || T.n_particles >= (1ull << 30))
        fail(APRGPU_ERR_CAPABILITY, "fill_tree: child links need fewer than 2^30 particles per access");
    apr->tree_links.ensure(sizeof(Links) * T.n_particles);
    FillArgs a = base_fill_args(apr);
    a.links = apr->tree_links.as<Links>();
    for (int lt = T.l_max; lt >= T.l_min; --lt) {
        set_fill_level(a, L, T, lt);
        if (a.n_work == 0) continue;
        const unsigned grid = std::min<unsigned>(blocks_for(a.n_work, 8), apr->ctx->sm_count * 16);
        k_fill_tree_level<true><<<grid, 256, 0, s>>>(a);
        count_launch(apr->ctx);
    }
    APR_CUDA(cudaGetLastError());
}

// validate's partition property over the interior levels (k_partition_check);
// the caller checks the coarsest level's own cells.
void tree_partition_check(aprgpu_apr* apr, int* dbl, unsigned long long* min_unc, cudaStream_t s) {
    const DevAccess& L = apr->leaf;
    const DevAccess& T = apr->tree;
    if (T.n_particles == 0) return;
    ensure_tree_links(apr, s);
    FillArgs a = base_fill_args(apr);
    a.links = apr->tree_links.as<Links>();
    for (int lt = T.l_max; lt >= T.l_min; --lt) {
        set_fill_level(a, L, T, lt);
        if (a.n_work == 0) continue;
        const unsigned grid = std::min<unsigned>(blocks_for(a.n_work, 8), apr->ctx->sm_count * 16);
        k_partition_check<<<grid, 256, 0, s>>>(a, dbl, min_unc);
        count_launch(apr->ctx);
    }
    APR_CUDA(cudaGetLastError());
}

// fp64 sums (vsum, wsum) of interior levels [lt_lo, lt_hi] (finest first),
// restricted to parent rows whose cells lie in the finest-level pixel planes
// [z_lo, z_hi) (z_hi < 0: every row).  Slab-decomposed callers run the levels
// whose cells fit in a slab locally, exchange the cut level's sums and run the
// coarser levels everywhere; fill_tree_device is all of it.
void fill_tree_sums(aprgpu_apr* apr, const float* leaf, int lt_lo, int lt_hi, int z_lo, int z_hi, cudaStream_t s,
                    float* tree_out) {
    aprgpu_ctx* ctx = apr->ctx;
    const DevAccess& L = apr->leaf;
    const DevAccess& T = apr->tree;
    if (T.n_particles == 0) return;
    if (!apr->vsum.p || apr->vsum.bytes < sizeof(double) * T.n_particles) {
        apr->vsum.ensure(sizeof(double) * T.n_particles);
        apr->wsum.ensure(sizeof(double) * T.n_particles);
    }
    FillArgs a = base_fill_args(apr);
    a.leaf_v = leaf;
    a.vsum = apr->vsum.as<double>();
    a.wsum = apr->wsum.as<double>();
    ensure_tree_links(apr, s);
    a.links = apr->tree_links.as<Links>();
    a.tree_out = tree_out;
    std::unique_lock<std::mutex> lk(apr->init_mu);
    if (apr->tree_level_first.empty()) {  // first node of each interior level, + the total (once per APR)
        std::vector<uint32_t> f(T.l_max + 2);
        for (int l = 0; l <= T.l_max + 1; ++l) {
            const uint64_t row = l <= T.l_max ? T.level_offset[l] : T.n_rows;
            APR_CUDA(cudaMemcpyAsync(&f[l], T.rb + row, 4, cudaMemcpyDeviceToHost, s));
        }
        APR_CUDA(cudaStreamSynchronize(s));
        apr->tree_level_first.assign(f.begin(), f.end());
    }
    lk.unlock();
    for (int lt = std::min(lt_hi, T.l_max); lt >= std::max(lt_lo, T.l_min); --lt) {
        set_fill_level(a, L, T, lt);
        a.pz_lo = z_hi < 0 ? 0 : (z_lo >> (a.glm - lt));
        a.pz_hi = z_hi < 0 ? (1 << 30) : ((z_hi + (1 << (a.glm - lt)) - 1) >> (a.glm - lt));
        if (a.n_work == 0) continue;
        const int64_t cs = int64_t(1) << (a.glm - a.c);  // child cell size
        static const bool flat_ok = [] {  // APRGPU_FILL_FLAT=0: always the row kernel
            const char* e = std::getenv("APRGPU_FILL_FLAT");
            return !(e && e[0] == '0');
        }();
        auto flat_level = [&](int l) {  // child cells of interior level l never clipped
            const int64_t c = int64_t(1) << (a.glm - l - 1);
            return flat_ok && z_hi < 0 && a.nz % c == 0 && a.nx % c == 0 && a.ny % c == 0;
        };
        const int lo = std::max(lt_lo, T.l_min);
        if (apr->tree_level_first[lt + 1] - apr->tree_level_first[lt] <= 2048) {  // (<= 2 nodes per thread: latency-bound levels)
            bool all = true;  // this level and every coarser one: one fused launch
            for (int l = lt; l >= lo && all; --l) all = flat_level(l);
            if (all) {
                CoarseLevels c{};
                for (int l = lt; l >= lo; --l, ++c.n) {
                    const double cl = static_cast<double>(int64_t(1) << (a.glm - l - 1));
                    c.n0[c.n] = static_cast<uint32_t>(apr->tree_level_first[l]);
                    c.n1[c.n] = static_cast<uint32_t>(apr->tree_level_first[l + 1]);
                    c.w[c.n] = cl * cl * cl;
                }
                k_fill_tree_coarse<<<1, 1024, 0, s>>>(a, c);
                count_launch(ctx);
                break;
            }
        }
        if (flat_level(lt)) {
            const uint32_t n0 = static_cast<uint32_t>(apr->tree_level_first[lt]);
            const uint32_t n1 = static_cast<uint32_t>(apr->tree_level_first[lt + 1]);
            const double w = static_cast<double>(cs) * static_cast<double>(cs) * static_cast<double>(cs);
            const unsigned grid = std::min<unsigned>(blocks_for(n1 - n0, 256), ctx->sm_count * 16);
            k_fill_tree_flat<<<grid, 256, 0, s>>>(a, n0, n1, w);
        } else {
            const unsigned grid = std::min<unsigned>(blocks_for(a.n_work, 8), ctx->sm_count * 16);
            k_fill_tree_level<false><<<grid, 256, 0, s>>>(a);
        }
        count_launch(ctx);
    }
    APR_CUDA(cudaGetLastError());
}

void fill_tree_finalize(aprgpu_apr* apr, float* tree, cudaStream_t s) {
    const DevAccess& T = apr->tree;
    if (T.n_particles == 0) return;
    k_tree_finalize<<<std::min<unsigned>(blocks_for(T.n_particles, 256), apr->ctx->sm_count * 8), 256, 0, s>>>(
        apr->vsum.as<double>(), apr->wsum.as<double>(), T.n_particles, tree);
    count_launch(apr->ctx);
    APR_CUDA(cudaGetLastError());
}

void fill_tree_device(aprgpu_apr* apr, const float* leaf, float* tree, cudaStream_t s) {
    // the float values are written with the sums (k_tree_finalize's division,
    // fused): one pass fewer over the interior nodes
    fill_tree_sums(apr, leaf, 0, 1 << 20, 0, -1, s, tree);
}

}  // namespace aprgpu
