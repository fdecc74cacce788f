// Dense reconstruction on the device: reconstruct_level / reconstruct_full /
// reconstruct_patch (reconstruct.hpp:73-129), the piecewise-constant pixel
// images the reference builds row by row with fill_level_row (:41-69).
//
// One warp per output row (z, x) of the level-l grid.  The row is zeroed, then
// filled in the reference's order -- the level-l leaves, the level l-1 leaves
// covering it, ..., the level l_min leaves, then (when tree values are given)
// the level-l interior nodes -- with a warp barrier between passes, so a cell
// covered twice (a malformed APR) keeps the reference's last writer.  Leaves at
// most 2 levels coarser are written one particle per lane (<= 4 cells, one
// vector store); 3-4 levels coarser a lane per cell, several particles per
// warp step; coarser ones one particle at a time, the warp across its 2^d cells.  Writes
// are row-contiguous; the zero pass and the fill of a row merge in L2, so the
// output is written to HBM about once: the kernel is bound by the output's
// size (4 bytes per cell).
#include "common.cuh"

namespace aprgpu {
namespace {

struct ReconArgs {
    AccessView leaf, tree;
    const float* values;
    const float* tree_values;  // null: no interior nodes (reconstruct_full)
    int l;
    // output rows: (oz, ox) of an out_nz x out_nx grid of rows of out_ny cells;
    // the level row is written at y offset pad
    int out_nz, out_nx, out_ny;
    int z0, x0, pad;  // output row (oz, ox) is level row (z0 + oz, x0 + ox) before reflection
    int pad_mode;     // APRGPU_PAD_ZERO / REFLECT (patch only)
    float* out;
};

__device__ __forceinline__ int reflect_i(int i, int n) {  // reflect_index (reconstruct.hpp:16-25)
    while (i < 0 || i >= n) i = i < 0 ? -i - 1 : 2 * n - 1 - i;
    return i;
}

// fill_level_row (reconstruct.hpp:41-69) of level row (z, x), y in [0, yd), into dst
__device__ void fill_row_warp(const ReconArgs& a, int z, int x, float* dst, int yd, int lane) {
    const int l = a.l;
    // every covering row's particle range at once: lane d loads depth d's
    uint32_t rb = 0, re = 0;
    if (lane <= l - a.leaf.l_min && l - lane <= a.leaf.l_max) {
        const LevelG g = a.leaf.g[l - lane];
        const int cz = z >> lane, cx = x >> lane;
        if (cz < g.zd && cx < g.xd) {
            const uint32_t row = g.row0 + static_cast<uint32_t>(cz) * g.xd + cx;
            rb = __ldg(a.leaf.rb + row);
            re = __ldg(a.leaf.rb + row + 1);
        }
    }
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {  // 16-byte zero stores where aligned
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int y = lane; y < (yd >> 2); y += 32) d4[y] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        for (int y = (yd & ~3) + lane; y < yd; y += 32) dst[y] = 0.0f;
    } else {
        for (int y = lane; y < yd; y += 32) dst[y] = 0.0f;
    }
    __syncwarp();
    for (int d = 0; d <= l - a.leaf.l_min; ++d) {
        const uint32_t b = __shfl_sync(0xffffffffu, rb, d), e = __shfl_sync(0xffffffffu, re, d);
        if (e <= b) continue;
        const bool al = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
        if (d <= 2) {  // one particle per lane, its 1 / 2 / 4 cells as one (aligned) store
            for (uint32_t i = b + lane; i < e; i += 32) {
                const int y0 = static_cast<int>(__ldg(a.leaf.y + i)) << d;
                const float v = __ldg(a.values + i);
                const int y1 = min(y0 + (1 << d), yd);
                if (al && d == 2 && y1 - y0 == 4) {
                    *reinterpret_cast<float4*>(dst + y0) = make_float4(v, v, v, v);
                } else if (al && d == 1 && y1 - y0 == 2) {
                    *reinterpret_cast<float2*>(dst + y0) = make_float2(v, v);
                } else {
                    for (int y = y0; y < y1; ++y) dst[y] = v;
                }
            }
        } else if (d <= 4) {  // 4 (d = 3) or 2 (d = 4) particles per warp step, a lane per cell
            const int c = 1 << d, per = 32 / c, k = lane / c, j = lane % c;
            for (uint32_t i0 = b; i0 < e; i0 += per) {
                const uint32_t i = i0 + k;
                if (i < e) {
                    const int y = (static_cast<int>(__ldg(a.leaf.y + i)) << d) + j;
                    if (y < yd) dst[y] = __ldg(a.values + i);
                }
            }
        } else {  // 32 particles' (y, value) loaded at once, then broadcast one by one
            for (uint32_t i0 = b; i0 < e; i0 += 32) {
                const int n = static_cast<int>(min(32u, e - i0));
                int yl = 0;
                float vl = 0.0f;
                if (lane < n) {
                    yl = __ldg(a.leaf.y + i0 + lane);
                    vl = __ldg(a.values + i0 + lane);
                }
                for (int k = 0; k < n; ++k) {
                    const int y0 = __shfl_sync(0xffffffffu, yl, k) << d;
                    const float v = __shfl_sync(0xffffffffu, vl, k);
                    const int y1 = min(y0 + (1 << d), yd);
                    for (int y = y0 + lane; y < y1; y += 32) dst[y] = v;
                }
            }
        }
        __syncwarp();
    }
    if (a.tree_values && l >= a.tree.l_min && l <= a.tree.l_max) {
        const LevelG g = a.tree.g[l];
        if (z < g.zd && x < g.xd) {
            const uint32_t row = g.row0 + static_cast<uint32_t>(z) * g.xd + x;
            const uint32_t b = __ldg(a.tree.rb + row), e = __ldg(a.tree.rb + row + 1);
            for (uint32_t i = b + lane; i < e; i += 32) {
                const int y = __ldg(a.tree.y + i);
                if (y < yd) dst[y] = __ldg(a.tree_values + i);
            }
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_reconstruct(ReconArgs a) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const LevelG g = a.leaf.g[a.l];
    const uint64_t nrows = static_cast<uint64_t>(a.out_nz) * a.out_nx;
    for (uint64_t r = warp; r < nrows; r += nwarps) {
        const int oz = static_cast<int>(r / a.out_nx), ox = static_cast<int>(r % a.out_nx);
        float* dst = a.out + r * a.out_ny;
        const int z = a.z0 + oz, x = a.x0 + ox;
        const bool inside = z >= 0 && z < g.zd && x >= 0 && x < g.xd;
        if (!inside && a.pad_mode == APRGPU_PAD_ZERO) {  // stays zero (reconstruct.hpp:116)
            for (int y = lane; y < a.out_ny; y += 32) dst[y] = 0.0f;
            continue;
        }
        float* row = dst + a.pad;
        fill_row_warp(a, inside ? z : reflect_i(z, g.zd), inside ? x : reflect_i(x, g.xd), row, g.yd, lane);
        if (a.pad) {  // y padding (reconstruct.hpp:121-125), from the finished row
            for (int p = lane; p < a.pad; p += 32) {
                const bool zero = a.pad_mode == APRGPU_PAD_ZERO;
                const float lo = zero ? 0.0f : row[reflect_i(p - a.pad, g.yd)];
                const float hi = zero ? 0.0f : row[reflect_i(g.yd + p, g.yd)];
                dst[p] = lo;
                row[g.yd + p] = hi;
            }
        }
    }
}

void launch(aprgpu_apr* apr, const ReconArgs& a, cudaStream_t s) {
    const uint64_t nrows = static_cast<uint64_t>(a.out_nz) * a.out_nx;
    if (!nrows || !a.out_ny) return;
    const unsigned grid = std::min<unsigned>(blocks_for(nrows * 32, 256), apr->ctx->sm_count * 16);
    k_reconstruct<<<grid, 256, 0, s>>>(a);
    count_launch(apr->ctx);
    APR_CUDA(cudaGetLastError());
}

ReconArgs base_args(const aprgpu_apr* apr, const float* values, const float* tree_values, int l, float* out) {
    ReconArgs a{};
    a.leaf = apr->leaf.view();
    a.tree = apr->tree.view();
    a.values = values;
    a.tree_values = apr->tree.n_particles ? tree_values : nullptr;
    a.l = l;
    a.out = out;
    return a;
}

}  // namespace

void reconstruct_level_device(aprgpu_apr* apr, const float* values, const float* tree_values, int l, float* out,
                              cudaStream_t s) {
    const DevAccess& L = apr->leaf;
    if (l < L.l_min || l > L.l_max) fail(APRGPU_ERR_RANGE, "reconstruct_level: level out of range");
    ReconArgs a = base_args(apr, values, tree_values, l, out);
    a.out_nz = L.zd[l];
    a.out_nx = L.xd[l];
    a.out_ny = L.yd[l];
    a.pad_mode = APRGPU_PAD_REFLECT;  // (every output row is inside the grid)
    launch(apr, a, s);
}

void reconstruct_patch_device(aprgpu_apr* apr, const float* values, const float* tree_values,
                              const aprgpu_patch_spec& sp, float* out, cudaStream_t s) {
    const DevAccess& L = apr->leaf;
    const int l = sp.level;
    if (l < L.l_min || l > L.l_max) fail(APRGPU_ERR_RANGE, "reconstruct_patch: level out of range");
    if (sp.z_begin < 0 || sp.z_end > L.zd[l] || sp.x_begin < 0 || sp.x_end > L.xd[l] || sp.z_begin > sp.z_end ||
        sp.x_begin > sp.x_end || sp.pad < 0)
        fail(APRGPU_ERR_RANGE, "reconstruct_patch: spec outside the level grid");
    if (sp.pad_mode != APRGPU_PAD_ZERO && sp.pad_mode != APRGPU_PAD_REFLECT) fail(APRGPU_ERR_RANGE, "bad pad mode");
    ReconArgs a = base_args(apr, values, tree_values, l, out);
    a.out_nz = sp.z_end - sp.z_begin + 2 * sp.pad;
    a.out_nx = sp.x_end - sp.x_begin + 2 * sp.pad;
    a.out_ny = L.yd[l] + 2 * sp.pad;
    a.z0 = sp.z_begin - sp.pad;
    a.x0 = sp.x_begin - sp.pad;
    a.pad = sp.pad;
    a.pad_mode = sp.pad_mode;
    launch(apr, a, s);
}

}  // namespace aprgpu
