// APR tiler on the device: the C4 workload ("C3 tiled 4x4x2 -> 4096x4096x2048",
// BASELINE.md; the paper's "concatenating copies").  Built
// straight into the device layout: C4 has 548 M particles, and building it
// from pixels would need 137 GB of f32 volume.
//
// Source: a cubic APR of edge n = 2^L.  Big dims (n*TZ, n*TX, n*TY), big
// l_max BL = compute_l_max(big dims), sh = BL - L.  Big level l holds, when
// tl = l - sh is a source level, in row (z, x) the concatenation over
// ty = 0..TY-1 of source row (tl, z mod 2^tl, x mod 2^tl) with every y shifted
// by ty * 2^tl; other big levels are empty.  The interior structure is then
// rebuilt by the device tree builder (coarse nodes span tiles).
// Appendix A (C4 tiler).
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace aprgpu {
namespace {

struct TileMap {
    AccessView src;
    int sh, ty_copies;
    int src_lmin, src_lmax;
};

// mode 0: counts[r]; mode 1: y (and values when src_v) of every big row
__global__ void k_tile_rows(int mode, TileMap m, LevelG bg, int l, uint32_t* __restrict__ counts,
                            const uint32_t* __restrict__ rb, uint16_t* __restrict__ y, const float* __restrict__ src_v,
                            float* __restrict__ v) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nrows = static_cast<uint64_t>(bg.zd) * bg.xd;
    const int tl = l - m.sh;
    const LevelG sg = m.src.g[tl];
    for (uint64_t r = warp; r < nrows; r += nwarps) {
        const int z = static_cast<int>(r / bg.xd), x = static_cast<int>(r % bg.xd);
        const uint32_t srow = sg.row0 + static_cast<uint32_t>(z % sg.zd) * sg.xd + (x % sg.xd);
        const uint32_t b = m.src.rb[srow], e = m.src.rb[srow + 1];
        const uint32_t n = e - b;
        if (mode == 0) {
            if (lane == 0) counts[bg.row0 + r] = n * m.ty_copies;
            continue;
        }
        uint32_t o = rb[bg.row0 + r];
        for (int t = 0; t < m.ty_copies; ++t, o += n)
            for (uint32_t k = lane; k < n; k += 32) {
                if (y) y[o + k] = static_cast<uint16_t>(m.src.y[b + k] + t * sg.yd);
                if (src_v) v[o + k] = src_v[b + k];
            }
    }
}

}  // namespace

// Builds the big leaf access of `big` from `src` (structure only when src_v is
// null) or, for an already tiled `big`, writes its values from src_v.
void tile_apr_device(aprgpu_ctx* ctx, const aprgpu_apr* src, int TZ, int TX, int TY, aprgpu_apr* big,
                     const float* src_v, float* big_v, cudaStream_t s) {
    const DevAccess& S = src->leaf;
    const int n = src->dims[0];
    if (src->dims[1] != n || src->dims[2] != n || (n & (n - 1)))
        fail(APRGPU_ERR_CAPABILITY, "tile_apr: the source must be a power-of-two cube");
    const int L = S.l_max;
    if ((1 << L) != n) fail(APRGPU_ERR_CAPABILITY, "tile_apr: source l_max does not match its edge");
    const int bz = n * TZ, bx = n * TX, by = n * TY;
    if (by > 65536) fail(APRGPU_ERR_CAPABILITY, "tile_apr: tiled y dimension exceeds the 16-bit index limit");
    int BL = 0;
    while ((1 << BL) < std::max(bz, std::max(bx, by))) ++BL;
    TileMap m{};
    m.src = S.view();
    m.sh = BL - L;
    m.ty_copies = TY;
    const bool build = src_v == nullptr;
    DevAccess& A = big->leaf;
    if (build) {
        big->dims[0] = bz;
        big->dims[1] = bx;
        big->dims[2] = by;
        big->geom_l_max = BL;
        A.l_max = BL;
        A.l_min = std::min(1, BL);
        A.zd.assign(BL + 1, 0);
        A.xd.assign(BL + 1, 0);
        A.yd.assign(BL + 1, 0);
        A.level_offset.assign(BL + 1, 0);
        uint64_t rows = 0;
        for (int l = 0; l <= BL; ++l) {
            A.zd[l] = grid_dim_dev(bz, BL, l);
            A.xd[l] = grid_dim_dev(bx, BL, l);
            A.yd[l] = grid_dim_dev(by, BL, l);
            A.level_offset[l] = l >= A.l_min ? rows : 0;
            if (l >= A.l_min) rows += static_cast<uint64_t>(A.zd[l]) * A.xd[l];
        }
        if (rows >= (1ull << 32) - 1) fail(APRGPU_ERR_CAPABILITY, "tile_apr: row count exceeds u32");
        A.n_rows = rows;
        APR_CUDA(cudaMalloc(&A.rb, sizeof(uint32_t) * (rows + 1)));
        GpuBuf counts, tmp;
        counts.ensure(sizeof(uint32_t) * (rows + 1));
        APR_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * (rows + 1), s));
        for (int l = A.l_min; l <= BL; ++l) {
            const int tl = l - m.sh;
            if (tl < S.l_min || tl > S.l_max) continue;
            const LevelG bg{A.zd[l], A.xd[l], A.yd[l], static_cast<uint32_t>(A.level_offset[l])};
            const uint64_t nr = static_cast<uint64_t>(bg.zd) * bg.xd;
            k_tile_rows<<<std::min<unsigned>(blocks_for(nr * 32, 256), ctx->sm_count * 32), 256, 0, s>>>(
                0, m, bg, l, counts.as<uint32_t>(), nullptr, nullptr, nullptr, nullptr);
            count_launch(ctx);
        }
        APR_CUDA(cudaGetLastError());
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.as<uint32_t>(), A.rb, static_cast<int64_t>(rows + 1), s);
        tmp.ensure(tb + 16);
        tb = tmp.bytes;
        APR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, counts.as<uint32_t>(), A.rb, static_cast<int64_t>(rows + 1), s));
        count_launch(ctx);
        uint32_t total = 0;
        APR_CUDA(cudaMemcpyAsync(&total, A.rb + rows, 4, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
        const uint64_t expect = static_cast<uint64_t>(S.n_particles) * TZ * TX * TY;
        if (total != expect) fail(APRGPU_ERR_INTEGRITY, "tile_apr: tiled particle count mismatch");
        A.n_particles = total;
        APR_CUDA(cudaMalloc(&A.y, 2ull * total + 2));
    }
    for (int l = A.l_min; l <= BL; ++l) {
        const int tl = l - m.sh;
        if (tl < S.l_min || tl > S.l_max) continue;
        const LevelG bg{A.zd[l], A.xd[l], A.yd[l], static_cast<uint32_t>(A.level_offset[l])};
        const uint64_t nr = static_cast<uint64_t>(bg.zd) * bg.xd;
        k_tile_rows<<<std::min<unsigned>(blocks_for(nr * 32, 256), ctx->sm_count * 32), 256, 0, s>>>(
            1, m, bg, l, nullptr, A.rb, build ? A.y : nullptr, src_v, big_v);
        count_launch(ctx);
    }
    APR_CUDA(cudaGetLastError());
    APR_CUDA(cudaStreamSynchronize(s));
    if (build) {
        build_work_lists(ctx, A);
        build_tile_lists(ctx, A);
        build_tree_structure(ctx, big);
        APR_CUDA(cudaStreamSynchronize(s));
    }
}

}  // namespace aprgpu
