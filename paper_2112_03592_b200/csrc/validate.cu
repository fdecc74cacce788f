// validate (apr.hpp:61-134) without the pixel volume.  The reference marks all
// N_pixels of the image to prove that the leaf cells partition it (C4: a
// 34 GB byte map); here the proof is O(particles + rows):
//
//   rows       (this file) one warp per leaf row: y strictly increasing and
//              inside the level grid (first violation by particle index, as
//              the reference's row scan reports it), and every cell's origin
//              inside the image ("particle cell outside the image domain");
//   partition  (tree.cu, k_partition_check) the interior structure built from
//              the leaves (init_tree_structure) is their ancestor closure, so
//              the leaves partition the image iff every in-image child of
//              every interior node is a leaf or an interior node, never both,
//              and the coarsest level's in-image cells likewise (host, tiny);
//              the smallest uncovered pixel is the smallest origin of an
//              uncovered cell.
#include "common.cuh"

namespace aprgpu {
namespace {

__global__ void __launch_bounds__(256) k_validate_rows(AccessView a, uint64_t n_rows, int nz, int nx, int ny,
                                                       unsigned long long* first_y, int* overflow) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < n_rows; r += nwarps) {
        int l = a.l_max;
        while (l > a.l_min && r < a.g[l].row0) --l;
        const LevelG g = a.g[l];
        const uint32_t loc = static_cast<uint32_t>(r) - g.row0;
        const int z = static_cast<int>(loc / g.xd), x = static_cast<int>(loc % g.xd);
        const uint32_t b = a.rb[r], e = a.rb[r + 1];
        if (e <= b) continue;
        const int64_t s = int64_t(1) << (a.l_max - l);  // cell_size(geom_l_max = l_max, l)
        if (z * s >= nz || x * s >= nx) atomicOr(overflow, 1);
        for (uint32_t i = b + lane; i < e; i += 32) {
            const int y = a.y[i];
            const int prev = i > b ? static_cast<int>(a.y[i - 1]) : -1;
            if (y <= prev) {
                atomicMin(first_y, static_cast<unsigned long long>(i) << 1);
            } else if (y >= g.yd) {
                atomicMin(first_y, (static_cast<unsigned long long>(i) << 1) | 1ull);
            } else if (y * s >= ny) {
                atomicOr(overflow, 1);
            }
        }
    }
}

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// Fallback partition check for a structure whose level grids are not the
// image's (validate still answers, by the reference's own method): one bit per
// pixel, every leaf cell's pixels set with atomicOr (an already-set bit is
// double coverage), then the first clear bit.  O(pixels); only for such
// mismatched structures.
__global__ void __launch_bounds__(256) k_cover_rows(AccessView a, uint64_t n_rows, int nz, int nx, int ny,
                                                    uint32_t* bits, int* dbl) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < n_rows; r += nwarps) {
        int l = a.l_max;
        while (l > a.l_min && r < a.g[l].row0) --l;
        const LevelG g = a.g[l];
        const uint32_t loc = static_cast<uint32_t>(r) - g.row0;
        const int64_t s = int64_t(1) << (a.l_max - l);
        const int64_t z0 = (loc / g.xd) * s, x0 = (loc % g.xd) * s;
        const uint32_t b = a.rb[r], e = a.rb[r + 1];
        for (uint32_t i = b + lane; i < e; i += 32) {
            const int64_t y0 = static_cast<int64_t>(a.y[i]) * s;
            if (z0 >= nz || x0 >= nx || y0 >= ny) continue;  // (reported by the row pass)
            const int64_t z1 = min64(z0 + s, nz), x1 = min64(x0 + s, nx), y1 = min64(y0 + s, ny);
            for (int64_t zz = z0; zz < z1; ++zz)
                for (int64_t xx = x0; xx < x1; ++xx) {
                    const uint64_t base = (static_cast<uint64_t>(zz) * nx + xx) * ny;
                    for (int64_t yy = y0; yy < y1;) {
                        const uint64_t p = base + yy;
                        const int nb = static_cast<int>(min64(32 - static_cast<int64_t>(p & 31), y1 - yy));
                        const uint32_t m = (nb == 32 ? ~0u : ((1u << nb) - 1u)) << (p & 31);
                        if (atomicOr(bits + (p >> 5), m) & m) atomicOr(dbl, 1);
                        yy += nb;
                    }
                }
        }
    }
}

__global__ void k_first_clear(const uint32_t* bits, uint64_t n_pixels, unsigned long long* first) {
    const uint64_t nw = (n_pixels + 31) >> 5;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = ~bits[w];
        if (w == nw - 1 && (n_pixels & 31)) v &= (1u << (n_pixels & 31)) - 1u;
        if (v) atomicMin(first, (w << 5) + __ffs(v) - 1);
    }
}

}  // namespace

void validate_cover_device(aprgpu_ctx* ctx, const DevAccess& L, const int dims[3], int* dbl,
                           unsigned long long* min_unc, cudaStream_t s) {
    const uint64_t n_pixels = static_cast<uint64_t>(dims[0]) * dims[1] * dims[2];
    GpuBuf bits;
    bits.ensure(4 * ((n_pixels + 31) / 32) + 4);
    APR_CUDA(cudaMemsetAsync(bits.p, 0, 4 * ((n_pixels + 31) / 32) + 4, s));
    if (L.n_rows) {
        const unsigned grid = std::min<unsigned>(blocks_for(L.n_rows, 8), ctx->sm_count * 16);
        k_cover_rows<<<grid, 256, 0, s>>>(L.view(), L.n_rows, dims[0], dims[1], dims[2], bits.as<uint32_t>(), dbl);
        count_launch(ctx);
    }
    k_first_clear<<<std::min<unsigned>(blocks_for((n_pixels + 31) / 32, 256), ctx->sm_count * 8), 256, 0, s>>>(
        bits.as<uint32_t>(), n_pixels, min_unc);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
    APR_CUDA(cudaStreamSynchronize(s));
    bits.release();
}

void validate_rows_device(aprgpu_ctx* ctx, const DevAccess& L, const int dims[3], unsigned long long* first_y,
                          int* overflow, cudaStream_t s) {
    if (L.n_rows == 0) return;
    const unsigned grid = std::min<unsigned>(blocks_for(L.n_rows, 8), ctx->sm_count * 16);
    k_validate_rows<<<grid, 256, 0, s>>>(L.view(), L.n_rows, dims[0], dims[1], dims[2], first_y, overflow);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
}

}  // namespace aprgpu
