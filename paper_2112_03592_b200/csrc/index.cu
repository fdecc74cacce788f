// Access-structure upload and the non-empty row index.
//
// Reference: LinearAccess (linear_access.hpp:52-96), nonempty_row_index
// (convolve.hpp:32-44) and the LevelInfo occupancy scan inside convolve_apr
// (convolve.hpp:234-261).
//
// Device layout: y_idx stays u16; the u64 cumulative row ends become a u32
// row-begin prefix rb[n_rows+1] (rb[0] = 0, rb[r+1] = xz_end[r]) so a row's
// range is two adjacent loads with no row-0 branch.  Per level the non-empty
// rows are compacted once at upload into an ascending row-id list (ascending
// row id == the reference's z-then-x order); that list is both the convolution
// work list and the source of nonempty_row_index.
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "internal.cuh"

namespace aprgpu {

AccessView DevAccess::view() const {
    AccessView v{};
    v.y = y;
    v.rb = rb;
    v.l_min = l_min;
    v.l_max = l_max;
    for (int l = 0; l <= l_max && l < kMaxLevels; ++l) {
        v.g[l].zd = zd[l];
        v.g[l].xd = xd[l];
        v.g[l].yd = yd[l];
        v.g[l].row0 = static_cast<uint32_t>(level_offset[l]);
    }
    return v;
}

void DevAccess::release() {
    cudaFree(y);
    cudaFree(rb);
    cudaFree(work);
    cudaFree(tiles);
    cudaFree(tile_meta);
    tile_meta = nullptr;
    for (int h = 0; h < 2; ++h) {
        cudaFree(tile_runs[h]);
        cudaFree(tile_run_off[h]);
        tile_runs[h] = nullptr;
        tile_run_off[h] = nullptr;
        cudaFree(tile_flat[h]);
        cudaFree(tile_flat_off[h]);
        tile_flat[h] = nullptr;
        tile_flat_off[h] = nullptr;
        for (int pm = 0; pm < 2; ++pm)
            for (int l = 0; l < kMaxLevels; ++l) {
                if (tile_map[h][pm][l]) {
                    cudaFree(tile_map[h][pm][l]->rec);
                    delete tile_map[h][pm][l];
                }
                tile_map[h][pm][l] = nullptr;
            }
    }
    for (MapWin* w : tile_map_retired) {
        cudaFree(w->rec);
        delete w;
    }
    tile_map_retired.clear();
    y = nullptr;
    rb = nullptr;
    work = nullptr;
    tiles = nullptr;
}

void GpuBuf::ensure(size_t n) {
    if (n <= bytes) return;
    release();
    APR_CUDA(cudaMalloc(&p, n));
    bytes = n;
}

void GpuBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

namespace {

__global__ void k_row_begin(const uint64_t* __restrict__ xz_end, uint64_t n_rows, uint32_t* __restrict__ rb,
                            int* __restrict__ bad) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = xz_end[r];
        const uint64_t b = r ? xz_end[r - 1] : 0;
        if (e < b) atomicOr(bad, 1);  // decreasing xz_end (validate, apr.hpp:76-80)
        rb[r + 1] = static_cast<uint32_t>(e);
        if (r == 0) rb[0] = 0;
    }
}

struct NonEmpty {
    const uint32_t* rb;
    __host__ __device__ bool operator()(uint32_t r) const { return rb[r + 1] > rb[r]; }
};

__global__ void k_row_spans(const uint32_t* __restrict__ work, uint64_t n, uint32_t row0, int xd,
                            const uint32_t* __restrict__ rb, const uint16_t* __restrict__ y, int32_t* z,
                            int32_t* x, uint16_t* ymin, uint16_t* ymax) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = work[i];
        const uint32_t loc = r - row0;
        z[i] = static_cast<int32_t>(loc / xd);
        x[i] = static_cast<int32_t>(loc % xd);
        ymin[i] = y[rb[r]];
        ymax[i] = y[rb[r + 1] - 1];
    }
}

}  // namespace

void build_row_begin(aprgpu_ctx* ctx, DevAccess& a, const uint64_t* xz_end_host) {
    if (a.n_particles >= (1ull << 32))
        fail(APRGPU_ERR_CAPABILITY, "particle count exceeds the u32 device row-offset range");
    APR_CUDA(cudaMalloc(&a.rb, sizeof(uint32_t) * (a.n_rows + 1)));
    if (a.n_rows == 0) {
        APR_CUDA(cudaMemsetAsync(a.rb, 0, sizeof(uint32_t), ctx->stream));
        return;
    }
    GpuBuf tmp;
    tmp.ensure(sizeof(uint64_t) * a.n_rows + 16);
    APR_CUDA(cudaMemcpyAsync(tmp.p, xz_end_host, sizeof(uint64_t) * a.n_rows, cudaMemcpyHostToDevice, ctx->stream));
    int* bad = reinterpret_cast<int*>(tmp.as<char>() + sizeof(uint64_t) * a.n_rows);
    APR_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    k_row_begin<<<std::min<unsigned>(blocks_for(a.n_rows, 256), 148 * 16), 256, 0, ctx->stream>>>(
        tmp.as<uint64_t>(), a.n_rows, a.rb, bad);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
    int hbad = 0;
    APR_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    APR_CUDA(cudaStreamSynchronize(ctx->stream));
    tmp.release();
    if (hbad) fail(APRGPU_ERR_INTEGRITY, "xz_end decreases");
    if (xz_end_host[a.n_rows - 1] != a.n_particles) fail(APRGPU_ERR_INTEGRITY, "xz_end[last] != y_idx length");
}

void build_work_lists(aprgpu_ctx* ctx, DevAccess& a) {
    a.work_off.assign(a.l_max + 2, 0);
    if (a.n_rows == 0) return;
    APR_CUDA(cudaMalloc(&a.work, sizeof(uint32_t) * a.n_rows));
    GpuBuf temp, nsel;
    nsel.ensure(sizeof(uint64_t) * (a.l_max + 1));
    size_t temp_bytes = 0;
    thrust::counting_iterator<uint32_t> it0(0);
    cub::DeviceSelect::If(nullptr, temp_bytes, it0, a.work, nsel.as<uint64_t>(), static_cast<int64_t>(a.n_rows),
                          NonEmpty{a.rb}, ctx->stream);
    temp.ensure(temp_bytes + 16);
    std::vector<uint64_t> counts(a.l_max + 1, 0);
    uint64_t off = 0;
    for (int l = a.l_min; l <= a.l_max; ++l) {
        a.work_off[l] = off;
        const uint64_t rows = static_cast<uint64_t>(a.zd[l]) * a.xd[l];
        if (rows == 0) continue;
        thrust::counting_iterator<uint32_t> it(static_cast<uint32_t>(a.level_offset[l]));
        size_t tb = temp.bytes;
        APR_CUDA(cub::DeviceSelect::If(temp.p, tb, it, a.work + off, nsel.as<uint64_t>() + l,
                                       static_cast<int64_t>(rows), NonEmpty{a.rb}, ctx->stream));
        count_launch(ctx);
        uint64_t c = 0;
        APR_CUDA(cudaMemcpyAsync(&c, nsel.as<uint64_t>() + l, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        APR_CUDA(cudaStreamSynchronize(ctx->stream));
        off += c;
    }
    a.work_off[a.l_max + 1] = off;
    // levels below l_min have empty ranges
    for (int l = 0; l < a.l_min; ++l) a.work_off[l] = 0;
}

void row_spans(aprgpu_ctx* ctx, const DevAccess& a, int level, int32_t* z, int32_t* x, uint16_t* ymin,
               uint16_t* ymax, uint64_t cap) {
    const uint64_t n = a.work_off[level + 1] - a.work_off[level];
    const uint64_t m = std::min(n, cap);
    if (m == 0) return;
    GpuBuf buf;
    buf.ensure(m * 12 + 64);
    int32_t* dz = buf.as<int32_t>();
    int32_t* dx = dz + m;
    uint16_t* dmin = reinterpret_cast<uint16_t*>(dx + m);
    uint16_t* dmax = dmin + m;
    k_row_spans<<<std::min<unsigned>(blocks_for(m, 256), 148 * 8), 256, 0, ctx->stream>>>(
        a.work + a.work_off[level], m, static_cast<uint32_t>(a.level_offset[level]), a.xd[level], a.rb, a.y, dz, dx,
        dmin, dmax);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
    APR_CUDA(cudaMemcpyAsync(z, dz, 4 * m, cudaMemcpyDeviceToHost, ctx->stream));
    APR_CUDA(cudaMemcpyAsync(x, dx, 4 * m, cudaMemcpyDeviceToHost, ctx->stream));
    APR_CUDA(cudaMemcpyAsync(ymin, dmin, 2 * m, cudaMemcpyDeviceToHost, ctx->stream));
    APR_CUDA(cudaMemcpyAsync(ymax, dmax, 2 * m, cudaMemcpyDeviceToHost, ctx->stream));
    APR_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace aprgpu
