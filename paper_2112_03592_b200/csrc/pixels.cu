// Dense pixel convolution on the device: convolve_pixels (convolve.hpp:48-98),
// the pixel-space baseline of the paper's APR-vs-pixels comparison
// (SURVEY §8f row 4).
//
// o(p) = sum_r w(r) u(p - r), true-convolution convention, the volume padded by
// reflect_index or zeros.  One CTA per 8 (z) x 8 (x) x kPy (y) output tile: the
// tile's (8 + 2hz) x (8 + 2hx) x (kPy + 2hy) input box is staged in shared
// memory (padding applied on load), then each thread evaluates 4 consecutive
// y outputs of one (z, x) column, taps in the reference's order (az, ax, ay)
// skipping zero weights (:86-88): EXACT = fp64 accumulation of exact products
// (bit-identical), FAST = fp32 FMA.  Extents up to kMaxStencilExtent = 13.
#include <cstdlib>

#include "common.cuh"

namespace aprgpu {
namespace {

constexpr int kPz = 8, kPx = 8, kPy = 64, kPixThreads = 256, kPixMaxK = 13;

struct PixArgs {
    const float* in;
    float* out;
    int nz, nx, ny;
    int kz, kx, ky;
    int pad;
    const float* w;  // kz * kx * ky
};

__device__ __forceinline__ int reflect_p(int i, int n) {  // reflect_index (reconstruct.hpp:16-25)
    while (i < 0 || i >= n) i = i < 0 ? -i - 1 : 2 * n - 1 - i;
    return i;
}

template <typename Acc>
__global__ void __launch_bounds__(kPixThreads) k_convolve_pixels(PixArgs a, int tyd, int txd) {
    extern __shared__ __align__(16) float box[];
    __shared__ float W[kPixMaxK * kPixMaxK * kPixMaxK];
    const int hz = a.kz / 2, hx = a.kx / 2, hy = a.ky / 2;
    const int BZ = kPz + 2 * hz, BX = kPx + 2 * hx, BY = kPy + 2 * hy;
    const int tid = threadIdx.x;
    const int ty = blockIdx.x % tyd, t2 = blockIdx.x / tyd;
    const int tx = t2 % txd, tz = t2 / txd;
    const int z0 = tz * kPz, x0 = tx * kPx, y0 = ty * kPy;
    const int KW = a.kz * a.kx * a.ky;
    for (int i = tid; i < KW; i += kPixThreads) W[i] = a.w[i];
    // stage the box: cell (bz, bx, by) is padded-volume (z0 + bz, x0 + bx, y0 + by),
    // i.e. input (z0 + bz - hz, ...) reflected or zero
    const int nb = BZ * BX * BY;
    for (int i = tid; i < nb; i += kPixThreads) {
        const int bz = i / (BX * BY), rem = i - bz * (BX * BY);
        const int bx = rem / BY, by = rem - bx * BY;
        int z = z0 + bz - hz, x = x0 + bx - hx, y = y0 + by - hy;
        const bool out = z < 0 || z >= a.nz || x < 0 || x >= a.nx || y < 0 || y >= a.ny;
        float v = 0.0f;
        if (!out) {
            v = __ldg(a.in + (static_cast<size_t>(z) * a.nx + x) * a.ny + y);
        } else if (a.pad == APRGPU_PAD_REFLECT && z < a.nz + 2 * hz && x < a.nx + 2 * hx && y < a.ny + 2 * hy) {
            z = reflect_p(z, a.nz);
            x = reflect_p(x, a.nx);
            y = reflect_p(y, a.ny);
            v = __ldg(a.in + (static_cast<size_t>(z) * a.nx + x) * a.ny + y);
        }
        box[i] = v;
    }
    __syncthreads();
    // 64 (z, x) columns x 16 groups of 4 y outputs
    for (int job = tid; job < kPz * kPx * (kPy / 4); job += kPixThreads) {
        const int col = job / (kPy / 4), g = job - col * (kPy / 4);
        const int oz = col / kPx, ox = col - oz * kPx, oy = 4 * g;
        if (z0 + oz >= a.nz || x0 + ox >= a.nx || y0 + oy >= a.ny) continue;
        Acc acc[4] = {Acc(0), Acc(0), Acc(0), Acc(0)};
        // output (oz, ox, oy + j) reads padded (z + 2hz - az, x + 2hx - ax, y + 2hy - ay)
        for (int az = 0; az < a.kz; ++az)
            for (int ax = 0; ax < a.kx; ++ax) {
                const float* row = box + ((oz + 2 * hz - az) * BX + (ox + 2 * hx - ax)) * BY + oy + 2 * hy;
                const float* wr = W + (az * a.kx + ax) * a.ky;
                for (int ay = 0; ay < a.ky; ++ay) {
                    const float wv = wr[ay];
                    if (wv == 0.0f) continue;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        acc[j] = fma(static_cast<Acc>(wv), static_cast<Acc>(row[j - ay]), acc[j]);
                }
            }
        float* dst = a.out + (static_cast<size_t>(z0 + oz) * a.nx + (x0 + ox)) * a.ny + y0 + oy;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (y0 + oy + j < a.ny) dst[j] = static_cast<float>(acc[j]);
    }
}

// Isotropic K^3 (K = 3, 5): the same tile, staged row by row (a warp per box
// row, lanes along y: coalesced loads, one reflection per row), weights in
// registers, each thread one (z, x) column x 8 consecutive y outputs from a
// sliding register window of 8 + K - 1 cells per (az, ax) row.
constexpr int kIsoPy = 64;
template <typename Acc, int K>
__global__ void __launch_bounds__(kPixThreads) k_convolve_pixels_iso(PixArgs a, int tyd, int txd) {
    constexpr int kPy = kIsoPy;
    constexpr int H = K / 2, BZ = kPz + 2 * H, BX = kPx + 2 * H, BY = kPy + 2 * H, RY = 8, NW = RY + K - 1;
    extern __shared__ __align__(16) float box[];  // BZ * BX * BY
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ty = blockIdx.x % tyd, t2 = blockIdx.x / tyd;
    const int tx = t2 % txd, tz = t2 / txd;
    const int z0 = tz * kPz, x0 = tx * kPx, y0 = ty * kPy;
    for (int r = warp; r < BZ * BX; r += kPixThreads / 32) {
        const int bz = r / BX, bx = r - bz * BX;
        int z = z0 + bz - H, x = x0 + bx - H;
        const bool row_out = z < 0 || z >= a.nz || x < 0 || x >= a.nx;
        float* dst = box + r * BY;
        if (row_out && a.pad == APRGPU_PAD_ZERO) {
            for (int by = lane; by < BY; by += 32) dst[by] = 0.0f;
            continue;
        }
        z = reflect_p(z, a.nz);
        x = reflect_p(x, a.nx);
        const float* src = a.in + (static_cast<size_t>(z) * a.nx + x) * a.ny;

        for (int by = lane; by < BY; by += 32) {
            const int y = y0 + by - H;
            float v = 0.0f;
            if (y >= 0 && y < a.ny) v = __ldg(src + y);
            else if (a.pad == APRGPU_PAD_REFLECT) v = __ldg(src + reflect_p(y, a.ny));
            dst[by] = v;
        }
    }
    float w[K * K * K];
#pragma unroll
    for (int i = 0; i < K * K * K; ++i) w[i] = __ldg(a.w + i);
    __syncthreads();
    for (int job = tid; job < kPz * kPx * (kPy / RY); job += kPixThreads) {
        const int col = job / (kPy / RY), g = job - col * (kPy / RY);
        const int oz = col / kPx, ox = col - oz * kPx, oy = RY * g;
        if (z0 + oz >= a.nz || x0 + ox >= a.nx || y0 + oy >= a.ny) continue;
        Acc acc[RY];
#pragma unroll
        for (int j = 0; j < RY; ++j) acc[j] = Acc(0);
#pragma unroll
        for (int az = 0; az < K; ++az)
#pragma unroll
            for (int ax = 0; ax < K; ++ax) {
                // output oy + j reads box y index oy + j + 2H - ay
                const float* row = box + ((oz + 2 * H - az) * BX + (ox + 2 * H - ax)) * BY + oy;
                float win[NW];
#pragma unroll
                for (int i = 0; i < NW; ++i) win[i] = row[i];
#pragma unroll
                for (int ay = 0; ay < K; ++ay) {
                    const float wv = w[(az * K + ax) * K + ay];
                    if (wv == 0.0f) continue;  // (convolve.hpp:86-88)
#pragma unroll
                    for (int j = 0; j < RY; ++j)
                        acc[j] = fma(static_cast<Acc>(wv), static_cast<Acc>(win[j + 2 * H - ay]), acc[j]);
                }
            }
        float* dst = a.out + (static_cast<size_t>(z0 + oz) * a.nx + (x0 + ox)) * a.ny + y0 + oy;
#pragma unroll
        for (int j = 0; j < RY; ++j)
            if (y0 + oy + j < a.ny) dst[j] = static_cast<float>(acc[j]);
    }
}

__device__ __forceinline__ void cp_async_4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// Isotropic K^3 (K = 3, 5), streamed along z (2.5-D blocking): a CTA owns a
// 32 (x) x 64 (y) column of outputs over kZc planes and keeps a ring of K + 2
// input planes -- the K the current output plane reads and the next two,
// prefetched with cp.async while the current plane is evaluated (padding
// applied on load).  Every input plane is read from HBM about once (x / y halo
// 1.1x, z halo 2H / kZc).  Lane = x row, warp = a run of 8 consecutive y
// outputs: a warp's window loads are 16-byte loads from 32 different rows
// whose stride (kPY = 76 floats, 12 banks) puts every quarter-warp on distinct
// banks -- conflict-free (lanes along y, 32 bytes apart, were 8-way conflicted).
// FAST keeps the K^3 weights in registers, EXACT reads them as doubles from
// shared memory (one broadcast load per tap).  SKIP: some weight is zero and
// is skipped like the reference (convolve.hpp:86-88) -- which only matters
// for non-finite inputs; otherwise no per-tap test.
constexpr int kSx = 32, kSy = 64, kZc = 32, kRY = 8, kPY = 76;
template <typename Acc, int K, bool SKIP>
__global__ void __launch_bounds__(kPixThreads) k_convolve_pixels_stream(PixArgs a, int txd, int tyd) {
    constexpr int D = 2;  // prefetch distance (planes)
    // a plane row: [4 - H unused][H halo][64 interior at a 16-byte boundary][H halo], kPY floats
    constexpr int H = K / 2, PX = kSx + 2 * H, OFF = 4 - H, PY = kPY, PLANE = PX * PY, RY = kRY,
                  NS = K + D, KW = K * K * K;
    static_assert(kSx * (kSy / RY) == kPixThreads && kSx == 32, "lane = x row, warp = y run");
    static_assert(PY >= kSy + 8 && PY % 4 == 0, "16-byte rows");
    extern __shared__ __align__(16) float ring[];  // NS planes
    __shared__ Acc Ws[KW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ty = blockIdx.x % tyd, t2 = blockIdx.x / tyd;
    const int tx = t2 % txd, tzc = t2 / txd;
    const int x0 = tx * kSx, y0 = ty * kSy, zc0 = tzc * kZc, zc1 = min(zc0 + kZc, a.nz);
    for (int i = tid; i < KW; i += kPixThreads) Ws[i] = static_cast<Acc>(a.w[i]);
    float wr[sizeof(Acc) == 4 ? KW : 1];  // FAST: the weights in registers
    if constexpr (sizeof(Acc) == 4) {
#pragma unroll
        for (int i = 0; i < KW; ++i) wr[i] = __ldg(a.w + i);
    }
    auto slot = [&](int z) { return ring + (((z % NS) + NS) % NS) * PLANE; };
    const bool vec = (a.ny & 3) == 0 && y0 + kSy <= a.ny;  // 16-byte aligned, whole interior in range
    // input plane z into its slot (reflected / zero outside the volume), asynchronously
    auto load = [&](int z) {
        float* pl = slot(z);
        const bool zout = z < 0 || z >= a.nz;
        const int zr = reflect_p(z, a.nz);
        for (int r = warp; r < PX; r += kPixThreads / 32) {
            const int x = x0 + r - H;
            float* dst = pl + r * PY + OFF;  // dst[c]: y = y0 + c - H
            if ((zout || x < 0 || x >= a.nx) && a.pad == APRGPU_PAD_ZERO) {
                for (int c = lane; c < kSy + 2 * H; c += 32) dst[c] = 0.0f;
                continue;
            }
            const float* src = a.in + (static_cast<size_t>(zr) * a.nx + reflect_p(x, a.nx)) * a.ny;
            if (vec) {  // the interior: 16-byte copies
                if (lane < kSy / 4)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     static_cast<unsigned>(__cvta_generic_to_shared(dst + H + 4 * lane))),
                                 "l"(src + y0 + 4 * lane)
                                 : "memory");
            } else {  // (ragged or unaligned rows)
                for (int c = H + lane; c < H + kSy; c += 32) {
                    const int y = y0 + c - H;
                    if (y < a.ny) cp_async_4(dst + c, src + y);
                    else if (a.pad == APRGPU_PAD_REFLECT) cp_async_4(dst + c, src + reflect_p(y, a.ny));
                    else dst[c] = 0.0f;
                }
            }
            if (lane >= 32 - 2 * H) {  // the halos (lanes the interior copies leave idle)
                const int k = lane - (32 - 2 * H);
                const int c = k < H ? k : kSy + k;
                const int y = y0 + c - H;
                if (y >= 0 && y < a.ny) cp_async_4(dst + c, src + y);
                else if (a.pad == APRGPU_PAD_REFLECT) cp_async_4(dst + c, src + reflect_p(y, a.ny));
                else dst[c] = 0.0f;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ox = lane, oy = warp * RY;  // this thread's outputs: row ox, y oy .. oy + 7
    // planes zc0 - H .. zc0 + H + D - 1 in flight; then one group per plane
    for (int z = zc0 - H; z < zc0 + H + D; ++z) {
        if (z < zc1 + H) load(z);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int z = zc0 + H; z < zc1 + H; ++z) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");  // all but the D newest groups
        __syncthreads();  // planes o - H .. o + H resident; the slot of o - H - 1 is free
        if (z + D < zc1 + H) load(z + D);  // prefetch D planes ahead
        else asm volatile("cp.async.commit_group;" ::: "memory");
        const int o = z - H;
        if (x0 + ox < a.nx && y0 + oy < a.ny) {
            Acc acc[RY];
#pragma unroll
            for (int j = 0; j < RY; ++j) acc[j] = Acc(0);
#pragma unroll
            for (int az = 0; az < K; ++az) {
                const float* plz = slot(o + H - az);  // input plane read with weight plane az
#pragma unroll
                for (int ax = 0; ax < K; ++ax) {
                    // outputs oy + j read cells c = oy + j + 2H - ay, c in [oy, oy + 7 + 2H]: the
                    // window from the 16-byte boundary at or below row + OFF + oy
                    const float* row = plz + (ox + 2 * H - ax) * PY;
                    constexpr int SH = OFF & 3, NL = (SH + RY + 2 * H + 3) & ~3;
                    Acc win[NL];  // (converted once per row, not per tap)
#pragma unroll
                    for (int i = 0; i < NL; i += 4) {
                        const float4 t = *reinterpret_cast<const float4*>(row + (OFF - SH) + oy + i);
                        win[i] = static_cast<Acc>(t.x);
                        win[i + 1] = static_cast<Acc>(t.y);
                        win[i + 2] = static_cast<Acc>(t.z);
                        win[i + 3] = static_cast<Acc>(t.w);
                    }
#pragma unroll
                    for (int ay = 0; ay < K; ++ay) {
                        const int wi = (az * K + ax) * K + ay;
                        Acc wa;
                        if constexpr (sizeof(Acc) == 4) wa = wr[wi]; else wa = Ws[wi];
                        if (SKIP && wa == Acc(0)) continue;  // (convolve.hpp:86-88)
#pragma unroll
                        for (int j = 0; j < RY; ++j) acc[j] = fma(wa, win[SH + j + 2 * H - ay], acc[j]);
                    }
                }
            }
            float* dst = a.out + (static_cast<size_t>(o) * a.nx + (x0 + ox)) * a.ny + y0 + oy;
            if (y0 + oy + RY <= a.ny && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < RY; j += 4)
                    __stcs(reinterpret_cast<float4*>(dst + j),
                           make_float4(static_cast<float>(acc[j]), static_cast<float>(acc[j + 1]),
                                       static_cast<float>(acc[j + 2]), static_cast<float>(acc[j + 3])));
            } else {
#pragma unroll
                for (int j = 0; j < RY; ++j)
                    if (y0 + oy + j < a.ny) dst[j] = static_cast<float>(acc[j]);
            }
        }
        __syncthreads();  // (the next prefetch overwrites this iteration's oldest plane)
    }
}

}  // namespace

void convolve_pixels_device(aprgpu_ctx* ctx, const float* in, int nz, int nx, int ny, const float* w_dev, int kz,
                            int kx, int ky, int pad, int accum, float* out, cudaStream_t s, bool any_zero_w) {
    if (kz > kPixMaxK || kx > kPixMaxK || ky > kPixMaxK)
        fail(APRGPU_ERR_CAPABILITY, "convolve_pixels: stencil extent exceeds the supported maximum");
    if (nz <= 0 || nx <= 0 || ny <= 0) return;
    PixArgs a{in, out, nz, nx, ny, kz, kx, ky, pad, w_dev};
    const int tzd = (nz + kPz - 1) / kPz, txd = (nx + kPx - 1) / kPx, tyd = (ny + kPy - 1) / kPy;
    const uint64_t blocks = static_cast<uint64_t>(tzd) * txd * tyd;
    if (blocks >= (1ull << 31)) fail(APRGPU_ERR_CAPABILITY, "convolve_pixels: volume too large");
    if (kz == kx && kx == ky && (kz == 3 || kz == 5) && !std::getenv("APRGPU_PIXELS_TILED")) {
        const bool ex = accum == APRGPU_ACCUM_EXACT;
        const int sxd = (nx + kSx - 1) / kSx, syd = (ny + kSy - 1) / kSy, szd = (nz + kZc - 1) / kZc;
        const unsigned g = static_cast<unsigned>(static_cast<uint64_t>(szd) * sxd * syd);
        const int h = kz / 2;
        const int rb = (kz + 2) * (kSx + 2 * h) * kPY * static_cast<int>(sizeof(float));
        static OncePerDevice sattr;
        sattr([] {
            const int mx = 7 * (kSx + 4) * kPY * static_cast<int>(sizeof(float));
#define APRGPU_SET_PIX(A, K_, S_) \
    APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_stream<A, K_, S_>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx))
            APRGPU_SET_PIX(double, 3, false);
            APRGPU_SET_PIX(double, 3, true);
            APRGPU_SET_PIX(float, 3, false);
            APRGPU_SET_PIX(float, 3, true);
            APRGPU_SET_PIX(double, 5, false);
            APRGPU_SET_PIX(double, 5, true);
            APRGPU_SET_PIX(float, 5, false);
            APRGPU_SET_PIX(float, 5, true);
#undef APRGPU_SET_PIX
        });
        const bool skip = any_zero_w;  // (a zero weight is skipped like the reference)
#define APRGPU_LAUNCH_PIX(A, K_) \
    (skip ? k_convolve_pixels_stream<A, K_, true><<<g, kPixThreads, rb, s>>>(a, sxd, syd) \
          : k_convolve_pixels_stream<A, K_, false><<<g, kPixThreads, rb, s>>>(a, sxd, syd))
        if (kz == 3) {
            if (ex) APRGPU_LAUNCH_PIX(double, 3); else APRGPU_LAUNCH_PIX(float, 3);
        } else {
            if (ex) APRGPU_LAUNCH_PIX(double, 5); else APRGPU_LAUNCH_PIX(float, 5);
        }
#undef APRGPU_LAUNCH_PIX
        count_launch(ctx);
        APR_CUDA(cudaGetLastError());
        return;
    }
    if (kz == kx && kx == ky && (kz == 3 || kz == 5)) {
        const bool ex = accum == APRGPU_ACCUM_EXACT;
        const int ityd = (ny + kIsoPy - 1) / kIsoPy;
        const unsigned g = static_cast<unsigned>(static_cast<uint64_t>(tzd) * txd * ityd);
        const int h = kz / 2;
        const int ib = (kPz + 2 * h) * (kPx + 2 * h) * (kIsoPy + 2 * h) * static_cast<int>(sizeof(float));
        static OncePerDevice iattr;
        iattr([] {
            const int mx = (kPz + 4) * (kPx + 4) * (kIsoPy + 4) * static_cast<int>(sizeof(float));
            APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_iso<double, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_iso<float, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_iso<double, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_iso<float, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        });
        if (kz == 3) {
            if (ex) k_convolve_pixels_iso<double, 3><<<g, kPixThreads, ib, s>>>(a, ityd, txd);
            else k_convolve_pixels_iso<float, 3><<<g, kPixThreads, ib, s>>>(a, ityd, txd);
        } else {
            if (ex) k_convolve_pixels_iso<double, 5><<<g, kPixThreads, ib, s>>>(a, ityd, txd);
            else k_convolve_pixels_iso<float, 5><<<g, kPixThreads, ib, s>>>(a, ityd, txd);
        }
        count_launch(ctx);
        APR_CUDA(cudaGetLastError());
        return;
    }
    const int bytes = (kPz + 2 * (kz / 2)) * (kPx + 2 * (kx / 2)) * (kPy + 2 * (ky / 2)) * static_cast<int>(sizeof(float));
    static OncePerDevice attr;
    attr([] {
        const int mx = (kPz + kPixMaxK - 1) * (kPx + kPixMaxK - 1) * (kPy + kPixMaxK - 1) * static_cast<int>(sizeof(float));
        APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    });
    if (accum == APRGPU_ACCUM_EXACT)
        k_convolve_pixels<double><<<static_cast<unsigned>(blocks), kPixThreads, bytes, s>>>(a, tyd, txd);
    else
        k_convolve_pixels<float><<<static_cast<unsigned>(blocks), kPixThreads, bytes, s>>>(a, tyd, txd);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
}

}  // namespace aprgpu
