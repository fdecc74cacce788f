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
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

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

constexpr int kSx = 32, kSy = 64, kRY = 8, kPY = 76, kZc = 128;

// Isotropic K^3 (K = 3, 5), z-register streaming (2.5-D blocking): a CTA owns
// a 32 (x) x 64 (y) column of outputs over kZc planes.  Lane = x row, warp = a
// run of RY consecutive y outputs; a warp's window loads are 16-byte loads
// from 32 rows whose stride (kPY = 76 floats, 12 banks) puts every
// quarter-warp on distinct banks.  Every input plane is read from shared
// memory ONCE per thread -- its K rows around the thread's x -- and scattered
// into the K output planes that read it, whose partial sums live in
// registers (acc[k]: output p - H + k, tap plane az = k).  Planes stream from
// the top down, so each output still receives its taps in the reference's
// (az, ax, ay) order (az = 0 reads plane o + H): EXACT stays bit-identical.
// The ring holds the current plane and D in flight (cp.async, one barrier per
// plane; a thread's share of a plane's copies -- x reflected, halo y
// reflected or zero -- is fixed for the whole column and computed once), and
// the weights are kernel parameters (constant-bank operands: no registers, no
// loads).  FAST pairs the y outputs into packed fp32x2 FMAs and takes 16 y
// outputs per thread (128 threads), EXACT 8 (256 threads).  Round 2 (C3 image,
// 1024^3, 3^3): the previous kernel (every output plane re-reading its K^2
// rows) 4.19 / 5.03 ms FAST / EXACT, this one 2.32 / 2.63 ms (58 / 51 % of
// HBM); D = 3, 32- or 64-plane columns and 288-byte bulk copies per row (TMA)
// all measured slower.
template <typename Acc, int KW>
struct PixW {
    Acc w[KW];
};

__device__ __forceinline__ float2 ffma2_p(float2 a, float2 b, float2 c) {  // fma.rn.f32x2 (sm_100)
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n"
        "mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n mov.b64 rc, {%6, %7};\n"
        "fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

// a plane slot: PX rows of kPY floats, rounded to 128 bytes (TMA destinations)
constexpr int plane_floats(int K) { return ((kSx + 2 * (K / 2)) * kPY + 31) & ~31; }

template <typename Acc, int K, bool SKIP, int RY = kRY>  // RY: y outputs per thread (warps = kSy / RY)
__global__ void __launch_bounds__(32 * kSy / RY, RY == 8 ? (sizeof(Acc) == 4 ? (K == 3 ? 4 : 3) : 2) : (sizeof(Acc) == 4 ? (K == 3 ? 5 : 3) : 2))
    k_convolve_pixels_zreg(PixArgs a, const __grid_constant__ PixW<Acc, K * K * K> W, int txd, int tyd, int zc,
                           const __grid_constant__ CUtensorMap tmap, int use_tma) {
    constexpr int D = 2;  // prefetch distance (planes)
    constexpr int NT = 32 * kSy / RY;
    constexpr int H = K / 2, PX = kSx + 2 * H, OFF = 4 - H, PY = kPY, PLANE = plane_floats(K), NS = D + 1;
    static_assert(kSx == 32 && kSy % RY == 0 && RY % 4 == 0, "lane = x row, warp = y run");
    extern __shared__ __align__(128) float ring[];  // NS planes
    __shared__ __align__(8) uint64_t bars[NS];      // TMA planes: one mbarrier per slot
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ty = blockIdx.x % tyd, t2 = blockIdx.x / tyd;
    const int tx = t2 % txd, tzc = t2 / txd;
    const int x0 = tx * kSx, y0 = ty * kSy, zc0 = tzc * zc, zc1 = min(zc0 + zc, a.nz);
    const bool vec = (a.ny & 3) == 0 && y0 + kSy <= a.ny;  // 16-byte aligned, whole interior in range
    const bool zpad = a.pad == APRGPU_PAD_ZERO;
    // TMA: ONE tensor copy per plane (the box of PX rows x kPY floats from
    // (x0 - H, y0 - 4), the slot's exact layout), issued by one thread on the
    // slot's mbarrier -- no per-thread copies through the LSU.  Its
    // out-of-range cells read as zero: right for zero padding everywhere; with
    // reflection only where every cell the outputs read is inside the volume
    // (else the cp.async path reflects)
    const bool tma_tile = use_tma && (zpad || (x0 - H >= 0 && x0 + kSx + H <= a.nx && y0 - H >= 0 &&
                                               y0 + kSy + H <= a.ny));
    auto tma_plane = [&](int z) { return tma_tile && (zpad || (z >= 0 && z < a.nz)); };
    if (tma_tile && tid == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    }
    __syncthreads();
    unsigned phase = 0;  // per slot: the parity of its next TMA completion
    // vec: a plane is PX rows x 16 interior chunks of 16 bytes + PX x 2H halo
    // cells; each thread's share (<= NDESC copies) is fixed for the whole z
    // column, so its source offsets within a plane (x reflected, halo y
    // reflected; -1: a zero) and slot offsets are computed once
    constexpr int NCH = PX * (kSy / 4), NCOPY = NCH + PX * 2 * H;
    constexpr int NDESC = (NCOPY + NT - 1) / NT;
    int sro[NDESC], dso[NDESC];
#pragma unroll
    for (int d = 0; d < NDESC; ++d) {
        const int i = tid + d * NT;
        sro[d] = -2;  // (none)
        dso[d] = 0;
        if (i >= NCOPY) continue;
        const int r = i < NCH ? i / (kSy / 4) : (i - NCH) / (2 * H);
        const int x = x0 + r - H;
        const bool xz = (x < 0 || x >= a.nx) && zpad;
        const int xo = reflect_p(x, a.nx) * a.ny;
        if (i < NCH) {
            const int c = i % (kSy / 4);
            dso[d] = r * PY + OFF + H + 4 * c;
            sro[d] = xz ? -1 : xo + y0 + 4 * c;
        } else {
            const int k = (i - NCH) % (2 * H);
            const int c = k < H ? k : kSy + k;  // box cell: y = y0 + c - H
            const int y = y0 + c - H;
            dso[d] = r * PY + OFF + c;
            sro[d] = xz || ((y < 0 || y >= a.ny) && zpad) ? -1 : xo + reflect_p(y, a.ny);
        }
    }
    auto load = [&](int z, int si) {  // input plane z into slot si (reflected / zero outside the volume)
        float* pl = ring + si * PLANE;
        const bool zout = z < 0 || z >= a.nz;
        const int zr = reflect_p(z, a.nz);
        if (tma_plane(z)) {
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (the slot's last reads)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[si])),
                             "r"(static_cast<unsigned>(PX * PY * sizeof(float)))
                             : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4}], [%5];" ::"r"(smem_u32(pl)),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(y0 - 4), "r"(x0 - H), "r"(z), "r"(smem_u32(&bars[si]))
                    : "memory");
            }
        } else if (vec) {
            const float* pb = a.in + static_cast<size_t>(zr) * a.nx * a.ny;
#pragma unroll
            for (int d = 0; d < NDESC; ++d) {
                if (sro[d] == -2) continue;
                const bool wide = tid + d * NT < NCH;
                if (sro[d] < 0 || (zout && zpad)) {
                    if (wide) *reinterpret_cast<float4*>(pl + dso[d]) = make_float4(0.f, 0.f, 0.f, 0.f);
                    else pl[dso[d]] = 0.0f;
                } else if (wide) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     static_cast<unsigned>(__cvta_generic_to_shared(pl + dso[d]))),
                                 "l"(pb + sro[d])
                                 : "memory");
                } else {
                    cp_async_4(pl + dso[d], pb + sro[d]);
                }
            }
        } else {  // (ragged or unaligned rows: element-wise)
            for (int r = warp; r < PX; r += NT / 32) {
                const int x = x0 + r - H;
                float* dst = pl + r * PY + OFF;  // dst[c]: y = y0 + c - H
                if ((zout || x < 0 || x >= a.nx) && zpad) {
                    for (int c = lane; c < kSy + 2 * H; c += 32) dst[c] = 0.0f;
                    continue;
                }
                const float* src = a.in + (static_cast<size_t>(zr) * a.nx + reflect_p(x, a.nx)) * a.ny;
                for (int c = lane; c < kSy + 2 * H; c += 32) {
                    const int y = y0 + c - H;
                    if (y >= 0 && y < a.ny) cp_async_4(dst + c, src + y);
                    else if (!zpad) cp_async_4(dst + c, src + reflect_p(y, a.ny));
                    else dst[c] = 0.0f;
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ox = lane, oy = warp * RY;
    const bool live = x0 + ox < a.nx && y0 + oy < a.ny;
    const int top = zc1 - 1 + H, bot = zc0 - H;  // planes top .. bot, descending
    int cur = top % NS;  // slot of plane p (top >= 1)
    for (int i = 0; i < D; ++i) {
        if (top - i >= bot) load(top - i, (top - i) % NS);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    constexpr int SH = OFF & 3, NL = (SH + RY + 2 * H + 3) & ~3;
    Acc acc[K][RY];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int j = 0; j < RY; ++j) acc[k][j] = Acc(0);
    float* dst = a.out + (static_cast<size_t>(top - H) * a.nx + (x0 + ox)) * a.ny + y0 + oy;
    const size_t zstride = static_cast<size_t>(a.nx) * a.ny;
    const bool vst = y0 + oy + RY <= a.ny && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && (zstride & 3) == 0;
    for (int p = top; p >= bot; --p) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");  // plane p landed (cp.async planes)
        if (tma_plane(p)) {  // (TMA planes)
            mbar_wait(&bars[cur], (phase >> cur) & 1u);
            phase ^= 1u << cur;
        }
        __syncthreads();  // ... for every thread; plane p + 1's slot is free
        const int nxt = cur == NS - 1 ? 0 : cur + 1;  // the slot of p + 1 == p - D (NS = D + 1)
        if (p - D >= bot) load(p - D, nxt);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        const float* pl = ring + cur * PLANE;
        cur = cur == 0 ? NS - 1 : cur - 1;
#pragma unroll
        for (int ax = 0; ax < K; ++ax) {
            const float* row = pl + (ox + 2 * H - ax) * PY + (OFF - SH) + oy;
            float win[NL];
#pragma unroll
            for (int i = 0; i < NL; i += 4) {
                const float4 t = *reinterpret_cast<const float4*>(row + i);
                win[i] = t.x;
                win[i + 1] = t.y;
                win[i + 2] = t.z;
                win[i + 3] = t.w;
            }
            // output p - H + k takes plane p with weight plane az = k
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int ay = 0; ay < K; ++ay) {
                    const Acc wa = W.w[(k * K + ax) * K + ay];
                    if (SKIP && wa == Acc(0)) continue;  // (convolve.hpp:86-88)
                    if constexpr (sizeof(Acc) == 4) {
#pragma unroll
                        for (int j = 0; j < RY; j += 2) {
                            const float2 r = ffma2_p(make_float2(wa, wa),
                                                     make_float2(win[SH + j + 2 * H - ay], win[SH + j + 1 + 2 * H - ay]),
                                                     make_float2(acc[k][j], acc[k][j + 1]));
                            acc[k][j] = r.x;
                            acc[k][j + 1] = r.y;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < RY; ++j)
                            acc[k][j] = fma(wa, static_cast<Acc>(win[SH + j + 2 * H - ay]), acc[k][j]);
                    }
                }
        }
        // output p + H (tap plane 2H) is complete; dst tracks output p - H, so it is 2H planes up
        const int o = p + H;
        if (live && o >= zc0 && o < zc1) {
            float* d = dst + 2 * H * zstride;
            if (vst) {
#pragma unroll
                for (int j = 0; j < RY; j += 4)
                    __stcs(reinterpret_cast<float4*>(d + j),
                           make_float4(static_cast<float>(acc[K - 1][j]), static_cast<float>(acc[K - 1][j + 1]),
                                       static_cast<float>(acc[K - 1][j + 2]), static_cast<float>(acc[K - 1][j + 3])));
            } else {
#pragma unroll
                for (int j = 0; j < RY; ++j)
                    if (y0 + oy + j < a.ny) d[j] = static_cast<float>(acc[K - 1][j]);
            }
        }
        dst -= zstride;
        // the sets move up one plane (register moves; unrolling the plane loop by K to rotate
        // them instead spilled at 64 registers and measured slower)
#pragma unroll
        for (int k = K - 1; k > 0; --k)
#pragma unroll
            for (int j = 0; j < RY; ++j) acc[k][j] = acc[k - 1][j];
#pragma unroll
        for (int j = 0; j < RY; ++j) acc[0][j] = Acc(0);
    }
}

}  // namespace

void convolve_pixels_device(aprgpu_ctx* ctx, const float* in, int nz, int nx, int ny, const float* w_dev, int kz,
                            int kx, int ky, int pad, int accum, float* out, cudaStream_t s, bool any_zero_w,
                            const float* w_host) {
    if (kz > kPixMaxK || kx > kPixMaxK || ky > kPixMaxK)
        fail(APRGPU_ERR_CAPABILITY, "convolve_pixels: stencil extent exceeds the supported maximum");
    if (nz <= 0 || nx <= 0 || ny <= 0) return;
    PixArgs a{in, out, nz, nx, ny, kz, kx, ky, pad, w_dev};
    const int tzd = (nz + kPz - 1) / kPz, txd = (nx + kPx - 1) / kPx, tyd = (ny + kPy - 1) / kPy;
    const uint64_t blocks = static_cast<uint64_t>(tzd) * txd * tyd;
    if (blocks >= (1ull << 31)) fail(APRGPU_ERR_CAPABILITY, "convolve_pixels: volume too large");
    if (kz == kx && kx == ky && (kz == 3 || kz == 5) && !std::getenv("APRGPU_PIXELS_TILED")) {
        const bool ex = accum == APRGPU_ACCUM_EXACT;
        static const int zc = [] {  // planes per CTA (APRGPU_PIXELS_ZC: A/B experiments)
            const char* e = std::getenv("APRGPU_PIXELS_ZC");
            return e ? std::max(1, std::atoi(e)) : kZc;
        }();
        const int ry = ex ? 8 : 16;  // y outputs per thread (A/B: FAST 2.35 -> 2.32 ms, EXACT 2.63 -> 2.76 ms at 16)
        const int sxd = (nx + kSx - 1) / kSx, syd = (ny + kSy - 1) / kSy, szd = (nz + zc - 1) / zc;
        const unsigned g = static_cast<unsigned>(static_cast<uint64_t>(szd) * sxd * syd);
        const int h = kz / 2;
        const int rb = 3 * (kz == 3 ? plane_floats(3) : plane_floats(5)) * static_cast<int>(sizeof(float));
        // the input as a 3-D tensor map for the TMA plane loads (ny * 4 bytes must be a 16-byte multiple)
        CUtensorMap tm{};
        int use_tma = 0;
        static const bool tma_on = [] {  // APRGPU_PIXELS_TMA=0: cp.async planes only (A/B)
            const char* e = std::getenv("APRGPU_PIXELS_TMA");
            return !(e && e[0] == '0');
        }();
        static PFN_cuTensorMapEncodeTiled encode = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess) {
                cudaGetLastError();
                fn = nullptr;
            }
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
        }();
        if (tma_on && encode && (ny & 3) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
            const cuuint64_t dims[3] = {static_cast<cuuint64_t>(ny), static_cast<cuuint64_t>(nx),
                                        static_cast<cuuint64_t>(nz)};
            const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ny) * 4, static_cast<cuuint64_t>(nx) * ny * 4};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(kPY), static_cast<cuuint32_t>(kSx + 2 * h), 1};
            const cuuint32_t es[3] = {1, 1, 1};
            use_tma = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        static OncePerDevice zattr;
        zattr([] {
            const int mx = 3 * plane_floats(5) * static_cast<int>(sizeof(float));
#define APRGPU_SET_PIX(A, K_, S_)                                                                                      \
    APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_zreg<A, K_, S_, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  mx));                                                                              \
    APR_CUDA(cudaFuncSetAttribute(k_convolve_pixels_zreg<A, K_, S_, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx))
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
        const bool skip = any_zero_w;
#define APRGPU_LAUNCH_PIX(A, K_)                                                                                \
    do {                                                                                                        \
        PixW<A, K_ * K_ * K_> pw;                                                                               \
        for (int i = 0; i < K_ * K_ * K_; ++i) pw.w[i] = static_cast<A>(w_host[i]);                             \
        if (ry == 16) {                                                                                         \
            if (skip) k_convolve_pixels_zreg<A, K_, true, 16><<<g, 128, rb, s>>>(a, pw, sxd, syd, zc, tm, use_tma);          \
            else k_convolve_pixels_zreg<A, K_, false, 16><<<g, 128, rb, s>>>(a, pw, sxd, syd, zc, tm, use_tma);              \
        } else {                                                                                                \
            if (skip) k_convolve_pixels_zreg<A, K_, true, 8><<<g, 256, rb, s>>>(a, pw, sxd, syd, zc, tm, use_tma);           \
            else k_convolve_pixels_zreg<A, K_, false, 8><<<g, 256, rb, s>>>(a, pw, sxd, syd, zc, tm, use_tma);               \
        }                                                                                                       \
    } while (0)
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
