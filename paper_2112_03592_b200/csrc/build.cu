// Device construction of APRs from pixels (the input side of the hot path):
//   generate_spheres   (synthetic.hpp:74-111, separable_gaussian :34-67)
//   build_apr          (build.hpp:290-312) with SigmaPolicy::constant(range),
//                      central-difference gradient, no smoothing passes:
//     gradient_magnitude (:42-75) -> level_function (:113-129) -> +1 safety
//     level -> solve_levels (:136-248) -> init_tree_structure -> sample_particles
//     (:252-284).
// Every floating-point step reproduces the reference's operation order with
// explicit round-to-nearest intrinsics (the reference oracle is compiled with
// -ffp-contract=off), so the structure and values match the reference build.
// Dense per-level grids live in HBM (int8 levels, fp64 sums only below the
// finest level): ~12 GB peak at 1024^3 instead of the reference's 34 GB host RSS.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <cmath>

#include "common.cuh"

namespace aprgpu {
namespace {

// ---- CounterRng (rng.hpp:8-55), host side ------------------------------------
uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
struct CounterRng {
    uint64_t seed, counter = 0;
    explicit CounterRng(uint64_t s) : seed(s) {}
    uint64_t next_u64() { return splitmix64(seed ^ splitmix64(counter++)); }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
};

struct Sphere {
    double cz, cx, cy, r2;
    float intensity;
};

__device__ __forceinline__ void decode(uint64_t i, int nx, int ny, int& z, int& x, int& y) {
    y = static_cast<int>(i % ny);
    const uint64_t t = i / ny;
    x = static_cast<int>(t % nx);
    z = static_cast<int>(t / nx);
}

__global__ void k_spheres(float* __restrict__ v, int nz, int nx, int ny, float background,
                          const Sphere* __restrict__ sp, int n_sp) {
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, nx, ny, z, x, y);
        float val = background;
        for (int s = 0; s < n_sp; ++s) {
            const double dz = static_cast<double>(z) - sp[s].cz;
            const double dx = static_cast<double>(x) - sp[s].cx;
            const double dy = static_cast<double>(y) - sp[s].cy;
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dz, dz), __dmul_rn(dx, dx)), __dmul_rn(dy, dy));
            if (d2 <= sp[s].r2) val = sp[s].intensity;
        }
        v[i] = val;
    }
}

__constant__ double c_gauss[32];

// one axis of separable_gaussian (synthetic.hpp:60-66): acc in double from 0,
// taps in i = -h..h order, reflect boundary
__global__ void k_blur_axis(const float* __restrict__ in, float* __restrict__ out, int nz, int nx, int ny, int axis,
                            int h) {
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    const int dim = axis == 0 ? nz : (axis == 1 ? nx : ny);
    const uint64_t stride = axis == 0 ? static_cast<uint64_t>(nx) * ny : (axis == 1 ? static_cast<uint64_t>(ny) : 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, nx, ny, z, x, y);
        const int c = axis == 0 ? z : (axis == 1 ? x : y);
        const uint64_t base = i - static_cast<uint64_t>(c) * stride;
        double acc = 0.0;
        for (int t = -h; t <= h; ++t) {
            const int cc = reflect_dev(c + t, dim);
            acc = __dadd_rn(acc, __dmul_rn(c_gauss[t + h], static_cast<double>(in[base + static_cast<uint64_t>(cc) * stride])));
        }
        out[i] = __double2float_rn(acc);
    }
}

// gradient_magnitude (build.hpp:42-75, CentralDiff, replicate boundary) fused
// with level_function (:113-129) and the constant-sigma +1 (:301-303)
__global__ void k_targets(const float* __restrict__ v, int8_t* __restrict__ T, int nz, int nx, int ny, double E,
                          double sigma, double omega, int l_min, int l_max) {
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    const uint64_t sz = static_cast<uint64_t>(nx) * ny;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, nx, ny, z, x, y);
        const uint64_t b = i - static_cast<uint64_t>(z) * sz - static_cast<uint64_t>(x) * ny - y;
        auto at = [&](int zz, int xx, int yy) { return v[b + static_cast<uint64_t>(zz) * sz + static_cast<uint64_t>(xx) * ny + yy]; };
        const int zp = min(z + 1, nz - 1), zm = max(z - 1, 0);
        const int xp = min(x + 1, nx - 1), xm = max(x - 1, 0);
        const int yp = min(y + 1, ny - 1), ym = max(y - 1, 0);
        // 0.5 * (float - float): the difference is a float operation, then promoted
        const double gz = __dmul_rn(0.5, static_cast<double>(__fsub_rn(at(zp, x, y), at(zm, x, y))));
        const double gx = __dmul_rn(0.5, static_cast<double>(__fsub_rn(at(z, xp, y), at(z, xm, y))));
        const double gy = __dmul_rn(0.5, static_cast<double>(__fsub_rn(at(z, x, yp), at(z, x, ym))));
        const double s = __dadd_rn(__dadd_rn(__dmul_rn(gz, gz), __dmul_rn(gx, gx)), __dmul_rn(gy, gy));
        const float g = __double2float_rn(__dsqrt_rn(s));
        int lev;
        if (static_cast<double>(g) <= 0.0) {
            lev = l_min;
        } else {
            const double L = __ddiv_rn(__dmul_rn(E, sigma), static_cast<double>(g));
            const int l = static_cast<int>(ceil(log2(__ddiv_rn(omega, L))));
            lev = min(max(l, l_min), l_max);
        }
        lev = min(lev + 1, l_max);                      // constant-sigma safety level
        T[i] = static_cast<int8_t>(min(max(lev, l_min), l_max));  // solve_levels clamp (:172)
    }
}

// ---- the general BuildParams path (apr.hpp:16-33) -----------------------------
__device__ __forceinline__ int clampi(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }

// gradient_magnitude (build.hpp:42-75): central differences or Sobel, replicate
// boundary; float result.  Sobel's coefficient products d*s*s are powers of two,
// so every term is exact and only the (a, b, c)-ordered sums round.
__global__ void k_gradient(const float* __restrict__ v, float* __restrict__ out, int nz, int nx, int ny, int sobel) {
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, nx, ny, z, x, y);
        auto at = [&](int zz, int xx, int yy) {
            return v[(static_cast<uint64_t>(zz) * nx + xx) * ny + yy];
        };
        double gz = 0.0, gx = 0.0, gy = 0.0;
        if (!sobel) {
            gz = __dmul_rn(0.5, static_cast<double>(__fsub_rn(at(clampi(z + 1, nz), x, y), at(clampi(z - 1, nz), x, y))));
            gx = __dmul_rn(0.5, static_cast<double>(__fsub_rn(at(z, clampi(x + 1, nx), y), at(z, clampi(x - 1, nx), y))));
            gy = __dmul_rn(0.5, static_cast<double>(__fsub_rn(at(z, x, clampi(y + 1, ny)), at(z, x, clampi(y - 1, ny)))));
        } else {
            const double sm[3] = {0.25, 0.5, 0.25}, dd[3] = {-0.5, 0.0, 0.5};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    for (int c = 0; c < 3; ++c) {
                        const double val = at(clampi(z + a - 1, nz), clampi(x + b - 1, nx), clampi(y + c - 1, ny));
                        gz = __dadd_rn(gz, __dmul_rn(__dmul_rn(__dmul_rn(dd[a], sm[b]), sm[c]), val));
                        gx = __dadd_rn(gx, __dmul_rn(__dmul_rn(__dmul_rn(sm[a], dd[b]), sm[c]), val));
                        gy = __dadd_rn(gy, __dmul_rn(__dmul_rn(__dmul_rn(sm[a], sm[b]), dd[c]), val));
                    }
        }
        const double s2 = __dadd_rn(__dadd_rn(__dmul_rn(gz, gz), __dmul_rn(gx, gx)), __dmul_rn(gy, gy));
        out[i] = __double2float_rn(__dsqrt_rn(s2));
    }
}

// detail::box_smooth (build.hpp:22-38): 3^3 mean, replicate boundary, fp64 sum
// in (dz, dx, dy) order; floor > 0 also applies local_scale's final
// max(s, float(floor)) (build.hpp:105).
__global__ void k_box_smooth(const float* __restrict__ v, float* __restrict__ out, int nz, int nx, int ny,
                             float floor_value, int use_floor) {
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, nx, ny, z, x, y);
        double acc = 0.0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dx = -1; dx <= 1; ++dx)
                for (int dy = -1; dy <= 1; ++dy)
                    acc = __dadd_rn(acc, static_cast<double>(
                                             v[(static_cast<uint64_t>(clampi(z + dz, nz)) * nx + clampi(x + dx, nx)) * ny +
                                               clampi(y + dy, ny)]));
        float r = __double2float_rn(__ddiv_rn(acc, 27.0));
        if (use_floor) r = fmaxf(r, floor_value);
        out[i] = r;
    }
}

// local_scale's local range (build.hpp:89-103): max - min of the in-domain
// (2r+1)^3 window, in float
__global__ void k_local_range(const float* __restrict__ v, float* __restrict__ out, int nz, int nx, int ny, int r) {
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, nx, ny, z, x, y);
        float lo = v[i], hi = lo;
        for (int zz = max(z - r, 0); zz <= min(z + r, nz - 1); ++zz)
            for (int xx = max(x - r, 0); xx <= min(x + r, nx - 1); ++xx)
                for (int yy = max(y - r, 0); yy <= min(y + r, ny - 1); ++yy) {
                    const float val = v[(static_cast<uint64_t>(zz) * nx + xx) * ny + yy];
                    lo = fminf(lo, val);
                    hi = fmaxf(hi, val);
                }
        out[i] = __fsub_rn(hi, lo);
    }
}

// level_function (build.hpp:113-129) over a gradient field and a sigma field
// (sigma == null: the constant sigma_c), the constant-sigma safety level
// (:301-303) when safety, and solve_levels' clamp (:172)
__global__ void k_levels(const float* __restrict__ grad, const float* __restrict__ sigma, double sigma_c,
                         int8_t* __restrict__ T, uint64_t n, double E, double omega, int l_min, int l_max, int safety) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double g = grad[i];
        int lev;
        if (g <= 0.0) {
            lev = l_min;
        } else {
            const double sg = sigma ? static_cast<double>(sigma[i]) : sigma_c;
            const double L = __ddiv_rn(__dmul_rn(E, sg), g);
            const int l = static_cast<int>(ceil(log2(__ddiv_rn(omega, L))));
            lev = min(max(l, l_min), l_max);
        }
        if (safety) lev = min(lev + 1, l_max);
        T[i] = static_cast<int8_t>(min(max(lev, l_min), l_max));
    }
}

struct Grid3 {
    int zd, xd, yd;
    __host__ __device__ uint64_t size() const { return static_cast<uint64_t>(zd) * xd * yd; }
};

// coarse[c] = max over the (clipped) 2x2x2 children of fine (max_reduce, :158-166)
__global__ void k_max_reduce(const int8_t* __restrict__ f, Grid3 fg, int8_t* __restrict__ c, Grid3 cg) {
    const uint64_t n = cg.size();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, cg.xd, cg.yd, z, x, y);
        int m = 0;  // grids start at 0 in the reference
        for (int a = 2 * z; a < min(2 * z + 2, fg.zd); ++a)
            for (int b = 2 * x; b < min(2 * x + 2, fg.xd); ++b)
                for (int d = 2 * y; d < min(2 * y + 2, fg.yd); ++d)
                    m = max(m, static_cast<int>(f[(static_cast<uint64_t>(a) * fg.xd + b) * fg.yd + d]));
        c[i] = static_cast<int8_t>(m);
    }
}

// need[l](c) = T[l](c) >= l  OR  some fine need cell reaches c through the 3^3
// dilation (solve_levels :181-203, as a gather)
__global__ void k_need(const int8_t* __restrict__ T, Grid3 g, int l, const uint8_t* __restrict__ fine_need, Grid3 fg,
                       uint8_t* __restrict__ need) {
    const uint64_t n = g.size();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, g.xd, g.yd, z, x, y);
        uint8_t r = T[i] >= l ? 1 : 0;
        if (!r && fine_need) {
            // positions p with p/2 == c inside the fine grid; sources f within 1 of some p
            const int pz0 = 2 * z, pz1 = min(2 * z + 1, fg.zd - 1);
            const int px0 = 2 * x, px1 = min(2 * x + 1, fg.xd - 1);
            const int py0 = 2 * y, py1 = min(2 * y + 1, fg.yd - 1);
            for (int a = max(pz0 - 1, 0); a <= min(pz1 + 1, fg.zd - 1) && !r; ++a)
                for (int b = max(px0 - 1, 0); b <= min(px1 + 1, fg.xd - 1) && !r; ++b)
                    for (int d = max(py0 - 1, 0); d <= min(py1 + 1, fg.yd - 1); ++d)
                        if (fine_need[(static_cast<uint64_t>(a) * fg.xd + b) * fg.yd + d]) {
                            r = 1;
                            break;
                        }
        }
        need[i] = r;
    }
}

struct NeedLevels {
    const uint8_t* need[kMaxLevels];
    Grid3 g[kMaxLevels];
};

// G(pixel) = finest level whose need covers the pixel (solve_levels :205-223)
__global__ void k_finest_demand(NeedLevels nl, int l_min, int l_max, int8_t* __restrict__ G, Grid3 pg) {
    const uint64_t n = pg.size();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, pg.xd, pg.yd, z, x, y);
        int e = l_min;
        for (int l = l_max; l > l_min; --l) {
            const int d = l_max - l;
            const Grid3 g = nl.g[l];
            if (nl.need[l][(static_cast<uint64_t>(z >> d) * g.xd + (x >> d)) * g.yd + (y >> d)]) {
                e = l;
                break;
            }
        }
        G[i] = static_cast<int8_t>(e);
    }
}

// leaf test (solve_levels :231-246): Gmax[l](c) <= l and (l == l_min or Gmax[l-1](c/2) > l-1)
__device__ __forceinline__ bool is_leaf(const int8_t* gl, Grid3 g, const int8_t* gp, Grid3 pg, int l, int l_min, int z,
                                        int x, int y) {
    if (gl[(static_cast<uint64_t>(z) * g.xd + x) * g.yd + y] > l) return false;
    if (l > l_min && gp[(static_cast<uint64_t>(z >> 1) * pg.xd + (x >> 1)) * pg.yd + (y >> 1)] <= l - 1) return false;
    return true;
}

// one warp per row (z,x) of level l: mode 0 counts leaves, mode 1 writes y
__global__ void k_leaf_rows(int mode, const int8_t* __restrict__ gl, Grid3 g, const int8_t* __restrict__ gp, Grid3 pg,
                            int l, int l_min, uint32_t* __restrict__ counts, const uint32_t* __restrict__ rb,
                            uint32_t row0, uint16_t* __restrict__ y_out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t rows = static_cast<uint64_t>(g.zd) * g.xd;
    for (uint64_t r = warp; r < rows; r += nw) {
        const int z = static_cast<int>(r / g.xd), x = static_cast<int>(r % g.xd);
        uint32_t pos = mode ? rb[row0 + r] : 0;
        uint32_t cnt = 0;
        for (int y0 = 0; y0 < g.yd; y0 += 32) {
            const int y = y0 + lane;
            const bool leaf = y < g.yd && is_leaf(gl, g, gp, pg, l, l_min, z, x, y);
            const unsigned m = __ballot_sync(kFull, leaf);
            if (mode && leaf) y_out[pos + __popc(m & ((1u << lane) - 1))] = static_cast<uint16_t>(y);
            pos += __popc(m);
            cnt += __popc(m);
        }
        if (!mode && lane == 0) counts[row0 + r] = cnt;
    }
}

// sample_particles (build.hpp:252-284): fp64 sum pyramid, children gathered in
// the reference's (z,x,y) visiting order; the finest level reads the volume.
__global__ void k_sum_reduce(const float* __restrict__ vf, const double* __restrict__ fs, Grid3 fg,
                             double* __restrict__ cs, Grid3 cg) {
    const uint64_t n = cg.size();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int z, x, y;
        decode(i, cg.xd, cg.yd, z, x, y);
        double s = 0.0;
        for (int a = 2 * z; a < min(2 * z + 2, fg.zd); ++a)
            for (int b = 2 * x; b < min(2 * x + 2, fg.xd); ++b)
                for (int d = 2 * y; d < min(2 * y + 2, fg.yd); ++d) {
                    const uint64_t fi = (static_cast<uint64_t>(a) * fg.xd + b) * fg.yd + d;
                    s = __dadd_rn(s, vf ? static_cast<double>(vf[fi]) : fs[fi]);
                }
        cs[i] = s;
    }
}

struct SumLevels {
    const double* s[kMaxLevels];
    Grid3 g[kMaxLevels];
};

__global__ void k_sample(AccessView a, SumLevels sl, const float* __restrict__ vol, int l_max, int nz, int nx, int ny,
                         const uint32_t* __restrict__ work, uint64_t n_work, int level, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const LevelG lg = a.g[level];
    const int s = 1 << (l_max - level);
    for (uint64_t wi = warp; wi < n_work; wi += nw) {
        const uint32_t row = work[wi];
        const uint32_t loc = row - lg.row0;
        const int z = static_cast<int>(loc / lg.xd), x = static_cast<int>(loc % lg.xd);
        const uint32_t b = a.rb[row], e = a.rb[row + 1];
        for (uint32_t i = b + lane; i < e; i += 32) {
            const int y = a.y[i];
            if (level == l_max) {
                out[i] = vol[(static_cast<uint64_t>(z) * nx + x) * ny + y];  // float(v / 1.0)
            } else {
                const Grid3 g = sl.g[level];
                const double sum = sl.s[level][(static_cast<uint64_t>(z) * g.xd + x) * g.yd + y];
                const double wz = min((z + 1) * s, nz) - z * s;
                const double wx = min((x + 1) * s, nx) - x * s;
                const double wy = min((y + 1) * s, ny) - y * s;
                out[i] = __double2float_rn(__ddiv_rn(sum, __dmul_rn(__dmul_rn(wz, wx), wy)));
            }
        }
    }
}

int compute_l_max(int nz, int nx, int ny) {
    const int m = std::max(nz, std::max(nx, ny));
    int l = 0;
    while ((1 << l) < m) ++l;
    return l;
}

unsigned grid_for(aprgpu_ctx* ctx, uint64_t n, unsigned per = 256) {
    return static_cast<unsigned>(std::min<uint64_t>((n + per - 1) / per, static_cast<uint64_t>(ctx->sm_count) * 32));
}

}  // namespace

// ---- entry points used by api.cu ----------------------------------------------
void generate_spheres_device(aprgpu_ctx* ctx, int nz, int nx, int ny, int count, double min_r, double max_r,
                             double background, double min_i, double max_i, double blur, uint64_t seed, float* out,
                             cudaStream_t s) {
    CounterRng rng(seed);
    std::vector<Sphere> sp(count);
    for (auto& q : sp) {  // synthetic.hpp:76-83
        const double r = rng.uniform(min_r, max_r);
        q.cz = rng.uniform(r, std::max<double>(nz - r, r));
        q.cx = rng.uniform(r, std::max<double>(nx - r, r));
        q.cy = rng.uniform(r, std::max<double>(ny - r, r));
        q.intensity = static_cast<float>(rng.uniform(min_i, max_i));
        q.r2 = r * r;
    }
    GpuBuf dsp, tmp;
    dsp.ensure(sizeof(Sphere) * std::max(count, 1));
    if (count) APR_CUDA(cudaMemcpyAsync(dsp.p, sp.data(), sizeof(Sphere) * count, cudaMemcpyHostToDevice, s));
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    k_spheres<<<grid_for(ctx, n), 256, 0, s>>>(out, nz, nx, ny, static_cast<float>(background), dsp.as<Sphere>(),
                                               count);
    count_launch(ctx);
    APR_CUDA(cudaGetLastError());
    if (blur > 0.0) {  // separable_gaussian (synthetic.hpp:34-67)
        const int size = 2 * static_cast<int>(std::ceil(3.0 * blur)) + 1;
        const int h = size / 2;
        if (size > 32) fail(APRGPU_ERR_CAPABILITY, "blur sigma too large");
        std::vector<double> g(size);
        double norm = 0.0;
        for (int i = -h; i <= h; ++i) {
            g[i + h] = std::exp(-0.5 * i * i / (blur * blur));
            norm += g[i + h];
        }
        for (double& w : g) w /= norm;
        APR_CUDA(cudaMemcpyToSymbolAsync(c_gauss, g.data(), sizeof(double) * size, 0, cudaMemcpyHostToDevice, s));
        tmp.ensure(sizeof(float) * n);
        float* a = out;
        float* b = tmp.as<float>();
        for (int axis = 0; axis < 3; ++axis) {
            k_blur_axis<<<grid_for(ctx, n), 256, 0, s>>>(a, b, nz, nx, ny, axis, h);
            count_launch(ctx);
            APR_CUDA(cudaGetLastError());
            std::swap(a, b);
        }
        if (a != out) APR_CUDA(cudaMemcpyAsync(out, a, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
    }
    APR_CUDA(cudaStreamSynchronize(s));
}

void build_apr_device(aprgpu_ctx* ctx, const float* vol, int nz, int nx, int ny, double rel_error, aprgpu_apr* apr,
                      GpuBuf& values_out, cudaStream_t s) {
    build_apr_device(ctx, vol, nz, nx, ny, nullptr, rel_error, apr, values_out, s);
}

// params == null: the spheres recipe, SigmaPolicy::constant(intensity_range(v))
void build_apr_device(aprgpu_ctx* ctx, const float* vol, int nz, int nx, int ny, const aprgpu_build_params* params,
                      double rel_error, aprgpu_apr* apr, GpuBuf& values_out, cudaStream_t s) {
    if (params) rel_error = params->rel_error;
    if (nz < 1 || nx < 1 || ny < 1) fail(APRGPU_ERR_RANGE, "build_apr: empty volume");
    if (ny > 65536) fail(APRGPU_ERR_CAPABILITY, "y dimension exceeds the 16-bit index limit");
    const int l_max = compute_l_max(nz, nx, ny);
    const int l_min = std::min(1, l_max);
    if (l_max >= kMaxLevels) fail(APRGPU_ERR_CAPABILITY, "too many levels");
    const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
    auto gdim = [&](int l) { return Grid3{grid_dim_dev(nz, l_max, l), grid_dim_dev(nx, l_max, l), grid_dim_dev(ny, l_max, l)}; };

    // intensity_range (pixel_volume.hpp:58) -> SigmaPolicy::constant(range) ->
    // local_scale's constant field float(max(range, 1e-3 * max(1e-30f, range)))
    GpuBuf red, redtmp;
    red.ensure(2 * sizeof(float));
    size_t tb = 0;
    cub::DeviceReduce::Min(nullptr, tb, vol, red.as<float>(), static_cast<int64_t>(n), s);
    redtmp.ensure(tb + 16);
    tb = redtmp.bytes;
    APR_CUDA(cub::DeviceReduce::Min(redtmp.p, tb, vol, red.as<float>(), static_cast<int64_t>(n), s));
    tb = redtmp.bytes;
    APR_CUDA(cub::DeviceReduce::Max(redtmp.p, tb, vol, red.as<float>() + 1, static_cast<int64_t>(n), s));
    float mm[2];
    APR_CUDA(cudaMemcpyAsync(mm, red.p, sizeof(mm), cudaMemcpyDeviceToHost, s));
    APR_CUDA(cudaStreamSynchronize(s));
    const float range = mm[1] - mm[0];
    const aprgpu_build_params bp =
        params ? *params : aprgpu_build_params{rel_error, 0, static_cast<double>(range), 2, 0.0, 0, 0};
    if (bp.sigma_mode != 0 && bp.sigma_mode != 1) fail(APRGPU_ERR_INVALID, "build_apr: bad sigma mode");
    if (bp.gradient_mode != 0 && bp.gradient_mode != 1) fail(APRGPU_ERR_INVALID, "build_apr: bad gradient mode");
    if (bp.smoothing_passes < 0 || bp.sigma_window < 0) fail(APRGPU_ERR_RANGE, "build_apr: negative pass count or window");
    // local_scale (build.hpp:80-108): floor = policy.floor, or 1e-3 x intensity range
    const double floor_value = bp.sigma_floor > 0.0 ? bp.sigma_floor : 1e-3 * std::max(1e-30f, range);
    const double sigma = static_cast<double>(static_cast<float>(std::max(bp.sigma_value, floor_value)));
    apr->params = bp;
    const double omega = static_cast<double>(1u << l_max);

    // dense per-level grids
    std::vector<GpuBuf> T(l_max + 1), need(l_max + 1), Gm(l_max + 1);
    T[l_max].ensure(n);
    if (bp.sigma_mode == 0 && bp.gradient_mode == 0 && bp.smoothing_passes == 0) {
        // fused: central differences -> constant sigma -> levels
        k_targets<<<grid_for(ctx, n), 256, 0, s>>>(vol, T[l_max].as<int8_t>(), nz, nx, ny, rel_error, sigma, omega,
                                                   l_min, l_max);
        count_launch(ctx);
    } else {
        GpuBuf grad, tmp, sig;
        grad.ensure(4 * n);
        k_gradient<<<grid_for(ctx, n), 256, 0, s>>>(vol, grad.as<float>(), nz, nx, ny, bp.gradient_mode);
        count_launch(ctx);
        for (int pass = 0; pass < bp.smoothing_passes; ++pass) {  // build.hpp:298
            tmp.ensure(4 * n);
            k_box_smooth<<<grid_for(ctx, n), 256, 0, s>>>(grad.as<float>(), tmp.as<float>(), nz, nx, ny, 0.0f, 0);
            count_launch(ctx);
            std::swap(grad.p, tmp.p);  // (GpuBuf is move-only: swap the owned buffers)
            std::swap(grad.bytes, tmp.bytes);
        }
        if (bp.sigma_mode == 1) {  // local range -> box_smooth -> floor
            sig.ensure(4 * n);
            tmp.ensure(4 * n);
            k_local_range<<<grid_for(ctx, n), 256, 0, s>>>(vol, tmp.as<float>(), nz, nx, ny, bp.sigma_window);
            k_box_smooth<<<grid_for(ctx, n), 256, 0, s>>>(tmp.as<float>(), sig.as<float>(), nz, nx, ny,
                                                          static_cast<float>(floor_value), 1);
            count_launch(ctx, 2);
        }
        k_levels<<<grid_for(ctx, n), 256, 0, s>>>(grad.as<float>(), bp.sigma_mode == 1 ? sig.as<float>() : nullptr,
                                                  sigma, T[l_max].as<int8_t>(), n, rel_error, omega, l_min, l_max,
                                                  bp.sigma_mode == 0 ? 1 : 0);
        count_launch(ctx);
        APR_CUDA(cudaStreamSynchronize(s));  // (the temporaries are freed on scope exit)
    }
    APR_CUDA(cudaGetLastError());
    for (int l = l_max - 1; l >= l_min; --l) {
        const Grid3 g = gdim(l);
        T[l].ensure(g.size());
        k_max_reduce<<<grid_for(ctx, g.size()), 256, 0, s>>>(T[l + 1].as<int8_t>(), gdim(l + 1), T[l].as<int8_t>(), g);
        count_launch(ctx);
    }
    for (int l = l_max; l >= l_min; --l) {
        const Grid3 g = gdim(l);
        need[l].ensure(g.size());
        k_need<<<grid_for(ctx, g.size()), 256, 0, s>>>(T[l].as<int8_t>(), g, l,
                                                        l < l_max ? need[l + 1].as<uint8_t>() : nullptr,
                                                        l < l_max ? gdim(l + 1) : g, need[l].as<uint8_t>());
        count_launch(ctx);
    }
    APR_CUDA(cudaGetLastError());
    for (auto& b : T) b.release();
    NeedLevels nl{};
    for (int l = l_min; l <= l_max; ++l) {
        nl.need[l] = need[l].as<uint8_t>();
        nl.g[l] = gdim(l);
    }
    Gm[l_max].ensure(n);
    k_finest_demand<<<grid_for(ctx, n), 256, 0, s>>>(nl, l_min, l_max, Gm[l_max].as<int8_t>(), gdim(l_max));
    count_launch(ctx);
    for (int l = l_max - 1; l >= l_min; --l) {
        const Grid3 g = gdim(l);
        Gm[l].ensure(g.size());
        k_max_reduce<<<grid_for(ctx, g.size()), 256, 0, s>>>(Gm[l + 1].as<int8_t>(), gdim(l + 1), Gm[l].as<int8_t>(), g);
        count_launch(ctx);
    }
    APR_CUDA(cudaGetLastError());
    APR_CUDA(cudaStreamSynchronize(s));
    for (auto& b : need) b.release();

    // leaf rows -> CSR (assemble_access, linear_access.hpp:101-130)
    DevAccess& A = apr->leaf;
    A.l_min = l_min;
    A.l_max = l_max;
    A.zd.assign(l_max + 1, 0);
    A.xd.assign(l_max + 1, 0);
    A.yd.assign(l_max + 1, 0);
    A.level_offset.assign(l_max + 1, 0);
    uint64_t rows = 0;
    for (int l = l_min; l <= l_max; ++l) {
        const Grid3 g = gdim(l);
        A.zd[l] = g.zd;
        A.xd[l] = g.xd;
        A.yd[l] = g.yd;
        A.level_offset[l] = rows;
        rows += static_cast<uint64_t>(g.zd) * g.xd;
    }
    A.n_rows = rows;
    GpuBuf counts, scan_tmp;
    counts.ensure(sizeof(uint32_t) * (rows + 1));
    APR_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * (rows + 1), s));
    APR_CUDA(cudaMalloc(&A.rb, sizeof(uint32_t) * (rows + 1)));
    for (int mode = 0; mode < 2; ++mode) {
        for (int l = l_min; l <= l_max; ++l) {
            const Grid3 g = gdim(l);
            const Grid3 pg = l > l_min ? gdim(l - 1) : g;
            const uint64_t r = static_cast<uint64_t>(g.zd) * g.xd;
            k_leaf_rows<<<grid_for(ctx, r * 32), 256, 0, s>>>(mode, Gm[l].as<int8_t>(), g,
                                                              l > l_min ? Gm[l - 1].as<int8_t>() : nullptr, pg, l, l_min,
                                                              counts.as<uint32_t>(), A.rb,
                                                              static_cast<uint32_t>(A.level_offset[l]), A.y);
            count_launch(ctx);
        }
        APR_CUDA(cudaGetLastError());
        if (mode == 0) {
            size_t sb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, sb, counts.as<uint32_t>(), A.rb, static_cast<int64_t>(rows + 1), s);
            scan_tmp.ensure(sb + 16);
            sb = scan_tmp.bytes;
            APR_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp.p, sb, counts.as<uint32_t>(), A.rb,
                                                   static_cast<int64_t>(rows + 1), s));
            uint32_t total = 0;
            APR_CUDA(cudaMemcpyAsync(&total, A.rb + rows, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            A.n_particles = total;
            APR_CUDA(cudaMalloc(&A.y, 2ull * total + 2));
        }
    }
    APR_CUDA(cudaStreamSynchronize(s));
    for (auto& b : Gm) b.release();
    counts.release();
    build_work_lists(ctx, A);
    build_tile_lists(ctx, A);
    build_tree_structure(ctx, apr);

    // sample_particles
    std::vector<GpuBuf> S(l_max + 1);
    SumLevels sl{};
    for (int l = l_max - 1; l >= l_min; --l) {
        const Grid3 g = gdim(l);
        S[l].ensure(sizeof(double) * g.size());
        k_sum_reduce<<<grid_for(ctx, g.size()), 256, 0, s>>>(l == l_max - 1 ? vol : nullptr,
                                                             l == l_max - 1 ? nullptr : S[l + 1].as<double>(),
                                                             gdim(l + 1), S[l].as<double>(), g);
        count_launch(ctx);
        sl.s[l] = S[l].as<double>();
        sl.g[l] = g;
    }
    APR_CUDA(cudaGetLastError());
    values_out.ensure(4 * A.n_particles + 4);
    const AccessView av = A.view();
    for (int l = l_min; l <= l_max; ++l) {
        const uint64_t nwk = A.work_off[l + 1] - A.work_off[l];
        if (!nwk) continue;
        k_sample<<<grid_for(ctx, nwk * 32), 256, 0, s>>>(av, sl, vol, l_max, nz, nx, ny, A.work + A.work_off[l], nwk, l,
                                                        values_out.as<float>());
        count_launch(ctx);
    }
    APR_CUDA(cudaGetLastError());
    APR_CUDA(cudaStreamSynchronize(s));
}

}  // namespace aprgpu
