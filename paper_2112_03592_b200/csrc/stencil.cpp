// Host-side stencil construction: presets and the restriction to coarser levels.
//
// restrict_stencil (stencil.hpp:127-160) computes, for a fine stencil w and a
// level gap delta (m = 2^delta), the coarse stencil acc[K] accumulated in
// double over all m^3 fine offsets o and all k^3 stencil taps r in the order
// (oz,ox,oy,rz,rx,ry), then rounded once to float.  That loop is O(m^3 k^3) --
// 26 min for one 3^3 pyramid at C4 (SURVEY.md §7 hard part 7).  Here:
//
//  * per axis, the fine offsets o with -floor_div(o - r, m) == K form the
//    contiguous range r in [o + (K-1)m + 1, o + Km]; so the number of o hitting
//    K for tap r is c(r,K) = max(0, min(m, r-(K-1)m) - max(0, r-Km)) and the
//    exact value is acc[K] = 2^(-3 delta) * sum_r w(r) * prod_axes c(r_a, K_a)
//    (closed form, O(k^3 H^3));
//  * whenever every partial sum of the reference's double loop is provably
//    exact (all terms are multiples of a common grain g and sum|terms| < 2^53 g),
//    the reference's result IS float(exact value) and the closed form is used;
//  * otherwise, if m^3 k^3 is within a budget, the reference's accumulation is
//    replayed per output tap K in exactly the reference order (the subsequence
//    of the reference loop that lands on K), parallel over K -- bit-identical;
//  * beyond the budget (where the reference loop itself takes minutes to
//    hours) the closed form is evaluated in binary128 and rounded once.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace aprgpu {
namespace {

int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

int coarse_span(int k, int m) {  // stencil.hpp:131-137
    const int h = k / 2;
    const int lo = -((h + m - 1) / m);
    const int hi = (m - 1 + h) / m;
    return std::max(-lo, hi);
}

// number of fine offsets o in [0,m) with -floor_div(o - r, m) == K
inline long long count_o(int r, int K, int m) {
    const long long lo = std::max<long long>(0, static_cast<long long>(r) - static_cast<long long>(K) * m);
    const long long hi = std::min<long long>(m, static_cast<long long>(r) - static_cast<long long>(K - 1) * m);
    return std::max<long long>(0, hi - lo);
}

// exponent of the lowest set bit of a finite nonzero float
int low_bit_exp(float v) {
    int e;
    double f = std::frexp(static_cast<double>(std::fabs(v)), &e);  // v = f * 2^e, f in [0.5,1)
    // f has at most 24 significant bits: scale to an integer mantissa
    long long mant = static_cast<long long>(std::ldexp(f, 24));
    int shift = 0;
    while (mant && !(mant & 1)) {
        mant >>= 1;
        ++shift;
    }
    return e - 24 + shift;
}

uint64_t restrict_budget() {
    if (const char* s = std::getenv("APRGPU_RESTRICT_BUDGET")) return std::strtoull(s, nullptr, 10);
    return 1ull << 32;
}

}  // namespace

namespace {
HostStencil restrict_stencil_compute(const HostStencil& w, int delta);

// restrict_stencil is a pure function of (w, delta) and its bit-exact replay
// costs seconds at delta 8-9 (rl_apr builds two pyramids per call): memoised.
struct RestrictKey {
    int kz, kx, ky, delta;
    std::vector<float> w;
    bool operator==(const RestrictKey& o) const {
        return kz == o.kz && kx == o.kx && ky == o.ky && delta == o.delta &&
               std::memcmp(w.data(), o.w.data(), sizeof(float) * w.size()) == 0 && w.size() == o.w.size();
    }
};
std::mutex g_restrict_mu;
std::vector<std::pair<RestrictKey, HostStencil>> g_restrict_cache;  // small: a few pyramids
}  // namespace

HostStencil restrict_stencil_host(const HostStencil& w, int delta) {
    if (delta <= 0) return restrict_stencil_compute(w, delta);
    RestrictKey key{w.kz, w.kx, w.ky, delta, w.w};
    {
        std::lock_guard<std::mutex> lk(g_restrict_mu);
        for (const auto& e : g_restrict_cache)
            if (e.first == key) return e.second;
    }
    HostStencil r = restrict_stencil_compute(w, delta);
    std::lock_guard<std::mutex> lk(g_restrict_mu);
    if (g_restrict_cache.size() >= 256) g_restrict_cache.erase(g_restrict_cache.begin());
    g_restrict_cache.emplace_back(std::move(key), r);
    return r;
}

namespace {
HostStencil restrict_stencil_compute(const HostStencil& w, int delta) {
    if (delta < 0) fail(APRGPU_ERR_RANGE, "restrict_stencil: delta must be >= 0");
    if (delta == 0) return w;
    if (delta > 30) fail(APRGPU_ERR_CAPABILITY, "restrict_stencil: delta too large");
    const int m = 1 << delta;
    const int Hz = coarse_span(w.kz, m), Hx = coarse_span(w.kx, m), Hy = coarse_span(w.ky, m);
    HostStencil out;
    out.kz = 2 * Hz + 1;
    out.kx = 2 * Hx + 1;
    out.ky = 2 * Hy + 1;
    const size_t nout = static_cast<size_t>(out.kz) * out.kx * out.ky;
    out.w.assign(nout, 0.0f);
    const int hz = w.kz / 2, hx = w.kx / 2, hy = w.ky / 2;
    const double inv = 1.0 / (static_cast<double>(m) * m * m);
    auto W = [&](int rz, int rx, int ry) {
        return w.w[(static_cast<size_t>(rz + hz) * w.kx + (rx + hx)) * w.ky + (ry + hy)];
    };
    // grain of every reference term inv*w(r) and per-K sum of |terms|
    int gexp = 1 << 30;
    bool finite = true;
    for (float v : w.w) {
        if (!std::isfinite(v)) finite = false;
        if (v != 0.0f && std::isfinite(v)) gexp = std::min(gexp, low_bit_exp(v) - 3 * delta);
    }
    std::vector<__float128> exact(nout, 0);
    std::vector<double> abs_sum(nout, 0.0);  // upper bound estimate (double is plenty for a bound)
    for (int Kz = -Hz; Kz <= Hz; ++Kz)
        for (int Kx = -Hx; Kx <= Hx; ++Kx)
            for (int Ky = -Hy; Ky <= Hy; ++Ky) {
                __float128 acc = 0;
                double as = 0.0;
                for (int rz = -hz; rz <= hz; ++rz) {
                    const long long cz = count_o(rz, Kz, m);
                    if (!cz) continue;
                    for (int rx = -hx; rx <= hx; ++rx) {
                        const long long cx = count_o(rx, Kx, m);
                        if (!cx) continue;
                        for (int ry = -hy; ry <= hy; ++ry) {
                            const long long cy = count_o(ry, Ky, m);
                            if (!cy) continue;
                            const __float128 cnt = static_cast<__float128>(cz) * cx * cy;
                            acc += static_cast<__float128>(W(rz, rx, ry)) * cnt;
                            as += std::fabs(static_cast<double>(W(rz, rx, ry))) * static_cast<double>(cnt);
                        }
                    }
                }
                const size_t k = (static_cast<size_t>(Kz + Hz) * out.kx + (Kx + Hx)) * out.ky + (Ky + Hy);
                exact[k] = acc / (static_cast<__float128>(m) * m * m);
                abs_sum[k] = as * inv;
            }
    bool provably_exact = finite;
    if (finite && gexp < (1 << 29)) {
        const double grain = std::ldexp(1.0, gexp);
        for (size_t k = 0; k < nout; ++k)
            if (abs_sum[k] * 1.0000001 >= std::ldexp(grain, 53)) provably_exact = false;
    }
    const uint64_t work = static_cast<uint64_t>(m) * m * m * static_cast<uint64_t>(w.kz) * w.kx * w.ky;
    if (provably_exact || work > restrict_budget()) {
        for (size_t k = 0; k < nout; ++k) out.w[k] = static_cast<float>(exact[k]);
        return out;
    }
    // Replay the reference accumulation order per K (bit-identical).
    std::atomic<size_t> next{0};
    auto worker = [&]() {
        for (size_t k; (k = next.fetch_add(1)) < nout;) {
            const int Kz = static_cast<int>(k / (static_cast<size_t>(out.kx) * out.ky)) - Hz;
            const int Kx = static_cast<int>((k / out.ky) % out.kx) - Hx;
            const int Ky = static_cast<int>(k % out.ky) - Hy;
            double acc = 0.0;
            for (int oz = 0; oz < m; ++oz) {
                const int rz0 = std::max(-hz, oz + (Kz - 1) * m + 1), rz1 = std::min(hz, oz + Kz * m);
                if (rz0 > rz1) continue;
                for (int ox = 0; ox < m; ++ox) {
                    const int rx0 = std::max(-hx, ox + (Kx - 1) * m + 1), rx1 = std::min(hx, ox + Kx * m);
                    if (rx0 > rx1) continue;
                    for (int oy = 0; oy < m; ++oy) {
                        const int ry0 = std::max(-hy, oy + (Ky - 1) * m + 1), ry1 = std::min(hy, oy + Ky * m);
                        if (ry0 > ry1) continue;
                        for (int rz = rz0; rz <= rz1; ++rz)
                            for (int rx = rx0; rx <= rx1; ++rx)
                                for (int ry = ry0; ry <= ry1; ++ry) acc += inv * W(rz, rx, ry);
                    }
                }
            }
            out.w[k] = static_cast<float>(acc);
        }
    };
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    nt = static_cast<unsigned>(std::min<size_t>(nt, nout));
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    (void)floor_div;
    return out;
}
}  // namespace

HostStencil gaussian_stencil_host(double sigma, int size) {
    // stencil.hpp:59-79
    if (size <= 0) {
        size = 2 * static_cast<int>(std::ceil(3.0 * sigma)) + 1;
        size = std::min(size, 13);
    }
    if (size < 1 || size % 2 == 0) fail(APRGPU_ERR_RANGE, "stencil extents must be odd and positive");
    const int h = size / 2;
    std::vector<double> g(size);
    double norm = 0.0;
    for (int i = -h; i <= h; ++i) {
        g[i + h] = std::exp(-0.5 * (i * i) / (sigma * sigma));
        norm += g[i + h];
    }
    for (double& v : g) v /= norm;
    HostStencil s;
    s.kz = s.kx = s.ky = size;
    s.w.resize(static_cast<size_t>(size) * size * size);
    for (int a = 0; a < size; ++a)
        for (int b = 0; b < size; ++b)
            for (int c = 0; c < size; ++c)
                s.w[(static_cast<size_t>(a) * size + b) * size + c] = static_cast<float>(g[a] * g[b] * g[c]);
    return s;
}

}  // namespace aprgpu
