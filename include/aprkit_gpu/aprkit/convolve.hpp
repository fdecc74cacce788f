// Drop-in for aprkit/convolve.hpp (reference: proj/include/aprkit/convolve.hpp).
//
// Put include/aprkit_gpu ahead of the reference's include directory: this file
// is then found for "aprkit/convolve.hpp", pulls the reference header in with
// #include_next (ConvolveOptions, RowSpan, convolve_pixels, detail::LevelSlab
// stay the reference's), and replaces the two hot-path entry points with the
// B200 path through the C-ABI (include/aprgpu.h):
//   convolve_apr        convolve.hpp:220-303  -> aprgpu_convolve
//   nonempty_row_index  convolve.hpp:32-44    -> aprgpu_row_index
//   convolve_pixels     convolve.hpp:48-98    -> aprgpu_convolve_pixels (the pixel baseline)
// Signatures, argument meaning and exceptions are the reference's.
#pragma once

#define convolve_apr convolve_apr_reference_cpu_
#define nonempty_row_index nonempty_row_index_reference_cpu_
#define convolve_pixels convolve_pixels_reference_cpu_
#include_next "aprkit/convolve.hpp"
#undef convolve_apr
#undef nonempty_row_index
#undef convolve_pixels

#include <algorithm>

#include "aprkit_gpu.hpp"

namespace aprkit {

// Dense pixel convolution on the device (convolve.hpp:48-98); EXACT unless
// $APRGPU_ACCUM=fast, like convolve_apr.  threads is accepted for API parity.
inline PixelVolume convolve_pixels(const PixelVolume& v, const Stencil& w, PadMode pad, int threads = 0) {
    (void)threads;
    if (w.kz > kMaxStencilExtent || w.kx > kMaxStencilExtent || w.ky > kMaxStencilExtent)
        throw CapabilityError("convolve_pixels: stencil extent exceeds the supported maximum");
    PixelVolume out(v.nz, v.nx, v.ny);
    if (out.size() == 0) return out;
    gpu::Runtime& rt = gpu::Runtime::get();
    gpu::check(aprgpu_convolve_pixels(rt.ctx(), v.values.data(), v.nz, v.nx, v.ny, w.weights.data(), w.kz, w.kx, w.ky,
                                      pad == PadMode::Zero ? APRGPU_PAD_ZERO : APRGPU_PAD_REFLECT, rt.accum(),
                                      out.values.data(), APRGPU_HOST, nullptr));
    return out;
}

// Exact per-level row occupancy, computed on the device (convolve.hpp:32-44).
inline std::vector<std::vector<RowSpan>> nonempty_row_index(const LinearAccess& a) {
    if (!gpu::well_formed(a)) return {};
    const std::array<int, 3> dims{a.z_dim[a.l_max], a.x_dim[a.l_max], a.y_dim[a.l_max]};
    const auto href_ = gpu::Runtime::get().upload(a, dims);
    aprgpu_apr* h = href_.get();
    std::vector<std::vector<RowSpan>> index(a.level_count());
    for (int l = a.l_min; l <= a.l_max; ++l) {
        std::uint64_t n = 0;
        gpu::check(aprgpu_row_index(h, l, nullptr, nullptr, nullptr, nullptr, 0, &n));
        std::vector<int32_t> z(n), x(n);
        std::vector<std::uint16_t> y0(n), y1(n);
        if (n) gpu::check(aprgpu_row_index(h, l, z.data(), x.data(), y0.data(), y1.data(), n, &n));
        auto& rows = index[l - a.l_min];
        rows.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) rows[i] = RowSpan{z[i], x[i], y0[i], y1[i]};
    }
    return index;
}

// APR-native convolution on the device (convolve.hpp:220-303).  opt.threads
// and opt.use_row_skip are accepted and never change the result (the device
// path is bit-identical to itself across launch configurations).  EXACT
// accumulation is bit-identical to the reference; $APRGPU_ACCUM=fast selects
// fp32 accumulation (tolerance-matched).  An empty tree_values with interior
// nodes present is filled on the device first (the reference reads stale
// buffer contents in that case, reconstruct.hpp:60 / convolve.hpp:139-142).
inline ParticleValues convolve_apr(const APR& apr, const ParticleValues& values, const ParticleValues& tree_values,
                                   const StencilPyramid& pyramid, PadMode pad = PadMode::Reflect,
                                   const ConvolveOptions& opt = {}) {
    (void)opt;
    const LinearAccess& a = apr.access;
    if (pyramid.l_min > a.l_min || pyramid.l_max < a.l_max)
        throw RangeError("convolve_apr: pyramid does not cover the APR levels");
    for (int l = a.l_min; l <= a.l_max; ++l) {
        const Stencil& w = pyramid.at(l);
        if (w.kz > kMaxStencilExtent || w.kx > kMaxStencilExtent || w.ky > kMaxStencilExtent)
            throw CapabilityError("convolve_apr: stencil extent exceeds the supported maximum");
    }
    if (values.size() != a.particle_count()) throw RangeError("convolve_apr: value count does not match the APR");
    gpu::Runtime& rt = gpu::Runtime::get();
    const auto href_ = rt.upload(apr);
    aprgpu_apr* h = href_.get();
    const std::uint64_t nt = gpu::count(h, APRGPU_TREE);
    ParticleValues tree_filled;
    const ParticleValues* tv = &tree_values;
    if (tree_values.size() != nt) {
        if (!tree_values.empty()) throw RangeError("convolve_apr: tree value count does not match the APR");
        tree_filled.resize(nt);
        gpu::check(aprgpu_fill_tree(h, values.data(), tree_filled.data(), APRGPU_HOST, nullptr));
        tv = &tree_filled;
    }
    ParticleValues out = gpu::result_vector(values.size());
    if (out.empty()) return out;
    // $APRGPU_DEVICES: z-slabs over several GPUs (halo = the largest half-width)
    int hw = 1;
    for (int l = a.l_min; l <= a.l_max; ++l) {
        const Stencil& w = pyramid.at(l);
        hw = std::max(hw, std::max(w.kz, std::max(w.kx, w.ky)) / 2);
    }
    if (const auto m = rt.multi(apr, std::max(hw, 2))) {
        std::vector<float> w;
        std::vector<int32_t> k3;
        for (const Stencil& st : pyramid.stencils) {
            w.insert(w.end(), st.weights.begin(), st.weights.end());
            k3.insert(k3.end(), {st.kz, st.kx, st.ky});
        }
        gpu::check(aprgpu_multi_convolve(m.get(), values.data(), tv->empty() ? nullptr : tv->data(), w.data(),
                                         k3.data(), pyramid.l_min, pyramid.l_max,
                                         pad == PadMode::Zero ? APRGPU_PAD_ZERO : APRGPU_PAD_REFLECT, rt.accum(),
                                         out.data()));
        return out;
    }
    gpu::DevicePyramid dp(pyramid);
    gpu::check(aprgpu_convolve(h, values.data(), tv->empty() ? nullptr : tv->data(), dp.get(),
                               pad == PadMode::Zero ? APRGPU_PAD_ZERO : APRGPU_PAD_REFLECT, rt.accum(), out.data(),
                               APRGPU_HOST, nullptr));
    return out;
}

}  // namespace aprkit
