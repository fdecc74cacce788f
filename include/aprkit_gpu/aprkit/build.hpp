// Drop-in for aprkit/build.hpp (reference: proj/include/aprkit/build.hpp).
//
// Found ahead of the reference header (see convolve.hpp here); keeps the
// stage functions (gradient_magnitude, local_scale, level_function,
// solve_levels, sample_particles) from the reference and replaces the
// pipeline on the input side of the hot path:
//   build_apr  build.hpp:290-312  -> aprgpu_build_apr_params: every stage on the
//              device (central differences or Sobel, smoothing passes, constant
//              or local-range sigma, the level solve, init_tree_structure,
//              sample_particles), structure and values bit-identical; the
//              APR comes back in the reference's host layout.
#pragma once

#define build_apr build_apr_reference_cpu_
#include_next "aprkit/build.hpp"
#undef build_apr

#include "aprkit_gpu.hpp"

namespace aprkit {

// threads is accepted for API parity; the result never depends on it.
inline std::pair<APR, ParticleValues> build_apr(const PixelVolume& v, const BuildParams& params, int threads = 0) {
    (void)threads;
    if (v.nz < 1 || v.nx < 1 || v.ny < 1) throw RangeError("build_apr: empty volume");
    if (v.ny > kMaxYDim) throw CapabilityError("y dimension exceeds the 16-bit index limit");
    aprgpu_build_params p{};
    p.rel_error = params.rel_error;
    p.sigma_mode = params.sigma.mode == SigmaMode::Constant ? 0 : 1;
    p.sigma_value = params.sigma.value;
    p.sigma_window = params.sigma.window_radius;
    p.sigma_floor = params.sigma.floor;
    p.gradient_mode = params.gradient == GradientMode::CentralDiff ? 0 : 1;
    p.smoothing_passes = params.smoothing_passes;
    aprgpu_apr* h = nullptr;
    gpu::check(aprgpu_build_apr_params(gpu::Runtime::get().ctx(), v.values.data(), v.nz, v.nx, v.ny, &p, APRGPU_HOST,
                                       &h));
    const std::unique_ptr<aprgpu_apr, int (*)(aprgpu_apr*)> own(h, aprgpu_apr_free);
    APR apr;
    apr.source_dims = {v.nz, v.nx, v.ny};
    apr.params = params;
    apr.access = gpu::download(h, APRGPU_LEAF);
    apr.tree_access = gpu::download(h, APRGPU_TREE);
    ParticleValues values(apr.access.particle_count());
    if (!values.empty()) gpu::check(aprgpu_apr_values(h, values.data(), APRGPU_HOST));
    return {std::move(apr), std::move(values)};
}

}  // namespace aprkit
