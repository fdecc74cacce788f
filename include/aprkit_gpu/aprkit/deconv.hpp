// Drop-in for aprkit/deconv.hpp (reference: proj/include/aprkit/deconv.hpp).
//
// Keeps RLConfig, detail::normalized_psf / rl_epsilon and rl_pixels from the
// reference and replaces rl_apr (deconv.hpp:75-107) by the device iteration
// (aprgpu_rl / aprgpu_rl_resume): tree refresh, conv(w) with the ratio fused
// into its epilogue, tree refresh, conv(flip w) with the multiply fused, all
// on the GPU.  The observer is served by resuming the device iteration every
// record_metrics_every iterations (bit-identical to an uninterrupted run).
#pragma once

#define rl_apr rl_apr_reference_cpu_
#include_next "aprkit/deconv.hpp"
#undef rl_apr

#include "aprkit_gpu.hpp"

namespace aprkit {

inline ParticleValues rl_apr(const APR& apr, const ParticleValues& observed, const RLConfig& cfg,
                             const std::function<void(int, const ParticleValues&)>& observer = nullptr) {
    detail::normalized_psf(cfg.psf);  // reference argument checks (RangeError)
    if (observed.size() != apr.access.particle_count())
        throw RangeError("rl_apr: observation count does not match the APR");
    gpu::Runtime& rt = gpu::Runtime::get();
    const auto href_ = rt.upload(apr);
    aprgpu_apr* h = href_.get();
    ParticleValues est = gpu::result_vector(observed.size());
    if (est.empty()) return est;
    const Stencil& w = cfg.psf;
    const int every = (observer && cfg.record_metrics_every > 0) ? cfg.record_metrics_every : cfg.iterations;
    int done = 0;
    if (cfg.iterations <= 0) {
        gpu::check(aprgpu_rl(h, observed.data(), w.weights.data(), w.kz, w.kx, w.ky, 0, cfg.epsilon, rt.accum(),
                             est.data(), APRGPU_HOST, nullptr));
        return est;
    }
    while (done < cfg.iterations) {
        const int n = std::min(every, cfg.iterations - done);
        gpu::check(aprgpu_rl_resume(h, observed.data(), done ? est.data() : nullptr, w.weights.data(), w.kz, w.kx,
                                    w.ky, n, cfg.epsilon, rt.accum(), est.data(), APRGPU_HOST, nullptr));
        done += n;
        if (observer && cfg.record_metrics_every > 0 && done % cfg.record_metrics_every == 0) observer(done, est);
    }
    return est;
}

}  // namespace aprkit
