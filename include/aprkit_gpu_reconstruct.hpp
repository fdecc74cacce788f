// Device implementations of the reconstruct.hpp drop-in
// (include/aprkit_gpu/aprkit/reconstruct.hpp); included once the runtime in
// aprkit_gpu.hpp is complete.
#pragma once

#include "aprkit/pixel_volume.hpp"

namespace aprkit {

// Piecewise-constant reconstruction on the level-l grid (reconstruct.hpp:73-84).
inline PixelVolume reconstruct_level(const APR& apr, const ParticleValues& values, const ParticleValues& tree_values,
                                     int l) {
    if (l < apr.access.l_min || l > apr.access.l_max) throw RangeError("reconstruct_level: level out of range");
    if (values.size() != apr.access.particle_count())
        throw RangeError("reconstruct_level: value count does not match the APR");
    const auto href_ = gpu::Runtime::get().upload(apr);
    aprgpu_apr* h = href_.get();
    const bool tree = !tree_values.empty();
    if (tree && tree_values.size() != gpu::count(h, APRGPU_TREE))
        throw RangeError("reconstruct_level: tree value count does not match the APR");
    PixelVolume out(apr.access.z_dim[l], apr.access.x_dim[l], apr.access.y_dim[l]);
    if (out.size())
        gpu::check(aprgpu_reconstruct_level(h, values.data(), tree ? tree_values.data() : nullptr, l,
                                            out.values.data(), APRGPU_HOST, nullptr));
    return out;
}

// Every pixel takes the value of its covering leaf (reconstruct.hpp:87-90).
inline PixelVolume reconstruct_full(const APR& apr, const ParticleValues& values) {
    static const ParticleValues no_tree;
    return reconstruct_level(apr, values, no_tree, apr.access.l_max);
}

// Dense window of reconstruct_level(l) plus padding (reconstruct.hpp:94-129).
inline PixelVolume reconstruct_patch(const APR& apr, const ParticleValues& values, const ParticleValues& tree_values,
                                     const PatchSpec& spec) {
    const LinearAccess& a = apr.access;
    const int l = spec.level;
    if (l < a.l_min || l > a.l_max) throw RangeError("reconstruct_patch: level out of range");
    if (spec.z_begin < 0 || spec.z_end > a.z_dim[l] || spec.x_begin < 0 || spec.x_end > a.x_dim[l] ||
        spec.z_begin > spec.z_end || spec.x_begin > spec.x_end || spec.pad < 0)
        throw RangeError("reconstruct_patch: spec outside the level grid");
    if (values.size() != a.particle_count()) throw RangeError("reconstruct_patch: value count does not match the APR");
    const auto href_ = gpu::Runtime::get().upload(apr);
    aprgpu_apr* h = href_.get();
    const bool tree = !tree_values.empty();
    if (tree && tree_values.size() != gpu::count(h, APRGPU_TREE))
        throw RangeError("reconstruct_patch: tree value count does not match the APR");
    PixelVolume out(spec.z_end - spec.z_begin + 2 * spec.pad, spec.x_end - spec.x_begin + 2 * spec.pad,
                    a.y_dim[l] + 2 * spec.pad, 0.0f);
    const aprgpu_patch_spec s{l, spec.z_begin, spec.z_end, spec.x_begin, spec.x_end, spec.pad,
                              spec.pad_mode == PadMode::Zero ? APRGPU_PAD_ZERO : APRGPU_PAD_REFLECT};
    if (out.size())
        gpu::check(aprgpu_reconstruct_patch(h, values.data(), tree ? tree_values.data() : nullptr, &s,
                                            out.values.data(), APRGPU_HOST, nullptr));
    return out;
}

}  // namespace aprkit
