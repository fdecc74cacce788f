// Drop-in for aprkit/tree.hpp (reference: proj/include/aprkit/tree.hpp).
//
// Found ahead of the reference header (see convolve.hpp here); keeps
// cell_footprint_volume and synchronized_parent_pass from the reference and
// replaces:
//   init_tree_structure  tree.hpp:26-82    -> built on the device (upload with no tree)
//   fill_tree            tree.hpp:110-150  -> aprgpu_fill_tree (fp64 in the reference's
//                                             per-parent order: bit-identical)
#pragma once

#define init_tree_structure init_tree_structure_reference_cpu_
#define fill_tree fill_tree_reference_cpu_
#include_next "aprkit/tree.hpp"
#undef init_tree_structure
#undef fill_tree

#include "aprkit_gpu.hpp"

namespace aprkit {

// Interior-node structure (tree.hpp:26-82), built on the device; bit-identical.
inline LinearAccess init_tree_structure(const LinearAccess& apr_access, const std::array<int, 3>& source_dims) {
    const auto href_ = gpu::Runtime::get().upload(apr_access, source_dims);
    aprgpu_apr* h = href_.get();
    return gpu::download(h, APRGPU_TREE);
}

// Footprint-weighted interior-node values (tree.hpp:110-150).  threads is
// accepted for API parity; the output never depends on it.
inline ParticleValues fill_tree(const APR& apr, const ParticleValues& leaf_values, int threads = 0) {
    (void)threads;
    if (leaf_values.size() != apr.access.particle_count())
        throw RangeError("fill_tree: leaf value count does not match the APR");
    const auto href_ = gpu::Runtime::get().upload(apr);
    aprgpu_apr* h = href_.get();
    ParticleValues out = gpu::result_vector(gpu::count(h, APRGPU_TREE));
    if (out.empty() || leaf_values.empty()) return out;
    gpu::check(aprgpu_fill_tree(h, leaf_values.data(), out.data(), APRGPU_HOST, nullptr));
    return out;
}

}  // namespace aprkit
