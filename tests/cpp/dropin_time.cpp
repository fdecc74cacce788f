// TEST INFRASTRUCTURE (not product code): times the C++ drop-in's
// convolve_apr -- the reference's own signature, pageable std::vector in and
// out -- on BASELINE config C3 (1024^3 spheres, 48 spheres, radii 24-80, blur
// 2, E = 0.1, the bench's recipe), 3^3 restricted Gaussian pyramid, EXACT
// (or $APRGPU_ACCUM=fast).  Built against the drop-in headers like the
// reference's own tests (tests/cpp/Makefile).  Prints one JSON line: the
// median and best wall time of N calls after 3 warm-up calls.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "aprkit/aprkit.hpp"

using namespace aprkit;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 1024;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 20;
    SphereSceneParams sc;
    sc.count = 48;
    sc.min_radius = 24.0;
    sc.max_radius = 80.0;
    sc.blur_sigma = 2.0;
    const PixelVolume v = generate_spheres(n, n, n, sc, 42);
    BuildParams bp;
    bp.rel_error = 0.1;
    bp.sigma = SigmaPolicy::constant(intensity_range(v));
    auto built = build_apr(v, bp);  // (drop-in: on the device)
    const APR& apr = built.first;
    const ParticleValues& leaf = built.second;
    const ParticleValues tree = fill_tree(apr, leaf);
    const StencilPyramid pyr =
        make_pyramid(gaussian_stencil(1.0, 3), apr.access.l_min, apr.access.l_max, PyramidMode::Restricted);
    ParticleValues out;
    for (int i = 0; i < 3; ++i) out = convolve_apr(apr, leaf, tree, pyr, PadMode::Reflect);
    std::vector<double> ms(reps);
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        out = convolve_apr(apr, leaf, tree, pyr, PadMode::Reflect);
        const auto t1 = std::chrono::steady_clock::now();
        ms[i] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    }
    std::sort(ms.begin(), ms.end());
    // the part of a call that is the API's own: a fresh result vector (std::vector<float>(n): page faults + zero fill)
    std::vector<double> am(reps);
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        ParticleValues tmp(leaf.size(), 0.0f);
        const auto t1 = std::chrono::steady_clock::now();
        am[i] = std::chrono::duration<double, std::milli>(t1 - t0).count() + tmp[i] * 0.0;
    }
    std::sort(am.begin(), am.end());
    std::vector<double> pm(reps);  // the drop-in's own result vectors (gpu::result_vector)
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        ParticleValues tmp = gpu::result_vector(leaf.size());
        const auto t1 = std::chrono::steady_clock::now();
        pm[i] = std::chrono::duration<double, std::milli>(t1 - t0).count() + tmp[i] * 0.0;
    }
    std::sort(pm.begin(), pm.end());
    double sum = 0.0;
    for (float x : out) sum += x;
    std::printf("{\"dropin_convolve_apr_ms_median\": %.4f, \"best_ms\": %.4f, \"plain_result_vector_ms_median\": %.4f, \"dropin_result_vector_ms_median\": %.4f, "
                "\"particles\": %zu, \"tree_nodes\": %zu, \"n\": %d, \"reps\": %d, \"checksum\": %.6e}\n",
                ms[reps / 2], ms[0], am[reps / 2], pm[reps / 2], leaf.size(), tree.size(), n, reps, sum);
    return 0;
}
