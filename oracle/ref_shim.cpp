// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product).
//
// Compiles the UNMODIFIED reference headers (/root/reference/proj/include/aprkit,
// plus the reference's test helpers /root/reference/proj/tests/helpers.hpp) where
// they lie and exposes them behind a flat extern "C" surface so that the Python
// test-suite and bench.py's CPU-baseline leg can call the real reference code
// through ctypes.  Built by oracle/Makefile into oracle/_ref/libaprref.so.
//
// Nothing here re-implements reference arithmetic: every function forwards to
// the reference symbol named in its comment.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "aprkit/aprkit.hpp"
#include "helpers.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

struct RefApr {
    aprkit::APR apr;
    aprkit::ParticleValues values;  // sampled leaf values when built from pixels
};

struct RefPyr {
    aprkit::StencilPyramid pyr;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const aprkit::RangeError& e) {
        g_err = e.what();
        return 1;
    } catch (const aprkit::CapabilityError& e) {
        g_err = e.what();
        return 2;
    } catch (const aprkit::IntegrityError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

aprkit::Stencil make_stencil(const float* w, int kz, int kx, int ky) {
    aprkit::Stencil s(kz, kx, ky);
    std::memcpy(s.weights.data(), w, sizeof(float) * s.weights.size());
    return s;
}

const aprkit::LinearAccess& pick(const RefApr* h, int which) {
    return which == 0 ? h->apr.access : h->apr.tree_access;
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---- RNG (rng.hpp:18-55) and test helpers (tests/helpers.hpp) ---------------
REF_API void* ref_rng_new(std::uint64_t seed) { return new aprkit::CounterRng(seed); }
REF_API void ref_rng_free(void* r) { delete static_cast<aprkit::CounterRng*>(r); }
REF_API std::uint64_t ref_rng_next_u64(void* r) { return static_cast<aprkit::CounterRng*>(r)->next_u64(); }
REF_API double ref_rng_uniform(void* r, double lo, double hi) {
    return static_cast<aprkit::CounterRng*>(r)->uniform(lo, hi);
}
REF_API std::int64_t ref_rng_uniform_int(void* r, std::int64_t lo, std::int64_t hi) {
    return static_cast<aprkit::CounterRng*>(r)->uniform_int(lo, hi);
}

// testutil::random_apr (helpers.hpp:23-52)
REF_API void* ref_random_apr(void* rng, int min_dim, int max_dim) {
    auto* h = new RefApr;
    h->apr = testutil::random_apr(*static_cast<aprkit::CounterRng*>(rng), min_dim, max_dim);
    return h;
}
// testutil::random_values (helpers.hpp:54-59)
REF_API void ref_random_values(void* rng, std::uint64_t n, double lo, double hi, float* out) {
    auto v = testutil::random_values(*static_cast<aprkit::CounterRng*>(rng), n, lo, hi);
    std::memcpy(out, v.data(), sizeof(float) * n);
}
// testutil::random_stencil (helpers.hpp:147-152)
REF_API void ref_random_stencil(void* rng, int kz, int kx, int ky, double lo, double hi, float* out) {
    auto s = testutil::random_stencil(*static_cast<aprkit::CounterRng*>(rng), kz, kx, ky, lo, hi);
    std::memcpy(out, s.weights.data(), sizeof(float) * s.weights.size());
}

// ---- APR construction -------------------------------------------------------
// solve_levels (build.hpp:136-248) + init_tree_structure (tree.hpp:26-82)
REF_API void* ref_apr_from_targets(const int* targets, int nz, int nx, int ny, int l_min, int l_max) {
    RefApr* out = nullptr;
    int st = guarded([&] {
        std::vector<int> t(targets, targets + static_cast<std::size_t>(nz) * nx * ny);
        auto h = std::make_unique<RefApr>();
        h->apr.source_dims = {nz, nx, ny};
        h->apr.access = aprkit::solve_levels(t, h->apr.source_dims, l_min, l_max);
        h->apr.tree_access = aprkit::init_tree_structure(h->apr.access, h->apr.source_dims);
        out = h.release();
    });
    return st == 0 ? out : nullptr;
}

// assemble an APR from raw leaf arrays; tree via init_tree_structure (tree.hpp:26)
REF_API void* ref_apr_from_arrays(int l_min, int l_max, const int* zd, const int* xd, const int* yd,
                                  const std::uint16_t* y_idx, std::uint64_t n_particles,
                                  const std::uint64_t* xz_end, std::uint64_t n_rows,
                                  const std::uint64_t* level_offset, int nz, int nx, int ny) {
    RefApr* out = nullptr;
    int st = guarded([&] {
        auto h = std::make_unique<RefApr>();
        aprkit::LinearAccess& a = h->apr.access;
        a.l_min = l_min;
        a.l_max = l_max;
        a.z_dim.assign(zd, zd + l_max + 1);
        a.x_dim.assign(xd, xd + l_max + 1);
        a.y_dim.assign(yd, yd + l_max + 1);
        a.y_idx.assign(y_idx, y_idx + n_particles);
        a.xz_end.assign(xz_end, xz_end + n_rows);
        a.level_offset.assign(level_offset, level_offset + l_max + 1);
        h->apr.source_dims = {nz, nx, ny};
        h->apr.tree_access = aprkit::init_tree_structure(a, h->apr.source_dims);
        out = h.release();
    });
    return st == 0 ? out : nullptr;
}

// generate_spheres (synthetic.hpp:74-111) -> build_apr (build.hpp:290-312) with
// SigmaPolicy::constant(intensity_range(v)), as SURVEY Appendix A / BASELINE.md
REF_API void* ref_build_spheres(int nz, int nx, int ny, int count, double rmin, double rmax,
                                double blur, double noise, std::uint64_t seed, double rel_error,
                                int threads) {
    RefApr* out = nullptr;
    int st = guarded([&] {
        aprkit::SphereSceneParams p;
        p.count = count;
        p.min_radius = rmin;
        p.max_radius = rmax;
        p.blur_sigma = blur;
        p.noise_sigma = noise;
        const aprkit::PixelVolume v = aprkit::generate_spheres(nz, nx, ny, p, seed);
        aprkit::BuildParams bp;
        bp.rel_error = rel_error;
        bp.sigma = aprkit::SigmaPolicy::constant(aprkit::intensity_range(v));
        auto built = aprkit::build_apr(v, bp, threads);
        auto h = std::make_unique<RefApr>();
        h->apr = std::move(built.first);
        h->values = std::move(built.second);
        out = h.release();
    });
    return st == 0 ? out : nullptr;
}

// generate_spheres only (synthetic.hpp:74-111)
REF_API int ref_generate_spheres(int nz, int nx, int ny, int count, double rmin, double rmax,
                                 double blur, double noise, std::uint64_t seed, float* out) {
    return guarded([&] {
        aprkit::SphereSceneParams p;
        p.count = count;
        p.min_radius = rmin;
        p.max_radius = rmax;
        p.blur_sigma = blur;
        p.noise_sigma = noise;
        const aprkit::PixelVolume v = aprkit::generate_spheres(nz, nx, ny, p, seed);
        std::memcpy(out, v.values.data(), sizeof(float) * v.values.size());
    });
}

// build_apr on a given pixel volume with constant sigma = intensity_range (build.hpp:290)
REF_API void* ref_build_apr(const float* vol, int nz, int nx, int ny, double rel_error, int threads) {
    RefApr* out = nullptr;
    int st = guarded([&] {
        aprkit::PixelVolume v(nz, nx, ny);
        std::memcpy(v.values.data(), vol, sizeof(float) * v.values.size());
        aprkit::BuildParams bp;
        bp.rel_error = rel_error;
        bp.sigma = aprkit::SigmaPolicy::constant(aprkit::intensity_range(v));
        auto built = aprkit::build_apr(v, bp, threads);
        auto h = std::make_unique<RefApr>();
        h->apr = std::move(built.first);
        h->values = std::move(built.second);
        out = h.release();
    });
    return st == 0 ? out : nullptr;
}

// build_apr with every BuildParams field (apr.hpp:16-33): sigma_mode 0 constant
// (sigma_value) / 1 local range (sigma_window, sigma_floor); gradient_mode 0
// central difference / 1 Sobel; smoothing_passes box passes on the gradient
REF_API void* ref_build_apr_params(const float* vol, int nz, int nx, int ny, double rel_error, int sigma_mode,
                                   double sigma_value, int sigma_window, double sigma_floor, int gradient_mode,
                                   int smoothing_passes, int threads) {
    RefApr* out = nullptr;
    int st = guarded([&] {
        aprkit::PixelVolume v(nz, nx, ny);
        std::memcpy(v.values.data(), vol, sizeof(float) * v.values.size());
        aprkit::BuildParams bp;
        bp.rel_error = rel_error;
        bp.sigma = sigma_mode == 0 ? aprkit::SigmaPolicy::constant(sigma_value)
                                   : aprkit::SigmaPolicy::local_range(sigma_window, sigma_floor);
        bp.gradient = gradient_mode == 0 ? aprkit::GradientMode::CentralDiff : aprkit::GradientMode::Sobel;
        bp.smoothing_passes = smoothing_passes;
        auto built = aprkit::build_apr(v, bp, threads);
        auto h = std::make_unique<RefApr>();
        h->apr = std::move(built.first);
        h->values = std::move(built.second);
        out = h.release();
    });
    return st == 0 ? out : nullptr;
}

// sample_particles (build.hpp:252-284)
REF_API int ref_sample_particles(void* hp, const float* vol, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        const auto& d = h->apr.source_dims;
        aprkit::PixelVolume v(d[0], d[1], d[2]);
        std::memcpy(v.values.data(), vol, sizeof(float) * v.values.size());
        auto s = aprkit::sample_particles(v, h->apr.access);
        std::memcpy(out, s.data(), sizeof(float) * s.size());
    });
}

REF_API void ref_apr_free(void* h) { delete static_cast<RefApr*>(h); }

// info[0..5] = l_min, l_max, n_particles, n_rows, (source dims via ref_apr_dims)
REF_API void ref_apr_info(void* hp, int which, std::int64_t* info) {
    const auto& a = pick(static_cast<RefApr*>(hp), which);
    info[0] = a.l_min;
    info[1] = a.l_max;
    info[2] = static_cast<std::int64_t>(a.particle_count());
    info[3] = static_cast<std::int64_t>(a.row_count());
}
REF_API void ref_apr_dims(void* hp, int* dims) {
    const auto& d = static_cast<RefApr*>(hp)->apr.source_dims;
    dims[0] = d[0];
    dims[1] = d[1];
    dims[2] = d[2];
}
REF_API void ref_apr_copy(void* hp, int which, std::uint16_t* y_idx, std::uint64_t* xz_end,
                          std::uint64_t* level_offset, int* zd, int* xd, int* yd) {
    const auto& a = pick(static_cast<RefApr*>(hp), which);
    std::memcpy(y_idx, a.y_idx.data(), 2 * a.y_idx.size());
    std::memcpy(xz_end, a.xz_end.data(), 8 * a.xz_end.size());
    std::memcpy(level_offset, a.level_offset.data(), 8 * a.level_offset.size());
    std::memcpy(zd, a.z_dim.data(), 4 * a.z_dim.size());
    std::memcpy(xd, a.x_dim.data(), 4 * a.x_dim.size());
    std::memcpy(yd, a.y_dim.data(), 4 * a.y_dim.size());
}
REF_API std::uint64_t ref_apr_values(void* hp, float* out) {
    auto* h = static_cast<RefApr*>(hp);
    if (out) std::memcpy(out, h->values.data(), 4 * h->values.size());
    return h->values.size();
}
// validate (apr.hpp:61-134); returns 1 if ok
REF_API int ref_validate(void* hp) { return aprkit::validate(static_cast<RefApr*>(hp)->apr).ok ? 1 : 0; }

// convolve_pixels (convolve.hpp:48-98); pad 0 Zero, 1 Reflect
REF_API int ref_convolve_pixels(const float* v, int nz, int nx, int ny, const float* w, int kz, int kx, int ky,
                                int pad, float* out) {
    return guarded([&] {
        aprkit::PixelVolume vol(nz, nx, ny);
        std::memcpy(vol.values.data(), v, 4 * vol.size());
        aprkit::Stencil st(kz, kx, ky);
        std::memcpy(st.weights.data(), w, 4 * st.weights.size());
        auto o = aprkit::convolve_pixels(vol, st, pad == 0 ? aprkit::PadMode::Zero : aprkit::PadMode::Reflect, 1);
        std::memcpy(out, o.values.data(), 4 * o.size());
    });
}

// save_apr (io.hpp:171-176) of a handle with the given leaf values
REF_API int ref_save_apr(void* hp, const float* values, const char* path) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues v(values, values + h->apr.access.particle_count());
        aprkit::save_apr(path, h->apr, v);
    });
}

// load_apr (io.hpp:178-183): 0 and the handle, or the exception's kind
// (1 IoError, 2 BadFormatError, 3 TruncatedFileError) and message
REF_API int ref_load_apr(const char* path, void** out, char* msg, std::uint64_t cap) {
    auto put = [&](const std::string& m) {
        if (msg && cap) {
            const std::size_t n = std::min<std::size_t>(cap - 1, m.size());
            std::memcpy(msg, m.data(), n);
            msg[n] = 0;
        }
    };
    try {
        auto h = std::make_unique<RefApr>();
        h->apr = aprkit::load_apr(path, h->values);
        *out = h.release();
        put("");
        return 0;
    } catch (const aprkit::TruncatedFileError& e) {
        put(e.what());
        return 3;
    } catch (const aprkit::BadFormatError& e) {
        put(e.what());
        return 2;
    } catch (const aprkit::IoError& e) {
        put(e.what());
        return 1;
    }
}

// validate (apr.hpp:61-134) of raw leaf arrays (no tree is built: malformed
// structures are the point); returns ok, the report's message into msg
REF_API int ref_validate_arrays(int l_min, int l_max, const int* zd, const int* xd, const int* yd,
                                const std::uint16_t* y_idx, std::uint64_t n_particles, const std::uint64_t* xz_end,
                                std::uint64_t n_rows, const std::uint64_t* level_offset, int nz, int nx, int ny,
                                char* msg, std::uint64_t cap) {
    aprkit::LinearAccess a;
    a.l_min = l_min;
    a.l_max = l_max;
    a.z_dim.assign(zd, zd + l_max + 1);
    a.x_dim.assign(xd, xd + l_max + 1);
    a.y_dim.assign(yd, yd + l_max + 1);
    a.y_idx.assign(y_idx, y_idx + n_particles);
    a.xz_end.assign(xz_end, xz_end + n_rows);
    a.level_offset.assign(level_offset, level_offset + l_max + 1);
    const auto rep = aprkit::validate(a, std::array<int, 3>{nz, nx, ny});
    if (msg && cap) {
        const std::size_t n = std::min<std::size_t>(cap - 1, rep.message.size());
        std::memcpy(msg, rep.message.data(), n);
        msg[n] = 0;
    }
    return rep.ok ? 1 : 0;
}

// ---- hot path ----------------------------------------------------------------
// fill_tree (tree.hpp:110-150)
REF_API int ref_fill_tree(void* hp, const float* leaf, int threads, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues v(leaf, leaf + h->apr.access.particle_count());
        auto t = aprkit::fill_tree(h->apr, v, threads);
        std::memcpy(out, t.data(), 4 * t.size());
    });
}

// nonempty_row_index (convolve.hpp:32-44); level-local list; returns count
REF_API std::int64_t ref_nonempty_row_index(void* hp, int level, int* z, int* x, std::uint16_t* ymin,
                                            std::uint16_t* ymax) {
    std::int64_t n = -1;
    guarded([&] {
        const auto& a = static_cast<RefApr*>(hp)->apr.access;
        auto idx = aprkit::nonempty_row_index(a);
        const auto& rows = idx.at(level - a.l_min);
        n = static_cast<std::int64_t>(rows.size());
        if (z)
            for (std::size_t i = 0; i < rows.size(); ++i) {
                z[i] = rows[i].z;
                x[i] = rows[i].x;
                ymin[i] = rows[i].y_min;
                ymax[i] = rows[i].y_max;
            }
    });
    return n;
}

// make_pyramid (stencil.hpp:176-191); mode: 0 Restricted, 1 Rescaled, 2 Uniform
REF_API void* ref_make_pyramid(const float* w, int kz, int kx, int ky, int l_min, int l_max, int mode) {
    RefPyr* out = nullptr;
    int st = guarded([&] {
        auto p = std::make_unique<RefPyr>();
        p->pyr = aprkit::make_pyramid(make_stencil(w, kz, kx, ky), l_min, l_max,
                                      static_cast<aprkit::PyramidMode>(mode));
        out = p.release();
    });
    return st == 0 ? out : nullptr;
}
// explicit_pyramid (stencil.hpp:193-202): weights concatenated level by level
REF_API void* ref_explicit_pyramid(const float* w, const int* k3, int l_min, int l_max) {
    RefPyr* out = nullptr;
    int st = guarded([&] {
        std::vector<aprkit::Stencil> st;
        std::size_t off = 0;
        for (int l = l_min; l <= l_max; ++l) {
            const int* k = k3 + 3 * (l - l_min);
            st.push_back(make_stencil(w + off, k[0], k[1], k[2]));
            off += static_cast<std::size_t>(k[0]) * k[1] * k[2];
        }
        auto p = std::make_unique<RefPyr>();
        p->pyr = aprkit::explicit_pyramid(std::move(st), l_min, l_max);
        out = p.release();
    });
    return st == 0 ? out : nullptr;
}
REF_API void ref_pyramid_free(void* p) { delete static_cast<RefPyr*>(p); }
REF_API int ref_pyramid_level(void* pp, int l, int* k3, float* w) {
    return guarded([&] {
        const auto& s = static_cast<RefPyr*>(pp)->pyr.at(l);
        k3[0] = s.kz;
        k3[1] = s.kx;
        k3[2] = s.ky;
        if (w) std::memcpy(w, s.weights.data(), 4 * s.weights.size());
    });
}

// restrict_stencil (stencil.hpp:127-160); out must hold the restricted extent
REF_API int ref_restrict_stencil(const float* w, int kz, int kx, int ky, int delta, int* k3, float* out) {
    return guarded([&] {
        auto r = aprkit::restrict_stencil(make_stencil(w, kz, kx, ky), delta);
        k3[0] = r.kz;
        k3[1] = r.kx;
        k3[2] = r.ky;
        if (out) std::memcpy(out, r.weights.data(), 4 * r.weights.size());
    });
}

// gaussian_stencil (stencil.hpp:59-79), box_stencil (:52); out sized k^3
REF_API int ref_gaussian_stencil(double sigma, int size, int* k, float* out) {
    return guarded([&] {
        auto s = aprkit::gaussian_stencil(sigma, size);
        *k = s.kz;
        if (out) std::memcpy(out, s.weights.data(), 4 * s.weights.size());
    });
}
REF_API int ref_box_stencil(int k, float* out) {
    return guarded([&] {
        auto s = aprkit::box_stencil(k);
        std::memcpy(out, s.weights.data(), 4 * s.weights.size());
    });
}

// convolve_apr (convolve.hpp:220-303)
REF_API int ref_convolve(void* hp, const float* values, const float* tree, void* pp, int pad,
                         int threads, int row_skip, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues v(values, values + h->apr.access.particle_count());
        aprkit::ParticleValues t(tree, tree + h->apr.tree_access.particle_count());
        aprkit::ConvolveOptions opt;
        opt.threads = threads;
        opt.use_row_skip = row_skip != 0;
        auto o = aprkit::convolve_apr(h->apr, v, t, static_cast<RefPyr*>(pp)->pyr,
                                      static_cast<aprkit::PadMode>(pad), opt);
        std::memcpy(out, o.data(), 4 * o.size());
    });
}

// reconstruct_level (reconstruct.hpp:73-84); out sized z_dim*x_dim*y_dim at l
REF_API int ref_reconstruct_level(void* hp, const float* values, const float* tree, int l, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues v(values, values + h->apr.access.particle_count());
        aprkit::ParticleValues t;  // tree NULL: no interior nodes (as reconstruct_full)
        if (tree) t.assign(tree, tree + h->apr.tree_access.particle_count());
        auto img = aprkit::reconstruct_level(h->apr, v, t, l);
        std::memcpy(out, img.values.data(), 4 * img.values.size());
    });
}

// reconstruct_full (reconstruct.hpp:87-90)
REF_API int ref_reconstruct_full(void* hp, const float* values, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues v(values, values + h->apr.access.particle_count());
        auto img = aprkit::reconstruct_full(h->apr, v);
        std::memcpy(out, img.values.data(), 4 * img.values.size());
    });
}

// reconstruct_patch (reconstruct.hpp:94-129); spec = level, z_begin, z_end,
// x_begin, x_end, pad, pad_mode (0 Zero, 1 Reflect)
REF_API int ref_reconstruct_patch(void* hp, const float* values, const float* tree, const int* spec, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues v(values, values + h->apr.access.particle_count());
        aprkit::ParticleValues t;
        if (tree) t.assign(tree, tree + h->apr.tree_access.particle_count());
        aprkit::PatchSpec sp;
        sp.level = spec[0];
        sp.z_begin = spec[1];
        sp.z_end = spec[2];
        sp.x_begin = spec[3];
        sp.x_end = spec[4];
        sp.pad = spec[5];
        sp.pad_mode = spec[6] == 0 ? aprkit::PadMode::Zero : aprkit::PadMode::Reflect;
        auto img = aprkit::reconstruct_patch(h->apr, v, t, sp);
        std::memcpy(out, img.values.data(), 4 * img.values.size());
    });
}

// rl_apr (deconv.hpp:75-107)
REF_API int ref_rl_apr(void* hp, const float* observed, const float* psf, int kz, int kx, int ky,
                       int iterations, double epsilon, int threads, float* out) {
    return guarded([&] {
        auto* h = static_cast<RefApr*>(hp);
        aprkit::ParticleValues u(observed, observed + h->apr.access.particle_count());
        aprkit::RLConfig cfg;
        cfg.iterations = iterations;
        cfg.psf = make_stencil(psf, kz, kx, ky);
        cfg.epsilon = epsilon;
        cfg.threads = threads;
        auto o = aprkit::rl_apr(h->apr, u, cfg);
        std::memcpy(out, o.data(), 4 * o.size());
    });
}

// resolve_threads (parallel.hpp:19-21): what threads=0 means on this host
REF_API int ref_resolve_threads(int requested) { return aprkit::resolve_threads(requested); }
