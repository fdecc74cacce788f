// include/aprkit_gpu.hpp -- C++ host runtime of the B200 drop-in for aprkit's
// hot path (APR-native convolution, arXiv 2112.03592).
//
// This header is the host side above the C-ABI (include/aprgpu.h): it keeps
// the reference's C++ types (aprkit::APR, LinearAccess, ParticleValues,
// StencilPyramid, PadMode, ConvolveOptions, RLConfig) and turns them into
// C-ABI calls, mapping status codes back onto aprkit's exception taxonomy
// (errors.hpp:9-41).  The drop-in headers under include/aprkit_gpu/aprkit/
// use it to replace convolve_apr / nonempty_row_index (convolve.hpp),
// fill_tree / init_tree_structure (tree.hpp) and rl_apr (deconv.hpp); a
// program compiled with -Iinclude/aprkit_gpu ahead of the reference's include
// directory gets the GPU path with no source change.
//
// Runtime model: one aprgpu context per process on device $APRGPU_DEVICE
// (default 0).  APRs are uploaded on first use and cached: a call first looks
// the APR up by the addresses and sizes of its arrays plus a sampled content
// check (O(1) per call -- aprkit's structures are immutable once built, SPEC
// §3), and only on a miss by a full content fingerprint, whose hit is then
// verified against the device copy before it is trusted.  Stencil pyramids
// are cached on the device by content.  With $APRGPU_DEVICES = "0,1,..." (more
// than one entry) convolve_apr runs on z-slabs over those devices
// (aprgpu_multi_*, peer-to-peer halos).  Accumulation: EXACT (fp64 in the
// reference's order, bit-identical) unless $APRGPU_ACCUM=fast.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>
#ifdef __linux__
#include <sys/mman.h>
#endif

#include "aprgpu.h"
#include "aprkit/apr.hpp"
#include "aprkit/errors.hpp"
#include "aprkit/linear_access.hpp"
#include "aprkit/reconstruct.hpp"
#include "aprkit/stencil.hpp"

namespace aprkit {
namespace gpu {

// C-ABI status -> the reference's exception types (errors.hpp:9-41).
[[noreturn]] inline void raise_status(int st) {
    const std::string m = aprgpu_last_error();
    switch (st) {
        case APRGPU_ERR_RANGE: throw RangeError(m);
        case APRGPU_ERR_CAPABILITY: throw CapabilityError(m);
        case APRGPU_ERR_INTEGRITY: throw IntegrityError(m);
        case APRGPU_ERR_OOM: throw std::bad_alloc();
        case APRGPU_ERR_IO: throw IoError(m);
        case APRGPU_ERR_BAD_FORMAT: throw BadFormatError(m);
        case APRGPU_ERR_TRUNCATED: throw TruncatedFileError(m);
        default: throw std::runtime_error("aprgpu: " + m);
    }
}

inline void check(int st) {
    if (st != APRGPU_OK) raise_status(st);
}

// A result vector of n zeros.  A large result is a fresh mapping, and its
// first touch -- one page fault per 4 KB, single-threaded in std::vector's
// constructor -- costs more than the whole device call (C3's 68 MB: ~22 ms
// against ~6 ms), so its pages are made huge where the kernel allows and
// faulted in by several threads first; the vector's own zero fill then runs
// at memory speed.  ($APRGPU_RESULT_THREADS, default min(8, cores / 2); 1
// keeps the plain constructor.)
inline ParticleValues result_vector(std::size_t n) {
    static const unsigned T = [] {
        const char* e = std::getenv("APRGPU_RESULT_THREADS");
        const unsigned hc = std::thread::hardware_concurrency();
        return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : std::min(8u, std::max(1u, hc / 2));
    }();
    ParticleValues v;
    if (T < 2 || n < (std::size_t(1) << 22)) {
        v.assign(n, 0.0f);
        return v;
    }
    v.reserve(n);  // (allocated, not yet touched)
    float* p = v.data();
#ifdef __linux__
    const std::uintptr_t b = (reinterpret_cast<std::uintptr_t>(p) + 4095) & ~std::uintptr_t(4095);
    const std::uintptr_t e = reinterpret_cast<std::uintptr_t>(p + n) & ~std::uintptr_t(4095);
    if (e > b) madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
#endif
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([=] {
            const std::size_t lo = n * t / T, hi = n * (t + 1) / T;
            std::memset(static_cast<void*>(p + lo), 0, 4 * (hi - lo));
        });
    for (auto& x : th) x.join();
    v.resize(n);
    return v;
}

inline aprgpu_access_desc describe(const LinearAccess& a) {
    aprgpu_access_desc d{};
    d.l_min = a.l_min;
    d.l_max = a.l_max;
    d.z_dim = a.z_dim.data();
    d.x_dim = a.x_dim.data();
    d.y_dim = a.y_dim.data();
    d.y_idx = a.y_idx.empty() ? nullptr : a.y_idx.data();
    d.n_particles = a.y_idx.size();
    d.xz_end = a.xz_end.empty() ? nullptr : a.xz_end.data();
    d.n_rows = a.xz_end.size();
    d.level_offset = a.level_offset.data();
    return d;
}

// An access structure the device can take: level vectors sized l_max + 1.
inline bool well_formed(const LinearAccess& a) {
    const std::size_t n = static_cast<std::size_t>(a.l_max) + 1;
    return a.l_min >= 0 && a.l_min <= a.l_max && a.z_dim.size() >= n && a.x_dim.size() >= n &&
           a.y_dim.size() >= n && a.level_offset.size() >= n;
}

// 64-bit content fingerprint (FNV-1a over 8-byte words).
class Fingerprint {
public:
    void bytes(const void* p, std::size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        std::size_t i = 0;
        for (; i + 8 <= n; i += 8) {
            std::uint64_t w;
            std::memcpy(&w, c + i, 8);
            mix(w);
        }
        std::uint64_t tail = 0;
        std::memcpy(&tail, c + i, n - i);
        mix(tail ^ (static_cast<std::uint64_t>(n) << 56));
    }
    template <class T>
    void vec(const std::vector<T>& v) {
        mix(v.size());
        if (!v.empty()) bytes(v.data(), v.size() * sizeof(T));
    }
    void access(const LinearAccess& a) {
        mix(static_cast<std::uint64_t>(a.l_min) << 32 | static_cast<std::uint32_t>(a.l_max));
        vec(a.z_dim);
        vec(a.x_dim);
        vec(a.y_dim);
        vec(a.y_idx);
        vec(a.xz_end);
        vec(a.level_offset);
    }
    std::uint64_t value() const { return h_; }

private:
    void mix(std::uint64_t w) {
        h_ ^= w;
        h_ *= 0x100000001b3ull;
        h_ ^= h_ >> 29;
    }
    std::uint64_t h_ = 0xcbf29ce484222325ull;
};

// Process-wide device runtime: context + LRU cache of uploaded APRs.
class Runtime {
public:
    static Runtime& get() {
        static Runtime rt;
        return rt;
    }

    aprgpu_ctx* ctx() { return ctx_; }

    int accum() const { return accum_; }

    // Device handle of an APR (uploaded on first use).  With an empty
    // tree_access the interior structure is built on the device
    // (init_tree_structure semantics).
    // Handles are shared: a call holds its APR for its duration, so an eviction
    // by another thread frees it only after the last holder is done.
    using Ref = std::shared_ptr<aprgpu_apr>;
    Ref upload(const APR& apr) {
        const bool tree = well_formed(apr.tree_access);
        const AddrKey ak = addr_key(apr.access, tree ? &apr.tree_access : nullptr, apr.source_dims);
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (auto it = cache_.begin(); it != cache_.end(); ++it)
                if (it->addr == ak) {
                    cache_.splice(cache_.begin(), cache_, it);
                    return cache_.front().ref;
                }
        }
        Fingerprint f;
        f.access(apr.access);
        if (tree) f.access(apr.tree_access);
        f.bytes(apr.source_dims.data(), sizeof(int) * 3);
        return lookup(f.value(), ak, [&](aprgpu_apr* h) { return same_structure(h, apr.access); },
                      [&](aprgpu_apr** out) {
                          if (!well_formed(apr.access)) throw RangeError("APR access structure has no levels");
                          const aprgpu_access_desc leaf = describe(apr.access);
                          aprgpu_access_desc td{};
                          if (tree) td = describe(apr.tree_access);
                          const int32_t dims[3] = {apr.source_dims[0], apr.source_dims[1], apr.source_dims[2]};
                          return aprgpu_upload_access(ctx_, &leaf, tree ? &td : nullptr, dims, out);
                      });
    }

    // A StencilPyramid on the device, cached by content.
    using PyrRef = std::shared_ptr<aprgpu_pyramid>;
    PyrRef pyramid(const StencilPyramid& p) {
        if (p.stencils.empty()) throw RangeError("StencilPyramid has no levels");
        std::vector<float> w;
        std::vector<int32_t> k3;
        for (const Stencil& st : p.stencils) {
            w.insert(w.end(), st.weights.begin(), st.weights.end());
            k3.insert(k3.end(), {st.kz, st.kx, st.ky});
        }
        Fingerprint f;
        f.vec(w);
        f.vec(k3);
        const std::uint64_t key = f.value() ^ (static_cast<std::uint64_t>(p.l_min) << 40) ^ p.l_max;
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = pyr_cache_.begin(); it != pyr_cache_.end(); ++it)
            if (it->key == key && it->l_min == p.l_min && it->w == w && it->k3 == k3) {
                pyr_cache_.splice(pyr_cache_.begin(), pyr_cache_, it);
                return pyr_cache_.front().ref;
            }
        aprgpu_pyramid* h = nullptr;
        check(aprgpu_pyramid_create_explicit(ctx_, w.data(), k3.data(), p.l_min, p.l_max, &h));
        pyr_cache_.push_front(PyrEntry{key, p.l_min, w, k3, PyrRef(h, [](aprgpu_pyramid* q) { aprgpu_pyramid_free(q); })});
        while (pyr_cache_.size() > kCacheSize * 2) pyr_cache_.pop_back();
        return pyr_cache_.front().ref;
    }

    // $APRGPU_DEVICES with more than one device: the APR's z-slabs (cached like
    // the single-device handles); null otherwise.
    using MultiRef = std::shared_ptr<aprgpu_multi>;
    MultiRef multi(const APR& apr, int halo) {
        if (devices_.size() < 2) return nullptr;
        const bool tree = well_formed(apr.tree_access);
        const AddrKey ak = addr_key(apr.access, tree ? &apr.tree_access : nullptr, apr.source_dims);
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = multi_cache_.begin(); it != multi_cache_.end(); ++it)
            if (it->first == ak && it->second.first >= halo) return it->second.second;
        const aprgpu_access_desc leaf = describe(apr.access);
        aprgpu_access_desc td{};
        if (tree) td = describe(apr.tree_access);
        const int32_t dims[3] = {apr.source_dims[0], apr.source_dims[1], apr.source_dims[2]};
        aprgpu_multi* m = nullptr;
        const int st = aprgpu_multi_create(devices_.data(), static_cast<int>(devices_.size()), &leaf,
                                           tree ? &td : nullptr, dims, halo, &m);
        if (st == APRGPU_ERR_RANGE) return nullptr;  // too thin to cut: one device does it
        check(st);
        multi_cache_.emplace_front(ak, std::make_pair(halo, MultiRef(m, [](aprgpu_multi* q) { aprgpu_multi_free(q); })));
        while (multi_cache_.size() > 2) multi_cache_.pop_back();
        return multi_cache_.front().second.second;
    }

    // Device handle of a bare access structure (leaf only; dims = its finest grid).
    Ref upload(const LinearAccess& a, const std::array<int, 3>& dims) {
        Fingerprint f;
        f.access(a);
        f.bytes(dims.data(), sizeof(int) * 3);
        f.bytes("access-only", 11);
        return lookup(f.value(), AddrKey{}, [&](aprgpu_apr* h) { return same_structure(h, a); },
                      [&](aprgpu_apr** out) {
                          if (!well_formed(a)) throw RangeError("access structure has no levels");
                          const aprgpu_access_desc leaf = describe(a);
                          const int32_t d3[3] = {dims[0], dims[1], dims[2]};
                          return aprgpu_upload_access(ctx_, &leaf, nullptr, d3, out);
                      });
    }

    ~Runtime() {
        cache_.clear();  // (the handles free themselves)
        pyr_cache_.clear();
        multi_cache_.clear();
        if (ctx_) aprgpu_ctx_free(ctx_);
    }

private:
    Runtime() {
        const char* dev = std::getenv("APRGPU_DEVICE");
        check(aprgpu_init(dev ? std::atoi(dev) : 0, &ctx_));
        const char* acc = std::getenv("APRGPU_ACCUM");
        accum_ = (acc && std::string(acc) == "fast") ? APRGPU_ACCUM_FAST : APRGPU_ACCUM_EXACT;
        if (const char* ds = std::getenv("APRGPU_DEVICES")) {  // "0,1,2,3": z-slabs over these devices
            for (const char* p = ds; *p;) {
                char* end = nullptr;
                const long d = std::strtol(p, &end, 10);
                if (end == p) break;
                devices_.push_back(static_cast<int>(d));
                p = *end ? end + 1 : end;
            }
        }
    }

    // The cheap identity of an APR: its arrays' addresses and sizes, its dims,
    // and a strided sample of its contents (the arrays are immutable once
    // built; the sample guards against a new APR reusing freed addresses).
    struct AddrKey {
        const void* p[4] = {};
        std::size_t n[4] = {};
        std::array<int, 3> dims{};
        std::uint64_t sample = 0;
        bool operator==(const AddrKey& o) const {
            for (int i = 0; i < 4; ++i)
                if (p[i] != o.p[i] || n[i] != o.n[i]) return false;
            return dims == o.dims && sample == o.sample && p[0] != nullptr;
        }
    };
    static AddrKey addr_key(const LinearAccess& a, const LinearAccess* t, const std::array<int, 3>& dims) {
        AddrKey k;
        k.p[0] = a.y_idx.data();
        k.n[0] = a.y_idx.size();
        k.p[1] = a.xz_end.data();
        k.n[1] = a.xz_end.size();
        if (t) {
            k.p[2] = t->y_idx.data();
            k.n[2] = t->y_idx.size();
            k.p[3] = t->xz_end.data();
            k.n[3] = t->xz_end.size();
        }
        k.dims = dims;
        Fingerprint f;  // 1024 strided samples of each array (+ the last entry)
        auto sample = [&f](const auto& v) {
            const std::size_t n = v.size();
            for (std::size_t i = 0, st = n / 1024 + 1; i < n; i += st) f.bytes(&v[i], sizeof(v[i]));
            if (n) f.bytes(&v[n - 1], sizeof(v[n - 1]));
        };
        sample(a.y_idx);
        sample(a.xz_end);
        sample(a.level_offset);
        if (t) {
            sample(t->y_idx);
            sample(t->xz_end);
        }
        k.sample = f.value();
        return k;
    }
    // Full verification of a content-fingerprint hit: the device structure
    // equals the host arrays (guards against 64-bit fingerprint collisions).
    static bool same_structure(aprgpu_apr* h, const LinearAccess& a) {
        aprgpu_access_info info{};
        if (aprgpu_access_get_info(h, APRGPU_LEAF, &info) != APRGPU_OK) return false;
        if (info.l_min != a.l_min || info.l_max != a.l_max || info.n_particles != a.y_idx.size() ||
            info.n_rows != a.xz_end.size())
            return false;
        const std::size_t n = static_cast<std::size_t>(info.l_max) + 1;
        std::vector<std::uint16_t> y(info.n_particles);
        std::vector<std::uint64_t> xz(info.n_rows), lo(n);
        std::vector<int32_t> zd(n), xd(n), yd(n);
        if (aprgpu_download_access(h, APRGPU_LEAF, y.data(), xz.data(), lo.data(), zd.data(), xd.data(), yd.data()) !=
            APRGPU_OK)
            return false;
        return y == a.y_idx && xz == a.xz_end;
    }

    template <class Verify, class Upload>
    Ref lookup(std::uint64_t key, const AddrKey& ak, Verify&& verify, Upload&& up) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = cache_.begin(); it != cache_.end(); ++it)
            if (it->key == key && verify(it->ref.get())) {
                it->addr = ak;  // (the same structure at new addresses)
                cache_.splice(cache_.begin(), cache_, it);
                return cache_.front().ref;
            }
        aprgpu_apr* h = nullptr;
        check(up(&h));
        cache_.push_front(Entry{key, ak, Ref(h, [](aprgpu_apr* p) { aprgpu_apr_free(p); })});
        while (cache_.size() > kCacheSize) cache_.pop_back();  // freed when its last holder lets go
        return cache_.front().ref;
    }

    struct Entry {
        std::uint64_t key;
        AddrKey addr;
        Ref ref;
    };
    struct PyrEntry {
        std::uint64_t key;
        int l_min;
        std::vector<float> w;
        std::vector<int32_t> k3;
        PyrRef ref;
    };
    static constexpr std::size_t kCacheSize = 8;
    aprgpu_ctx* ctx_ = nullptr;
    int accum_ = APRGPU_ACCUM_EXACT;
    std::vector<int> devices_;
    std::mutex mu_;
    std::list<Entry> cache_;
    std::list<PyrEntry> pyr_cache_;
    std::list<std::pair<AddrKey, std::pair<int, MultiRef>>> multi_cache_;
};

// A StencilPyramid held on the device (cached by content in the Runtime).
class DevicePyramid {
public:
    explicit DevicePyramid(const StencilPyramid& p) : ref_(Runtime::get().pyramid(p)) {}
    aprgpu_pyramid* get() const { return ref_.get(); }

private:
    Runtime::PyrRef ref_;
};

inline std::uint64_t count(aprgpu_apr* h, int which) {
    aprgpu_access_info info{};
    check(aprgpu_access_get_info(h, which, &info));
    return info.n_particles;
}

inline LinearAccess download(aprgpu_apr* h, int which) {
    aprgpu_access_info info{};
    check(aprgpu_access_get_info(h, which, &info));
    LinearAccess a;
    a.l_min = info.l_min;
    a.l_max = info.l_max;
    const std::size_t n = static_cast<std::size_t>(info.l_max) + 1;
    a.z_dim.resize(n);
    a.x_dim.resize(n);
    a.y_dim.resize(n);
    a.level_offset.resize(n);
    a.y_idx.resize(info.n_particles);
    a.xz_end.resize(info.n_rows);
    check(aprgpu_download_access(h, which, a.y_idx.data(), a.xz_end.data(), a.level_offset.data(), a.z_dim.data(),
                                 a.x_dim.data(), a.y_dim.data()));
    return a;
}

}  // namespace gpu
}  // namespace aprkit

// The reconstruct.hpp drop-in (include/aprkit_gpu/aprkit/reconstruct.hpp) is
// pulled in by this header's own #include of "aprkit/reconstruct.hpp", before
// the runtime above exists; its device implementations follow here.
#define APRKIT_GPU_RUNTIME_DONE 1
#ifdef APRKIT_GPU_RECONSTRUCT_OVERLAY
#include "aprkit_gpu_reconstruct.hpp"
#endif
#ifdef APRKIT_GPU_APR_OVERLAY
#include "aprkit_gpu_apr.hpp"
#endif
