// Multi-GPU z-slabs behind the C-ABI: one
// process drives several devices -- or several slabs of one device -- with
// level-aware halos copied peer to peer (cudaMemcpyPeerAsync: NVLink / NVSwitch
// between GPUs, a device copy within one).  This is the C++ drop-in's
// multi-GPU path (torch.distributed's NCCL version is paper_2112_03592_b200/slab.py,
// one process per GPU); both follow the same plan:
//
//  * the finest-level pixel planes are cut into blocks of 2^c planes, slab s
//    owns a contiguous run of blocks; levels >= lc = l_max - c are PARTITIONED
//    (a cell never straddles two slabs), levels < lc REPLICATED (tiny);
//  * rows are z-major in the CSR, so the rows [za, zb) of a level are one
//    contiguous particle range: every transfer is one contiguous copy.
//
// A convolution (convolve_apr, convolve.hpp:220-303) on N slabs:
//   1. per slab, H2D of its owned leaf / interior values and the replicated
//      prefix; the INTERIOR of the slab -- planes at least halo * 2^(l_max-lc)
//      from a cut -- convolves at once (its stencils never leave the slab);
//   2. per internal cut, the halo rows of every partitioned level (halo level-l
//      rows = halo * 2^(l_max - l) planes) are copied from the neighbour as soon
//      as the neighbour's upload has landed, on a copy stream;
//   3. the slab's two boundary bands convolve after their halos arrive;
//   4. D2H of the owned outputs (slab 0 also returns the replicated levels).
// Every output reads only cells within the stencil half-width of its own
// cell, which the slab plus its halo hold, so each owned output is
// bit-identical to the single-domain result (EXACT mode).
#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"

namespace aprgpu {
namespace {

struct Range {
    uint64_t b = 0, e = 0;
};

// Host copy of the row geometry of one access structure (what the plan needs).
struct HostRows {
    int l_min = 0, l_max = -1;
    std::vector<int> zd, xd;
    std::vector<uint64_t> level_offset, xz_end;
    uint64_t n = 0;

    void load(const aprgpu_access_desc* d) {
        if (!d) return;
        l_min = d->l_min;
        l_max = d->l_max;
        zd.assign(d->z_dim, d->z_dim + l_max + 1);
        xd.assign(d->x_dim, d->x_dim + l_max + 1);
        level_offset.assign(d->level_offset, d->level_offset + l_max + 1);
        xz_end.assign(d->xz_end, d->xz_end + d->n_rows);
        n = d->n_particles;
    }
    bool empty() const { return xz_end.empty(); }
    uint64_t begin(uint64_t r) const { return r ? xz_end[r - 1] : 0; }
    // particles of rows z in [za, zb) of level l (contiguous, z-major)
    Range rows(int l, int za, int zb) const {
        if (empty() || l < l_min || l > l_max) return {};
        za = std::max(0, std::min(za, zd[l]));
        zb = std::max(za, std::min(zb, zd[l]));
        const uint64_t r0 = level_offset[l] + static_cast<uint64_t>(za) * xd[l];
        const uint64_t r1 = level_offset[l] + static_cast<uint64_t>(zb) * xd[l];
        return {begin(r0), begin(r1)};
    }
};

struct Transfer {
    int src, dst;
    bool tree;
    Range r;
};

// The z-slab plan (slab.py SlabPlan.make, restated).
struct Plan {
    int n = 1, l_max = 0, c = 0, lc = 0, halo = 1;
    std::vector<std::pair<int, int>> bounds;  // per slab: finest planes [z_lo, z_hi)

    std::pair<int, int> rows(int l, int s) const {
        const int sh = l_max - l;
        return {bounds[s].first >> sh, (bounds[s].second + (1 << sh) - 1) >> sh};
    }
    std::vector<Range> owned(const HostRows& a, int s) const {
        std::vector<Range> out;
        if (a.empty()) return out;
        for (int l = std::max(lc, a.l_min); l <= a.l_max; ++l) {
            const auto r = rows(l, s);
            out.push_back(a.rows(l, r.first, r.second));
        }
        return out;
    }
    Range replicated(const HostRows& a) const {
        if (a.empty() || lc <= a.l_min) return {};
        return {0, a.rows(std::min(lc, a.l_max + 1) - 1, 0, 1 << 30).e};
    }
    void transfers(const HostRows& a, bool tree, std::vector<Transfer>& out) const {
        if (a.empty()) return;
        for (int l = std::max(lc, a.l_min); l <= a.l_max; ++l)
            for (int s = 0; s + 1 < n; ++s) {
                const auto lo = rows(l, s), hi = rows(l, s + 1);
                const Range up = a.rows(l, std::max(lo.first, lo.second - halo), lo.second);  // s -> s+1
                if (up.e > up.b) out.push_back({s, s + 1, tree, up});
                const Range dn = a.rows(l, hi.first, std::min(hi.second, hi.first + halo));  // s+1 -> s
                if (dn.e > dn.b) out.push_back({s + 1, s, tree, dn});
            }
    }
};

struct SlabDev {
    int device = 0;
    aprgpu_ctx* ctx = nullptr;
    aprgpu_apr* apr = nullptr;
    cudaStream_t compute = nullptr, copy = nullptr;
    cudaEvent_t uploaded = nullptr, halos = nullptr;
    GpuBuf values, tree, out;
};

}  // namespace
}  // namespace aprgpu

struct aprgpu_multi {
    aprgpu::Plan plan;
    aprgpu::HostRows leaf, tree;
    std::vector<aprgpu::SlabDev> slabs;
    std::vector<aprgpu::Transfer> xfer;
    uint64_t n_leaf = 0, n_tree = 0;
    std::mutex mu;  // one call at a time (the slabs' buffers and streams)
};

namespace aprgpu {
namespace {

void free_multi(aprgpu_multi* m) {
    for (auto& s : m->slabs) {
        DeviceGuard g(s.device);
        if (s.compute) cudaStreamSynchronize(s.compute);
        if (s.copy) cudaStreamSynchronize(s.copy);
        s.values.release();
        s.tree.release();
        s.out.release();
        if (s.uploaded) cudaEventDestroy(s.uploaded);
        if (s.halos) cudaEventDestroy(s.halos);
        if (s.compute) cudaStreamDestroy(s.compute);
        if (s.copy) cudaStreamDestroy(s.copy);
        if (s.apr) aprgpu_apr_free(s.apr);
        if (s.ctx) aprgpu_ctx_free(s.ctx);
    }
    m->slabs.clear();
}

void check(int st) {
    if (st != APRGPU_OK) fail(st, last_error_slot());
}

}  // namespace
}  // namespace aprgpu

extern "C" {

int aprgpu_multi_create(const int* devices, int n_slabs, const aprgpu_access_desc* leaf,
                        const aprgpu_access_desc* tree, const int32_t source_dims[3], int halo, aprgpu_multi** out) {
    using namespace aprgpu;
    aprgpu_multi* m = nullptr;
    const int st = guard("aprgpu_multi_create", [&] {
        need(devices && leaf && source_dims && out && n_slabs >= 1, "null argument");
        need(halo >= 1 && halo <= 6, "halo must be 1..6 rows (half-width of a stencil <= 13)");
        m = new aprgpu_multi;
        m->leaf.load(leaf);
        m->n_leaf = leaf->n_particles;
        if (leaf->l_min < 0 || leaf->l_max < leaf->l_min || leaf->l_max >= kMaxLevels)
            fail(APRGPU_ERR_RANGE, "multi: bad level range");
        // the plan: the largest block 2^c such that every slab gets >= halo blocks
        Plan& p = m->plan;
        p.n = n_slabs;
        p.halo = halo;
        int geom = 0;
        while ((1 << geom) < std::max(source_dims[0], std::max(source_dims[1], source_dims[2]))) ++geom;
        p.l_max = std::max(leaf->l_max, geom);
        const int nz = source_dims[0];
        p.c = -1;
        for (int cc = p.l_max; cc >= 0; --cc) {
            const int nb = (nz + (1 << cc) - 1) >> cc;
            if (nb / n_slabs >= halo) {
                p.c = cc;
                break;
            }
        }
        if (p.c < 0) fail(APRGPU_ERR_RANGE, "multi: the volume is too thin for this many slabs");
        p.lc = p.l_max - p.c;
        const int nb = (nz + (1 << p.c) - 1) >> p.c;
        for (int s = 0; s < n_slabs; ++s) {
            const int b0 = static_cast<int>(static_cast<int64_t>(s) * nb / n_slabs);
            const int b1 = static_cast<int>(static_cast<int64_t>(s + 1) * nb / n_slabs);
            p.bounds.push_back({std::min(b0 << p.c, nz), std::min(b1 << p.c, nz)});
        }
        m->slabs.resize(n_slabs);
        for (int s = 0; s < n_slabs; ++s) {
            SlabDev& d = m->slabs[s];
            d.device = devices[s];
            check(aprgpu_init(d.device, &d.ctx));
            check(aprgpu_upload_access(d.ctx, leaf, tree, source_dims, &d.apr));
            // its per-tile state only for its own slab's tiles
            check(aprgpu_apr_restrict(d.apr, p.lc, p.bounds[s].first, p.bounds[s].second));
            DeviceGuard g(d.device);
            APR_CUDA(cudaStreamCreateWithFlags(&d.compute, cudaStreamNonBlocking));
            APR_CUDA(cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking));
            APR_CUDA(cudaEventCreateWithFlags(&d.uploaded, cudaEventDisableTiming));
            APR_CUDA(cudaEventCreateWithFlags(&d.halos, cudaEventDisableTiming));
            for (int o = 0; o < n_slabs; ++o)  // peer access between distinct GPUs (NVLink / NVSwitch)
                if (devices[o] != d.device) {
                    int ok = 0;
                    cudaDeviceCanAccessPeer(&ok, d.device, devices[o]);
                    if (ok) {
                        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[o], 0);
                        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) APR_CUDA(e);
                        cudaGetLastError();
                    }
                }
        }
        // the interior structure as uploaded (or built on the device)
        aprgpu_access_info ti{};
        check(aprgpu_access_get_info(m->slabs[0].apr, APRGPU_TREE, &ti));
        m->n_tree = ti.n_particles;
        if (ti.n_particles) {
            const int n = ti.l_max + 1;
            std::vector<uint16_t> y(ti.n_particles);
            std::vector<uint64_t> xz(ti.n_rows), lo(n);
            std::vector<int32_t> zd(n), xd(n), yd(n);
            check(aprgpu_download_access(m->slabs[0].apr, APRGPU_TREE, y.data(), xz.data(), lo.data(), zd.data(),
                                         xd.data(), yd.data()));
            aprgpu_access_desc td{ti.l_min, ti.l_max, zd.data(), xd.data(), yd.data(), y.data(), ti.n_particles,
                                  xz.data(), ti.n_rows, lo.data()};
            m->tree.load(&td);
        }
        p.transfers(m->leaf, false, m->xfer);
        p.transfers(m->tree, true, m->xfer);
        for (auto& d : m->slabs) {
            DeviceGuard g(d.device);
            d.values.ensure(4 * m->n_leaf + 16);
            d.tree.ensure(4 * m->n_tree + 16);
            d.out.ensure(4 * m->n_leaf + 16);
        }
        *out = m;
    });
    if (st != APRGPU_OK && m) {
        free_multi(m);
        delete m;
    }
    return st;
}

int aprgpu_multi_free(aprgpu_multi* m) {
    return aprgpu::guard([&] {
        if (!m) return;
        aprgpu::free_multi(m);
        delete m;
    });
}

int aprgpu_multi_info(const aprgpu_multi* m, int* n_slabs, int* cut_level, int32_t* z_bounds) {
    return aprgpu::guard([&] {
        aprgpu::need(m, "null argument");
        if (n_slabs) *n_slabs = m->plan.n;
        if (cut_level) *cut_level = m->plan.lc;
        if (z_bounds)
            for (int s = 0; s < m->plan.n; ++s) {
                z_bounds[2 * s] = m->plan.bounds[s].first;
                z_bounds[2 * s + 1] = m->plan.bounds[s].second;
            }
    });
}

int aprgpu_multi_convolve(aprgpu_multi* m, const float* values, const float* tree_values, const float* w,
                          const int32_t* k3, int l_min, int l_max, int pad_mode, int accum, float* out) {
    using namespace aprgpu;
    return guard("aprgpu_multi_convolve", [&] {
        need(m && values && w && k3 && out, "null argument");
        need(tree_values || m->n_tree == 0, "tree values are required");
        need(pad_mode == APRGPU_PAD_ZERO || pad_mode == APRGPU_PAD_REFLECT, "bad pad mode");
        need(accum == APRGPU_ACCUM_EXACT || accum == APRGPU_ACCUM_FAST, "bad accumulation mode");
        std::lock_guard<std::mutex> lk(m->mu);
        const Plan& p = m->plan;
        // halo depth in pixels: the halo's level-lc rows cover every partitioned level's halo
        const int margin = p.halo << (p.l_max - p.lc);
        for (int l = std::max(p.lc, l_min); l <= l_max; ++l) {
            const int* k = k3 + 3 * (l - l_min);
            if (std::max(k[0], std::max(k[1], k[2])) / 2 > p.halo)
                fail(APRGPU_ERR_RANGE, "multi: a stencil half-width exceeds the slabs' halo");
        }
        // per-device pyramids (explicit levels), freed at the end of the call
        std::vector<aprgpu_pyramid*> pyr(p.n, nullptr);
        struct Free {
            std::vector<aprgpu_pyramid*>& v;
            ~Free() {
                for (auto* q : v)
                    if (q) aprgpu_pyramid_free(q);
            }
        } free_pyr{pyr};
        for (int s = 0; s < p.n; ++s)
            check(aprgpu_pyramid_create_explicit(m->slabs[s].ctx, w, k3, l_min, l_max, &pyr[s]));
        const Range rl = p.replicated(m->leaf), rt = p.replicated(m->tree);
        auto h2d = [](float* dst, const float* src, Range r, cudaStream_t st) {
            if (r.e > r.b) APR_CUDA(cudaMemcpyAsync(dst + r.b, src + r.b, 4 * (r.e - r.b), cudaMemcpyHostToDevice, st));
        };
        auto conv = [&](int s, int z_lo, int z_hi, bool rep) {
            SlabDev& d = m->slabs[s];
            if (z_hi <= z_lo && !rep) return;
            Slab slab;
            slab.lc = p.lc;
            slab.z_lo = z_lo;
            slab.z_hi = std::max(z_lo, z_hi);
            slab.rep = rep;
            EpiArgs epi;
            convolve_device(d.apr, d.values.as<float>(), d.tree.as<float>(), pyr[s], pad_mode, accum,
                            d.out.as<float>(), epi, d.compute, slab);
        };
        // 1. uploads, then the interior of every slab
        std::unique_ptr<NvtxRange> ph(new NvtxRange("aprgpu_multi: uploads + interior bands"));
        for (int s = 0; s < p.n; ++s) {
            SlabDev& d = m->slabs[s];
            DeviceGuard g(d.device);
            h2d(d.values.as<float>(), values, rl, d.compute);
            for (const Range& r : p.owned(m->leaf, s)) h2d(d.values.as<float>(), values, r, d.compute);
            h2d(d.tree.as<float>(), tree_values, rt, d.compute);
            for (const Range& r : p.owned(m->tree, s)) h2d(d.tree.as<float>(), tree_values, r, d.compute);
            APR_CUDA(cudaEventRecord(d.uploaded, d.compute));
            const int lo = p.bounds[s].first + (s > 0 ? margin : 0);
            const int hi = p.bounds[s].second - (s + 1 < p.n ? margin : 0);
            conv(s, lo, hi, true);
        }
        // 2. halos: each destination's copy stream waits for its source's upload
        ph.reset(new NvtxRange("aprgpu_multi: halo exchange (peer copies)"));
        for (int s = 0; s < p.n; ++s) {
            SlabDev& d = m->slabs[s];
            DeviceGuard g(d.device);
            for (const Transfer& t : m->xfer) {
                if (t.dst != s) continue;
                const SlabDev& src = m->slabs[t.src];
                APR_CUDA(cudaStreamWaitEvent(d.copy, src.uploaded, 0));
                float* dp = (t.tree ? d.tree : d.values).as<float>() + t.r.b;
                const float* sp = (t.tree ? src.tree : src.values).as<float>() + t.r.b;
                APR_CUDA(cudaMemcpyPeerAsync(dp, d.device, sp, src.device, 4 * (t.r.e - t.r.b), d.copy));
            }
            APR_CUDA(cudaEventRecord(d.halos, d.copy));
        }
        // 3. the boundary bands, 4. the owned outputs back
        ph.reset(new NvtxRange("aprgpu_multi: boundary bands + download"));
        for (int s = 0; s < p.n; ++s) {
            SlabDev& d = m->slabs[s];
            DeviceGuard g(d.device);
            APR_CUDA(cudaStreamWaitEvent(d.compute, d.halos, 0));
            const int z0 = p.bounds[s].first, z1 = p.bounds[s].second;
            if (s > 0) conv(s, z0, std::min(z0 + margin, z1), false);
            if (s + 1 < p.n) conv(s, std::max(z1 - margin, s > 0 ? z0 + margin : z0), z1, false);
            auto d2h = [&](Range r) {
                if (r.e > r.b)
                    APR_CUDA(cudaMemcpyAsync(out + r.b, d.out.as<float>() + r.b, 4 * (r.e - r.b),
                                             cudaMemcpyDeviceToHost, d.compute));
            };
            if (s == 0) d2h(rl);
            for (const Range& r : p.owned(m->leaf, s)) d2h(r);
        }
        for (auto& d : m->slabs) {
            DeviceGuard g(d.device);
            APR_CUDA(cudaStreamSynchronize(d.compute));
            APR_CUDA(cudaStreamSynchronize(d.copy));
        }
    });
}

}  // extern "C"
