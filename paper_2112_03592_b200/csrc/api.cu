// The C-ABI (include/aprgpu.h): contexts, structure upload/download, stencil
// pyramids, and the host/device-pointer front doors of fill_tree, convolve_apr
// and rl_apr.  Exceptions never cross this boundary; aprgpu::Error carries the
// status code that the reference-side shim maps back to aprkit's exceptions.
#include <algorithm>
#include <thread>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "common.cuh"

namespace aprgpu {
std::string& last_error_slot() {
    static thread_local std::string msg;
    return msg;
}
}  // namespace aprgpu

namespace {

using aprgpu::DeviceGuard;
using aprgpu::fail;
using aprgpu::guard;
using aprgpu::need;
#define g_last_error (aprgpu::last_error_slot())

int host_compute_l_max(int nz, int nx, int ny) {
    const int m = std::max(nz, std::max(nx, ny));
    int l = 0;
    while ((1 << l) < m) ++l;
    return l;
}

void upload_one(aprgpu_ctx* ctx, const aprgpu_access_desc* d, aprgpu::DevAccess& a, bool tiles) {
    need(d != nullptr, "null access descriptor");
    need(d->l_min >= 0 && d->l_min <= d->l_max, "l_min > l_max");
    if (d->l_max >= aprgpu::kMaxLevels) fail(APRGPU_ERR_CAPABILITY, "too many levels");
    need(d->z_dim && d->x_dim && d->y_dim && d->level_offset, "null dims");
    need(d->n_rows == 0 || d->xz_end, "null xz_end");
    need(d->n_particles == 0 || d->y_idx, "null y_idx");
    a.l_min = d->l_min;
    a.l_max = d->l_max;
    a.zd.assign(d->z_dim, d->z_dim + d->l_max + 1);
    a.xd.assign(d->x_dim, d->x_dim + d->l_max + 1);
    a.yd.assign(d->y_dim, d->y_dim + d->l_max + 1);
    a.level_offset.assign(d->level_offset, d->level_offset + d->l_max + 1);
    uint64_t expect = 0;
    for (int l = a.l_min; l <= a.l_max; ++l) {  // validate, apr.hpp:66-73
        if (a.level_offset[l] != expect) fail(APRGPU_ERR_INTEGRITY, "level_offset mismatch");
        if (a.yd[l] > 65536) fail(APRGPU_ERR_CAPABILITY, "y dimension exceeds the 16-bit index limit");
        expect += static_cast<uint64_t>(a.zd[l]) * a.xd[l];
    }
    if (expect != d->n_rows) fail(APRGPU_ERR_INTEGRITY, "xz_end length does not match level grids");
    if (d->n_rows >= (1ull << 32) - 1) fail(APRGPU_ERR_CAPABILITY, "row count exceeds u32");
    a.n_particles = d->n_particles;
    a.n_rows = d->n_rows;
    APR_CUDA(cudaMalloc(&a.y, 2 * a.n_particles + 2));
    if (a.n_particles)
        APR_CUDA(cudaMemcpyAsync(a.y, d->y_idx, 2 * a.n_particles, cudaMemcpyHostToDevice, ctx->stream));
    if (a.n_rows == 0 && a.n_particles) fail(APRGPU_ERR_INTEGRITY, "particles present but no rows");
    aprgpu::build_row_begin(ctx, a, d->xz_end);
    aprgpu::build_work_lists(ctx, a);
    if (tiles) aprgpu::build_tile_lists(ctx, a);
}

void free_apr(aprgpu_apr* apr) {
    if (apr->scratch_ev) cudaEventDestroy(apr->scratch_ev);
    if (apr->index_ev) cudaEventDestroy(apr->index_ev);
    apr->scratch_ev = nullptr;
    apr->leaf.release();
    apr->tree.release();
    for (aprgpu::GpuBuf* b : {&apr->vsum, &apr->wsum, &apr->tree_links, &apr->h_in, &apr->h_tree, &apr->h_out, &apr->rl_u,
                              &apr->rl_ratio, &apr->rl_tv, &apr->tmp, &apr->built_values})
        b->release();
}

// One user of an APR's scratch at a time (fill_tree's fp64 sums, the staging
// buffers of host-pointer calls, RL state): the lock serialises the callers on
// the host, the event orders their work across their streams (a device-pointer
// fill on one stream completes before the next caller's kernels touch the sums).
struct ScratchGuard {
    std::lock_guard<std::mutex> lk;
    cudaEvent_t& ev;
    cudaStream_t s;
    // the APR's shared scratch (fill_tree sums, host staging, RL state) by default;
    // a scratch of its own (mutex + event) otherwise
    ScratchGuard(aprgpu_apr* a, cudaStream_t st) : ScratchGuard(a->exec_mu, a->scratch_ev, st) {}
    ScratchGuard(std::mutex& mu, cudaEvent_t& e, cudaStream_t st) : lk(mu), ev(e), s(st) {
        if (!ev)
            APR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        else
            APR_CUDA(cudaStreamWaitEvent(s, ev, 0));
    }
    ~ScratchGuard() { cudaEventRecord(ev, s); }
};

aprgpu::HostStencil make_host_stencil(const float* w, int kz, int kx, int ky) {
    if (kz < 1 || kx < 1 || ky < 1 || kz % 2 == 0 || kx % 2 == 0 || ky % 2 == 0)
        fail(APRGPU_ERR_RANGE, "stencil extents must be odd and positive");  // Stencil ctor, stencil.hpp:24-25
    need(w != nullptr, "null stencil weights");
    aprgpu::HostStencil s;
    s.kz = kz;
    s.kx = kx;
    s.ky = ky;
    s.w.assign(w, w + static_cast<size_t>(kz) * kx * ky);
    return s;
}

// Rank-1 factors of a stencil from its marginals: w[a][b][c] ~ Mz[a] Mx[b] My[c]
// / S^2 (S = sum of w).  Accepted when every weight matches to 5e-7 relative
// (a truncated Gaussian, stencil.hpp:59-79, and its restrictions are products
// of per-axis factors); appended to sep as floats fz = Mz/S, fx = Mx/S, fy = My.
bool separable_factors(const float* w, int kz, int kx, int ky, std::vector<float>& sep) {
    std::vector<double> mz(kz, 0.0), mx(kx, 0.0), my(ky, 0.0);
    double sum = 0.0;
    for (int a = 0; a < kz; ++a)
        for (int b = 0; b < kx; ++b)
            for (int c = 0; c < ky; ++c) {
                const double v = w[(static_cast<size_t>(a) * kx + b) * ky + c];
                if (v < 0.0) return false;
                mz[a] += v;
                mx[b] += v;
                my[c] += v;
                sum += v;
            }
    if (!(sum > 0.0)) return false;
    std::vector<float> fz(kz), fx(kx), fy(ky);
    for (int a = 0; a < kz; ++a) fz[a] = static_cast<float>(mz[a] / sum);
    for (int b = 0; b < kx; ++b) fx[b] = static_cast<float>(mx[b] / sum);
    for (int c = 0; c < ky; ++c) fy[c] = static_cast<float>(my[c]);
    for (int a = 0; a < kz; ++a)
        for (int b = 0; b < kx; ++b)
            for (int c = 0; c < ky; ++c) {
                const double v = w[(static_cast<size_t>(a) * kx + b) * ky + c];
                const double f = static_cast<double>(fz[a]) * fx[b] * fy[c];
                if (std::fabs(f - v) > 5e-7 * std::fabs(v)) return false;
            }
    sep.insert(sep.end(), fz.begin(), fz.end());
    sep.insert(sep.end(), fx.begin(), fx.end());
    sep.insert(sep.end(), fy.begin(), fy.end());
    return true;
}

void pyramid_upload(aprgpu_pyramid* p) {
    DeviceGuard g(p->ctx->device);
    const size_t n = p->w_host.size();
    APR_CUDA(cudaMalloc(&p->w_dev, sizeof(float) * (n + 1)));
    APR_CUDA(cudaMalloc(&p->wd_dev, sizeof(double) * (n + 1)));
    std::vector<double> wd(p->w_host.begin(), p->w_host.end());
    APR_CUDA(cudaMemcpy(p->w_dev, p->w_host.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
    APR_CUDA(cudaMemcpy(p->wd_dev, wd.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    std::vector<float> sep;
    p->sep_off.assign(p->off.size(), -1);
    for (size_t i = 0; i < p->off.size(); ++i) {
        const int* k = &p->k3[3 * i];
        const size_t at = sep.size();
        if (separable_factors(p->w_host.data() + p->off[i], k[0], k[1], k[2], sep))
            p->sep_off[i] = static_cast<int64_t>(at);
    }
    APR_CUDA(cudaMalloc(&p->sep_dev, sizeof(float) * (sep.size() + 1)));
    if (!sep.empty())
        APR_CUDA(cudaMemcpy(p->sep_dev, sep.data(), sizeof(float) * sep.size(), cudaMemcpyHostToDevice));
}

void push_level(aprgpu_pyramid* p, const aprgpu::HostStencil& s) {
    p->off.push_back(p->w_host.size());
    p->k3.insert(p->k3.end(), {s.kz, s.kx, s.ky});
    p->w_host.insert(p->w_host.end(), s.w.begin(), s.w.end());
}

// u = max(in, 0) (deconv.hpp:89), and the same into est unless est is null
// (a resumed run keeps its running estimate).  in may alias est: every
// element is read before it is written, by the same thread.
__global__ void k_clamp_copy(const float* in, float* __restrict__ u, float* est, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = in[i];
        const float c = v < 0.0f ? 0.0f : v;  // std::max(v, 0.0f), deconv.hpp:89
        u[i] = c;
        if (est) est[i] = c;
    }
}

// Exactness test + exact sum of the RL observations (see aprgpu_rl_resume).
constexpr int kNoLowBit = 1 << 20;
struct MeanStats {
    double abs_sum;        // sum |v| (any order: an upper bound of every partial sum)
    int neg_gexp_max;      // kNoLowBit - (smallest low-bit exponent); 0 = all values zero
    int nonfinite;
    unsigned long long isum;  // sum of v / 2^g as two's-complement int64 (order-free, exact)
};

__device__ __forceinline__ int low_bit_exp(float v) {  // exponent of the lowest set bit of v (v != 0, finite)
    const uint32_t b = __float_as_uint(v);
    const int e = static_cast<int>((b >> 23) & 0xff);
    uint32_t m = b & 0x7fffff;
    if (e) m |= 0x800000;
    return (e ? e : 1) - 150 + __ffs(static_cast<int>(m)) - 1;
}

// block reductions: one atomic per block (a per-thread fp64 / int64 atomic on
// one address serialises the whole grid)
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : sh[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;  // valid in thread 0
}

__global__ void __launch_bounds__(256) k_mean_bound(const float* __restrict__ u, uint64_t n, MeanStats* st) {
    __shared__ double shd[8];
    __shared__ int shi[8];
    double as = 0.0;
    int gmin = kNoLowBit;
    int bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = u[i];
        if (!isfinite(v)) {
            bad = 1;
            continue;
        }
        as += fabs(static_cast<double>(v));
        if (v != 0.0f) gmin = min(gmin, low_bit_exp(v));
    }
    as = block_reduce(as, [](double x, double y) { return x + y; }, shd);
    gmin = block_reduce(gmin, [](int x, int y) { return min(x, y); }, shi);
    bad = block_reduce(bad, [](int x, int y) { return x | y; }, shi);
    if (threadIdx.x == 0) {
        atomicAdd(&st->abs_sum, as);  // (order-free: only compared against a bound with margin)
        if (gmin != kNoLowBit) atomicMax(&st->neg_gexp_max, kNoLowBit - gmin);
        if (bad) atomicOr(&st->nonfinite, 1);
    }
}

__global__ void __launch_bounds__(256) k_mean_exact(const float* __restrict__ u, uint64_t n, MeanStats* st) {
    __shared__ long long shl[8];
    if (st->nonfinite || st->neg_gexp_max == 0) return;
    const int g = kNoLowBit - st->neg_gexp_max;
    if (!(st->abs_sum < ldexp(1.0, 53 + g) * 0.999999)) return;
    long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        acc += static_cast<long long>(ldexp(static_cast<double>(u[i]), -g));  // exact: |v / 2^g| < 2^53
    acc = block_reduce(acc, [](long long x, long long y) { return x + y; }, shl);  // integer: order-free
    if (threadIdx.x == 0) atomicAdd(&st->isum, static_cast<unsigned long long>(acc));
}

// any value < 0 -> st->nonfinite = 1 (aprgpu_sequential_sum's argument check)
__global__ void k_min_check(const float* __restrict__ u, uint64_t n, MeanStats* st) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (u[i] < 0.0f) st->nonfinite = 1;
}

}  // namespace

namespace {

__global__ void k_gather_rb(const uint32_t* __restrict__ rb, const uint64_t* __restrict__ rows, uint64_t* __restrict__ out,
                            int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = rb[rows[i]];
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

}  // namespace

namespace aprgpu {

HostPool::HostPool(int n) {
    for (int i = 0; i < n; ++i)
        th_.emplace_back([this] {
            uint64_t seen = 0;
            for (;;) {
                std::function<void()> job;
                {
                    std::unique_lock<std::mutex> lk(m_);
                    cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                    if (stop_) return;
                    seen = gen_;
                    job = job_;
                }
                job();
                std::lock_guard<std::mutex> lk(m_);
                if (--busy_ == 0) done_.notify_all();
            }
        });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> lk(m_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
}

void HostPool::start(std::function<void()> job) {
    std::lock_guard<std::mutex> lk(m_);
    job_ = std::move(job);
    busy_ = static_cast<int>(th_.size());
    ++gen_;
    cv_.notify_all();
}

void HostPool::wait() {
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return busy_ == 0; });
}

}  // namespace aprgpu

namespace {

// The z-chunk plan of a host-pointer convolution (see convolve_host_pipelined).
bool host_pipe_plan(aprgpu_apr* apr, int chunks, cudaStream_t s) {
    const aprgpu::DevAccess& L = apr->leaf;
    const aprgpu::DevAccess& T = apr->tree;
    const int nzf = L.zd[L.l_max];
    int S = 8;  // >= the tile height at l_max
    while (2 * S * chunks <= nzf) S *= 2;
    const int K = (nzf + S - 1) / S;
    if (K < 2) return false;
    int lg = 0;
    while ((1 << lg) < S) ++lg;
    // levels >= lc: a tile (8 rows) never spans two chunks, so a chunk's outputs
    // are final after its own pass; its halo (<= 6 rows) lies in the neighbours
    const int lc = std::max(L.l_max - (lg - 3), L.l_min);
    auto& P = apr->host_pipe;
    if (P.S == S && P.K == K) return true;
    std::vector<uint64_t> rows;
    auto add_rows = [&](const aprgpu::DevAccess& A, int lo) {
        for (int l = lo; l <= A.l_max; ++l) {
            const int sh = L.l_max - l;
            for (int j = 0; j <= K; ++j) {
                const int64_t zp = std::min<int64_t>(static_cast<int64_t>(j) * S, nzf);
                const int64_t zb = std::min<int64_t>((zp + (int64_t(1) << sh) - 1) >> sh, A.zd[l]);
                rows.push_back(A.level_offset[l] + static_cast<uint64_t>(zb) * A.xd[l]);
            }
        }
    };
    const int tlo = std::max(lc, T.l_min);
    add_rows(L, lc);
    const size_t nleafrows = rows.size();
    if (T.n_particles) add_rows(T, tlo);
    const size_t ntreerows = rows.size() - nleafrows;
    rows.push_back(L.level_offset[lc]);
    if (T.n_particles) rows.push_back(tlo <= T.l_max ? T.level_offset[tlo] : T.n_rows);
    aprgpu::GpuBuf d_rows, d_out;
    d_rows.ensure(8 * rows.size());
    d_out.ensure(8 * rows.size());
    APR_CUDA(cudaMemcpyAsync(d_rows.p, rows.data(), 8 * rows.size(), cudaMemcpyHostToDevice, s));
    std::vector<uint64_t> got(rows.size());
    // (leaf rows index the leaf rb, the rest the interior rb)
    k_gather_rb<<<1, 256, 0, s>>>(L.rb, d_rows.as<uint64_t>(), d_out.as<uint64_t>(), static_cast<int>(nleafrows));
    if (ntreerows)
        k_gather_rb<<<1, 256, 0, s>>>(T.rb, d_rows.as<uint64_t>() + nleafrows, d_out.as<uint64_t>() + nleafrows,
                                      static_cast<int>(ntreerows));
    k_gather_rb<<<1, 32, 0, s>>>(L.rb, d_rows.as<uint64_t>() + nleafrows + ntreerows,
                                 d_out.as<uint64_t>() + nleafrows + ntreerows, 1);
    if (T.n_particles)
        k_gather_rb<<<1, 32, 0, s>>>(T.rb, d_rows.as<uint64_t>() + nleafrows + ntreerows + 1,
                                     d_out.as<uint64_t>() + nleafrows + ntreerows + 1, 1);
    aprgpu::count_launch(apr->ctx, 2 + (ntreerows ? 1 : 0) + (T.n_particles ? 1 : 0));
    APR_CUDA(cudaGetLastError());
    APR_CUDA(cudaMemcpyAsync(got.data(), d_out.p, 8 * rows.size(), cudaMemcpyDeviceToHost, s));
    APR_CUDA(cudaStreamSynchronize(s));
    P.S = S;
    P.K = K;
    P.lc = lc;
    P.leaf_b.assign(got.begin(), got.begin() + nleafrows);
    P.tree_b.assign(got.begin() + nleafrows, got.begin() + nleafrows + ntreerows);
    P.leaf_pre = got[nleafrows + ntreerows];
    P.tree_pre = T.n_particles ? got[nleafrows + ntreerows + 1] : 0;
    return true;
}

// convolve_apr with host pointers, pipelined over z-chunks of the volume: the
// inputs stream in chunk by chunk on one copy stream, chunk j's tiles convolve
// (Slab restriction, as the multi-GPU path) once chunks <= j+1 have arrived, and
// chunk j's outputs stream back on a second copy stream while later chunks
// convolve -- so the PCIe copies in both directions overlap each other and the
// kernels.  Outputs are bit-identical to the one-shot path (every output is
// computed from the same inputs by the same kernel; levels < lc, a few
// thousand particles, are recomputed by every pass and copied back last).
// Page-locked buffers are copied directly.  Pageable ones (a std::vector: the
// C++ drop-in) go through the context's pinned staging: its worker threads
// copy chunk j in while the device already copies and convolves the chunks
// before it, and copy chunk j's outputs out as soon as they have landed -- a
// plain cudaMemcpy of pageable memory would serialise all of it.  C3 on one
// B200: 2.80 ms one-shot -> 2.36 ms pinned (PCIe: the two directions share the
// link's budget, so the overlap is partial).  Returns false when the volume
// is too small to be worth chunking (or the staging would exceed
// $APRGPU_STAGE_MAX_MB, default 4096).
bool convolve_host_pipelined(aprgpu_apr* apr, const float* values, const float* tree_values,
                             const aprgpu_pyramid* pyr, int pad, int accum, float* out, cudaStream_t s) {
    const int chunks = env_int("APRGPU_HOST_CHUNKS", 8);
    const int min_np = env_int("APRGPU_HOST_PIPELINE_MIN", 1 << 20);
    const uint64_t np = apr->leaf.n_particles, nt = apr->tree.n_particles;
    if (chunks < 2 || np < static_cast<uint64_t>(std::max(min_np, 0)) || !s) return false;
    auto pinned = [](const void* p) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return at.type == cudaMemoryTypeHost;
    };
    // staging per array: a page-locked array is copied directly, a pageable one
    // through the pinned staging (the C++ drop-in hands in pageable inputs and a
    // page-locked output buffer)
    const bool st_val = !pinned(values), st_tree = nt && !pinned(tree_values), st_out = !pinned(out);
    const bool staged = st_val || st_tree || st_out;
    const size_t stage_need = 4 * (2 * np + nt);
    if (staged && stage_need > static_cast<size_t>(std::max(env_int("APRGPU_STAGE_MAX_MB", 4096), 0)) << 20)
        return false;
    aprgpu_ctx* ctx = apr->ctx;
    std::lock_guard<std::mutex> lk(ctx->pipe_mu);
    aprgpu::NvtxRange nr(staged ? "aprgpu: host pipeline (pageable, staged)" : "aprgpu: host pipeline (pinned)");
    if (!host_pipe_plan(apr, chunks, s)) return false;
    const auto& P = apr->host_pipe;
    const int K = P.K;
    if (!ctx->copy_in) APR_CUDA(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
    if (!ctx->copy_out) APR_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
    while (ctx->events.size() < static_cast<size_t>(3 * K + 2)) {
        cudaEvent_t e;
        APR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->events.push_back(e);
    }
    cudaEvent_t start = ctx->events[0];
    cudaEvent_t* e_in = ctx->events.data() + 1;
    cudaEvent_t* e_conv = ctx->events.data() + 1 + K;
    cudaEvent_t* e_out = ctx->events.data() + 1 + 2 * K;  // K + 1: each chunk's outputs, then the rest
    float* d_in = apr->h_in.as<float>();
    float* d_tree = apr->h_tree.as<float>();
    float* d_out = apr->h_out.as<float>();
    const aprgpu::DevAccess& L = apr->leaf;
    const aprgpu::DevAccess& T = apr->tree;
    const int tlo = std::max(P.lc, T.l_min);
    const int ntl = nt ? std::max(T.l_max - tlo + 1, 0) : 0;
    // the host side of the copies: the caller's buffers, or the pinned staging
    const float* h_val = values;
    const float* h_tree = tree_values;
    float* h_out = out;
    if (staged) {
        if (ctx->stage_bytes < stage_need) {
            if (ctx->stage) cudaFreeHost(ctx->stage);
            ctx->stage = nullptr;
            ctx->stage_bytes = 0;
            APR_CUDA(cudaHostAlloc(&ctx->stage, stage_need, cudaHostAllocDefault));
            ctx->stage_bytes = stage_need;
        }
        if (!ctx->pool) {
            const int hc = static_cast<int>(std::thread::hardware_concurrency());
            ctx->pool = new aprgpu::HostPool(std::max(1, env_int("APRGPU_HOST_THREADS", std::min(8, std::max(1, hc / 2)))));
        }
        float* st = static_cast<float*>(ctx->stage);
        if (st_val) h_val = st;
        if (st_tree) h_tree = st + np;
        if (st_out) h_out = st + np + nt;
    }
    // few, large copies: the finest level's rows carry ~90 % of the particles,
    // so chunk 0 takes every coarser level whole and each later chunk one
    // contiguous range of the finest level (leaf and interior alike); outputs
    // come back per chunk for the two finest levels, the rest at the end
    auto LB = [&](int l, int jj) { return P.leaf_b[(l - P.lc) * (K + 1) + jj]; };
    auto TB = [&](int jj) { return P.tree_b[(ntl - 1) * (K + 1) + jj]; };
    struct Range {
        int arr;  // 0 leaf values, 1 tree values, 2 outputs
        uint64_t b, e;
    };
    std::vector<std::vector<Range>> in_r(K), out_r(K + 1);
    const bool two = L.l_max - 1 >= P.lc;
    for (int j = 0; j < K; ++j) {
        in_r[j].push_back({0, j ? LB(L.l_max, j) : 0, LB(L.l_max, j + 1)});
        if (nt) {
            if (ntl) in_r[j].push_back({1, j ? TB(j) : 0, TB(j + 1)});
            else if (j == 0) in_r[j].push_back({1, 0, nt});
        }
        out_r[j].push_back({2, LB(L.l_max, j), LB(L.l_max, j + 1)});
        if (two) out_r[j].push_back({2, LB(L.l_max - 1, j), LB(L.l_max - 1, j + 1)});
    }
    out_r[K].push_back({2, 0, two ? LB(L.l_max - 1, 0) : LB(L.l_max, 0)});
    // staged: the host copies, as pieces of <= 1 MB in chunk order
    struct Piece {
        float* dst;
        const float* src;
        size_t n;
        int chunk;
    };
    std::vector<Piece> pin, pout;
    std::vector<std::atomic<int>> left(K);
    if (staged) {
        constexpr size_t kPiece = 1 << 18;  // floats
        auto cut = [&](std::vector<Piece>& v, float* dst, const float* src, uint64_t b, uint64_t e, int c) {
            for (uint64_t x = b; x < e; x += kPiece) v.push_back({dst + x, src + x, std::min<uint64_t>(kPiece, e - x), c});
        };
        for (int j = 0; j < K; ++j) {
            const size_t n0 = pin.size();
            for (const Range& r : in_r[j])
                if (r.arr == 0 ? st_val : st_tree)
                    cut(pin, const_cast<float*>(r.arr == 0 ? h_val : h_tree), r.arr == 0 ? values : tree_values, r.b,
                        r.e, j);
            left[j].store(static_cast<int>(pin.size() - n0));
        }
        if (st_out)
            for (int j = 0; j <= K; ++j)
                for (const Range& r : out_r[j]) cut(pout, out, h_out, r.b, r.e, j);
    }
    std::atomic<size_t> next{0};
    struct Join {  // an error below must not leave the workers on this frame's pieces
        aprgpu::HostPool* p;
        ~Join() {
            if (p) p->wait();
        }
    } join{staged ? ctx->pool : nullptr};
    if (staged)
        ctx->pool->start([&] {
            for (size_t i; (i = next.fetch_add(1)) < pin.size();) {
                std::memcpy(pin[i].dst, pin[i].src, 4 * pin[i].n);
                left[pin[i].chunk].fetch_sub(1, std::memory_order_release);
            }
        });
    APR_CUDA(cudaEventRecord(start, s));
    APR_CUDA(cudaStreamWaitEvent(ctx->copy_in, start, 0));
    APR_CUDA(cudaStreamWaitEvent(ctx->copy_out, start, 0));
    aprgpu::EpiArgs epi;
    auto conv = [&](int j) {  // chunk j's tiles (inputs <= j+1 landed), then its outputs back
        APR_CUDA(cudaStreamWaitEvent(s, e_in[std::min(j + 1, K - 1)], 0));
        aprgpu::Slab slab;
        slab.lc = P.lc;
        slab.z_lo = j * P.S;
        slab.z_hi = j == K - 1 ? (1 << 30) : (j + 1) * P.S;
        aprgpu::convolve_device(apr, d_in, d_tree, pyr, pad, accum, d_out, epi, s, slab);
        APR_CUDA(cudaEventRecord(e_conv[j], s));
        APR_CUDA(cudaStreamWaitEvent(ctx->copy_out, e_conv[j], 0));
        for (const Range& r : out_r[j])
            if (r.e > r.b)
                APR_CUDA(cudaMemcpyAsync(h_out + r.b, d_out + r.b, 4 * (r.e - r.b), cudaMemcpyDeviceToHost, ctx->copy_out));
        APR_CUDA(cudaEventRecord(e_out[j], ctx->copy_out));
    };
    for (int j = 0; j < K; ++j) {
        if (staged)
            while (left[j].load(std::memory_order_acquire) > 0) std::this_thread::yield();
        for (const Range& r : in_r[j]) {
            float* d = r.arr == 0 ? d_in : d_tree;
            const float* h = r.arr == 0 ? h_val : h_tree;
            if (r.e > r.b)
                APR_CUDA(cudaMemcpyAsync(d + r.b, h + r.b, 4 * (r.e - r.b), cudaMemcpyHostToDevice, ctx->copy_in));
        }
        APR_CUDA(cudaEventRecord(e_in[j], ctx->copy_in));
        if (j >= 1) conv(j - 1);
    }
    conv(K - 1);
    for (const Range& r : out_r[K])
        if (r.e > r.b)
            APR_CUDA(cudaMemcpyAsync(h_out + r.b, d_out + r.b, 4 * (r.e - r.b), cudaMemcpyDeviceToHost, ctx->copy_out));
    APR_CUDA(cudaEventRecord(e_out[K], ctx->copy_out));
    if (staged) {  // outputs out of the staging, chunk by chunk as they land
        ctx->pool->wait();
        next.store(0);
        std::atomic<int> bad{0};
        ctx->pool->start([&] {
            for (size_t i; (i = next.fetch_add(1)) < pout.size();) {
                if (cudaEventSynchronize(e_out[pout[i].chunk]) != cudaSuccess) {
                    bad.store(1);
                    continue;
                }
                std::memcpy(pout[i].dst, pout[i].src, 4 * pout[i].n);
            }
        });
        ctx->pool->wait();
        if (bad.load()) fail(APRGPU_ERR_CUDA, "pipelined convolve: a device-to-host copy failed");
    }
    APR_CUDA(cudaStreamSynchronize(ctx->copy_out));
    APR_CUDA(cudaStreamSynchronize(s));
    return true;
}

}  // namespace

extern "C" {

const char* aprgpu_last_error(void) { return g_last_error.c_str(); }

int aprgpu_host_alloc(uint64_t bytes, void** out) {
    return guard([&] {
        need(out != nullptr, "null out");
        *out = nullptr;
        if (bytes) APR_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
    });
}

int aprgpu_host_free(void* p) {
    return guard([&] {
        if (p) APR_CUDA(cudaFreeHost(p));
    });
}
int aprgpu_version(void) { return 1; }

int aprgpu_init(int device, aprgpu_ctx** out) {
    return guard([&] {
        need(out != nullptr, "null out");
        int n = 0;
        APR_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(APRGPU_ERR_RANGE, "no such CUDA device");
        DeviceGuard g(device);
        auto* c = new aprgpu_ctx;
        c->device = device;
        APR_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        APR_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        *out = c;
    });
}

int aprgpu_ctx_free(aprgpu_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        DeviceGuard g(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
        if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
        for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
        delete ctx->pool;
        if (ctx->stage) cudaFreeHost(ctx->stage);
        delete ctx;
    });
}

int aprgpu_ctx_stream(aprgpu_ctx* ctx, void** stream_out) {
    return guard([&] {
        need(ctx && stream_out, "null argument");
        *stream_out = ctx->stream;
    });
}

int aprgpu_launch_count(aprgpu_ctx* ctx, uint64_t* out) {
    return guard([&] {
        need(ctx && out, "null argument");
        *out = ctx->launches.load();
    });
}

int aprgpu_upload_access(aprgpu_ctx* ctx, const aprgpu_access_desc* leaf, const aprgpu_access_desc* tree,
                         const int32_t source_dims[3], aprgpu_apr** out) {
    aprgpu_apr* apr = nullptr;
    int st = guard("aprgpu_upload_access", [&] {
        need(ctx && leaf && source_dims && out, "null argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        DeviceGuard g(ctx->device);
        apr = new aprgpu_apr;
        apr->ctx = ctx;
        for (int i = 0; i < 3; ++i) apr->dims[i] = source_dims[i];
        if (source_dims[2] > 65536) fail(APRGPU_ERR_CAPABILITY, "y dimension exceeds the 16-bit index limit");
        upload_one(ctx, leaf, apr->leaf, true);
        apr->geom_l_max = std::max(apr->leaf.l_max, host_compute_l_max(source_dims[0], source_dims[1], source_dims[2]));
        if (tree) {
            upload_one(ctx, tree, apr->tree, false);
            aprgpu::verify_tree_links(ctx, apr);
        } else {
            aprgpu::build_tree_structure(ctx, apr);
        }
        APR_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = apr;
    });
    if (st != APRGPU_OK && apr) {
        free_apr(apr);
        delete apr;
    }
    return st;
}

// The level grids are the image's (assemble_access geometry), which the
// interior-structure partition check relies on.
bool grids_match(const aprgpu_access_desc* d, const int32_t dims[3]) {
    int lm = 0;
    while ((1 << lm) < std::max(dims[0], std::max(dims[1], dims[2]))) ++lm;
    if (lm != d->l_max) return false;
    for (int l = d->l_min; l <= d->l_max; ++l) {
        const int64_t s = int64_t(1) << (d->l_max - l);
        if (d->z_dim[l] != (dims[0] + s - 1) / s || d->x_dim[l] != (dims[1] + s - 1) / s ||
            d->y_dim[l] != (dims[2] + s - 1) / s)
            return false;
    }
    return true;
}

// validate (apr.hpp:61-134), O(particles + rows) on the device; the reference's
// checks in its order, with its messages.
int aprgpu_validate_access(aprgpu_ctx* ctx, const aprgpu_access_desc* d, const int32_t source_dims[3], int* ok,
                           char* msg, size_t msg_cap) {
    aprgpu_apr* tmp = nullptr;
    int st = guard("aprgpu_validate_access", [&] {
        need(ctx && d && source_dims && ok, "null argument");
        std::string m;
        auto verdict = [&](std::string v) { m = std::move(v); };
        // apr.hpp:62-83 (host: O(levels + rows))
        if (d->l_min > d->l_max) {
            verdict("l_min > l_max");
        } else {
            uint64_t expect = 0;
            for (int l = d->l_min; l <= d->l_max && m.empty(); ++l) {
                if (d->level_offset[l] != expect) verdict("level_offset mismatch at level " + std::to_string(l));
                expect += static_cast<uint64_t>(d->z_dim[l]) * d->x_dim[l];
            }
            if (m.empty() && d->n_rows != expect) verdict("xz_end length does not match level grids");
            uint64_t prev = 0;
            for (uint64_t r = 0; r < d->n_rows && m.empty(); ++r) {
                if (d->xz_end[r] < prev) verdict("xz_end decreases at row " + std::to_string(r));
                prev = d->xz_end[r];
            }
            if (m.empty() && d->n_rows && d->xz_end[d->n_rows - 1] != d->n_particles)
                verdict("xz_end[last] != y_idx length");
            if (m.empty() && !d->n_rows && d->n_particles) verdict("particles present but no rows");
        }
        const uint64_t n_pixels = static_cast<uint64_t>(source_dims[0]) * source_dims[1] * source_dims[2];
        if (m.empty()) {
            std::lock_guard<std::mutex> lk(ctx->mu);
            DeviceGuard g(ctx->device);
            cudaStream_t s = ctx->stream;
            tmp = new aprgpu_apr;
            tmp->ctx = ctx;
            for (int i = 0; i < 3; ++i) tmp->dims[i] = source_dims[i];
            upload_one(ctx, d, tmp->leaf, false);
            // rows (apr.hpp:85-101) and cell origins (:112-116)
            struct Flags {
                unsigned long long first_y, min_unc;
                int overflow, dbl;
            };
            aprgpu::GpuBuf fb;
            fb.ensure(sizeof(Flags));
            const Flags init{~0ull, ~0ull, 0, 0};
            APR_CUDA(cudaMemcpyAsync(fb.p, &init, sizeof(Flags), cudaMemcpyHostToDevice, s));
            Flags* f = fb.as<Flags>();
            aprgpu::validate_rows_device(ctx, tmp->leaf, source_dims, &f->first_y, &f->overflow, s);
            Flags h{};
            APR_CUDA(cudaMemcpyAsync(&h, fb.p, sizeof(Flags), cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            if (h.first_y != ~0ull) {
                const uint64_t i = h.first_y >> 1;
                // the row of particle i: the first row ending after it
                const uint64_t r = static_cast<uint64_t>(
                    std::upper_bound(d->xz_end, d->xz_end + d->n_rows, i) - d->xz_end);
                int l = d->l_max;
                while (l > d->l_min && r < d->level_offset[l]) --l;
                const uint64_t loc = r - d->level_offset[l];
                const int z = static_cast<int>(loc / d->x_dim[l]), x = static_cast<int>(loc % d->x_dim[l]);
                if (h.first_y & 1)
                    verdict("y index out of level grid in level " + std::to_string(l));
                else
                    verdict("non-increasing y in row (" + std::to_string(l) + ", " + std::to_string(z) + ", " +
                            std::to_string(x) + ")");
            } else if (n_pixels == 0) {
                // success (apr.hpp:106)
            } else if (h.overflow) {
                verdict("particle cell outside the image domain");
            } else if (!grids_match(d, source_dims)) {
                // level grids that are not the image's: the reference's cover map, on the device
                aprgpu::validate_cover_device(ctx, tmp->leaf, source_dims, &f->dbl, &f->min_unc, s);
                APR_CUDA(cudaMemcpyAsync(&h, fb.p, sizeof(Flags), cudaMemcpyDeviceToHost, s));
                APR_CUDA(cudaStreamSynchronize(s));
                if (h.dbl)
                    verdict("double coverage: overlapping particle cells");
                else if (h.min_unc != ~0ull)
                    verdict("uncovered pixel at flat index " + std::to_string(h.min_unc));
            } else {
                // partition (apr.hpp:103-131) through the leaves' interior structure
                tmp->geom_l_max = tmp->leaf.l_max;
                aprgpu::build_tree_structure(ctx, tmp);
                aprgpu::tree_partition_check(tmp, &f->dbl, &f->min_unc, s);
                APR_CUDA(cudaMemcpyAsync(&h, fb.p, sizeof(Flags), cudaMemcpyDeviceToHost, s));
                // the coarsest level's own cells: each in-image cell exactly one leaf or node
                const aprgpu::DevAccess& T = tmp->tree;
                const int top = T.n_particles ? T.l_min : d->l_min;
                std::vector<uint16_t> ty;
                std::vector<uint32_t> trb;
                if (T.n_particles && top <= T.l_max) {
                    const uint64_t r0 = T.level_offset[top], nr = static_cast<uint64_t>(T.zd[top]) * T.xd[top];
                    trb.resize(nr + 1);
                    APR_CUDA(cudaMemcpyAsync(trb.data(), T.rb + r0, 4 * (nr + 1), cudaMemcpyDeviceToHost, s));
                    APR_CUDA(cudaStreamSynchronize(s));
                    ty.resize(trb[nr] - trb[0]);
                    if (!ty.empty())
                        APR_CUDA(cudaMemcpy(ty.data(), T.y + trb[0], 2 * ty.size(), cudaMemcpyDeviceToHost));
                }
                APR_CUDA(cudaStreamSynchronize(s));
                const int64_t cs = int64_t(1) << (d->l_max - top);
                const int tzd = static_cast<int>((source_dims[0] + cs - 1) / cs),
                          txd = static_cast<int>((source_dims[1] + cs - 1) / cs),
                          tyd = static_cast<int>((source_dims[2] + cs - 1) / cs);
                for (int z = 0; z < tzd; ++z)
                    for (int x = 0; x < txd; ++x)
                        for (int y = 0; y < tyd; ++y) {
                            int c = 0;
                            if (top >= d->l_min && z < d->z_dim[top] && x < d->x_dim[top]) {
                                const uint64_t r = d->level_offset[top] + static_cast<uint64_t>(z) * d->x_dim[top] + x;
                                const uint64_t b = r ? d->xz_end[r - 1] : 0, e = d->xz_end[r];
                                c += std::binary_search(d->y_idx + b, d->y_idx + e, static_cast<uint16_t>(y)) ? 1 : 0;
                            }
                            if (!trb.empty() && z < T.zd[top] && x < T.xd[top]) {
                                const uint64_t r = static_cast<uint64_t>(z) * T.xd[top] + x;
                                const uint16_t* yb = ty.data() + (trb[r] - trb[0]);
                                const uint16_t* ye = ty.data() + (trb[r + 1] - trb[0]);
                                c += std::binary_search(yb, ye, static_cast<uint16_t>(y)) ? 1 : 0;
                            }
                            if (c > 1) h.dbl = 1;
                            if (c == 0) {
                                const unsigned long long p =
                                    (static_cast<unsigned long long>(z * cs) * source_dims[1] + x * cs) *
                                        source_dims[2] + y * cs;
                                h.min_unc = std::min(h.min_unc, p);
                            }
                        }
                if (h.dbl)
                    verdict("double coverage: overlapping particle cells");
                else if (h.min_unc != ~0ull)
                    verdict("uncovered pixel at flat index " + std::to_string(h.min_unc));
            }
            fb.release();
        }
        *ok = m.empty() ? 1 : 0;
        if (msg && msg_cap) {
            const size_t n = std::min(msg_cap - 1, m.size());
            std::memcpy(msg, m.data(), n);
            msg[n] = '\0';
        }
    });
    if (tmp) {
        free_apr(tmp);
        delete tmp;
    }
    return st;
}

int aprgpu_apr_free(aprgpu_apr* apr) {
    return guard([&] {
        if (!apr) return;
        DeviceGuard g(apr->ctx->device);
        cudaStreamSynchronize(apr->ctx->stream);
        free_apr(apr);
        delete apr;
    });
}

int aprgpu_apr_dims(const aprgpu_apr* apr, int32_t dims_out[3]) {
    return guard([&] {
        need(apr && dims_out, "null argument");
        for (int i = 0; i < 3; ++i) dims_out[i] = apr->dims[i];
    });
}

int aprgpu_access_get_info(const aprgpu_apr* apr, int which, aprgpu_access_info* out) {
    return guard([&] {
        need(apr && out, "null argument");
        need(which == APRGPU_LEAF || which == APRGPU_TREE, "bad access selector");
        const aprgpu::DevAccess& a = which == APRGPU_LEAF ? apr->leaf : apr->tree;
        out->l_min = a.l_min;
        out->l_max = a.l_max;
        out->n_particles = a.n_particles;
        out->n_rows = a.n_rows;
    });
}

int aprgpu_apr_map_tiles(const aprgpu_apr* apr, uint64_t* built, uint64_t* n_tiles) {
    return guard([&] {
        need(apr && built && n_tiles, "null argument");
        std::lock_guard<std::mutex> lk(apr->ctx->mu);
        const aprgpu::DevAccess& L = apr->leaf;
        uint64_t b = 0;
        for (int h = 0; h < 2; ++h)
            for (int pm = 0; pm < 2; ++pm)
                for (int l = 0; l < aprgpu::kMaxLevels; ++l)
                    if (const auto* w = L.tile_map[h][pm][l]) b += w->a1 - w->a0;
        *built = b;
        *n_tiles = L.tile_off.empty() ? 0 : L.tile_off.back();
    });
}

int aprgpu_apr_restrict(aprgpu_apr* apr, int cut_level, int32_t z_lo, int32_t z_hi) {
    return guard([&] {
        need(apr != nullptr, "null argument");
        need(z_lo <= z_hi, "aprgpu_apr_restrict: empty plane range");
        std::lock_guard<std::mutex> lk(apr->ctx->mu);
        const aprgpu::DevAccess& L = apr->leaf;
        bool built = L.tile_meta != nullptr || L.tile_runs[0] || L.tile_runs[1];
        for (int h = 0; h < 2; ++h)
            for (int pm = 0; pm < 2; ++pm)
                for (int l = 0; l < aprgpu::kMaxLevels; ++l) built = built || L.tile_map[h][pm][l];
        if (built) aprgpu::fail(APRGPU_ERR_RANGE, "aprgpu_apr_restrict: call before the first convolution");
        apr->tile_slab.lc = cut_level;
        apr->tile_slab.z_lo = z_lo;
        apr->tile_slab.z_hi = z_hi;
    });
}

int aprgpu_download_access(const aprgpu_apr* apr, int which, uint16_t* y_idx, uint64_t* xz_end,
                           uint64_t* level_offset, int32_t* z_dim, int32_t* x_dim, int32_t* y_dim) {
    return guard("aprgpu_download_access", [&] {
        need(apr != nullptr, "null argument");
        need(which == APRGPU_LEAF || which == APRGPU_TREE, "bad access selector");
        DeviceGuard g(apr->ctx->device);
        const aprgpu::DevAccess& a = which == APRGPU_LEAF ? apr->leaf : apr->tree;
        cudaStream_t s = apr->ctx->stream;
        if (y_idx && a.n_particles) APR_CUDA(cudaMemcpyAsync(y_idx, a.y, 2 * a.n_particles, cudaMemcpyDeviceToHost, s));
        if (xz_end && a.n_rows) {
            std::vector<uint32_t> rb(a.n_rows + 1);
            APR_CUDA(cudaMemcpyAsync(rb.data(), a.rb, 4 * (a.n_rows + 1), cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            for (uint64_t r = 0; r < a.n_rows; ++r) xz_end[r] = rb[r + 1];
        }
        APR_CUDA(cudaStreamSynchronize(s));
        for (int l = 0; l <= a.l_max; ++l) {
            if (level_offset) level_offset[l] = a.level_offset[l];
            if (z_dim) z_dim[l] = a.zd[l];
            if (x_dim) x_dim[l] = a.xd[l];
            if (y_dim) y_dim[l] = a.yd[l];
        }
    });
}

int aprgpu_row_index(const aprgpu_apr* apr, int level, int32_t* z, int32_t* x, uint16_t* y_min, uint16_t* y_max,
                     uint64_t cap, uint64_t* count) {
    return guard("aprgpu_row_index", [&] {
        need(apr && count, "null argument");
        const aprgpu::DevAccess& a = apr->leaf;
        if (level < a.l_min || level > a.l_max) fail(APRGPU_ERR_RANGE, "row_index: level out of range");
        DeviceGuard g(apr->ctx->device);
        *count = a.work_off[level + 1] - a.work_off[level];
        if (z && x && y_min && y_max && cap) aprgpu::row_spans(apr->ctx, a, level, z, x, y_min, y_max, cap);
    });
}

int aprgpu_rebuild_index(aprgpu_apr* apr, void* stream) {
    return guard("aprgpu_rebuild_index", [&] {
        need(apr, "null argument");
        DeviceGuard g(apr->ctx->device);
        cudaStream_t s = aprgpu::pick_stream(apr->ctx, stream);
        // (its own scratch: the index step may overlap fill_tree on another stream)
        ScratchGuard sg(apr->index_mu, apr->index_ev, s);
        aprgpu::rebuild_index_device(apr, s);
    });
}

int aprgpu_fill_tree(aprgpu_apr* apr, const float* leaf, float* tree, int ptr_kind, void* stream) {
    return guard("aprgpu_fill_tree", [&] {
        need(apr && leaf && (tree || apr->tree.n_particles == 0), "null argument");
        DeviceGuard g(apr->ctx->device);
        cudaStream_t s = aprgpu::pick_stream(apr->ctx, stream);
        const uint64_t np = apr->leaf.n_particles, nt = apr->tree.n_particles;
        ScratchGuard sg(apr, s);
        if (ptr_kind == APRGPU_DEVICE) {
            aprgpu::fill_tree_device(apr, leaf, tree, s);
            return;
        }
        need(ptr_kind == APRGPU_HOST, "bad pointer kind");
        apr->h_in.ensure(4 * np + 4);
        apr->h_tree.ensure(4 * nt + 4);
        APR_CUDA(cudaMemcpyAsync(apr->h_in.p, leaf, 4 * np, cudaMemcpyHostToDevice, s));
        aprgpu::fill_tree_device(apr, apr->h_in.as<float>(), apr->h_tree.as<float>(), s);
        if (nt) APR_CUDA(cudaMemcpyAsync(tree, apr->h_tree.p, 4 * nt, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
    });
}

int aprgpu_restrict_stencil(const float* w, int kz, int kx, int ky, int delta, int32_t out_k3[3], float* out) {
    return guard([&] {
        need(out_k3 != nullptr, "null argument");
        const aprgpu::HostStencil r = aprgpu::restrict_stencil_host(make_host_stencil(w, kz, kx, ky), delta);
        out_k3[0] = r.kz;
        out_k3[1] = r.kx;
        out_k3[2] = r.ky;
        if (out) std::memcpy(out, r.w.data(), sizeof(float) * r.w.size());
    });
}

int aprgpu_gaussian_stencil(double sigma, int size, int32_t* k_out, float* out) {
    return guard([&] {
        const aprgpu::HostStencil s = aprgpu::gaussian_stencil_host(sigma, size);
        if (k_out) *k_out = s.kz;
        if (out) std::memcpy(out, s.w.data(), sizeof(float) * s.w.size());
    });
}

int aprgpu_box_stencil(int k, float* out) {
    return guard([&] {
        if (k < 1 || k % 2 == 0) fail(APRGPU_ERR_RANGE, "stencil extents must be odd and positive");
        need(out != nullptr, "null argument");
        const float v = 1.0f / static_cast<float>(k) / k / k;  // stencil.hpp:52-55
        for (int i = 0; i < k * k * k; ++i) out[i] = v;
    });
}

int aprgpu_sobel_stencil(int axis, float* out) {
    return guard([&] {
        if (axis < 0 || axis > 2) fail(APRGPU_ERR_RANGE, "sobel axis must be 0, 1 or 2");
        need(out != nullptr, "null argument");
        static const double smooth[3] = {0.25, 0.5, 0.25};
        static const double diff[3] = {-0.5, 0.0, 0.5};
        for (int a = 0; a < 3; ++a)  // stencil.hpp:83-98
            for (int b = 0; b < 3; ++b)
                for (int c = 0; c < 3; ++c) {
                    const double wz = axis == 0 ? diff[a] : smooth[a];
                    const double wx = axis == 1 ? diff[b] : smooth[b];
                    const double wy = axis == 2 ? diff[c] : smooth[c];
                    out[(a * 3 + b) * 3 + c] = static_cast<float>(wz * wx * wy);
                }
    });
}

int aprgpu_sequential_sum(aprgpu_ctx* ctx, const float* values, uint64_t n, int ptr_kind, double* out, void* stream) {
    return guard("aprgpu_sequential_sum", [&] {
        need(ctx && out && (values || n == 0), "null argument");
        need(ptr_kind == APRGPU_HOST || ptr_kind == APRGPU_DEVICE, "bad pointer kind");
        DeviceGuard g(ctx->device);
        cudaStream_t s = aprgpu::pick_stream(ctx, stream);
        aprgpu::GpuBuf staged, scratch;
        const float* u = values;
        if (ptr_kind == APRGPU_HOST && n) {
            staged.ensure(4 * n);
            APR_CUDA(cudaMemcpyAsync(staged.p, values, 4 * n, cudaMemcpyHostToDevice, s));
            u = staged.as<float>();
        }
        if (n) {  // the same check as rl_apr's (non-negative, finite)
            scratch.ensure(64);
            MeanStats* ms = scratch.as<MeanStats>();
            APR_CUDA(cudaMemsetAsync(ms, 0, sizeof(MeanStats), s));
            const unsigned grid = std::min<unsigned>(aprgpu::blocks_for(n, 256), ctx->sm_count * 8);
            k_mean_bound<<<grid, 256, 0, s>>>(u, n, ms);
            aprgpu::count_launch(ctx);
            MeanStats h{};
            APR_CUDA(cudaMemcpyAsync(&h, ms, sizeof(MeanStats), cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            if (h.nonfinite) fail(APRGPU_ERR_RANGE, "aprgpu_sequential_sum: non-finite value");
            k_min_check<<<grid, 256, 0, s>>>(u, n, ms);
            aprgpu::count_launch(ctx);
            APR_CUDA(cudaMemcpyAsync(&h, ms, sizeof(MeanStats), cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            if (h.nonfinite) fail(APRGPU_ERR_RANGE, "aprgpu_sequential_sum: negative value");
        }
        *out = aprgpu::sequential_sum_device(ctx, u, n, scratch, s);
    });
}

int aprgpu_pyramid_create(aprgpu_ctx* ctx, const float* w, int kz, int kx, int ky, int l_min, int l_max, int mode,
                          aprgpu_pyramid** out) {
    aprgpu_pyramid* p = nullptr;
    int st = guard([&] {
        need(ctx && out, "null argument");
        need(l_min >= 0 && l_min <= l_max && l_max < aprgpu::kMaxLevels, "bad level range");
        const aprgpu::HostStencil base = make_host_stencil(w, kz, kx, ky);
        p = new aprgpu_pyramid;
        p->ctx = ctx;
        p->l_min = l_min;
        p->l_max = l_max;
        p->mode = mode;
        for (int l = l_min; l <= l_max; ++l) {  // make_pyramid, stencil.hpp:176-191
            const int delta = l_max - l;
            if (mode == APRGPU_PYR_RESTRICTED) {
                push_level(p, aprgpu::restrict_stencil_host(base, delta));
            } else if (mode == APRGPU_PYR_RESCALED) {
                aprgpu::HostStencil r = base;  // rescale_stencil, stencil.hpp:114-120
                const float scale = std::ldexp(1.0f, -delta);
                for (float& v : r.w) v *= scale;
                push_level(p, r);
            } else if (mode == APRGPU_PYR_UNIFORM || mode == APRGPU_PYR_EXPLICIT) {
                push_level(p, base);
            } else {
                fail(APRGPU_ERR_INVALID, "unknown pyramid mode");
            }
        }
        pyramid_upload(p);
        *out = p;
    });
    if (st != APRGPU_OK && p) aprgpu_pyramid_free(p);
    return st;
}

int aprgpu_pyramid_create_explicit(aprgpu_ctx* ctx, const float* w, const int32_t* k3, int l_min, int l_max,
                                   aprgpu_pyramid** out) {
    aprgpu_pyramid* p = nullptr;
    int st = guard([&] {
        need(ctx && w && k3 && out, "null argument");
        need(l_min >= 0 && l_min <= l_max && l_max < aprgpu::kMaxLevels, "bad level range");
        p = new aprgpu_pyramid;
        p->ctx = ctx;
        p->l_min = l_min;
        p->l_max = l_max;
        p->mode = APRGPU_PYR_EXPLICIT;
        size_t off = 0;
        for (int l = l_min; l <= l_max; ++l) {
            const int32_t* k = k3 + 3 * (l - l_min);
            aprgpu::HostStencil s = make_host_stencil(w + off, k[0], k[1], k[2]);
            off += s.w.size();
            push_level(p, s);
        }
        pyramid_upload(p);
        *out = p;
    });
    if (st != APRGPU_OK && p) aprgpu_pyramid_free(p);
    return st;
}

int aprgpu_pyramid_free(aprgpu_pyramid* p) {
    return guard([&] {
        if (!p) return;
        cudaFree(p->w_dev);
        cudaFree(p->wd_dev);
        cudaFree(p->sep_dev);
        delete p;
    });
}

int aprgpu_pyramid_level(const aprgpu_pyramid* p, int level, int32_t k3[3], float* w) {
    return guard([&] {
        need(p && k3, "null argument");
        if (level < p->l_min || level > p->l_max) fail(APRGPU_ERR_RANGE, "StencilPyramid: level out of range");
        const int li = level - p->l_min;
        for (int i = 0; i < 3; ++i) k3[i] = p->k3[3 * li + i];
        if (w) {
            const size_t n = static_cast<size_t>(k3[0]) * k3[1] * k3[2];
            std::memcpy(w, p->w_host.data() + p->off[li], sizeof(float) * n);
        }
    });
}

int aprgpu_convolve(aprgpu_apr* apr, const float* values, const float* tree_values, const aprgpu_pyramid* pyr,
                    int pad_mode, int accum, float* out, int ptr_kind, void* stream) {
    return guard("aprgpu_convolve", [&] {
        need(apr && values && pyr && out, "null argument");
        need(tree_values || apr->tree.n_particles == 0, "tree values are required");
        need(pad_mode == APRGPU_PAD_ZERO || pad_mode == APRGPU_PAD_REFLECT, "bad pad mode");
        need(accum == APRGPU_ACCUM_EXACT || accum == APRGPU_ACCUM_FAST, "bad accumulation mode");
        need(pyr->ctx == apr->ctx, "pyramid belongs to another context");
        DeviceGuard g(apr->ctx->device);
        aprgpu::check_pyramid(apr, pyr);
        cudaStream_t s = aprgpu::pick_stream(apr->ctx, stream);
        const uint64_t np = apr->leaf.n_particles, nt = apr->tree.n_particles;
        aprgpu::EpiArgs epi;
        if (ptr_kind == APRGPU_DEVICE) {
            aprgpu::convolve_device(apr, values, tree_values, pyr, pad_mode, accum, out, epi, s);
            return;
        }
        need(ptr_kind == APRGPU_HOST, "bad pointer kind");
        ScratchGuard sg(apr, s);
        apr->h_in.ensure(4 * np + 4);
        apr->h_tree.ensure(4 * nt + 4);
        apr->h_out.ensure(4 * np + 4);
        if (convolve_host_pipelined(apr, values, tree_values, pyr, pad_mode, accum, out, s)) return;
        APR_CUDA(cudaMemcpyAsync(apr->h_in.p, values, 4 * np, cudaMemcpyHostToDevice, s));
        if (nt) APR_CUDA(cudaMemcpyAsync(apr->h_tree.p, tree_values, 4 * nt, cudaMemcpyHostToDevice, s));
        aprgpu::convolve_device(apr, apr->h_in.as<float>(), apr->h_tree.as<float>(), pyr, pad_mode, accum,
                                apr->h_out.as<float>(), epi, s);
        APR_CUDA(cudaMemcpyAsync(out, apr->h_out.p, 4 * np, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

namespace {
// Shared body of the reconstruction entry points: host pointers are staged
// through device buffers (values, tree values, the output volume).
template <typename F>
void reconstruct_call(aprgpu_apr* apr, const float* values, const float* tree_values, float* out, uint64_t cells,
                      int ptr_kind, void* stream, F run) {
    need(apr && values && out, "null argument");
    need(ptr_kind == APRGPU_HOST || ptr_kind == APRGPU_DEVICE, "bad pointer kind");
    DeviceGuard g(apr->ctx->device);
    cudaStream_t s = aprgpu::pick_stream(apr->ctx, stream);
    if (ptr_kind == APRGPU_DEVICE) {
        run(values, tree_values, out, s);
        return;
    }
    const uint64_t np = apr->leaf.n_particles, nt = apr->tree.n_particles;
    ScratchGuard sg(apr, s);
    apr->h_in.ensure(4 * np + 4);
    APR_CUDA(cudaMemcpyAsync(apr->h_in.p, values, 4 * np, cudaMemcpyHostToDevice, s));
    const float* tv = nullptr;
    if (tree_values && nt) {
        apr->h_tree.ensure(4 * nt + 4);
        APR_CUDA(cudaMemcpyAsync(apr->h_tree.p, tree_values, 4 * nt, cudaMemcpyHostToDevice, s));
        tv = apr->h_tree.as<float>();
    }
    aprgpu::GpuBuf dev_out;
    dev_out.ensure(4 * cells + 4);
    run(apr->h_in.as<float>(), tv, dev_out.as<float>(), s);
    APR_CUDA(cudaMemcpyAsync(out, dev_out.p, 4 * cells, cudaMemcpyDeviceToHost, s));
    APR_CUDA(cudaStreamSynchronize(s));
    dev_out.release();
}
}  // namespace

extern "C" {

int aprgpu_reconstruct_level(aprgpu_apr* apr, const float* values, const float* tree_values, int level, float* out,
                             int ptr_kind, void* stream) {
    return guard("aprgpu_reconstruct_level", [&] {
        need(apr != nullptr, "null argument");
        const aprgpu::DevAccess& L = apr->leaf;
        if (level < L.l_min || level > L.l_max) aprgpu::fail(APRGPU_ERR_RANGE, "reconstruct_level: level out of range");
        const uint64_t cells = static_cast<uint64_t>(L.zd[level]) * L.xd[level] * L.yd[level];
        reconstruct_call(apr, values, tree_values, out, cells, ptr_kind, stream,
                         [&](const float* v, const float* tv, float* o, cudaStream_t s) {
                             aprgpu::reconstruct_level_device(apr, v, tv, level, o, s);
                         });
    });
}

int aprgpu_reconstruct_patch(aprgpu_apr* apr, const float* values, const float* tree_values,
                             const aprgpu_patch_spec* spec, float* out, int ptr_kind, void* stream) {
    return guard("aprgpu_reconstruct_patch", [&] {
        need(apr && spec, "null argument");
        const aprgpu::DevAccess& L = apr->leaf;
        const int l = spec->level;
        if (l < L.l_min || l > L.l_max) aprgpu::fail(APRGPU_ERR_RANGE, "reconstruct_patch: level out of range");
        if (spec->z_begin < 0 || spec->z_end > L.zd[l] || spec->x_begin < 0 || spec->x_end > L.xd[l] ||
            spec->z_begin > spec->z_end || spec->x_begin > spec->x_end || spec->pad < 0)
            aprgpu::fail(APRGPU_ERR_RANGE, "reconstruct_patch: spec outside the level grid");
        const uint64_t cells = static_cast<uint64_t>(spec->z_end - spec->z_begin + 2 * spec->pad) *
                               (spec->x_end - spec->x_begin + 2 * spec->pad) * (L.yd[l] + 2 * spec->pad);
        reconstruct_call(apr, values, tree_values, out, cells, ptr_kind, stream,
                         [&](const float* v, const float* tv, float* o, cudaStream_t s) {
                             aprgpu::reconstruct_patch_device(apr, v, tv, *spec, o, s);
                         });
    });
}

int aprgpu_rl(aprgpu_apr* apr, const float* observed, const float* psf, int kz, int kx, int ky, int iterations,
              double epsilon, int accum, float* out, int ptr_kind, void* stream) {
    return aprgpu_rl_resume(apr, observed, nullptr, psf, kz, kx, ky, iterations, epsilon, accum, out, ptr_kind,
                            stream);
}

int aprgpu_rl_resume(aprgpu_apr* apr, const float* observed, const float* estimate_in, const float* psf, int kz,
                     int kx, int ky, int iterations, double epsilon, int accum, float* out, int ptr_kind,
                     void* stream) {
    return guard("aprgpu_rl_resume", [&] {
        need(apr && observed && psf && out, "null argument");
        need(ptr_kind == APRGPU_HOST || ptr_kind == APRGPU_DEVICE, "bad pointer kind");
        need(accum == APRGPU_ACCUM_EXACT || accum == APRGPU_ACCUM_FAST, "bad accumulation mode");
        DeviceGuard g(apr->ctx->device);
        aprgpu_ctx* ctx = apr->ctx;
        cudaStream_t s = aprgpu::pick_stream(ctx, stream);
        ScratchGuard sg(apr, s);
        // normalized_psf (deconv.hpp:26-34)
        aprgpu::HostStencil w = make_host_stencil(psf, kz, kx, ky);
        for (float v : w.w)
            if (v < 0.0f) fail(APRGPU_ERR_RANGE, "RL psf weights must be non-negative");
        double sum = 0.0;
        for (float v : w.w) sum += v;
        if (sum <= 0.0) fail(APRGPU_ERR_RANGE, "RL psf must have positive sum");
        for (float& v : w.w) v = static_cast<float>(v / sum);
        aprgpu::HostStencil wt = w;  // flip_stencil, stencil.hpp:101-110
        for (int a = 0; a < kz; ++a)
            for (int b = 0; b < kx; ++b)
                for (int c = 0; c < ky; ++c)
                    wt.w[(static_cast<size_t>(kz - 1 - a) * kx + (kx - 1 - b)) * ky + (ky - 1 - c)] =
                        w.w[(static_cast<size_t>(a) * kx + b) * ky + c];
        const int l_min = apr->leaf.l_min, l_max = apr->leaf.l_max;
        aprgpu_pyramid *pw = nullptr, *pwt = nullptr;
        int st = aprgpu_pyramid_create(ctx, w.w.data(), kz, kx, ky, l_min, l_max, APRGPU_PYR_RESTRICTED, &pw);
        if (st) fail(st, g_last_error);
        st = aprgpu_pyramid_create(ctx, wt.w.data(), kz, kx, ky, l_min, l_max, APRGPU_PYR_RESTRICTED, &pwt);
        if (st) {
            aprgpu_pyramid_free(pw);
            fail(st, g_last_error);
        }
        const uint64_t np = apr->leaf.n_particles, nt = apr->tree.n_particles;
        // clamped observations u and the running estimate
        apr->rl_u.ensure(4 * np + 4);
        apr->rl_ratio.ensure(4 * np + 4);
        apr->rl_tv.ensure(4 * nt + 4);
        apr->h_out.ensure(4 * np + 4);
        std::vector<float> host_obs;
        const float* obs_dev = observed;
        if (ptr_kind == APRGPU_HOST) {
            apr->h_in.ensure(4 * np + 4);
            APR_CUDA(cudaMemcpyAsync(apr->h_in.p, observed, 4 * np, cudaMemcpyHostToDevice, s));
            obs_dev = apr->h_in.as<float>();
        }
        float* est = ptr_kind == APRGPU_DEVICE ? out : apr->h_out.as<float>();
        float* u = apr->rl_u.as<float>();
        // resume: the running estimate replaces the clamped observation, so the
        // clamp writes u only (estimate_in may be out itself: an in-place resume)
        k_clamp_copy<<<std::min<unsigned>(aprgpu::blocks_for(np, 256), ctx->sm_count * 8), 256, 0, s>>>(
            obs_dev, u, estimate_in ? nullptr : est, np);
        aprgpu::count_launch(ctx);
        APR_CUDA(cudaGetLastError());
        if (estimate_in && estimate_in != est)
            APR_CUDA(cudaMemcpyAsync(est, estimate_in, 4 * np,
                                     ptr_kind == APRGPU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
        // mean of the clamped observations in the reference's sequential order
        // (deconv.hpp:90-92).  When every partial sum of that double loop is
        // provably exact (all values are multiples of 2^g and sum|v| < 2^(53+g))
        // the sequential sum IS the exact sum, computed on the device as an
        // order-free int64 sum of v / 2^g; otherwise the loop is replayed on the
        // device (seqsum.cu), bit for bit.
        double mean = 0.0;
        if (epsilon <= 0.0) {
            apr->tmp.ensure(64);
            MeanStats* ms = apr->tmp.as<MeanStats>();
            APR_CUDA(cudaMemsetAsync(ms, 0, sizeof(MeanStats), s));
            const unsigned grid = std::min<unsigned>(aprgpu::blocks_for(np, 256), ctx->sm_count * 8);
            k_mean_bound<<<grid, 256, 0, s>>>(u, np, ms);
            k_mean_exact<<<grid, 256, 0, s>>>(u, np, ms);
            aprgpu::count_launch(ctx, 2);
            MeanStats h{};
            APR_CUDA(cudaMemcpyAsync(&h, ms, sizeof(MeanStats), cudaMemcpyDeviceToHost, s));
            APR_CUDA(cudaStreamSynchronize(s));
            const int g = kNoLowBit - h.neg_gexp_max;  // smallest low-bit exponent of the values
            const bool exact = !h.nonfinite && (np == 0 || h.neg_gexp_max == 0 ||
                                                h.abs_sum < std::ldexp(1.0, 53 + g) * 0.999999);
            if (exact) {
                mean = h.neg_gexp_max == 0 ? 0.0 : std::ldexp(static_cast<double>(static_cast<int64_t>(h.isum)), g);
            } else if (!h.nonfinite) {
                // the partial sums round: the loop replayed on the device (seqsum.cu)
                aprgpu::GpuBuf scratch;
                mean = aprgpu::sequential_sum_device(ctx, u, np, scratch, s);
            } else {  // (NaN / inf observations: the loop on the host)
                host_obs.resize(np);
                APR_CUDA(cudaMemcpyAsync(host_obs.data(), u, 4 * np, cudaMemcpyDeviceToHost, s));
                APR_CUDA(cudaStreamSynchronize(s));
                for (float v : host_obs) mean += v;
            }
            mean /= static_cast<double>(std::max<uint64_t>(np, 1));
        }
        const double eps = epsilon > 0.0 ? epsilon : 1e-6 * std::max(mean, 1e-30);  // rl_epsilon, deconv.hpp:36-38
        float* ratio = apr->rl_ratio.as<float>();
        float* tv = apr->rl_tv.as<float>();
        auto iteration = [&] {
            aprgpu::fill_tree_device(apr, est, tv, s);
            aprgpu::EpiArgs e1;
            e1.mode = aprgpu::EPI_RL_RATIO;
            e1.u = u;
            e1.eps = eps;
            aprgpu::convolve_device(apr, est, tv, pw, APRGPU_PAD_REFLECT, accum, ratio, e1, s);
            aprgpu::fill_tree_device(apr, ratio, tv, s);
            aprgpu::EpiArgs e2;
            e2.mode = aprgpu::EPI_RL_MULT;
            e2.est = est;
            aprgpu::convolve_device(apr, ratio, tv, pwt, APRGPU_PAD_REFLECT, accum, nullptr, e2, s);
        };
        // The first iteration runs eagerly (it builds the lazily cached maps,
        // links and attributes); the rest replay it as one CUDA graph (~24
        // kernels per iteration, no launch gaps).  APRGPU_RL_GRAPH=0: eager.
        const char* ge = std::getenv("APRGPU_RL_GRAPH");
        const bool use_graph = !(ge && ge[0] == '0') && s != nullptr;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        uint64_t graph_kernels = 0;  // our kernels per replay
        try {
            for (int k = 1; k <= iterations; ++k) {
                if (k == 1 || !use_graph) {
                    iteration();
                    continue;
                }
                if (!exec) {
                    const uint64_t l0 = ctx->launches.load();
                    APR_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                    try {
                        iteration();
                    } catch (...) {
                        cudaStreamEndCapture(s, &graph);
                        throw;
                    }
                    APR_CUDA(cudaStreamEndCapture(s, &graph));
                    APR_CUDA(cudaGraphInstantiate(&exec, graph, 0));
                    graph_kernels = ctx->launches.load() - l0;  // captured, not run: counted per replay
                    ctx->launches.fetch_sub(graph_kernels);
                }
                APR_CUDA(cudaGraphLaunch(exec, s));
                aprgpu::count_launch(ctx, graph_kernels);
            }
        } catch (...) {
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
            aprgpu_pyramid_free(pw);
            aprgpu_pyramid_free(pwt);
            throw;
        }
        if (exec) APR_CUDA(cudaGraphExecDestroy(exec));
        if (graph) APR_CUDA(cudaGraphDestroy(graph));
        if (ptr_kind == APRGPU_HOST) APR_CUDA(cudaMemcpyAsync(out, est, 4 * np, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
        aprgpu_pyramid_free(pw);
        aprgpu_pyramid_free(pwt);
    });
}

int aprgpu_fill_tree_sums(aprgpu_apr* apr, const float* leaf, int lt_lo, int lt_hi, int z_lo, int z_hi,
                          void* stream) {
    return guard("aprgpu_fill_tree_sums", [&] {
        need(apr && (leaf || apr->leaf.n_particles == 0), "null argument");
        DeviceGuard g(apr->ctx->device);
        aprgpu::fill_tree_sums(apr, leaf, lt_lo, lt_hi, z_lo, z_hi, aprgpu::pick_stream(apr->ctx, stream));
    });
}

int aprgpu_tree_scratch(aprgpu_apr* apr, double** vsum, double** wsum) {
    return guard([&] {
        need(apr && vsum && wsum, "null argument");
        DeviceGuard g(apr->ctx->device);
        const uint64_t nt = apr->tree.n_particles;
        if (!apr->vsum.p || apr->vsum.bytes < sizeof(double) * nt) {
            apr->vsum.ensure(sizeof(double) * nt + 8);
            apr->wsum.ensure(sizeof(double) * nt + 8);
        }
        *vsum = apr->vsum.as<double>();
        *wsum = apr->wsum.as<double>();
    });
}

int aprgpu_fill_tree_finalize(aprgpu_apr* apr, float* tree, void* stream) {
    return guard("aprgpu_fill_tree_finalize", [&] {
        need(apr && (tree || apr->tree.n_particles == 0), "null argument");
        DeviceGuard g(apr->ctx->device);
        aprgpu::fill_tree_finalize(apr, tree, aprgpu::pick_stream(apr->ctx, stream));
    });
}

int aprgpu_convolve_slab(aprgpu_apr* apr, const float* values, const float* tree_values, const aprgpu_pyramid* pyr,
                         int pad_mode, int accum, int lc, int z_lo, int z_hi, float* out, void* stream) {
    return aprgpu_convolve_slab_band(apr, values, tree_values, pyr, pad_mode, accum, lc, z_lo, z_hi, 1, out, stream);
}

int aprgpu_convolve_slab_band(aprgpu_apr* apr, const float* values, const float* tree_values,
                              const aprgpu_pyramid* pyr, int pad_mode, int accum, int lc, int z_lo, int z_hi,
                              int replicated, float* out, void* stream) {
    return guard("aprgpu_convolve_slab_band", [&] {
        need(apr && values && pyr && out, "null argument");
        need(tree_values || apr->tree.n_particles == 0, "tree values are required");
        need(pad_mode == APRGPU_PAD_ZERO || pad_mode == APRGPU_PAD_REFLECT, "bad pad mode");
        need(accum == APRGPU_ACCUM_EXACT || accum == APRGPU_ACCUM_FAST, "bad accumulation mode");
        need(pyr->ctx == apr->ctx, "pyramid belongs to another context");
        need(z_lo >= 0 && z_lo <= z_hi, "bad slab");
        DeviceGuard g(apr->ctx->device);
        aprgpu::Slab slab;
        slab.lc = lc;
        slab.z_lo = z_lo;
        slab.z_hi = z_hi;
        slab.rep = replicated != 0;
        aprgpu::EpiArgs epi;
        aprgpu::convolve_device(apr, values, tree_values, pyr, pad_mode, accum, out, epi,
                                aprgpu::pick_stream(apr->ctx, stream), slab);
    });
}

int aprgpu_generate_spheres(aprgpu_ctx* ctx, int nz, int nx, int ny, int count, double min_radius,
                            double max_radius, double background, double min_intensity, double max_intensity,
                            double blur_sigma, uint64_t seed, float* out, int ptr_kind) {
    return guard("aprgpu_generate_spheres", [&] {
        need(ctx && out, "null argument");
        need(nz > 0 && nx > 0 && ny > 0 && count >= 0, "bad dimensions");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
        if (ptr_kind == APRGPU_DEVICE) {
            aprgpu::generate_spheres_device(ctx, nz, nx, ny, count, min_radius, max_radius, background, min_intensity,
                                            max_intensity, blur_sigma, seed, out, ctx->stream);
            return;
        }
        need(ptr_kind == APRGPU_HOST, "bad pointer kind");
        aprgpu::GpuBuf buf;
        buf.ensure(4 * n);
        aprgpu::generate_spheres_device(ctx, nz, nx, ny, count, min_radius, max_radius, background, min_intensity,
                                        max_intensity, blur_sigma, seed, buf.as<float>(), ctx->stream);
        APR_CUDA(cudaMemcpy(out, buf.p, 4 * n, cudaMemcpyDeviceToHost));
    });
}

int aprgpu_build_apr(aprgpu_ctx* ctx, const float* volume, int nz, int nx, int ny, double rel_error, int ptr_kind,
                     aprgpu_apr** out) {
    aprgpu_build_params p{rel_error, -1, 0.0, 0, 0.0, 0, 0};  // (sigma_mode -1: the spheres recipe)
    return aprgpu_build_apr_params(ctx, volume, nz, nx, ny, &p, ptr_kind, out);
}

int aprgpu_build_apr_params(aprgpu_ctx* ctx, const float* volume, int nz, int nx, int ny,
                            const aprgpu_build_params* params, int ptr_kind, aprgpu_apr** out) {
    aprgpu_apr* apr = nullptr;
    int st = guard("aprgpu_build_apr_params", [&] {
        need(ctx && volume && out, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        apr = new aprgpu_apr;
        apr->ctx = ctx;
        apr->dims[0] = nz;
        apr->dims[1] = nx;
        apr->dims[2] = ny;
        const float* vol = volume;
        aprgpu::GpuBuf staged;
        if (ptr_kind == APRGPU_HOST) {
            const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
            staged.ensure(4 * n);
            APR_CUDA(cudaMemcpy(staged.p, volume, 4 * n, cudaMemcpyHostToDevice));
            vol = staged.as<float>();
        } else {
            need(ptr_kind == APRGPU_DEVICE, "bad pointer kind");
        }
        need(params != nullptr, "null build parameters");
        const bool recipe = params->sigma_mode == -1;
        aprgpu::build_apr_device(ctx, vol, nz, nx, ny, recipe ? nullptr : params, params->rel_error, apr,
                                 apr->built_values, ctx->stream);
        APR_CUDA(cudaStreamSynchronize(ctx->stream));  // (the staged volume is freed on return)
        apr->geom_l_max = std::max(apr->leaf.l_max, host_compute_l_max(nz, nx, ny));
        *out = apr;
    });
    if (st != APRGPU_OK && apr) {
        free_apr(apr);
        delete apr;
    }
    return st;
}

int aprgpu_tile_apr(aprgpu_apr* src, int tz, int tx, int ty, aprgpu_apr** out) {
    aprgpu_apr* big = nullptr;
    int st = guard("aprgpu_tile_apr", [&] {
        need(src && out && tz > 0 && tx > 0 && ty > 0, "bad argument");
        aprgpu_ctx* ctx = src->ctx;
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        big = new aprgpu_apr;
        big->ctx = ctx;
        aprgpu::tile_apr_device(ctx, src, tz, tx, ty, big, nullptr, nullptr, ctx->stream);
        *out = big;
    });
    if (st != APRGPU_OK && big) {
        free_apr(big);
        delete big;
    }
    return st;
}

int aprgpu_tile_values(aprgpu_apr* src, aprgpu_apr* big, int tz, int tx, int ty, const float* src_values,
                       float* big_values) {
    return guard("aprgpu_tile_values", [&] {
        need(src && big && src_values && big_values, "null argument");
        need(src->ctx == big->ctx, "APRs belong to different contexts");
        DeviceGuard g(src->ctx->device);
        if (big->dims[0] != src->dims[0] * tz || big->dims[1] != src->dims[1] * tx || big->dims[2] != src->dims[2] * ty)
            fail(APRGPU_ERR_RANGE, "tile_values: big APR is not this tiling of the source");
        aprgpu::tile_apr_device(src->ctx, src, tz, tx, ty, big, src_values, big_values, src->ctx->stream);
    });
}

int aprgpu_convolve_pixels(aprgpu_ctx* ctx, const float* in, int nz, int nx, int ny, const float* w, int kz, int kx,
                           int ky, int pad_mode, int accum, float* out, int ptr_kind, void* stream) {
    return guard("aprgpu_convolve_pixels", [&] {
        need(ctx && in && w && out, "null argument");
        need(pad_mode == APRGPU_PAD_ZERO || pad_mode == APRGPU_PAD_REFLECT, "bad pad mode");
        need(accum == APRGPU_ACCUM_EXACT || accum == APRGPU_ACCUM_FAST, "bad accumulation mode");
        need(ptr_kind == APRGPU_HOST || ptr_kind == APRGPU_DEVICE, "bad pointer kind");
        need(nz >= 0 && nx >= 0 && ny >= 0, "negative volume dims");
        const aprgpu::HostStencil hs = make_host_stencil(w, kz, kx, ky);
        if (kz > 13 || kx > 13 || ky > 13)
            fail(APRGPU_ERR_CAPABILITY, "convolve_pixels: stencil extent exceeds the supported maximum");
        DeviceGuard g(ctx->device);
        cudaStream_t s = aprgpu::pick_stream(ctx, stream);
        const uint64_t n = static_cast<uint64_t>(nz) * nx * ny;
        aprgpu::GpuBuf wd, vin, vout;
        wd.ensure(4 * hs.w.size());
        APR_CUDA(cudaMemcpyAsync(wd.p, hs.w.data(), 4 * hs.w.size(), cudaMemcpyHostToDevice, s));
        const float* src = in;
        float* dst = out;
        if (ptr_kind == APRGPU_HOST) {
            vin.ensure(4 * n + 4);
            vout.ensure(4 * n + 4);
            APR_CUDA(cudaMemcpyAsync(vin.p, in, 4 * n, cudaMemcpyHostToDevice, s));
            src = vin.as<float>();
            dst = vout.as<float>();
        }
        bool any_zero = false;  // (zero weights are skipped like the reference, convolve.hpp:86-88)
        for (float v : hs.w) any_zero = any_zero || v == 0.0f;
        aprgpu::convolve_pixels_device(ctx, src, nz, nx, ny, wd.as<float>(), kz, kx, ky, pad_mode, accum, dst, s,
                                       any_zero, hs.w.data());
        if (ptr_kind == APRGPU_HOST) APR_CUDA(cudaMemcpyAsync(out, dst, 4 * n, cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));  // (the weights' buffer is released on return)
    });
}

int aprgpu_load_apr(aprgpu_ctx* ctx, const char* path, aprgpu_apr** out) {
    return guard("aprgpu_load_apr", [&] {
        need(ctx && path && out, "null argument");
        DeviceGuard g(ctx->device);
        std::string msg;
        const int st = aprgpu::load_apr_host(ctx, path, out, msg);
        if (st != APRGPU_OK) fail(st, msg);
    });
}

int aprgpu_save_apr(aprgpu_apr* apr, const char* path, const float* values, int ptr_kind) {
    return guard("aprgpu_save_apr", [&] {
        need(apr && path && (values || apr->leaf.n_particles == 0), "null argument");
        need(ptr_kind == APRGPU_HOST || ptr_kind == APRGPU_DEVICE, "bad pointer kind");
        DeviceGuard g(apr->ctx->device);
        std::vector<float> host;
        const float* v = values;
        if (ptr_kind == APRGPU_DEVICE) {
            host.resize(apr->leaf.n_particles);
            APR_CUDA(cudaMemcpy(host.data(), values, 4 * host.size(), cudaMemcpyDeviceToHost));
            v = host.data();
        }
        std::string msg;
        const int st = aprgpu::save_apr_host(apr, path, v, msg);
        if (st != APRGPU_OK) fail(st, msg);
    });
}

int aprgpu_apr_params(const aprgpu_apr* apr, aprgpu_build_params* out) {
    return guard([&] {
        need(apr && out, "null argument");
        *out = apr->params;
    });
}

int aprgpu_apr_values(const aprgpu_apr* apr, float* out, int ptr_kind) {
    return guard([&] {
        need(apr && out, "null argument");
        if (!apr->built_values.p) fail(APRGPU_ERR_INVALID, "this APR was neither built (aprgpu_build_apr) nor loaded");
        DeviceGuard g(apr->ctx->device);
        const uint64_t n = apr->leaf.n_particles;
        APR_CUDA(cudaMemcpy(out, apr->built_values.p, 4 * n,
                            ptr_kind == APRGPU_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
