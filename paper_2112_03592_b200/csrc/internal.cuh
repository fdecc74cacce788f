// Internal declarations shared by the aprgpu translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "aprgpu.h"
#include <nvtx3/nvToolsExt.h>

namespace aprgpu {

constexpr int kMaxLevels = APRGPU_MAX_LEVELS;
constexpr int kMaxExtent = APRGPU_MAX_EXTENT;

// ---- errors: thrown inside the library, converted to status at the C-ABI ----
struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};
[[noreturn]] inline void fail(int st, const std::string& m) { throw Error(st, m); }

#define APR_CUDA(expr)                                                                             \
    do {                                                                                           \
        cudaError_t e__ = (expr);                                                                  \
        if (e__ != cudaSuccess) {                                                                  \
            if (e__ == cudaErrorMemoryAllocation)                                                  \
                ::aprgpu::fail(APRGPU_ERR_OOM, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
            ::aprgpu::fail(APRGPU_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));  \
        }                                                                                          \
    } while (0)

// ---- C-ABI plumbing (api.cu, multi.cu) --------------------------------------
std::string& last_error_slot();  // thread-local message of the last failed call

// NVTX ranges (header-only NVTX 3: free unless a tool -- Nsight Systems,
// `ncu --nvtx` -- is attached): one per compute entry point of the C-ABI,
// named after it, and one per internal phase (gather-map builds, the host
// pipeline's chunks, the multi-device passes), nested inside it.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Runs f, converting exceptions into the C-ABI status (and the thread's message).
template <class F>
int guard(F&& f) {
    try {
        f();
        return APRGPU_OK;
    } catch (const Error& e) {
        last_error_slot() = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        last_error_slot() = e.what();
        return APRGPU_ERR_OOM;
    } catch (const std::exception& e) {
        last_error_slot() = e.what();
        return APRGPU_ERR_INVALID;
    }
}

// guard() inside an NVTX range named after the entry point
template <class F>
int guard(const char* range, F&& f) {
    NvtxRange r(range);
    return guard(std::forward<F>(f));
}

inline void need(bool cond, const char* what) {
    if (!cond) fail(APRGPU_ERR_INVALID, what);
}

struct DeviceGuard {  // make a device current for the call, restore on exit
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ---- device-resident access structure ---------------------------------------
// Per level: grid dims and the index of the level's first row.  Row r of the
// structure covers particles [rb[r], rb[r+1]) -- the reference's xz_end shifted
// by one with a leading 0 (so no row-0 branch), narrowed to u32.
struct LevelG {
    int zd, xd, yd;
    uint32_t row0;
};

struct AccessView {  // passed by value to kernels
    const uint16_t* y;
    const uint32_t* rb;
    int l_min, l_max;
    LevelG g[kMaxLevels];
};

struct DevAccess {
    int l_min = 0, l_max = 0;
    std::vector<int> zd, xd, yd;           // l_max+1
    std::vector<uint64_t> level_offset;    // l_max+1
    uint64_t n_particles = 0, n_rows = 0;
    uint16_t* y = nullptr;                 // device [n_particles]
    uint32_t* rb = nullptr;                // device [n_rows+1]
    // per-level non-empty rows (global row ids), ascending == (z,x) order
    uint32_t* work = nullptr;              // device
    std::vector<uint64_t> work_off;        // l_max+2 offsets into work
    // per-level occupied (8z x 8x x 16y) output tiles of the box-tile kernel
    uint32_t* tiles = nullptr;             // device, linear tile ids per level
    std::vector<uint64_t> tile_off;        // l_max+2 offsets into tiles
    std::vector<int> tile_dims;            // 3 per level: tile grid (z, x, y)
    uint8_t* tile_meta = nullptr;          // device, one byte per tile (coarse depth, fill flags); lazy
    // per tile, the non-empty source rows of its (H = 1, 2) box: {first particle, row slot | count << 16}
    uint2* tile_runs[2] = {nullptr, nullptr};
    uint32_t* tile_run_off[2] = {nullptr, nullptr};  // n_tiles + 1 offsets into tile_runs
    // per level, for each tile z-row tz = 0 .. tzd: the first local index of a tile with z-row >= tz
    // (tiles are ordered (tz, tx, ty)), so a z-slab's tiles are one contiguous range
    std::vector<uint32_t> tile_zfirst;
    std::vector<uint64_t> tile_zfirst_off;  // l_max+1 offsets into tile_zfirst
    // resident gather maps of the box-tile kernel, [H-1][pad][level] (lazy; conv_tile.cu): records for the
    // tiles [a0, a1) (absolute tile indices) -- a slab's launches build only the tiles they compute
    struct MapWin {
        uint32_t* rec = nullptr;
        uint64_t a0 = 0, a1 = 0;
    };
    MapWin* tile_map[2][2][kMaxLevels] = {};
    std::vector<MapWin*> tile_map_retired;  // windows a wider one replaced (in-flight launches may read them)
    // per H: every tile's flattened sources (leaf particles, then interior nodes), tiles padded to 4
    uint32_t* tile_flat[2] = {nullptr, nullptr};
    uint32_t* tile_flat_off[2] = {nullptr, nullptr};  // n_tiles + 1 offsets into tile_flat
    uint64_t tile_flat_n[2] = {0, 0};                 // entries of tile_flat
    uint32_t tile_flat_cap[2] = {0, 0};               // its per-tile stride (the largest tile's chunks)
    uint8_t tile_map_fail[2][2][kMaxLevels] = {};  // a level that reconstructs (no map)
    int tile_map_ng[2][kMaxLevels] = {};            // per H and level: largest per-tile chunk count
    AccessView view() const;
    void release();
};

struct GpuBuf {  // owned device allocation (freed on release() or destruction; move-only)
    void* p = nullptr;
    size_t bytes = 0;
    GpuBuf() = default;
    GpuBuf(const GpuBuf&) = delete;
    GpuBuf& operator=(const GpuBuf&) = delete;
    GpuBuf(GpuBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    ~GpuBuf() { release(); }
    void ensure(size_t n);
    void release();
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// z-slab restriction of a convolution: levels >= lc compute only
// the tiles / rows that touch finest-level pixel planes [z_lo, z_hi); coarser
// levels are computed whole.  lc > l_max: no restriction.
struct Slab {
    int lc = 1 << 20, z_lo = 0, z_hi = 1 << 30;
    bool rep = true;  // compute the replicated levels < lc too (multi.cu's boundary passes skip them)
};

// Host worker threads of a context (api.cu): run one job at a time on every
// worker, asynchronously to the caller (start ... wait).  Used by the
// pageable host-pointer convolution to stage chunks through pinned memory.
class HostPool {
  public:
    explicit HostPool(int n);
    ~HostPool();
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;
    void start(std::function<void()> job);  // job() runs once on each worker
    void wait();
    int size() const { return static_cast<int>(th_.size()); }

  private:
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::function<void()> job_;
    uint64_t gen_ = 0;
    int busy_ = 0;
    bool stop_ = false;
};

}  // namespace aprgpu

struct aprgpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // host-pointer convolutions: copy streams and events of the z-chunk pipeline (lazy)
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<cudaEvent_t> events;
    std::mutex pipe_mu;  // one pipelined call at a time per context (shares the streams and events)
    // pageable host-pointer convolutions: pinned staging (inputs, then outputs) and the threads
    // that copy through it (lazy; both under pipe_mu)
    void* stage = nullptr;
    size_t stage_bytes = 0;
    aprgpu::HostPool* pool = nullptr;
    std::mutex mu;
    std::atomic<uint64_t> launches{0};
    int sm_count = 148;
};

struct aprgpu_apr {
    aprgpu_ctx* ctx = nullptr;
    int dims[3] = {0, 0, 0};
    int geom_l_max = 0;
    aprgpu::DevAccess leaf, tree;
    // scratch (grown on demand)
    aprgpu::GpuBuf vsum, wsum;             // fill_tree fp64 sums [n_tree]
    aprgpu::GpuBuf tree_links;             // per interior node, its children (tree.cu); lazy
    std::vector<uint64_t> tree_level_first;  // first node of each interior level + the total (tree.cu); lazy
    std::mutex init_mu;                      // guards the lazy per-APR caches above (links, level starts)
    // per-APR scratch (fill_tree's fp64 sums, host-call staging, RL state): one
    // call at a time, and stream-ordered across callers' streams (api.cu ScratchGuard)
    std::mutex exec_mu;
    cudaEvent_t scratch_ev = nullptr;
    aprgpu::GpuBuf h_in, h_tree, h_out;    // staging for host-pointer calls
    aprgpu::GpuBuf rl_u, rl_ratio, rl_tv;  // RL state
    aprgpu::GpuBuf tmp;                    // misc
    aprgpu::GpuBuf built_values;           // leaf values sampled by aprgpu_build_apr / read by aprgpu_load_apr
    aprgpu::GpuBuf index_scratch;          // aprgpu_rebuild_index (the paper protocol's per-call index step)
    std::mutex index_mu;                   // ... and its own scratch guard (api.cu ScratchGuard)
    // aprgpu_apr_restrict: the z-slab whose tiles this APR's per-tile state covers (default: all)
    aprgpu::Slab tile_slab;
    cudaEvent_t index_ev = nullptr;
    // z-chunk plan of host-pointer convolutions (api.cu, HostPipe): chunk of S
    // finest planes; levels >= lc split per chunk, [l - lc][j] = first particle
    // of chunk j's rows at level l (j = 0..K)
    struct HostPipe {
        int S = 0, K = 0, lc = 0;
        std::vector<uint64_t> leaf_b, tree_b;
        uint64_t leaf_pre = 0, tree_pre = 0;  // particles of the levels < lc (a prefix)
    } host_pipe;
    // BuildParams (apr.hpp:28-33): the reference's defaults unless built or loaded
    aprgpu_build_params params{0.1, 0, 1.0, 2, 0.0, 0, 0};
};

struct aprgpu_pyramid {
    aprgpu_ctx* ctx = nullptr;
    int l_min = 0, l_max = 0, mode = 0;
    std::vector<int> k3;                   // 3 per level
    std::vector<float> w_host;             // all weights, level by level
    std::vector<uint64_t> off;             // per level offset into w_host
    float* w_dev = nullptr;                // device copy (float)
    double* wd_dev = nullptr;              // device copy (double)
    // rank-1 (separable) levels: float factors fz[kz], fx[kx], fy[ky] with
    // w == fz (x) fx (x) fy to within 5e-7 relative per weight (a Gaussian and
    // its restrictions); offset into sep_dev per level, or -1.  Only the FAST
    // 5^3 apply uses them (tolerance-matched; EXACT keeps the weights).
    std::vector<int64_t> sep_off;
    float* sep_dev = nullptr;
};

namespace aprgpu {

// launches.cu / index.cu
void build_row_begin(aprgpu_ctx* ctx, DevAccess& a, const uint64_t* xz_end_host);
void build_work_lists(aprgpu_ctx* ctx, DevAccess& a);
void row_spans(aprgpu_ctx* ctx, const DevAccess& a, int level, int32_t* z, int32_t* x, uint16_t* ymin,
               uint16_t* ymax, uint64_t cap);

// conv_tile.cu
void build_tile_lists(aprgpu_ctx* ctx, DevAccess& a);
void conv_tile_levels(aprgpu_apr* apr, const aprgpu_pyramid* pyr, const float* values, const float* tree_values,
                      int pad, int accum, float* out, const struct EpiArgs& epi, const struct Slab& slab,
                      cudaStream_t s, bool* done);

void rebuild_index_device(aprgpu_apr* apr, cudaStream_t s);

// reconstruct.cu
void reconstruct_level_device(aprgpu_apr* apr, const float* values, const float* tree_values, int l, float* out,
                              cudaStream_t s);
void reconstruct_patch_device(aprgpu_apr* apr, const float* values, const float* tree_values,
                              const aprgpu_patch_spec& spec, float* out, cudaStream_t s);

// tree.cu
void build_tree_structure(aprgpu_ctx* ctx, aprgpu_apr* apr);
void verify_tree_links(aprgpu_ctx* ctx, aprgpu_apr* apr);
void fill_tree_device(aprgpu_apr* apr, const float* leaf, float* tree, cudaStream_t s);

// seqsum.cu: the reference's sequential double sum (`double m = 0; for (float
// v : u) m += v;`, deconv.hpp:90-91) of n non-negative finite device floats,
// bit for bit (synchronises the stream; scratch grows to 16 B per 2048 values)
double sequential_sum_device(aprgpu_ctx* ctx, const float* u, uint64_t n, GpuBuf& scratch, cudaStream_t s);
void fill_tree_sums(aprgpu_apr* apr, const float* leaf, int lt_lo, int lt_hi, int z_lo, int z_hi, cudaStream_t s,
                    float* tree_out = nullptr);
void fill_tree_finalize(aprgpu_apr* apr, float* tree, cudaStream_t s);
void ensure_tree_links(aprgpu_apr* apr, cudaStream_t s);
void tree_partition_check(aprgpu_apr* apr, int* dbl, unsigned long long* min_unc, cudaStream_t s);

// pixels.cu: convolve_pixels (convolve.hpp:48-98); w_dev = kz*kx*ky device floats
void convolve_pixels_device(aprgpu_ctx* ctx, const float* in, int nz, int nx, int ny, const float* w_dev, int kz,
                            int kx, int ky, int pad, int accum, float* out, cudaStream_t s, bool any_zero_w,
                            const float* w_host);  // (w_host: the weights again, for kernel parameters)

// io.cpp: the .apr container (docs/FORMATS.md)
int load_apr_host(aprgpu_ctx* ctx, const char* path, aprgpu_apr** out, std::string& msg);
int save_apr_host(const aprgpu_apr* apr, const char* path, const float* values, std::string& msg);

// validate.cu: the per-row part of validate (apr.hpp:85-101) plus the cell
// origins' domain check; first_y = min(particle << 1 | out-of-grid)
void validate_rows_device(aprgpu_ctx* ctx, const DevAccess& L, const int dims[3], unsigned long long* first_y,
                          int* overflow, cudaStream_t s);
// the partition check by a per-pixel bitmap (structures whose grids are not the image's)
void validate_cover_device(aprgpu_ctx* ctx, const DevAccess& L, const int dims[3], int* dbl,
                           unsigned long long* min_unc, cudaStream_t s);


// conv.cu
enum Epilogue { EPI_STORE = 0, EPI_RL_RATIO = 1, EPI_RL_MULT = 2 };
struct EpiArgs {
    int mode = EPI_STORE;
    const float* u = nullptr;  // RL observed (ratio epilogue)
    double eps = 0.0;
    float* est = nullptr;      // RL estimate (multiply epilogue; also the output)
};
void convolve_device(aprgpu_apr* apr, const float* values, const float* tree_values, const aprgpu_pyramid* pyr,
                     int pad, int accum, float* out, const EpiArgs& epi, cudaStream_t s, const Slab& slab = Slab());
void check_pyramid(const aprgpu_apr* apr, const aprgpu_pyramid* pyr);

// build.cu
void generate_spheres_device(aprgpu_ctx* ctx, int nz, int nx, int ny, int count, double min_r, double max_r,
                             double background, double min_i, double max_i, double blur, uint64_t seed, float* out,
                             cudaStream_t s);
void build_apr_device(aprgpu_ctx* ctx, const float* vol, int nz, int nx, int ny, double rel_error, aprgpu_apr* apr,
                      GpuBuf& values_out, cudaStream_t s);
void build_apr_device(aprgpu_ctx* ctx, const float* vol, int nz, int nx, int ny, const aprgpu_build_params* params,
                      double rel_error, aprgpu_apr* apr, GpuBuf& values_out, cudaStream_t s);

// tile.cu
void tile_apr_device(aprgpu_ctx* ctx, const aprgpu_apr* src, int TZ, int TX, int TY, aprgpu_apr* big,
                     const float* src_v, float* big_v, cudaStream_t s);

// stencil.cpp (host)
struct HostStencil {
    int kz = 1, kx = 1, ky = 1;
    std::vector<float> w;
};
HostStencil restrict_stencil_host(const HostStencil& w, int delta);
HostStencil gaussian_stencil_host(double sigma, int size);

// Lazily built per-APR device caches are double-checked: read without the
// lock (acquire), built and published under it (release) only after the
// kernels that fill them have completed -- so a reader on another thread and
// stream never sees a pointer to unfilled memory.
template <class T>
inline T* acquire_ptr(T* const& p) { return __atomic_load_n(&p, __ATOMIC_ACQUIRE); }
template <class T>
inline void publish_ptr(T*& p, T* v) { __atomic_store_n(&p, v, __ATOMIC_RELEASE); }

// Kernel attributes (dynamic shared-memory limit, carveout) are per device:
// `set` runs once per device ordinal (a context may live on any GPU of the
// process).  Setting an attribute twice is harmless, so racing callers need no
// lock -- only the published bit is ordered.
struct OncePerDevice {
    std::atomic<uint64_t> done{0};
    template <class F>
    void operator()(F&& set) {
        int dev = 0;
        APR_CUDA(cudaGetDevice(&dev));
        const uint64_t bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return;
        set();
        done.fetch_or(bit, std::memory_order_acq_rel);
    }
};

inline void count_launch(aprgpu_ctx* ctx, uint64_t n = 1) { ctx->launches.fetch_add(n, std::memory_order_relaxed); }

inline cudaStream_t pick_stream(aprgpu_ctx* ctx, void* s) {
    return s ? static_cast<cudaStream_t>(s) : ctx->stream;
}

inline unsigned blocks_for(uint64_t n, unsigned per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace aprgpu
