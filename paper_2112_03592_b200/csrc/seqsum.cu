// The reference's sequential double sum of non-negative floats, on the device.
//
// rl_apr's mean (deconv.hpp:90-91: `double mean = 0; for (float v : u) mean
// += v;`, u clamped to >= 0 at :89) rounds after every addition, so its value
// depends on the order.  aprgpu_rl_resume first tries the order-free exact
// sum (every partial sum provably exact); when that bound fails -- C4's 548 M
// observations do -- this file replays the loop bit for bit in parallel:
//
//  * s never decreases (v >= 0).  While s stays in one binade [2^e, 2^(e+1))
//    every partial sum is a multiple of u = ulp(s) = 2^(e-52), and adding v
//    rounds (s + v)/u to an integer: s/u + round(v/u) -- except when v/u is
//    exactly half-odd, where round-half-even looks at the parity of the total
//    (s/u + floor(v/u)) and lands on the even neighbour.  So an element is a
//    map p -> increment (p = parity of s/u), the parity after it is (p + inc)
//    & 1, and maps compose associatively: C(p) = A(p) + B((p + A(p)) & 1).
//  * A window of the array is cut into chunks of kSeqChunk elements, each
//    reduced to its map (k_seq_chunks), and one block scans the chunk maps in
//    order from the current state (k_seq_scan) until s/u would reach 2^53,
//    i.e. the sum leaves its binade.  That chunk is replayed by plain
//    sequential double additions (k_seq_serial) from its exact incoming sum,
//    which also covers the start (s = 0 has no binade) -- then the next binade.
//  * Increments saturate at 2^62 (a saturated map always crosses), so no
//    overflow; the state lives on the device, the host only reads the cursor.
//
// Binade crossings are few (about log2 of the sum's growth) and each window
// starts at twice the cursor, so the array is read about twice in total.
#include <cmath>

#include "internal.cuh"

namespace aprgpu {
namespace {

constexpr int kSeqChunk = 2048;
constexpr int kSeqThreads = 256;  // 8 consecutive elements per thread
constexpr unsigned long long kSat = 1ull << 62;
constexpr unsigned long long kTop = 1ull << 53;  // s/u reaching 2^53 = the next binade

struct SeqMap {  // increment (in units of u) for an incoming parity 0 / 1
    unsigned long long i0, i1;
};

__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
    const unsigned long long c = a + b;  // (a, b <= 2^62: no wrap)
    return c < kSat ? c : kSat;
}

__device__ __forceinline__ SeqMap compose(const SeqMap& a, const SeqMap& b) {  // a first, then b
    SeqMap c;
    c.i0 = sat_add(a.i0, (a.i0 & 1) ? b.i1 : b.i0);
    c.i1 = sat_add(a.i1, (a.i1 & 1) ? b.i0 : b.i1);  // parity after a from p = 1: (1 + i1) & 1
    return c;
}

// binade exponent e of s > 0 (s in [2^e, 2^(e+1)))
__device__ __forceinline__ int binade(double s) {
    int e;
    frexp(s, &e);  // s = f * 2^e, f in [0.5, 1)
    return e - 1;
}

// One element's map under u = 2^(e-52) (q = v / u, exact scaling by a power of two).
__device__ __forceinline__ SeqMap element_map(float v, int e) {
    const double q = ldexp(static_cast<double>(v), 52 - e);
    if (!(q < 9007199254740992.0)) return SeqMap{kSat, kSat};  // >= 2^53: crosses by itself
    const double f = floor(q), fr = q - f;                       // exact
    const unsigned long long n = static_cast<unsigned long long>(f);
    if (fr < 0.5) return SeqMap{n, n};
    if (fr > 0.5) return SeqMap{n + 1, n + 1};
    // a tie: the total s/u + n + 1/2 rounds to the even neighbour
    return SeqMap{n + (n & 1), n + ((n + 1) & 1)};
}

struct SeqState {
    double s;                  // the running sum after element k - 1
    unsigned long long k;      // cursor
    unsigned long long cross;  // 1: the chunk at k crosses a binade (serial replay next)
};

// Map of each chunk of the window [k, k + nchunks * kSeqChunk), in chunk order.
__global__ void __launch_bounds__(kSeqThreads) k_seq_chunks(const float* __restrict__ u, unsigned long long n,
                                                            const SeqState* __restrict__ st, SeqMap* __restrict__ maps) {
    __shared__ SeqMap sh[kSeqThreads / 32];
    const double s = st->s;
    const unsigned long long k0 = st->k + static_cast<unsigned long long>(blockIdx.x) * kSeqChunk;
    const int e = s > 0.0 ? binade(s) : 0;
    SeqMap m{0, 0};
    const unsigned long long b = k0 + static_cast<unsigned long long>(threadIdx.x) * (kSeqChunk / kSeqThreads);
#pragma unroll
    for (int j = 0; j < kSeqChunk / kSeqThreads; ++j) {
        const unsigned long long i = b + j;
        if (i < n) {
            const float v = u[i];
            // (s = 0: zeros keep it 0; the first nonzero element starts the sum -> serial)
            m = compose(m, s > 0.0 ? element_map(v, e) : (v != 0.0f ? SeqMap{kSat, kSat} : SeqMap{0, 0}));
        }
    }
    // ordered reduction: lanes in order, then warps in order
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        SeqMap o;
        o.i0 = __shfl_down_sync(0xffffffffu, m.i0, d);
        o.i1 = __shfl_down_sync(0xffffffffu, m.i1, d);
        if ((lane & (2 * d - 1)) == 0) m = compose(m, o);
    }
    if (lane == 0) sh[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        SeqMap t = sh[0];
        for (int w = 1; w < kSeqThreads / 32; ++w) t = compose(t, sh[w]);
        maps[blockIdx.x] = t;
    }
}

// One block: the chunk maps of the window in order from the current sum; stops
// at the first chunk after which s/u would reach 2^53 (or at the window's end).
__global__ void __launch_bounds__(1024) k_seq_scan(const SeqMap* __restrict__ maps, unsigned long long nchunks,
                                                   unsigned long long n, SeqState* st) {
    __shared__ SeqMap sc[1024];
    __shared__ unsigned long long first;
    const double s = st->s;
    const unsigned long long k = st->k;
    // s / u, in [2^52, 2^53) (s = 0: 0, and every chunk map is 0 or saturated)
    const int e = s > 0.0 ? binade(s) : 0;
    unsigned long long S = static_cast<unsigned long long>(ldexp(s, 52 - e));
    const int t = threadIdx.x;
    for (unsigned long long c0 = 0; c0 < nchunks; c0 += 1024) {
        const unsigned long long c = c0 + t;
        sc[t] = c < nchunks ? maps[c] : SeqMap{0, 0};
        if (t == 0) first = ~0ull;
        __syncthreads();
        for (int d = 1; d < 1024; d <<= 1) {  // inclusive ordered scan (Hillis-Steele)
            SeqMap v = sc[t];
            if (t >= d) v = compose(sc[t - d], v);
            __syncthreads();
            sc[t] = v;
            __syncthreads();
        }
        const unsigned long long p = S & 1;
        const unsigned long long after = sat_add(S, p ? sc[t].i1 : sc[t].i0);
        if (c < nchunks && after >= kTop) atomicMin(&first, c);
        __syncthreads();
        if (first != ~0ull) {
            if (t == 0) {
                const unsigned long long j = first - c0;
                const unsigned long long before = j == 0 ? S : S + (p ? sc[j - 1].i1 : sc[j - 1].i0);
                st->s = ldexp(static_cast<double>(before), e - 52);  // (< 2^53: exact)
                st->k = k + first * kSeqChunk;
                st->cross = 1;
            }
            return;
        }
        S += p ? sc[1023].i1 : sc[1023].i0;  // (< 2^53)
        __syncthreads();
    }
    if (t == 0) {
        st->s = ldexp(static_cast<double>(S), e - 52);
        const unsigned long long end = k + nchunks * kSeqChunk;
        st->k = end < n ? end : n;
        st->cross = 0;
    }
}

// The crossing chunk, replayed: one warp, the sum in every lane (the reference's
// additions, in order).
__global__ void k_seq_serial(const float* __restrict__ u, unsigned long long n, SeqState* st) {
    if (!st->cross) return;
    double s = st->s;
    const unsigned long long k = st->k, end = k + kSeqChunk < n ? k + kSeqChunk : n;
    const int lane = threadIdx.x;
    for (unsigned long long b = k; b < end; b += 32) {
        const unsigned long long i = b + lane;
        const float x = i < end ? u[i] : 0.0f;
        const int m = static_cast<int>(end - b < 32 ? end - b : 32);
        for (int j = 0; j < m; ++j) s = __dadd_rn(s, static_cast<double>(__shfl_sync(0xffffffffu, x, j)));
    }
    if (lane == 0) {
        st->s = s;
        st->k = end;
        st->cross = 0;
    }
}

}  // namespace

double sequential_sum_device(aprgpu_ctx* ctx, const float* u, uint64_t n, GpuBuf& scratch, cudaStream_t s) {
    if (n == 0) return 0.0;
    const uint64_t nchunks_all = (n + kSeqChunk - 1) / kSeqChunk;
    scratch.ensure(64 + sizeof(SeqMap) * nchunks_all);
    SeqState* st = scratch.as<SeqState>();
    SeqMap* maps = reinterpret_cast<SeqMap*>(scratch.as<char>() + 64);
    APR_CUDA(cudaMemsetAsync(st, 0, sizeof(SeqState), s));
    SeqState h{};
    uint64_t w = 256;  // window, chunks
    for (;;) {
        k_seq_serial<<<1, 32, 0, s>>>(u, n, st);  // (the start, and after a crossing)
        APR_CUDA(cudaMemcpyAsync(&h, st, sizeof(SeqState), cudaMemcpyDeviceToHost, s));
        APR_CUDA(cudaStreamSynchronize(s));
        count_launch(ctx);
        if (h.k >= n) break;
        const uint64_t left = (n - h.k + kSeqChunk - 1) / kSeqChunk;
        w = std::min<uint64_t>(std::max<uint64_t>(w, h.k / kSeqChunk), left);  // the next crossing: ~2x the cursor
        k_seq_chunks<<<static_cast<unsigned>(w), kSeqThreads, 0, s>>>(u, n, st, maps);
        k_seq_scan<<<1, 1024, 0, s>>>(maps, w, n, st);
        count_launch(ctx, 2);
        APR_CUDA(cudaGetLastError());
        w = std::min<uint64_t>(2 * w, nchunks_all);
    }
    return h.s;
}

}  // namespace aprgpu
