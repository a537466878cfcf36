// radix_sort.cu -- stable LSD radix sort of (uint64 key, uint32 value) pairs and u32 scans.
//
// Step a3 of the hot path: the linear cell ids of §4.3 are
// sorted on device so that the points of each non-empty cell become one contiguous range of
// A.  Stability (ties keep the ascending point-id order of the input) makes A deterministic
// (reading R14).  Only the key_bits actually used by prod|g_j| are sorted.
//
// Per 8-bit digit pass (HBM-bound; 3 kernels):
//   hist    : each CTA histograms its TILE of digits in shared memory -> counts[digit][cta]
//   scan    : exclusive scan over counts in digit-major order -> scatter base per (digit, cta)
//   scatter : each CTA re-reads its tile in order and places every item at
//             base[digit][cta] + (rank among equal digits before it in the tile), the rank
//             computed with __match_any_sync inside a warp plus per-warp digit counts in smem.
#include "sj_common.cuh"

namespace sj {

namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kTile = kSortThreads * kSortItems;

__global__ void __launch_bounds__(kSortThreads)
k_radix_hist(const uint64_t *__restrict__ keys, uint32_t n, int shift, uint32_t *__restrict__ counts,
             uint32_t nblocks)
{
    __shared__ uint32_t h[kRadix];
    for (int i = threadIdx.x; i < kRadix; i += kSortThreads) h[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int r = 0; r < kSortItems; ++r) {
        uint64_t i = base + (uint64_t)r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & (kRadix - 1)], 1u);
    }
    __syncthreads();
    for (int dg = threadIdx.x; dg < kRadix; dg += kSortThreads)
        counts[(uint64_t)dg * nblocks + blockIdx.x] = h[dg];
}

__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                uint64_t *__restrict__ kout, uint32_t *__restrict__ vout, uint32_t n, int shift,
                const uint32_t *__restrict__ offsets, uint32_t nblocks)
{
    __shared__ uint32_t s_base[kRadix];
    __shared__ uint32_t s_wcnt[kSortWarps][kRadix];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int dg = tid; dg < kRadix; dg += kSortThreads)
        s_base[dg] = offsets[(uint64_t)dg * nblocks + blockIdx.x];
    const unsigned lt_mask = (1u << lane) - 1u;
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = base + (uint64_t)r * kSortThreads + tid;
        const bool valid = i < n;
        uint64_t k = 0;
        uint32_t v = 0;
        int dg = kRadix;  // sentinel for invalid lanes
        if (valid) {
            k = kin[i];
            v = vin[i];
            dg = (int)((k >> shift) & (kRadix - 1));
        }
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const int leader = __ffs(peers) - 1;
        const uint32_t rank_w = __popc(peers & lt_mask);
        for (int w = 0; w < kSortWarps; ++w) s_wcnt[w][tid] = 0;  // kSortThreads == kRadix
        __syncthreads();
        if (valid && lane == leader) s_wcnt[warp][dg] = __popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t pre = 0;
            for (int w = 0; w < warp; ++w) pre += s_wcnt[w][dg];
            const uint32_t pos = s_base[dg] + pre + rank_w;
            kout[pos] = k;
            vout[pos] = v;
        }
        __syncthreads();
        {
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) tot += s_wcnt[w][tid];
            s_base[tid] += tot;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- u32 scans (3-phase)
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *s_warp, uint32_t *total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = (lane < (int)(blockDim.x >> 5)) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;  // inclusive prefix of warp totals
    }
    __syncthreads();
    const uint32_t warp_off = warp ? s_warp[warp - 1] : 0;
    if (total) *total = s_warp[(blockDim.x >> 5) - 1];
    const uint32_t r = warp_off + x - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const uint32_t *__restrict__ in, uint64_t n, uint32_t *__restrict__ block_sums)
{
    __shared__ uint32_t s_warp[32];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {
        uint64_t i = base + (uint64_t)r * kScanThreads + threadIdx.x;
        if (i < n) acc += in[i];
    }
    uint32_t tot;
    block_exclusive_scan(acc, s_warp, &tot);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// single CTA: exclusive scan of block sums in place
__global__ void __launch_bounds__(kScanThreads)
k_scan_sums(uint32_t *__restrict__ sums, uint64_t m)
{
    __shared__ uint32_t s_warp[32];
    uint32_t carry = 0;
    for (uint64_t base = 0; base < m; base += kScanThreads) {
        uint64_t i = base + threadIdx.x;
        uint32_t v = (i < m) ? sums[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan(v, s_warp, &tot);
        if (i < m) sums[i] = carry + ex;
        carry += tot;
    }
}

template <bool INCLUSIVE>
__global__ void __launch_bounds__(kScanThreads)
k_scan_apply(const uint32_t *__restrict__ in, uint32_t *__restrict__ out, uint64_t n,
             const uint32_t *__restrict__ block_off)
{
    __shared__ uint32_t s_warp[32];
    // each thread owns kScanItems consecutive items
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {
        uint64_t i = base + r;
        v[r] = (i < n) ? in[i] : 0;
        acc += v[r];
    }
    uint32_t run = block_off[blockIdx.x] + block_exclusive_scan(acc, s_warp, nullptr);
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {
        uint64_t i = base + r;
        if (INCLUSIVE) run += v[r];
        if (i < n) out[i] = run;
        if (!INCLUSIVE) run += v[r];
    }
}

void scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, bool inclusive, cudaStream_t s)
{
    if (n == 0) return;
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    Scratch<uint32_t> sums(nb, s);
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, sums.p);
    SJ_LAUNCHED();
    k_scan_sums<<<1, kScanThreads, 0, s>>>(sums.p, nb);
    SJ_LAUNCHED();
    if (inclusive)
        k_scan_apply<true><<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, sums.p);
    else
        k_scan_apply<false><<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, sums.p);
    SJ_LAUNCHED();
}

}  // namespace

void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s)
{
    scan_u32(in, out, n, false, s);
}

void inclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s)
{
    scan_u32(in, out, n, true, s);
}

void radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp,
                      uint32_t n, int key_bits, cudaStream_t s, bool *result_in_tmp)
{
    *result_in_tmp = false;
    if (n <= 1 || key_bits <= 0) return;
    const uint32_t nb = (n + kTile - 1) / kTile;
    Scratch<uint32_t> counts((size_t)kRadix * nb, s);
    Scratch<uint32_t> offs((size_t)kRadix * nb, s);
    uint64_t *ka = keys, *kb = keys_tmp;
    uint32_t *va = vals, *vb = vals_tmp;
    for (int shift = 0; shift < key_bits; shift += kRadixBits) {
        k_radix_hist<<<nb, kSortThreads, 0, s>>>(ka, n, shift, counts.p, nb);
        SJ_LAUNCHED();
        exclusive_scan_u32(counts.p, offs.p, (uint64_t)kRadix * nb, s);
        k_radix_scatter<<<nb, kSortThreads, 0, s>>>(ka, va, kb, vb, n, shift, offs.p, nb);
        SJ_LAUNCHED();
        std::swap(ka, kb);
        std::swap(va, vb);
        *result_in_tmp = !*result_in_tmp;
    }
}

}  // namespace sj
