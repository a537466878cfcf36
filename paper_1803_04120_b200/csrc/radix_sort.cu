// radix_sort.cu -- stable LSD radix sort of (uint64 key, uint32 value) pairs and u32 scans.
//
// Step a3 of the hot path: the linear cell ids of §4.3 are
// sorted on device so that the points of each non-empty cell become one contiguous range of
// A.  Stability (ties keep the ascending point-id order of the input) makes A deterministic
// (reading R14).  Only the key_bits actually used by prod|g_j| are sorted.
//
// ceil(key_bits/11) passes of <= 11-bit digits (41-bit 6-D keys: 4 passes); per pass (HBM-bound):
//   hist    : each CTA histograms its 4096-item tile in shared memory -> counts[digit][cta]
//   scan    : exclusive scan over counts in digit-major order -> scatter base per (digit, cta)
//   scatter : each warp ranks its 512 consecutive items in registers (__match_any_sync + warp
//             private digit counters, no CTA barrier per round), one CTA prefix over the warps,
//             then every item goes to base[digit][cta] + its stable rank.
#include "scan.cuh"

namespace sj {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortRounds = 16;                       // items per thread
constexpr int kWarpTile = 32 * kSortRounds;           // 512 consecutive items per warp
constexpr int kTile = kSortWarps * kWarpTile;         // 4096 items per CTA

template <int BITS>
__global__ void __launch_bounds__(kSortThreads)
k_radix_hist(const uint64_t *__restrict__ keys, uint32_t n, int shift, uint32_t *__restrict__ counts,
             uint32_t ntiles)
{
    constexpr int R = 1 << BITS;
    __shared__ uint32_t h[R];
    for (int i = threadIdx.x; i < R; i += kSortThreads) h[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int r = 0; r < kTile / kSortThreads; ++r) {
        const uint64_t i = base + (uint64_t)r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & (R - 1)], 1u);
    }
    __syncthreads();
    for (int dg = threadIdx.x; dg < R; dg += kSortThreads) counts[(uint64_t)dg * ntiles + blockIdx.x] = h[dg];
}

// Stable scatter of one digit pass.  Each warp ranks its own 512 consecutive items round by
// round (32 items per round, __match_any_sync for equal digits, a warp-private running count per
// digit in shared memory) -- no CTA barrier inside the rounds; one CTA-wide exclusive prefix over
// the warps per digit then turns warp ranks into tile ranks.  Item order == rank order within a
// digit, so the pass is stable (A ties keep ascending point ids, reading R14).
template <int BITS>
__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
                uint32_t *__restrict__ vout, uint32_t n, int shift, const uint32_t *__restrict__ offsets,
                uint32_t ntiles)
{
    constexpr int R = 1 << BITS;
    extern __shared__ uint32_t s_cnt[];               // [kSortWarps][R]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *wc = s_cnt + warp * R;
    for (int i = lane; i < R; i += 32) wc[i] = 0;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    const uint64_t wbase = (uint64_t)blockIdx.x * kTile + (uint64_t)warp * kWarpTile;
    uint64_t k[kSortRounds];
    uint32_t v[kSortRounds], rk[kSortRounds];
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        k[r] = valid ? kin[i] : 0;
        v[r] = (valid && vin) ? vin[i] : 0;
    }
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t dg = valid ? (uint32_t)((k[r] >> shift) & (R - 1)) : (uint32_t)R;
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const uint32_t before = valid ? wc[dg] : 0u;
        rk[r] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0u) wc[dg] = before + __popc(peers);   // group leader
        __syncwarp();
    }
    __syncthreads();
    // per digit: tile offset = global offset of (digit, tile) + counts of the warps before
    for (int dg = threadIdx.x; dg < R; dg += kSortThreads) {
        uint32_t run = offsets[(uint64_t)dg * ntiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = s_cnt[w * R + dg];
            s_cnt[w * R + dg] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        if (i < n) {
            const uint32_t dg = (uint32_t)((k[r] >> shift) & (R - 1));
            const uint32_t pos = wc[dg] + rk[r];
            kout[pos] = k[r];
            if (vout) vout[pos] = v[r];
        }
    }
}

// ---------------------------------------------------------------- u32 scans (single pass)
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// Single-pass scan with decoupled look-back (one launch instead of reduce + apply): CTA c handles
// tiles c, c + grid, ... in order (grid <= resident CTAs, so every tile a look-back waits for is
// being processed by a running CTA); tile t publishes its aggregate, looks back over the tiles
// before it (a warp reads 32 statuses at a time, stopping at the first inclusive prefix), then
// publishes its inclusive prefix.  status[t] = flag << 32 | value (flag 1: aggregate, 2:
// inclusive prefix; the array is zeroed first).
template <bool INCLUSIVE>
__global__ void __launch_bounds__(kScanThreads, 2)
k_scan_1pass(const uint32_t *__restrict__ in, uint32_t *__restrict__ out, uint64_t n, uint64_t ntiles,
             unsigned long long *status, uint32_t *__restrict__ out2, uint32_t *__restrict__ zero_in)
{
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_excl;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t base = t * kScanTile + (uint64_t)threadIdx.x * kScanItems;
        uint32_t v[kScanItems];
        uint32_t acc = 0;
        if (base + kScanItems <= n && !(reinterpret_cast<uintptr_t>(in + base) & 15u)) {
            const uint4 q = *reinterpret_cast<const uint4 *>(in + base);
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
#pragma unroll
            for (int r = 0; r < kScanItems; ++r) v[r] = (base + r < n) ? in[base + r] : 0u;
        }
#pragma unroll
        for (int r = 0; r < kScanItems; ++r) acc += v[r];
        if (zero_in) {
#pragma unroll
            for (int r = 0; r < kScanItems; ++r)
                if (base + r < n) zero_in[base + r] = 0u;
        }
        uint32_t tot;
        const uint32_t excl = block_exclusive_scan(acc, s_warp, &tot);
        if (threadIdx.x < 32) {
            // warp 0: publish, look back, publish the inclusive prefix
            const unsigned lane = threadIdx.x;
            if (lane == 0)
                atomicExch(status + t, ((unsigned long long)(t == 0 ? 2u : 1u) << 32) | tot);
            uint32_t prefix = 0;
            if (t > 0) {
                int64_t j = (int64_t)t - 1;
                while (true) {
                    // statuses j - lane (lane 0 nearest); spin until none up to the nearest
                    // inclusive prefix is empty
                    unsigned long long st = 0;
                    const int64_t k = j - (int64_t)lane;
                    unsigned incl = 0;
                    while (true) {
                        st = k >= 0 ? __ldcg(status + k) : (2ull << 32);
                        const unsigned empty = __ballot_sync(0xffffffffu, (st >> 32) == 0);
                        incl = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                        const unsigned need = incl ? ((2u << (__ffs(incl) - 1)) - 1u) : 0xffffffffu;
                        if (!(empty & need)) break;
                    }
                    // sum lanes 0 .. first inclusive lane (inclusive), all aggregates before it
                    const int stop = incl ? __ffs(incl) - 1 : 31;
                    uint32_t val = (lane <= (unsigned)stop) ? (uint32_t)st : 0u;
#pragma unroll
                    for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    prefix += val;
                    if (incl) break;
                    j -= 32;
                }
                if (lane == 0) atomicExch(status + t, (2ull << 32) | (uint32_t)(prefix + tot));
            }
            if (lane == 0) s_excl = prefix;
        }
        __syncthreads();
        uint32_t run = s_excl + excl;
        __syncthreads();                                       // s_excl / s_warp reused next tile
#pragma unroll
        for (int r = 0; r < kScanItems; ++r) {
            const uint64_t i = base + r;
            if (INCLUSIVE) run += v[r];
            if (i < n) {
                out[i] = run;
                if (out2) out2[i] = run;
            }
            if (!INCLUSIVE) run += v[r];
        }
    }
}

void scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, bool inclusive, cudaStream_t s,
              uint32_t *out2 = nullptr, uint32_t *zero_in = nullptr)
{
    if (n == 0) return;
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    int dev = 0;
    SJ_CUDA(cudaGetDevice(&dev));
    const uint64_t resident = 2ull * (uint64_t)device_sm_count(dev);       // __launch_bounds__(1024, 2)
    const unsigned grid = (unsigned)std::min<uint64_t>(nb, resident);
    Scratch<unsigned long long> status(nb, s);
    SJ_CUDA(cudaMemsetAsync(status.p, 0, sizeof(unsigned long long) * nb, s));
    if (inclusive)
        k_scan_1pass<true><<<grid, kScanThreads, 0, s>>>(in, out, n, nb, status.p, out2, zero_in);
    else
        k_scan_1pass<false><<<grid, kScanThreads, 0, s>>>(in, out, n, nb, status.p, out2, zero_in);
    SJ_LAUNCHED();
}

}  // namespace

void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s)
{
    scan_u32(in, out, n, false, s);
}

void exclusive_scan_u32_consume(uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s)
{
    scan_u32(in, out, n, false, s, nullptr, in);
}

void exclusive_scan_u32_dup(const uint32_t *in, uint32_t *out, uint32_t *out2, uint64_t n, cudaStream_t s)
{
    scan_u32(in, out, n, false, s, out2);
}

void inclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s)
{
    scan_u32(in, out, n, true, s);
}

namespace {
template <int BITS>
void radix_pass(const uint64_t *ka, const uint32_t *va, uint64_t *kb, uint32_t *vb, uint32_t n, int shift,
                uint32_t *counts, uint32_t *offs, uint32_t nt, cudaStream_t s)
{
    constexpr int R = 1 << BITS;
    k_radix_hist<BITS><<<nt, kSortThreads, 0, s>>>(ka, n, shift, counts, nt);
    SJ_LAUNCHED();
    exclusive_scan_u32(counts, offs, (uint64_t)R * nt, s);
    const size_t smem = sizeof(uint32_t) * kSortWarps * R;
    set_max_dyn_smem(reinterpret_cast<const void *>(k_radix_scatter<BITS>), (int)smem);
    k_radix_scatter<BITS><<<nt, kSortThreads, smem, s>>>(ka, va, kb, vb, n, shift, offs, nt);
    SJ_LAUNCHED();
}
}  // namespace

// Stable LSD radix sort over the low key_bits bits: ceil(key_bits/11) passes of equal width
// (<= 11 bits: 2048 buckets, 64 KB of warp counters per CTA).
void radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp,
                      uint32_t n, int key_bits, cudaStream_t s, bool *result_in_tmp)
{
    *result_in_tmp = false;
    if (n <= 1 || key_bits <= 0) return;
    const uint32_t nt = (n + kTile - 1) / kTile;
    const int passes = (key_bits + 10) / 11;
    const int bits = (key_bits + passes - 1) / passes;   // 1..11
    Scratch<uint32_t> counts((size_t)(1u << bits) * nt, s);
    Scratch<uint32_t> offs((size_t)(1u << bits) * nt, s);
    uint64_t *ka = keys, *kb = keys_tmp;
    uint32_t *va = vals, *vb = vals_tmp;
    for (int p = 0; p < passes; ++p) {
        const int shift = p * bits;
        switch (bits) {
#define SJ_PASS(B) case B: radix_pass<B>(ka, va, kb, vb, n, shift, counts.p, offs.p, nt, s); break;
            SJ_PASS(1) SJ_PASS(2) SJ_PASS(3) SJ_PASS(4) SJ_PASS(5) SJ_PASS(6)
            SJ_PASS(7) SJ_PASS(8) SJ_PASS(9) SJ_PASS(10) SJ_PASS(11)
#undef SJ_PASS
        default: fail(SJ_ERR_ARG, "bad radix width");
        }
        std::swap(ka, kb);
        std::swap(va, vb);
        *result_in_tmp = !*result_in_tmp;
    }
}

// ---------------------------------------------------------------- prefix-bucket sort (sparse keys)
// For keys whose top-k-dimension prefix splits the points into small buckets (the caller has
// already histogrammed the prefixes, fused into k_keys):
//   1. exclusive scan -> bucket starts (and a copy used as per-bucket cursors); scatter with an
//      atomic cursor per bucket (order inside a bucket arbitrary);
//   2. one thread per bucket of <= kBucketMax items sorts it by (key, id) (insertion sort); larger
//      buckets are queued and sorted by one CTA each in shared memory (bitonic, <= kBigMax items).
// The result is the (key, id)-ascending order -- exactly what the stable LSD sort produces, so A is
// unchanged (reading R14).  No host round trip: a bucket larger than kBigMax sets *overflow and
// is left unsorted; the caller checks the flag at its next sync and rebuilds with the LSD sort.
namespace {
constexpr uint32_t kBucketMax = 64;
constexpr uint32_t kBigMax = 4096;          // 4096 x (8 + 4) B = 48 KB of shared memory
constexpr int kBigThreads = 512;

// Packed mode (idb > 0): the item travels as ONE 64-bit word (key - prefix*div) << idb | id -- within
// a bucket the prefix is common, so u64 order == (key, id) order -- instead of a key and an id
// written to two random places.
// The position of item i is start[prefix] + rank[i]: the rank came back from the key pass's histogram
// atomic, so this pass is a plain streaming scatter (no atomic round trip per item).
__global__ void __launch_bounds__(256)
k_bucket_scatter(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ rank, uint32_t n, uint64_t div,
                 double inv, const uint32_t *__restrict__ start, uint64_t *__restrict__ kout, int idb)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = kin[i];
    uint64_t q = (uint64_t)((double)k * inv);          // prefix = k / div (double estimate, corrected)
    if (q * div > k) --q;
    else if ((q + 1) * div <= k) ++q;
    const uint32_t pos = __ldg(start + q) + rank[i];
    kout[pos] = ((k - q * div) << idb) | i;           // ids are the input positions
}

// big[0] = number of queued big buckets, big[1..] = their ids.
// Besides sorting, each bucket reports its cells (distinct keys): local[i] = index of item i's cell
// among the bucket's cells, cellcnt[b] = the bucket's cell count -- the exclusive scan of cellcnt
// is the prefix directory and gives every item its global cell number (no head-flag pass/scan).
__global__ void __launch_bounds__(256)
k_bucket_sort(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, const uint32_t *__restrict__ start,
              uint64_t P, uint64_t *__restrict__ kout, uint32_t *__restrict__ vout, uint32_t *__restrict__ big,
              uint32_t big_cap, uint32_t *__restrict__ local, uint32_t *__restrict__ cellcnt, int idb, uint64_t div)
{
    const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= P) return;
    const uint32_t s = start[b], e = start[b + 1];
    if (e - s > kBucketMax) {
        const uint32_t slot = atomicAdd(big, 1u);
        if (slot < big_cap) big[1 + slot] = (uint32_t)b;
        return;                                        // cellcnt[b] written by the big-bucket kernel
    }
    if (idb && e - s <= 8u) {
        // packed items of a small bucket (the common case: ~2 per prefix on sparse data): sorted in
        // registers by an unrolled odd-even transposition network, unpacked, cells numbered
        const uint32_t m = e - s;
        uint64_t r[8];
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) r[i] = i < m ? kin[s + i] : ~0ull;
#pragma unroll
        for (int round = 0; round < 8; ++round) {
#pragma unroll
            for (int i = round & 1; i + 1 < 8; i += 2) {
                const uint64_t a = r[i], c = r[i + 1];
                r[i] = a < c ? a : c;
                r[i + 1] = a < c ? c : a;
            }
        }
        const uint64_t base = b * div, mask = (1ull << idb) - 1ull;
        uint32_t c = 0;
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
            if (i < m) {
                if (i > 0 && (r[i] >> idb) != (r[i - 1] >> idb)) ++c;
                kout[s + i] = base + (r[i] >> idb);
                vout[s + i] = (uint32_t)(r[i] & mask);
                local[s + i] = c;
            }
        }
        cellcnt[b] = m ? c + 1 : 0;
        return;
    }
    if (idb) {
        // packed items: insertion sort in place (u64 order), then unpack into the output range
        uint64_t *w = const_cast<uint64_t *>(kin);
        for (uint32_t i = s + 1; i < e; ++i) {
            const uint64_t x = w[i];
            uint32_t j = i;
            while (j > s && w[j - 1] > x) {
                w[j] = w[j - 1];
                --j;
            }
            w[j] = x;
        }
        const uint64_t base = b * div, mask = (1ull << idb) - 1ull;
        for (uint32_t i = s; i < e; ++i) {
            const uint64_t x = w[i];
            kout[i] = base + (x >> idb);
            vout[i] = (uint32_t)(x & mask);
        }
    } else {
    // insertion sort by (key, id) directly in the output range (a few L1-resident entries)
    for (uint32_t i = s; i < e; ++i) {
        const uint64_t ki = kin[i];
        const uint32_t vi = vin[i];
        uint32_t j = i;
        while (j > s) {
            const uint64_t kj = kout[j - 1];
            const uint32_t vj = vout[j - 1];
            if (kj < ki || (kj == ki && vj < vi)) break;
            kout[j] = kj;
            vout[j] = vj;
            --j;
        }
        kout[j] = ki;
        vout[j] = vi;
    }
    }
    uint32_t c = 0;
    uint64_t prev = 0;
    for (uint32_t i = s; i < e; ++i) {
        const uint64_t k = kout[i];
        if (i > s && k != prev) ++c;
        local[i] = c;
        prev = k;
    }
    cellcnt[b] = (e > s) ? c + 1 : 0;
}

// One CTA per queued big bucket (grid-stride over the queue): bitonic sort of (key, id) in shared
// memory, padded to a power of two with (UINT64_MAX, UINT32_MAX); then the cells of the bucket
// (head flags, CTA-wide scan) -> local[], cellcnt[b].
__global__ void __launch_bounds__(kBigThreads)
k_bucket_sort_big(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                  const uint32_t *__restrict__ start, const uint32_t *__restrict__ big, uint32_t big_cap,
                  uint64_t *__restrict__ kout, uint32_t *__restrict__ vout, uint32_t *__restrict__ overflow,
                  uint32_t *__restrict__ local, uint32_t *__restrict__ cellcnt, int idb, uint64_t div)
{
    extern __shared__ __align__(16) uint64_t s_big[];   // [kBigMax] keys, [kBigMax] ids, warp sums
    uint64_t *sk = s_big;
    uint32_t *sv = reinterpret_cast<uint32_t *>(s_big + kBigMax);
    uint32_t *s_warp = sv + kBigMax;
    const uint32_t nbig = min(big[0], big_cap);
    if (big[0] > big_cap && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(overflow, 1u);
    constexpr uint32_t kPer = kBigMax / kBigThreads;   // 8 consecutive items per thread in the scan
    for (uint32_t qi = blockIdx.x; qi < nbig; qi += gridDim.x) {
        const uint32_t b = big[1 + qi];
        const uint32_t s = start[b], m = start[b + 1] - s;
        if (m > kBigMax) {
            // flagged: the build is redone with the LSD sort.  Keep the cell numbering in range
            // meanwhile (one cell for the whole bucket) so the compaction stays in bounds.
            if (threadIdx.x == 0) {
                atomicOr(overflow, 1u);
                cellcnt[b] = 1;
            }
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) local[s + i] = 0;
            continue;
        }
        uint32_t m2 = 1;
        while (m2 < m) m2 <<= 1;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < m2; i += blockDim.x) {
            sk[i] = i < m ? kin[s + i] : ~0ull;
            sv[i] = (i < m && !idb) ? vin[s + i] : ~0u;          // packed: ids inside sk, sv constant
        }
        __syncthreads();
        for (uint32_t size = 2; size <= m2; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < m2 / 2; i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const uint64_t ka = sk[lo], kb = sk[hi];
                    const uint32_t va = sv[lo], vb = sv[hi];
                    const bool gt = ka > kb || (ka == kb && va > vb);
                    if (gt == up) {
                        sk[lo] = kb; sk[hi] = ka;
                        sv[lo] = vb; sv[hi] = va;
                    }
                }
                __syncthreads();
            }
        }
        if (idb) {
            const uint64_t base = (uint64_t)b * div, mask = (1ull << idb) - 1ull;
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                kout[s + i] = base + (sk[i] >> idb);
                vout[s + i] = (uint32_t)(sk[i] & mask);
            }
        } else {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                kout[s + i] = sk[i];
                vout[s + i] = sv[i];
            }
        }
        // cells: thread t owns items [t*kPer, t*kPer + kPer); head = first item or key change
        uint32_t flags = 0, cnt = 0;
#pragma unroll
        for (uint32_t r = 0; r < kPer; ++r) {
            const uint32_t i = threadIdx.x * kPer + r;
            const bool head = i < m && i > 0 && (sk[i] >> idb) != (sk[i - 1] >> idb);   // keys only (idb = 0: plain)
            flags |= (head ? 1u : 0u) << r;
            cnt += head ? 1u : 0u;
        }
        uint32_t incl = cnt;                             // block inclusive scan of cnt
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((threadIdx.x & 31) >= (uint32_t)o) incl += y;
        }
        if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = incl;
        __syncthreads();
        uint32_t woff = 0;
        for (uint32_t w = 0; w < (threadIdx.x >> 5); ++w) woff += s_warp[w];
        uint32_t run = woff + incl - cnt;
#pragma unroll
        for (uint32_t r = 0; r < kPer; ++r) {
            const uint32_t i = threadIdx.x * kPer + r;
            run += (flags >> r) & 1u;
            if (i < m) local[s + i] = run;
        }
        if (threadIdx.x == blockDim.x - 1) cellcnt[b] = woff + incl + 1;   // heads after item 0, + 1
        __syncthreads();
    }
}
}  // namespace

// hist: per-prefix point counts (P + 1 entries, the last one 0); vals holds every point's rank in its
// bucket (from the key pass's histogram atomic) on entry and the sorted ids on exit.
// local[n]: cell index of each sorted item within its bucket; cellcnt[P+1]: cells per bucket (the
// caller scans it into the prefix directory).
void bucket_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp, uint32_t n,
                       uint64_t div, uint64_t P, uint32_t *hist, uint32_t *overflow, uint32_t *local,
                       uint32_t *cellcnt, cudaStream_t s)
{
    if (n == 0) return;
    HostTrace tr("bsort");
    const double inv = 1.0 / (double)div;
    // at most n / (kBucketMax + 1) buckets are big
    const uint32_t big_cap = n / (kBucketMax + 1) + 1;
    Scratch<uint32_t> start((size_t)P + 1, s), big((size_t)big_cap + 1, s);
    SJ_CUDA(cudaMemsetAsync(big.p, 0, sizeof(uint32_t), s));
    SJ_CUDA(cudaMemsetAsync(cellcnt + P, 0, sizeof(uint32_t), s));
    tr.dev("start", s);
    exclusive_scan_u32(hist, start.p, (uint64_t)P + 1, s);
    tr.dev("bucket scan", s);
    const uint32_t g = (n + 255) / 256;
    // packed items when (bits of key - prefix*div) + (bits of an id) <= 64
    int lowb = 0, idb = 0;
    while (lowb < 64 && ((div - 1) >> lowb)) ++lowb;
    while (idb < 32 && ((uint64_t)(n - 1) >> idb)) ++idb;
    if (idb == 0) idb = 1;
    if (lowb + idb > 64) fail(SJ_ERR_CUDA, "bucket sort needs packed items (internal error)");
    k_bucket_scatter<<<g, 256, 0, s>>>(keys, vals, n, div, inv, start.p, keys_tmp, idb);
    SJ_LAUNCHED();
    tr.dev("scatter", s);
    k_bucket_sort<<<(uint32_t)((P + 255) / 256), 256, 0, s>>>(keys_tmp, vals_tmp, start.p, P, keys, vals, big.p,
                                                               big_cap, local, cellcnt, idb, div);
    SJ_LAUNCHED();
    tr.dev("bucket sort", s);
    constexpr size_t kBigSmem = kBigMax * (sizeof(uint64_t) + sizeof(uint32_t)) + sizeof(uint32_t) * (kBigThreads / 32);
    set_max_dyn_smem(reinterpret_cast<const void *>(k_bucket_sort_big), (int)kBigSmem);
    k_bucket_sort_big<<<296, kBigThreads, kBigSmem, s>>>(keys_tmp, vals_tmp, start.p, big.p, big_cap, keys, vals,
                                                         overflow, local, cellcnt, idb, div);
    SJ_LAUNCHED();
    tr.dev("big buckets", s);
}

}  // namespace sj
