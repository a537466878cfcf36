// index_build.cu -- steps a1-a4 of the hot path: the sparse epsilon-grid index.
//
// PAPER.md §4.2 "Index Properties" (lines 155-168), §4.3 "Index Components" (170-173, 181):
// only non-empty cells are stored: B = sorted linear ids, G = per-cell ranges into A,
// A = point ids grouped by cell, M_j = occupied coordinates per dimension.  Readings
// (DESIGN.md): R6 cell width w = eps + 2^-44 (eps + R); R7 c_j = 1 + floor(fl(fl(x_j-min_j)/w)),
// |g_j| = 3 + floor(fl(fl(max_j-min_j)/w)) (one empty pad cell each side);
// R8 dimension 1 fastest; R9 M_j as occupied sets; R14 A ordered by (linear id, point id).
//
// Kernels (all HBM-bound; algorithmic bytes in DESIGN.md §Roofline):
//   k_minmax                        : exact per-dimension min/max + non-finite check (a1)
//   k_keys                          : cell coordinates -> linear id, identity ids, mask bytes (a2)
//   radix sort                      : stable LSD over key_bits (a3, radix_sort.cu)
//   k_heads + inclusive scan        : cell index of every A-position (a4)
//   k_compact_gather                : B, G starts, SoA coordinates X[j][k] = D[A[k]][j] (a4)
//   k_dir_hist + exclusive scan     : prefix directory bounding every B search (a4)
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>

#include "scan.cuh"

namespace sj {

namespace {

constexpr int kThreads = 256;

// Order-preserving map of a (non-NaN) double to uint64, so min/max become integer atomics.
__device__ __forceinline__ unsigned long long ord_key(double x)
{
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Geometry computed ON THE DEVICE from the min/max (same IEEE operations as host_geometry, so the
// host's copy -- read while k_keys already runs -- must agree bit for bit): cell width, |g_j|,
// strides, key bits, the prefix-directory plan (k, P, pstride) and the sort strategy.  This takes
// the host round trip between the min/max pass and the key pass off the GPU's critical path.
struct DevGeom {
    double w;
    double mins[SJ_MAX_DIM], maxs[SJ_MAX_DIM];
    uint64_t cpd[SJ_MAX_DIM], strides[SJ_MAX_DIM], pstride[SJ_MAX_DIM];
    uint64_t mask_off[SJ_MAX_DIM + 1];
    uint64_t P, div;
    int key_bits, k, use_bucket, masks_on;
    int status;                  // 0 ok, 1 non-finite coordinate, 2 key overflow
};
static_assert(sizeof(DevGeom) % 8 == 0, "DevGeom is copied as 64-bit words");
static_assert(sizeof(DevGeom) <= 2048, "DevGeom fits below the doorbell");

__device__ __forceinline__ double ord_to_double(unsigned long long k)
{
    const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)u);
}

// SJ_DEBUG_SYNC=1: synchronise and check after the build's phases (fault localisation)
static bool debug_sync()
{
    static const bool on = [] { const char *e = std::getenv("SJ_DEBUG_SYNC"); return e && *e && *e != '0'; }();
    return on;
}

// directory size cap: P_k <= max(mult * N, 2^16) entries (SJ_DIR_CAP overrides mult)

static uint32_t dir_cap_mult()
{
    static const uint32_t m = [] {
        const char *e = std::getenv("SJ_DIR_CAP");
        const long v = e ? std::strtol(e, nullptr, 10) : 0;
        return (uint32_t)(v >= 1 && v <= 64 ? v : 4);
    }();
    return m;
}

// the full directory (k = d) is taken when it has at most kFullDirMult entries per point
constexpr uint32_t kFullDirMult = 8;

constexpr int kSmemMaskWords = 2048;   // 64 K bits, 8 KB of shared memory
// context slot layout of the build: min/max partials (<= 4 * SMs blocks), then the DevGeom
constexpr size_t kGeomOffset = 4 * 256 * (2 * SJ_MAX_DIM + 1) * sizeof(unsigned long long);
constexpr size_t kEstOffset = kGeomOffset + 4096;          // pinned staging of aux + estimate buckets
constexpr size_t kBellOffset = 2048;                       // host slots: DevGeom at 0, the doorbell here
constexpr size_t kMaxEstBuckets = 1100;
constexpr size_t kAuxEstOffset = 64;                       // estimate buckets, bytes after aux
constexpr int kAuxWords = 8;                               // aux: |G|, tasks, populous, overflow, masks-trivial
constexpr size_t kBuildSlotBytes = kEstOffset + kAuxEstOffset + 8 * kMaxEstBuckets;

// prefix-bucket items travel packed as ONE 64-bit word ((key - prefix*div) << idb | id): possible when
// the low key part and the point id fit together (bits(div - 1) + bits(n - 1) <= 64)
__host__ __device__ __forceinline__ int id_bits(uint32_t n)
{
    int b = 1;
    while (b < 32 && ((uint64_t)(n - 1) >> b)) ++b;
    return b;
}
__host__ __device__ __forceinline__ int low_bits(uint64_t div)
{
    int b = 0;
    while (b < 64 && ((div - 1) >> b)) ++b;
    return b;
}
__host__ __device__ __forceinline__ bool bucket_items_pack(uint64_t div, uint32_t n)
{
    return low_bits(div) + id_bits(n) <= 64;
}

__device__ __noinline__ void geometry_products(const uint64_t *cpd, int d, uint32_t n, int allow_bucket,
                                               int want_masks, uint32_t cap_mult, DevGeom &G);

// executed by the whole (last) CTA of k_minmax_geom (256 threads); not inlined, so its registers
// do not limit the occupancy of the min/max loop
__device__ __noinline__ void geometry_block(const unsigned long long *__restrict__ part, uint32_t parts, int d,
                                               double eps, uint32_t n, int allow_bucket, int want_masks,
                                               uint32_t cap_mult, DevGeom *__restrict__ g, DevGeom *hgeom,
                                               volatile uint32_t *hbell, uint32_t epoch)
{
    // reduce the per-block partials of k_minmax: min over [0, d), max over [d, 2d), or of [2d];
    // each thread folds whole rows (independent loads in flight), then warp and CTA reductions
    __shared__ unsigned long long s_red[2 * SJ_MAX_DIM + 1][8];
    __shared__ unsigned long long mm[2 * SJ_MAX_DIM + 1];
    unsigned long long acc[2 * SJ_MAX_DIM + 1];
#pragma unroll
    for (int v = 0; v <= 2 * SJ_MAX_DIM; ++v) acc[v] = v < d ? ~0ull : 0ull;
    for (uint32_t b = threadIdx.x; b < parts; b += blockDim.x) {
        const unsigned long long *row = part + (uint64_t)b * (2 * d + 1);
#pragma unroll
        for (int v = 0; v <= 2 * SJ_MAX_DIM; ++v) {
            if (v > 2 * d) break;
            const unsigned long long x = __ldcg(row + v);     // written by other CTAs: bypass L1
            acc[v] = v < d ? min(acc[v], x) : max(acc[v], x);
        }
    }
#pragma unroll
    for (int v = 0; v <= 2 * SJ_MAX_DIM; ++v) {
        if (v > 2 * d) break;
        for (int o = 16; o; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, acc[v], o);
            acc[v] = v < d ? min(acc[v], y) : max(acc[v], y);
        }
        if ((threadIdx.x & 31) == 0) s_red[v][threadIdx.x >> 5] = acc[v];
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // warp 0: lanes finish the reduction per value, then lane j < d handles dimension j (its
    // division in parallel with the others); lane 0 does the products
    const int lane = threadIdx.x;
    if (lane <= 2 * d) {
        unsigned long long a = s_red[lane][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = lane < d ? min(a, s_red[lane][w]) : max(a, s_red[lane][w]);
        mm[lane] = a;
    }
    __syncwarp();
    __shared__ DevGeom G;
    if (lane == 0) {
        uint64_t *z = reinterpret_cast<uint64_t *>(&G);
        for (size_t i2 = 0; i2 < sizeof(DevGeom) / 8; ++i2) z[i2] = 0;
    }
    __syncwarp();
    const bool bad = mm[2 * d] != 0;
    double range = 0.0;
    if (lane < d) {
        const double mn = ord_to_double(mm[lane]), mx = ord_to_double(mm[d + lane]);
        G.mins[lane] = mn;
        G.maxs[lane] = mx;
        range = __dsub_rn(mx, mn);
    }
    double R = range;
    for (int o = 16; o; o >>= 1) R = fmax(R, __shfl_xor_sync(0xffffffffu, R, o));
    const double er = __dadd_rn(eps, R);
    const double w = __dadd_rn(eps, __dmul_rn(er, 0x1p-44));       // = eps + ldexp(er, -44) (exact scaling)
    double t = 0.0;
    if (lane < d) t = floor(__ddiv_rn(range, w));
    const bool tbad = lane < d && !(t < 9.0e18);
    const bool any_tbad = __any_sync(0xffffffffu, tbad);
    const uint64_t mycpd = (lane < d && !tbad) ? 3ull + (uint64_t)t : 0ull;
    uint64_t cpd[SJ_MAX_DIM];
#pragma unroll
    for (int j = 0; j < SJ_MAX_DIM; ++j) cpd[j] = __shfl_sync(0xffffffffu, mycpd, j);
    if (lane == 0) {
        G.w = w;
        if (bad) G.status = 1;
        else if (any_tbad) G.status = 2;
        else geometry_products(cpd, d, n, allow_bucket, want_masks, cap_mult, G);
    }
    __syncwarp();
    const uint64_t *src = reinterpret_cast<const uint64_t *>(&G);
    uint64_t *dst = reinterpret_cast<uint64_t *>(g);
    for (size_t i2 = lane; i2 < sizeof(DevGeom) / 8; i2 += 32) dst[i2] = src[i2];
    if (hgeom) {
        // the host's copy straight into mapped pinned memory, then the doorbell: the host polls it
        // instead of an event + D2H copy between this kernel and the key pass (which would stop the
        // key pass from launching programmatically behind this one)
        uint64_t *hdst = reinterpret_cast<uint64_t *>(hgeom);
        for (size_t i2 = lane; i2 < sizeof(DevGeom) / 8; i2 += 32) hdst[i2] = src[i2];
        __threadfence_system();
        __syncwarp();
        if (lane == 0) *hbell = epoch;
    }
}

// a1: exact per-dimension min/max + non-finite flag, then -- in the LAST CTA to finish -- the geometry
// (geometry_block) and the zeroing of the index's small masks / aux / estimate buckets.  D is read as
// ONE flat array of n*D doubles, fully coalesced: the grid's thread count is a multiple of D (host),
// so every element a thread visits has the same dimension t mod D.  Each CTA writes its partial
// (order-preserving integer images): part[b][0..D) = ord(min), [D..2D) = ord(max), [2D] = non-finite.
template <int D>
__global__ void __launch_bounds__(kThreads, 4)
k_minmax_geom(const double *__restrict__ pts, uint32_t n, unsigned long long *__restrict__ part,
              unsigned int *__restrict__ done, double eps, int allow_bucket, int want_masks, uint32_t cap_mult,
              DevGeom *__restrict__ g, uint32_t *__restrict__ zero_words, uint32_t nzero, DevGeom *hgeom,
              volatile uint32_t *hbell, uint32_t epoch)
{
#ifndef SJ_PDL_TRIGGER_END
    pdl_trigger();                   // the key pass may launch now (it loads its rows, then waits)
#endif
    const uint64_t total = (uint64_t)n * D;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
    // 16-byte loads: thread t reads the element pairs v = t, t+S, ... (elements 2v, 2v+1, always of
    // dimensions 2t mod D and (2t+1) mod D: 2S is a multiple of D).  Every round issues U loads
    // together (predicated, the out-of-range ones repeat the first), so a thread waits for
    // ceil(pairs / (U*S)) memory latencies -- 3 at 2 M x 6-D -- instead of one per tail element.
    // (the odd last element of an odd total belongs to dimension D-1: CTA 0 folds it in below)
    __shared__ double s_mn[2 * kThreads], s_mx[2 * kThreads];
    bool bad = false;
    const bool vec = (reinterpret_cast<uintptr_t>(pts) & 15u) == 0;
    if (vec) {
        const double2 *p2 = reinterpret_cast<const double2 *>(pts);
        const uint64_t T2 = total >> 1;
        double mna = INFINITY, mxa = -INFINITY, mnb = INFINITY, mxb = -INFINITY;
        constexpr int U = 8;
#pragma unroll 1
        for (uint64_t v0 = t; v0 < T2; v0 += U * S) {
            double2 x[U];
            x[0] = p2[v0];
#pragma unroll
            for (int u = 1; u < U; ++u) x[u] = v0 + u * S < T2 ? p2[v0 + u * S] : x[0];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                bad |= !isfinite(x[u].x) || !isfinite(x[u].y);
                mna = fmin(mna, x[u].x);
                mxa = fmax(mxa, x[u].x);
                mnb = fmin(mnb, x[u].y);
                mxb = fmax(mxb, x[u].y);
            }
        }
        s_mn[2 * threadIdx.x] = mna;
        s_mx[2 * threadIdx.x] = mxa;
        s_mn[2 * threadIdx.x + 1] = mnb;
        s_mx[2 * threadIdx.x + 1] = mxb;
    } else {
        double mn = INFINITY, mx = -INFINITY;
#pragma unroll 1
        for (uint64_t e = t; e < total; e += S) {
            const double x = pts[e];
            bad |= !isfinite(x);
            mn = fmin(mn, x);
            mx = fmax(mx, x);
        }
        s_mn[threadIdx.x] = mn;
        s_mx[threadIdx.x] = mx;
    }
    if (vec && (total & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) bad |= !isfinite(pts[total - 1]);
    const bool any_bad = __syncthreads_or(bad);
    unsigned long long *out = part + (uint64_t)blockIdx.x * (2 * D + 1);
    if (threadIdx.x < D) {
        const int j = threadIdx.x;
        // the slots cover elements base .. base + L - 1 of the flat array (mod D: their dimensions)
        const uint32_t L = vec ? 2 * kThreads : kThreads;
        const uint32_t base = (uint32_t)(((uint64_t)blockIdx.x * L) % D);
        double a = INFINITY, b = -INFINITY;
        for (uint32_t l = (uint32_t)((j + D - (int)base) % D); l < L; l += D) {
            a = fmin(a, s_mn[l]);
            b = fmax(b, s_mx[l]);
        }
        if (vec && (total & 1ull) && blockIdx.x == 0 && j == D - 1) {
            const double x = pts[total - 1];
            a = fmin(a, x);
            b = fmax(b, x);
        }
        out[j] = ord_key(a);            // +inf / -inf when the CTA saw no element of dimension j
        out[D + j] = ord_key(b);
    }
    if (threadIdx.x == 0) out[2 * D] = any_bad ? 1ull : 0ull;
#ifdef SJ_PDL_TRIGGER_END
    pdl_trigger();
#endif
    // last CTA: geometry from all partials
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (uint32_t i = threadIdx.x; i < nzero; i += blockDim.x) zero_words[i] = 0u;
    geometry_block(part, gridDim.x, D, eps, n, allow_bucket, want_masks, cap_mult, g, hgeom, hbell, epoch);
    if (threadIdx.x == 0) *done = 0u;                 // ready for the next build on this context
}

// lane 0 of k_geometry: everything that needs only products and sums of the |g_j|
__device__ __noinline__ void geometry_products(const uint64_t *cpd, int d, uint32_t n, int allow_bucket,
                                               int want_masks, uint32_t cap_mult, DevGeom &G)
{
    unsigned __int128 prod = 1;
    for (int j = 0; j < d; ++j) {
        G.cpd[j] = cpd[j];
        prod *= cpd[j];
        if (prod >> 64) { G.status = 2; return; }
    }
    G.strides[0] = 1;
    for (int j = 1; j < d; ++j) G.strides[j] = G.strides[j - 1] * cpd[j - 1];
    const unsigned __int128 maxkey = prod - 1;
    const uint64_t hi = (uint64_t)(maxkey >> 64), lo = (uint64_t)maxkey;
    G.key_bits = hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
    // directory plan (plan_dir): the full directory (k = d) when prod_j |g_j| <= kFullDirMult * N,
    // else the largest k with prod_{top k} |g_j| <= max(4N, 2^16)
    const uint64_t cap = max((uint64_t)cap_mult * n, (uint64_t)1 << 16);
    unsigned __int128 P = 1;
    if (prod <= (unsigned __int128)kFullDirMult * n) {
        P = prod;
        G.k = d;
    } else {
        for (int kk = 1; kk <= d; ++kk) {
            const unsigned __int128 Q = P * cpd[d - kk];
            if (Q > cap) break;
            P = Q;
            G.k = kk;
        }
    }
    G.P = (uint64_t)P;
    G.div = 1;
    for (int j = 0; j < d - G.k; ++j) G.div *= cpd[j];
    uint64_t ps = 1;                                   // pstride_j = prod_{d-k <= m < j} |g_m|
    for (int j = 0; j < d; ++j) {
        G.pstride[j] = (j >= d - G.k) ? ps : 0;
        if (j >= d - G.k) ps *= cpd[j];
    }
    G.use_bucket = allow_bucket && G.k >= 1 && (double)n <= 2.0 * (double)G.P && G.P <= (1ull << 22) &&
                   G.key_bits <= 62 && bucket_items_pack(G.div, n);
    uint64_t mt = 0;
    for (int j = 0; j < d; ++j) { G.mask_off[j] = mt; mt += cpd[j]; }
    G.mask_off[d] = mt;
    G.masks_on = want_masks && mt <= 32ull * kSmemMaskWords;
}

// floor(fl(t / w)) for t >= 0 (reading R7's rounded quotient) without a division in the common case:
// y = fl(t * fl(1/w)) is within 1.5 * 2^-52 * t/w of t/w and the correctly rounded fl(t/w) within
// 2^-53 * t/w, so both lie in [y - d, y + d] with d = 2^-49 y (the computed ends, rounded, still
// bracket that); when floor() is the same at both ends it is the floor of fl(t/w).  Otherwise (y within
// ~2^-49 relative of an integer) the exact division decides.  Pinned by the bit-exact index tests.
__device__ __forceinline__ double cell_floor(double t, double w, double inv_w)
{
    const double y = __dmul_rn(t, inv_w);
    const double d = __dmul_rn(y, 0x1p-49);
    const double lo = floor(__dsub_rn(y, d));
    if (lo == floor(__dadd_rn(y, d))) return lo;
    return floor(__ddiv_rn(t, w));
}

// Cell coordinate c_j = 1 + floor(fl(fl(x_j - min_j) / w))  (reading R7), linear id with
// dimension 1 fastest (R8): key = sum_j c_j * stride_j (exact: < prod |g_j| < 2^64).
// Masks M_j as one bitmap over all dimensions (bit mask_off[j] + c): each CTA ORs
// into a shared copy and flushes only the non-zero words, so the few hot words are not hammered by
// every point (masks larger than kSmemMaskWords words: k_masks_global after the geometry sync).
// bhist (prefix-bucket sort only): points per top-k prefix sum_j c_j * pstride_j, fused here so
// the sort needs no histogram pass of its own.  Geometry from the device (k_geometry).
template <int D>
__global__ void __launch_bounds__(kThreads)
k_keys(const double *__restrict__ pts, uint32_t n, const DevGeom *g, uint64_t *__restrict__ keys,
       uint32_t *__restrict__ ids, uint32_t *__restrict__ masks, uint32_t *__restrict__ bhist)
{
    __shared__ uint32_t s_mask[kSmemMaskWords];
    __shared__ double s_min[D];
    __shared__ uint64_t s_str[D], s_pstr[D], s_moff[D];
    // the point's row does not depend on the min/max pass: under programmatic dependent launch it is
    // loaded while k_minmax_geom's last CTA still computes the geometry, then we wait for that grid
    const uint64_t base = (uint64_t)blockIdx.x * kThreads;
    const uint32_t cnt = (uint32_t)min((uint64_t)kThreads, (uint64_t)n - base);
    const uint64_t i = base + threadIdx.x;
    double xr[D];
    if (threadIdx.x < cnt) {
        bool loaded = false;
        if constexpr (D % 2 == 0) {
            if ((reinterpret_cast<uintptr_t>(pts) & 15u) == 0) {   // 16-B aligned rows: vector loads
#pragma unroll
                for (int j = 0; j < D; j += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(pts + i * D + j);
                    xr[j] = v.x;
                    xr[j + 1] = v.y;
                }
                loaded = true;
            }
        }
        if (!loaded) {
#pragma unroll
            for (int j = 0; j < D; ++j) xr[j] = pts[i * D + j];
        }
    }
    // The geometry is written by the primary grid (k_minmax_geom's last CTA): read it only after the
    // wait, through L2 (__ldcg).  (With g declared const __restrict__ the compiler hoisted the status
    // load above griddepcontrol.wait as a read-only .CONSTANT load: a small build whose key pass
    // launched early read the previous build's status -- e.g. a failed build's -- and skipped its keys.)
    pdl_wait();
    // one coherent read per CTA (into shared memory): the same few words read through L2 by every
    // thread of every CTA cost the key pass ~40 us of L2 hot-spot serialisation
    __shared__ int s_status, s_masks_on, s_use_bucket, s_k;
    __shared__ double s_w;
    __shared__ uint64_t s_moffD;
    if (threadIdx.x == 0) {
        s_status = __ldcg(&g->status);
        s_masks_on = __ldcg(&g->masks_on);
        s_use_bucket = __ldcg(&g->use_bucket);
        s_k = __ldcg(&g->k);
        s_w = __ldcg(&g->w);
        s_moffD = __ldcg(&g->mask_off[D]);
    }
    if (threadIdx.x < D) {
        s_min[threadIdx.x] = __ldcg(&g->mins[threadIdx.x]);
        s_str[threadIdx.x] = __ldcg(&g->strides[threadIdx.x]);
        s_pstr[threadIdx.x] = __ldcg(&g->pstride[threadIdx.x]);
        s_moff[threadIdx.x] = __ldcg(&g->mask_off[threadIdx.x]);
    }
    __syncthreads();
    if (s_status) return;
    const bool use_masks = s_masks_on != 0;
    const bool use_hist = s_use_bucket != 0;
    const int dir_k = s_k;
    const double w = s_w;
    const double inv_w = 1.0 / w;
    const uint32_t mask_words = (uint32_t)((s_moffD + 31) / 32);
    if (use_masks)
        for (uint32_t w2 = threadIdx.x; w2 < mask_words; w2 += blockDim.x) s_mask[w2] = 0;
    __syncthreads();
    if (threadIdx.x < cnt) {
        uint64_t key = 0, prefix = 0;
        uint32_t rank = (uint32_t)i;
        // top dimension first: the prefix is complete after the dir_k top dims, so the bucket path's
        // histogram atomic -- whose old value is the point's rank in its bucket (the scatter then
        // needs no atomic of its own) -- is in flight while the low dimensions are divided
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            const int j = D - 1 - jj;
            const double x = xr[j];
            const double t = cell_floor(__dsub_rn(x, s_min[j]), w, inv_w);
            const uint64_t c = 1ull + (uint64_t)t;
            key += c * s_str[j];
            prefix += c * s_pstr[j];
            if (use_hist && jj == dir_k - 1) rank = atomicAdd(bhist + prefix, 1u);
            if (use_masks) {
                const uint64_t bit = s_moff[j] + c;
                const uint32_t m = 1u << (bit & 31);
                if (!(s_mask[bit >> 5] & m)) atomicOr(s_mask + (bit >> 5), m);   // (set already: skip the atomic)
            }
        }
        keys[i] = key;
        ids[i] = rank;                      // bucket path: the rank; LSD: the values (input positions)
    }
    if (use_masks) {
        __syncthreads();
        for (uint32_t w2 = threadIdx.x; w2 < mask_words; w2 += blockDim.x)
            if (s_mask[w2] && (__ldcg(masks + w2) & s_mask[w2]) != s_mask[w2]) atomicOr(masks + w2, s_mask[w2]);
    }
}

// masks too large for shared memory (host-launched after the geometry sync): global atomics
template <int D>
__global__ void __launch_bounds__(kThreads)
k_masks_global(const double *__restrict__ pts, uint32_t n, DevIndex ix, uint32_t *__restrict__ masks)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const double t = floor(__ddiv_rn(__dsub_rn(pts[i * D + j], ix.mins[j]), ix.w));
        const uint64_t bit = ix.mask_off[j] + 1ull + (uint64_t)t;
        atomicOr(masks + (bit >> 5), 1u << (bit & 31));
    }
}

__global__ void __launch_bounds__(kThreads)
k_heads(const uint64_t *__restrict__ keys, uint32_t n, uint32_t *__restrict__ flags)
{
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    flags[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1u : 0u;
}

__device__ __forceinline__ uint64_t quot_small(uint64_t x, uint64_t d, double inv)   // floor(x/d), x/d < 2^50
{
    uint64_t q = (uint64_t)((double)x * inv);
    if (q * d > x) --q;
    else if ((q + 1) * d <= x) ++q;
    return q;
}

// occ_set_cell (below) from the key and its top-k prefix alone, no full key decode: the grouped
// index c_L + |g_L| (c_lo + |g_lo| rest) with prefix = c_L + |g_L| rest and c_lo (c_lo2) the
// digits of the key's low part key - prefix * dir_div
__device__ __forceinline__ void occ_set_prefix(const DevIndex &ix, uint64_t key, uint64_t prefix, uint32_t *occ,
                                               uint32_t *occ2)
{
    const int L = ix.d - ix.dir_k;
    const uint64_t gL = ix.cpd[L], glo = ix.cpd[L - 1];
    const uint64_t rest = quot_small(prefix, gL, ix.inv_cpd[L]);
    const uint64_t cL = prefix - rest * gL;
    const uint64_t low = key - prefix * ix.dir_div;
    const uint64_t clo = quot_small(low, ix.strides[L - 1], ix.inv_stride[L - 1]);
    const uint64_t q = cL + gL * (clo + glo * rest);
    atomicOr(occ + ((q - gL) >> 5), 1u << ((q - gL) & 31));
    atomicOr(occ + (q >> 5), 1u << (q & 31));
    atomicOr(occ + ((q + gL) >> 5), 1u << ((q + gL) & 31));
    if (occ2) {
        const uint64_t glo2 = ix.cpd[L - 2];
        const uint64_t low2 = low - clo * ix.strides[L - 1];
        const uint64_t clo2 = quot_small(low2, ix.strides[L - 2], ix.inv_stride[L - 2]);
        const uint64_t q2 = cL + gL * (clo2 + glo2 * rest);
        atomicOr(occ2 + ((q2 - gL) >> 5), 1u << ((q2 - gL) & 31));
        atomicOr(occ2 + (q2 >> 5), 1u << (q2 & 31));
        atomicOr(occ2 + ((q2 + gL) >> 5), 1u << ((q2 + gL) & 31));
    }
}

// Occupancy bitmaps over (top-k prefix, c_lo), lo = d-k-1 (occ) / d-k-2 (occ2), stored DILATED along
// c_lo: a cell sets the bits of c_lo - 1, c_lo, c_lo + 1 (index(c) +- the stride of c_lo, see
// apply_dir_geometry), so the refine asks "is any cell of that prefix in the window c_lo + {-1,0,1}?"
// with one bit test -- and, the lowest top dimension being the fastest index, for the three top
// offsets that differ only in c_{d-k} with one load.  (c_lo is in [1, |g|-2]: the window never
// leaves the prefix; the pad cells are empty.)
template <int D>
__device__ __forceinline__ void occ_set_cell(const DevIndex &ix, const uint64_t (&c)[D], uint32_t *occ, uint32_t *occ2)
{
    const int L = D - ix.dir_k;
    uint64_t q = 0, q2 = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        q += c[j] * ix.occ_mul[j];
        q2 += c[j] * ix.occ2_mul[j];
    }
    uint64_t st = 0, st2 = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        if (j == L - 1) st = ix.occ_mul[j];
        if (j == L - 2) st2 = ix.occ2_mul[j];
    }
    atomicOr(occ + ((q - st) >> 5), 1u << ((q - st) & 31));
    atomicOr(occ + (q >> 5), 1u << (q & 31));
    atomicOr(occ + ((q + st) >> 5), 1u << ((q + st) & 31));
    if (occ2) {
        atomicOr(occ2 + ((q2 - st2) >> 5), 1u << ((q2 - st2) & 31));
        atomicOr(occ2 + (q2 >> 5), 1u << (q2 & 31));
        atomicOr(occ2 + ((q2 + st2) >> 5), 1u << ((q2 + st2) & 31));
    }
}

// pcell holds the inclusive scan of head flags on entry (1-based cell number) and the
// 0-based cell index on exit.  At the head of each cell h (one thread per cell):
//   B[h], G[h]; populous-cell count (dense tasks); its packed coordinates (decoded from the key)
//   and Alg. 1 line-6 mask word (bit j: c_j - 1 not in M_j; bit 8+j: c_j + 1 not in M_j); the
//   prefix-directory histogram (cells per top-k prefix) and the occupancy bit of its top-(k+1)
//   prefix.  Every thread: the SoA gather X[j][k] = D[A[k]][j].
template <int D>
__global__ void __launch_bounds__(kThreads)
k_compact_gather(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ A,
                 const double *__restrict__ pts, uint32_t n, uint32_t *__restrict__ pcell,
                 uint64_t *__restrict__ B, uint32_t *__restrict__ G, double *__restrict__ X,
                 uint64_t *__restrict__ ccoord, uint32_t *__restrict__ cmask, DevIndex ix, uint32_t dense_T,
                 uint32_t *__restrict__ n_dense_cells, uint32_t *__restrict__ dirhist, uint32_t *__restrict__ occ,
                 bool bucket_cells, double dir_inv)
{
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t a = A[k];
    const uint64_t key = keys[k];
    uint32_t h;
    // the key's top-k prefix (exact quotient: double estimate + one integer correction)
    uint64_t b = (uint64_t)((double)key * dir_inv);
    if (b * ix.dir_div > key) --b;
    else if ((b + 1) * ix.dir_div <= key) ++b;
    if (bucket_cells) {             // cell = directory start of the key's top-k prefix + index within it
        h = __ldg(ix.dir + b) + pcell[k];
        if (h >= n) return;         // only after a flagged bucket overflow (the build is redone)
    } else {                        // inclusive scan of head flags (1-based)
        h = pcell[k] - 1u;
    }
    pcell[k] = h;
    if (k == 0 || keys[k - 1] != key) {
        B[h] = key;
        G[h] = (uint32_t)k;
        // populous cell (>= dense_T points)?  one extra load: its (dense_T-1)-th successor
        if (n_dense_cells && k + dense_T - 1 < n && keys[k + dense_T - 1] == key) atomicAdd(n_dense_cells, 1u);
        if (ccoord) {
            uint64_t c[D];
            key_to_coords<D>(ix, key, c);
            uint64_t packed = 0;
            uint32_t mb = 0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                packed |= c[j] << ix.cshift[j];
                if (ix.masks) {
                    const uint64_t lo = ix.mask_off[j] + c[j] - 1ull, hi = lo + 2ull;
                    if (!((ix.masks[lo >> 5] >> (lo & 31)) & 1u)) mb |= 1u << j;
                    if (!((ix.masks[hi >> 5] >> (hi & 31)) & 1u)) mb |= 1u << (j + 8);
                }
            }
            ccoord[h] = packed;
            cmask[h] = mb;
        }
        if (dirhist) atomicAdd(dirhist + b, 1u);
        if (occ) occ_set_prefix(ix, key, b, occ, const_cast<uint32_t *>(ix.occ2));
    }
    if (k == n - 1) {
        G[h + 1] = n;
        if (h + 1 < n) B[h + 1] = 1ull << 63;   // sentinel (keys < 2^62 when the build estimates)
    }
    const double *src = pts + (uint64_t)a * D;
    if (D % 2 == 0 && (reinterpret_cast<uintptr_t>(pts) & 15u) == 0) {   // 16-B aligned rows: vector loads
#pragma unroll
        for (int j = 0; j < D; j += 2) {
            const double2 v = *reinterpret_cast<const double2 *>(src + j);
            X[(uint64_t)j * n + k] = v.x;
            X[(uint64_t)(j + 1) * n + k] = v.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) X[(uint64_t)j * n + k] = src[j];
    }
}


struct BuildArgs {
    const double *pts = nullptr;
    uint32_t n = 0;
    unsigned long long *mm = nullptr;
    unsigned int *done = nullptr;
    double eps = 0.0;
    int allow_bucket = 0, want_masks = 0;
    uint32_t *zero_words = nullptr;
    uint32_t nzero = 0;
    uint32_t *nonfinite = nullptr;
    uint64_t *keys = nullptr;
    uint32_t *ids = nullptr;
    uint32_t *masks = nullptr;
    const DevGeom *geom = nullptr;
    uint32_t *bhist = nullptr;
    const uint32_t *A = nullptr;
    uint32_t *pcell = nullptr;
    uint64_t *B = nullptr;
    uint32_t *G = nullptr;
    double *X = nullptr;
    uint64_t *ccoord = nullptr;
    uint32_t *cmask = nullptr;
    uint32_t *ndense = nullptr;
    uint32_t *dirhist = nullptr;
    bool bucket_cells = false;   // pcell holds the cell index within the top-k prefix; dir is final
    double dir_inv = 0.0;
    uint32_t *occ = nullptr;
    DevGeom *hgeom = nullptr;              // mapped pinned copy of the geometry + its doorbell
    volatile uint32_t *hbell = nullptr;
    uint32_t epoch = 0;
};

template <int D>
void launch_dim(int which, dim3 g, cudaStream_t s, const DevIndex &ix, const BuildArgs &a)
{
    if (which == 0) {
        k_minmax_geom<D><<<g, kThreads, 0, s>>>(a.pts, a.n, a.mm, a.done, a.eps, a.allow_bucket, a.want_masks,
                                                 dir_cap_mult(), const_cast<DevGeom *>(a.geom), a.zero_words, a.nzero,
                                                 a.hgeom, a.hbell, a.epoch);
    } else if (which == 1) {
        launch_pdl(k_keys<D>, g, dim3(kThreads), 0, s, a.pts, a.n, a.geom, a.keys, a.ids, a.masks, a.bhist);
    } else if (which == 3) {
        k_masks_global<D><<<g, kThreads, 0, s>>>(a.pts, a.n, ix, a.masks);
    } else {
        k_compact_gather<D><<<g, kThreads, 0, s>>>(a.keys, a.A, a.pts, a.n, a.pcell, a.B, a.G, a.X, a.ccoord, a.cmask,
                                                   ix, 16u, a.ndense, a.dirhist, a.occ, a.bucket_cells, a.dir_inv);
    }
    SJ_LAUNCHED();
}

void launch(int d, int which, dim3 g, cudaStream_t s, const DevIndex &ix, const BuildArgs &a)
{
    switch (d) {
    case 2: launch_dim<2>(which, g, s, ix, a); break;
    case 3: launch_dim<3>(which, g, s, ix, a); break;
    case 4: launch_dim<4>(which, g, s, ix, a); break;
    case 5: launch_dim<5>(which, g, s, ix, a); break;
    case 6: launch_dim<6>(which, g, s, ix, a); break;
    default: fail(SJ_ERR_DIM, "d must be in [2,6]");
    }
}


// Host-side geometry (a1 epilogue): R, w, |g_j|, strides, key bits.  Exact same IEEE
// operations as written in DESIGN.md R6/R7.
void host_geometry(int d, double eps, const double *mins, const double *maxs, sj_index_view &v)
{
    double R = 0.0;
    double ranges[SJ_MAX_DIM];
    for (int j = 0; j < d; ++j) {
        volatile double r = maxs[j] - mins[j];
        ranges[j] = r;
        if (r > R) R = r;
    }
    volatile double er = eps + R;
    volatile double w = eps + std::ldexp((double)er, -44);
    v.w = w;
    long double prod = 1.0L;
    unsigned __int128 iprod = 1;
    for (int j = 0; j < d; ++j) {
        volatile double q = ranges[j] / (double)w;
        const double t = std::floor((double)q);
        if (!(t < 9.0e18)) fail(SJ_ERR_KEY_OVERFLOW, "cells per dimension overflow: use a larger eps");
        v.cpd[j] = 3ull + (uint64_t)t;
        prod *= (long double)v.cpd[j];
        if (prod >= 18446744073709551616.0L)
            fail(SJ_ERR_KEY_OVERFLOW, "prod |g_j| >= 2^64: linear cell ids overflow uint64; use a larger eps");
        iprod *= v.cpd[j];
    }
    v.strides[0] = 1;
    for (int j = 1; j < d; ++j) v.strides[j] = v.strides[j - 1] * v.cpd[j - 1];
    // bits needed for linear ids in [0, prod-1]
    unsigned __int128 maxkey = iprod - 1;
    int bits = 0;
    while (maxkey > 0) { ++bits; maxkey >>= 1; }
    v.key_bits = bits;
}

}  // namespace

// ---- prefix directory plan (host): DESIGN.md §6 "bounded search".  The largest k such that the
// number of top-k coordinate prefixes P_k = prod_{j >= d-k} |g_j| stays <= max(4N, 2^16) (<= 16 B
// per point, so the index stays O(|D|)); every B lookup of the refine is bounded to
// one prefix's range.  The same k/P drive the prefix-bucket sort.  The occupancy bitmap over the
// top-(k+1) prefixes is planned when it costs <= 8 B per point and filters (the +-1 window of 3
// sub-prefixes is expected occupied with probability ~3N/P_{k+1} < SJ_OCC_MAXFILL: 6-D eps=1: 0.06; eps=8:
// 0.53 -> not built).
#ifndef SJ_OCC_MAXFILL
#define SJ_OCC_MAXFILL 0.5     // 6-D eps=4: 0.35 -> built (join 2.59 -> 1.72 ms); eps=8: 0.53 -> not (built: slower)
#endif
struct DirPlan {
    int k = 0;
    uint64_t P = 1;
    uint64_t div = 1;            // stride of dimension d-k: key / div = prefix
    bool occ = false;
    uint64_t occ_cpd = 0, occ_div = 0;
    size_t occ_words = 0;
    bool occ2 = false;           // (top-k prefix, c_{d-k-2}) bitmap, only with occ and >= 2 low dims
    uint64_t occ2_cpd = 0;
    size_t occ2_words = 0;
};

DirPlan plan_dir(const sj_index_view &v)
{
    DirPlan dp;
    const int d = v.d;
    const uint64_t n = v.n;
    const unsigned __int128 cap = std::max<uint64_t>((uint64_t)dir_cap_mult() * n, 1ull << 16);
    unsigned __int128 P = 1;
    unsigned __int128 prod = 1;
    for (int j = 0; j < d; ++j) prod *= v.cpd[j];
    if (prod <= (unsigned __int128)kFullDirMult * n) {
        // the full directory: every row of three cells is ONE O(1) lookup (dense-rows mode; 6-D
        // eps = 8: 15^6 = 11.4 M entries, join 8.6 -> 4.1 ms against the k = 5 cell scan)
        P = prod;
        dp.k = d;
    } else {
        for (int kk = 1; kk <= d; ++kk) {
            const unsigned __int128 Q = P * v.cpd[d - kk];
            if (Q > cap) break;
            P = Q;
            dp.k = kk;
        }
    }
    dp.P = (uint64_t)P;
    for (int j = 0; j < d - dp.k; ++j) dp.div *= v.cpd[j];
    if (dp.k >= 1 && dp.k < d) {
        const unsigned __int128 P1 = P * v.cpd[d - dp.k - 1];
        if (P1 <= (unsigned __int128)64 * std::max<uint64_t>(n, 1ull << 16) &&
            3.0 * (double)n < SJ_OCC_MAXFILL * (double)(uint64_t)P1) {
            dp.occ = true;
            dp.occ_cpd = v.cpd[d - dp.k - 1];
            dp.occ_div = dp.div / dp.occ_cpd;
            dp.occ_words = (size_t)((P1 + 31) / 32) + 2;     // +2: the refine's 64-bit window loads
            if (d - dp.k >= 2) {
                const unsigned __int128 P2 = P * v.cpd[d - dp.k - 2];
                if (P2 <= (unsigned __int128)64 * std::max<uint64_t>(n, 1ull << 16)) {
                    dp.occ2 = true;
                    dp.occ2_cpd = v.cpd[d - dp.k - 2];
                    dp.occ2_words = (size_t)((P2 + 31) / 32) + 2;
                }
            }
        }
    }
    return dp;
}

// Geometry-derived constants of the directory in kernel form.
void apply_dir_geometry(DevIndex &ix, const sj_index_view &v, const DirPlan &dp)
{
    const int d = v.d;
    ix.dir_k = dp.k;
    ix.dir_P = dp.P;
    ix.dir_div = dp.div;
    for (int j = 0; j < SJ_MAX_DIM; ++j) ix.pstride[j] = (j < d && j >= d - dp.k) ? v.strides[j] / dp.div : 0;
    uint32_t ntop = 1;
    for (int j = 0; j < dp.k; ++j) ntop *= 3;
    ix.dir_ntop = ntop;
    for (int j = 0; j < d; ++j) ix.inv_cpd[j] = 1.0 / (double)v.cpd[j];
    ix.lowR[0] = 0;
    for (int j = 0; j < d; ++j) ix.lowR[j + 1] = ix.lowR[j] + (int64_t)(j < d - dp.k ? v.strides[j] : 0);
    ix.occ_div = dp.occ ? dp.occ_div : 0;
    ix.occ_cpd = dp.occ ? dp.occ_cpd : 0;
    ix.occ2_cpd = dp.occ2 ? dp.occ2_cpd : 0;
    // bitmap index = c_L + |g_L| * (c_lo + |g_lo| * (prefix - c_L) / |g_L|), L = d-k (the lowest top
    // dimension), lo = L-1 (occ) or L-2 (occ2): the three top offsets that differ only in c_L are
    // ADJACENT bits, so the refine tests them with one load (DESIGN.md §6 "grouped occupancy")
    const int Lt = d - dp.k;
    for (int j = 0; j < SJ_MAX_DIM; ++j) {
        const bool top = j < d && j >= Lt;
        const uint64_t cL = dp.k >= 1 ? v.cpd[Lt] : 1;
        ix.occ_mul[j] = !dp.occ ? 0 : (j == Lt ? 1 : (top ? ix.pstride[j] * ix.occ_cpd : (j == Lt - 1 ? cL : 0)));
        ix.occ2_mul[j] = !dp.occ2 ? 0 : (j == Lt ? 1 : (top ? ix.pstride[j] * ix.occ2_cpd : (j == Lt - 2 ? cL : 0)));
    }
    // key -> coordinates by double reciprocals when every quotient < 2^50 and keys < 2^63
    bool fast = v.key_bits <= 63;
    for (int j = 1; j < d; ++j) fast = fast && v.cpd[j] < (1ull << 50);
    ix.key_fastdiv = fast ? 1 : 0;
    for (int j = 0; j < d; ++j) ix.inv_stride[j] = 1.0 / (double)v.strides[j];
}

// dir (P+1 entries) and the occupancy bitmap (zeroed), owned by the index.
void alloc_dir(sj_index *idx, const DirPlan &dp, cudaStream_t s)
{
    uint32_t *dir = static_cast<uint32_t *>(dev_alloc(sizeof(uint32_t) * ((size_t)dp.P + 1), s));
    idx->bufs[idx->nbufs++] = dir;
    idx->view.dir = dir;
    idx->dev.dir = dir;
    // the bitmaps come zeroed from the zeroed-buffer cache when one is there (released bitmaps are
    // zeroed when their index is freed), else fresh + memset
    auto zeroed = [&](size_t bytes, int slot) -> uint32_t * {
        size_t got = 0;
        void *p = zbuf_get(idx->device, bytes, &got);
        if (p) {
            idx->zbufs[slot] = p;
            idx->zbytes[slot] = got;
            return static_cast<uint32_t *>(p);
        }
        if (!alloc_hook_set()) {
            SJ_CUDA(cudaMalloc(&p, bytes));
            idx->zbufs[slot] = p;
            idx->zbytes[slot] = bytes;
        } else {
            p = dev_alloc(bytes, s);
            idx->bufs[idx->nbufs++] = p;
        }
        SJ_CUDA(cudaMemsetAsync(p, 0, bytes, s));
        return static_cast<uint32_t *>(p);
    };
    idx->dev.occ = nullptr;
    if (dp.occ) idx->dev.occ = zeroed(sizeof(uint32_t) * dp.occ_words, 0);
    idx->dev.occ2 = nullptr;
    if (dp.occ2) idx->dev.occ2 = zeroed(sizeof(uint32_t) * dp.occ2_words, 1);
}

namespace {
// floor(x / d) for quotients < 2^50: double estimate (|error| <= 1) + integer correction
__device__ __forceinline__ uint64_t div_small_quot(uint64_t x, uint64_t d, double inv)
{
    uint64_t q = (uint64_t)((double)x * inv);
    if (q * d > x) --q;
    else if ((q + 1) * d <= x) ++q;
    return q;
}

// dir[q] = #cells with prefix < q = exclusive prefix sum of the per-prefix cell histogram
__global__ void __launch_bounds__(kThreads)
k_dir_hist(const uint64_t *__restrict__ B, const uint32_t *__restrict__ nG, uint64_t div, double inv,
           uint32_t *__restrict__ hist)
{
    const uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= *nG) return;
    atomicAdd(hist + div_small_quot(B[h], div, inv), 1u);
}

// occupancy bits of an imported index (the build sets them in its compaction): coordinates
// decoded from each cell's key, then occ_set_cell
template <int D>
__global__ void __launch_bounds__(kThreads)
k_occ_import(const DevIndex ix, const uint64_t *__restrict__ B, const uint32_t *__restrict__ nG, uint32_t *occ,
             uint32_t *occ2)
{
    const uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= *nG) return;
    uint64_t c[D];
    uint64_t rem = B[h];
#pragma unroll
    for (int j = D - 1; j >= 1; --j) {
        c[j] = rem / ix.strides[j];
        rem -= c[j] * ix.strides[j];
    }
    c[0] = rem;
    occ_set_cell<D>(ix, c, occ, occ2);
}

// Are the masks M_j trivial (every coordinate c in [1, |g_j|-2] occupied, in every dimension)?  Then
// they exclude no adjacent cell (uniform data) and the refine need not consult them (*flag = 1).
__global__ void __launch_bounds__(256)
k_masks_full(const DevIndex ix, uint32_t *__restrict__ flag)
{
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int j = 0; j < ix.d; ++j) {
        const uint64_t lo = ix.mask_off[j] + 1, hi = ix.mask_off[j] + ix.cpd[j] - 2;   // inclusive
        for (uint64_t b = lo + threadIdx.x; b <= hi; b += blockDim.x)
            if (!((__ldcg(ix.masks + (b >> 5)) >> (b & 31)) & 1u)) s_bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) *flag = s_bad ? 0u : 1u;
}

// dense tasks, in A-order: cells with >= T points are cut into <= 32-query tasks; count, exclusive
// scan (over the N upper bound, zero past |G|), fill
__global__ void __launch_bounds__(kThreads)
k_dense_count(const uint32_t *__restrict__ G, const uint32_t *__restrict__ nG, uint32_t T, uint32_t *__restrict__ cnt)
{
    const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= *nG) return;
    const uint32_t n = G[h + 1] - G[h];
    cnt[h] = n >= T ? (n + 31u) / 32u : 0u;
}

__global__ void __launch_bounds__(kThreads)
k_dense_fill(const uint32_t *__restrict__ G, const uint32_t *__restrict__ nG, uint32_t T,
             const uint32_t *__restrict__ off, uint32_t *__restrict__ tasks)
{
    const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= *nG) return;
    const uint32_t s = G[h], n = G[h + 1] - s;
    if (n < T) return;
    const uint32_t o = off[h];
    for (uint32_t i = 0; i < (n + 31u) / 32u; ++i) tasks[o + i] = s + 32u * i;
}
}  // namespace


// Device-built directory -> dir (exclusive scan of the per-prefix cell histogram); then the single
// host sync reads |G| (aux[0]), the populous-cell count (aux[2]) and the bucket-sort overflow flag
// (aux[3]) into h_aux.  Dense-cell tasks (cells with >= kDenseT points cut into <= 32-query tasks,
// one warp each in k_refine_dense) are built in A-order when the compaction saw populous cells (the
// import path, which has no such count, always builds them).
constexpr uint32_t kDenseT = 16;
void launch_masks_full(const DevIndex &ix, uint32_t *flag, cudaStream_t s)
{
    k_masks_full<<<1, 256, 0, s>>>(ix, flag);
    SJ_LAUNCHED();
}

void finish_aux(sj_index *idx, cudaStream_t s, uint32_t *aux, const DirPlan &dp, const uint32_t *dirhist,
                bool force_dense, uint32_t *h_aux, void *h_stage = nullptr, size_t stage_bytes = 0,
                bool check_masks = true, const volatile unsigned int *bell = nullptr, unsigned int epoch = 0)
{
    sj_index_view &v = idx->view;
    DevIndex &ix = idx->dev;
    if (dirhist) exclusive_scan_u32(dirhist, const_cast<uint32_t *>(ix.dir), (uint64_t)dp.P + 1, s);
    // aux[4]: the masks exclude nothing (the build checks on its side stream; the import here)
    if (check_masks && ix.masks && v.mask_offsets[v.d] <= 32ull * kSmemMaskWords) launch_masks_full(ix, aux + 4, s);
    if (h_stage && bell && wait_doorbell(bell, epoch, s)) {
        // the estimate's last CTA published aux + the buckets into h_stage
        std::atomic_thread_fence(std::memory_order_acquire);
        std::memcpy(h_aux, const_cast<const void *>(static_cast<volatile void *>(h_stage)), kAuxWords * sizeof(uint32_t));
    } else if (h_stage) {
        // one copy into pinned memory: aux and whatever the caller placed after it (the build's
        // estimate buckets)
        SJ_CUDA(cudaMemcpyAsync(h_stage, aux, stage_bytes, cudaMemcpyDeviceToHost, s));
        SJ_CUDA(cudaStreamSynchronize(s));
        std::memcpy(h_aux, h_stage, kAuxWords * sizeof(uint32_t));
    } else {
        SJ_CUDA(cudaMemcpyAsync(h_aux, aux, kAuxWords * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SJ_CUDA(cudaStreamSynchronize(s));
    }
    // trivial masks: the kernels skip them (the view keeps them: S never depends on masks)
    if (h_aux[4]) ix.masks = nullptr;
    uint32_t *tasks = nullptr;
    uint32_t ntasks = 0;
    if (!h_aux[3] && (h_aux[2] > 0 || force_dense)) {
        const uint64_t nGh = h_aux[0];
        const uint32_t gG = (uint32_t)((nGh + kThreads - 1) / kThreads);
        Scratch<uint32_t> cnt((size_t)nGh + 1, s), off((size_t)nGh + 1, s);
        SJ_CUDA(cudaMemsetAsync(cnt.p + nGh, 0, sizeof(uint32_t), s));
        k_dense_count<<<gG, kThreads, 0, s>>>(v.G, aux, kDenseT, cnt.p);
        SJ_LAUNCHED();
        exclusive_scan_u32(cnt.p, off.p, nGh + 1, s);
        SJ_CUDA(cudaMemcpyAsync(&ntasks, off.p + nGh, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SJ_CUDA(cudaStreamSynchronize(s));
        if (ntasks) {
            tasks = static_cast<uint32_t *>(dev_alloc(sizeof(uint32_t) * ntasks, s));
            idx->bufs[idx->nbufs++] = tasks;
            k_dense_fill<<<gG, kThreads, 0, s>>>(v.G, aux, kDenseT, off.p, tasks);
            SJ_LAUNCHED();
            SJ_CUDA(cudaStreamSynchronize(s));
        }
    }
    h_aux[1] = ntasks;
    const uint32_t nG = h_aux[0];
    v.n_cells = nG;
    ix.nG = nG;
    v.dir_k = dp.k;
    v.dir_entries = dp.P + 1;
    v.dir = ix.dir;
    // mode: a dense directory gives O(1) rows; small prefix ranges (<= 8 cells on average) are
    // cheapest to scan cell by cell (sparse high-d data); otherwise bounded row searches.
    const double avg_range = (double)nG / (double)dp.P;
    if (dp.k == v.d) ix.search_mode = kSearchDenseRows;
    else if (avg_range <= 8.0 && (double)dp.div < 4.0e15) ix.search_mode = kSearchCellScan;
    else ix.search_mode = kSearchRows;
    ix.dense_tasks = tasks;
    ix.n_dense_tasks = ntasks;
    ix.dense_T = kDenseT;
}



sj_index *build_index_impl2(const double *points, uint64_t n, int d, double eps, const sj_build_opts &o,
                            bool allow_bucket);

sj_index *build_index_impl(const double *points, uint64_t n, int d, double eps, const sj_build_opts &o)
{
    return build_index_impl2(points, n, d, eps, o, true);
}

sj_index *build_index_impl2(const double *points, uint64_t n, int d, double eps, const sj_build_opts &o,
                            bool allow_bucket)
{
    // ---- argument validation before any allocation (sj.h contract)
    if (d < 2 || d > SJ_MAX_DIM) fail(SJ_ERR_DIM, "d must be in [2,6] (PAPER.md:391)");
    if (!points) fail(SJ_ERR_ARG, "points is NULL");
    if (n == 0 || n >= (1ull << 32)) fail(SJ_ERR_ARG, "N must satisfy 1 <= N < 2^32");
    if (!std::isfinite(eps) || !(eps > 0.0)) fail(SJ_ERR_ARG, "eps must be finite and > 0");
    {
        volatile double e2 = eps * eps;
        if (!std::isnormal((double)e2)) fail(SJ_ERR_ARG, "fl(eps*eps) must be a normal double");
    }
    const int ndev = device_count();
    if (ndev == 0) fail(SJ_ERR_STATE, "no CUDA device available (the library has no CPU fallback)");
    if (o.device < 0 || o.device >= ndev) fail(SJ_ERR_ARG, "bad device ordinal");
    SJ_CUDA(cudaSetDevice(o.device));

    HostTrace tr("build");
    // the build runs on the caller's stream, or on a pooled library stream; the pooled context also
    // lends its pinned slot memory and an event (device geometry read-back)
    static_assert(sizeof(DevGeom) <= 4096, "DevGeom fits its slot");
    CtxGuard cg{acquire_ctx(o.device, 2, 4, kBuildSlotBytes)};   // stream 1: geometry read-back, mask check
    cudaStream_t s = o.stream ? static_cast<cudaStream_t>(o.stream) : cg.c->streams[0];
    if (!o.stream) {
        // NULL = the library stream, ordered after the work already queued on the legacy default
        // stream (e.g. torch's default stream producing the points), which a non-blocking library
        // stream would not otherwise wait for
        SJ_CUDA(cudaEventRecord(cg.c->events[1], cudaStreamLegacy));
        SJ_CUDA(cudaStreamWaitEvent(s, cg.c->events[1], 0));
    }

    const uint32_t N = (uint32_t)n;
    // phase events (pooled); handed to the index, which turns them into timings on request
    struct Events {
        int dev;
        cudaEvent_t e[7];
        explicit Events(int d) : dev(d) { for (auto &x : e) x = nullptr; for (auto &x : e) x = event_get(dev); }
        ~Events() { for (auto &x : e) event_put(dev, x); }
        void rec(int i, cudaStream_t st) { SJ_CUDA(cudaEventRecord(e[i], st)); }
    } ev(o.device);
    ev.rec(0, s);
    tr.dev("start", s);

    sj_index *idx = new sj_index();
    idx->device = o.device;
    auto own = [&](void *p) { idx->bufs[idx->nbufs++] = p; return p; };
    uint32_t h_aux[kAuxWords] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int nsm = device_sm_count(o.device);
    bool l2p = false;              // the input is marked L2-persisting on s (see below)
    try {
        // ---- inputs on device
        const double *pts = points;
        Scratch<double> d_pts;
        if (!o.points_on_device) {
            d_pts.p = dalloc<double>((size_t)n * d, s);
            d_pts.s = s;
            SJ_CUDA(cudaMemcpyAsync(d_pts.p, points, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
            pts = d_pts.p;
        }
        ev.rec(1, s);

        // every N-sized array in two arenas.  The index's arena is laid out for the multi-GPU
        // broadcast (sj_index_view.packed): [X | A | pcell | G | small masks | aux | B]; with B last,
        // the bytes up to B + 8|G| are the whole index (B is sized for the upper bound N cells so
        // that no host round trip for |G| is needed during the build).  The scratch arena holds the
        // keys, sort buffers and bucket histogram.
        auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
        const size_t b_A = al(4 * n), b_pc = al(4 * n), b_B = al(8 * n), b_G = al(4 * (n + 1)), b_X = al(8 * n * d),
                     b_mk = al(4 * kSmemMaskWords),
                     b_aux = al(kAuxEstOffset + 8 * kMaxEstBuckets);   // aux + the build's estimate buckets
        const size_t o_X = 0, o_A = o_X + b_X, o_pc = o_A + b_A, o_G = o_pc + b_pc, o_mk = o_G + b_G,
                     o_aux = o_mk + b_mk, o_B = o_aux + b_aux;
        char *arena = static_cast<char *>(own(dev_alloc(o_B + b_B, s)));
        idx->arena = arena;
        uint32_t *A = reinterpret_cast<uint32_t *>(arena + o_A);
        uint32_t *pcell = reinterpret_cast<uint32_t *>(arena + o_pc);
        uint64_t *B = reinterpret_cast<uint64_t *>(arena + o_B);
        uint32_t *G = reinterpret_cast<uint32_t *>(arena + o_G);
        double *X = reinterpret_cast<double *>(arena + o_X);
        uint64_t *ccoord = nullptr;
        uint32_t *cmask = nullptr;
        uint32_t *small_masks = reinterpret_cast<uint32_t *>(arena + o_mk);
        // aux: [0] = |G|, [1] = #dense tasks, [2] = #populous cells, [3] = bucket-sort overflow
        uint32_t *aux = reinterpret_cast<uint32_t *>(arena + o_aux);
        const uint64_t hcap = std::max<uint64_t>((uint64_t)std::max(dir_cap_mult(), kFullDirMult) * n, 1ull << 16);
        const size_t s_k = al(8 * n), s_i = al(4 * n), s_h = al(4 * (hcap + 2));
        // the build's temporaries: the per-device cached scratch buffer (released after the final
        // stream sync below), else pool memory.  Layout: [bucket histogram | keys | keys_tmp/items |
        // ids_tmp | flags].  The histogram sits at
        // offset 0 and every build leaves it zero (the bucket path's finish kernel re-zeroes the cursors
        // it used), so a reused scratch buffer needs no zeroing pass; `zero` is the known-zero prefix.
        // (The bucket path leaves cells-per-bucket there; the directory scan consumes and zeroes it.)
        struct BuildScratch {
            int dev;
            char *p = nullptr;
            bool cached = false;
            size_t zero = 0, leave_zero = 0;
            cudaStream_t s;
            BuildScratch(int d, size_t bytes, cudaStream_t st) : dev(d), s(st)
            {
                p = static_cast<char *>(scratch_acquire(dev, bytes, &zero));
                cached = p != nullptr;
                if (!cached) {
                    p = static_cast<char *>(dev_alloc(bytes, s));
                    zero = 0;
                }
            }
            ~BuildScratch()
            {
                if (cached) {
                    if (!leave_zero) cudaStreamSynchronize(s);   // (a completed build ends synced)
                    scratch_release(dev, p, leave_zero);
                } else {
                    dev_free(p, s);
                }
            }
        } scratch(o.device, s_h + 2 * s_k + 2 * s_i, s);
        uint32_t *bhist = reinterpret_cast<uint32_t *>(scratch.p);
        uint64_t *keys = reinterpret_cast<uint64_t *>(scratch.p + s_h);
        uint64_t *keys_tmp = reinterpret_cast<uint64_t *>(scratch.p + s_h + s_k);
        uint32_t *ids_tmp = reinterpret_cast<uint32_t *>(scratch.p + s_h + 2 * s_k);
        uint32_t *flags = reinterpret_cast<uint32_t *>(scratch.p + s_h + 2 * s_k + s_i);
        if (scratch.zero < s_h) SJ_CUDA(cudaMemsetAsync(bhist, 0, s_h, s));
        // ---- a1: exact per-dimension min/max + finiteness (one kernel, integer atomics), then the
        // geometry on the device (k_geometry) and the key pass right behind it; the host reads the
        // geometry (one small D2H copy, waited on by an event) while the key pass runs.
        // grid: a multiple of 3 and 5 CTAs (so the thread count is a multiple of d), <= 1020 partials
        // one wave: <= 4 resident CTAs per SM (__launch_bounds__(256, 4)), a multiple of 15
        const uint32_t pcap = std::max<uint32_t>(15u, std::min<uint32_t>(1020u, (uint32_t)(4 * nsm) / 15u * 15u));
        uint32_t parts = (uint32_t)std::min<uint64_t>((n * d + kThreads * 16 - 1) / (kThreads * 16), pcap);
        parts = std::max<uint32_t>(15u, (parts + 14u) / 15u * 15u);
        parts = std::min<uint32_t>(parts, pcap);
        // min/max partials, the device geometry and the last-CTA counter live in the context's slots
        unsigned long long *part = static_cast<unsigned long long *>(cg.c->d_slots);
        DevGeom *dgeom = reinterpret_cast<DevGeom *>(static_cast<char *>(cg.c->d_slots) + kGeomOffset);
        unsigned int *done = reinterpret_cast<unsigned int *>(static_cast<char *>(cg.c->d_slots) + kGeomOffset + 4096 - 16);
        DevIndex ix{};
        ix.d = d;
        ix.n = N;
        BuildArgs ba;
        ba.pts = pts;
        ba.n = N;
        ba.mm = part;
        ba.done = done;
        ba.eps = eps;
        ba.allow_bucket = allow_bucket ? 1 : 0;
        ba.want_masks = o.build_masks ? 1 : 0;
        ba.geom = dgeom;
        ba.zero_words = small_masks;            // small masks, aux and the build's estimate buckets
        ba.nzero = (uint32_t)((b_mk + b_aux) / 4);
        // the input is read three times (min/max, keys, the gather's random rows): keep it in L2 as
        // persisting lines until the gather is enqueued (library stream only: a caller's stream keeps
        // its own attributes)
        l2p = !o.stream;
        if (l2p) l2_persist_begin(o.device, s, pts, sizeof(double) * n * d);
        // the geometry comes back through mapped pinned memory + a doorbell the host polls (no
        // stream operation between the min/max pass and the key pass: see geometry_block)
        DevGeom *hgeom = static_cast<DevGeom *>(cg.c->h_slots);
        volatile uint32_t *hbell = reinterpret_cast<volatile uint32_t *>(static_cast<char *>(cg.c->h_slots) + kBellOffset);
        {
            void *dh = nullptr;
            SJ_CUDA(cudaHostGetDevicePointer(&dh, cg.c->h_slots, 0));
            ba.hgeom = static_cast<DevGeom *>(dh);
            ba.hbell = reinterpret_cast<volatile uint32_t *>(static_cast<char *>(dh) + kBellOffset);
            ba.epoch = ++cg.c->doorbell;
        }
        cudaStream_t s_side = cg.c->streams[1];
        launch(d, 0, dim3(parts), s, ix, ba);
        tr.dev("minmax + geometry", s);

        tr.mark("minmax + geometry enqueued");
        const dim3 grid((unsigned)((n + kThreads - 1) / kThreads));

        // ---- a2: keys (+ small masks, + prefix histogram of the bucket sort)
        ba.keys = keys;
        ba.ids = A;
        ba.masks = small_masks;
        ba.geom = dgeom;
        ba.bhist = bhist;
        launch(d, 1, grid, s, ix, ba);
        ev.rec(2, s);
        ev.rec(3, s);
        SJ_CUDA(cudaEventRecord(cg.c->events[2], s));          // keys (and the small masks) done
        tr.dev("keys", s);
        if (debug_sync()) { SJ_CUDA(cudaStreamSynchronize(s)); std::fprintf(stderr, "[sj-debug] keys ok\n"); }
        tr.mark("minmax/geometry/keys enqueued");
        {
            // poll the doorbell (the stream is queried now and then, so a failed launch is reported
            // instead of waited for)
            uint64_t spins = 0;
            while (*hbell != ba.epoch) {
                if ((++spins & 255u) == 0) {
                    const cudaError_t e = cudaStreamQuery(s);
                    if (e == cudaSuccess) break;
                    if (e != cudaErrorNotReady) SJ_CUDA(e);
                }
            }
            if (*hbell != ba.epoch) {           // (the stream drained without ringing: read it back)
                SJ_CUDA(cudaMemcpy(hgeom, dgeom, sizeof(DevGeom), cudaMemcpyDeviceToHost));
            }
            std::atomic_thread_fence(std::memory_order_acquire);
        }
        tr.mark("geometry read");
        const DevGeom hg = *const_cast<const DevGeom *>(hgeom);
        if (hg.status == 1) fail(SJ_ERR_NONFINITE, "a coordinate is NaN or infinite");

        sj_index_view v{};
        v.d = d;
        v.device = o.device;
        v.n = n;
        v.eps = eps;
        {
            volatile double e2 = eps * eps;
            v.eps2 = e2;
        }
        {
            double h_mm[2 * SJ_MAX_DIM];
            for (int j = 0; j < d; ++j) {
                h_mm[j] = hg.mins[j];
                v.mins[j] = hg.mins[j];
            }
            for (int j = 0; j < d; ++j) h_mm[d + j] = hg.maxs[j];
            host_geometry(d, eps, h_mm, h_mm + d, v);   // throws SJ_ERR_KEY_OVERFLOW like the device
        }
        bool same = hg.status == 0 && hg.w == v.w && hg.key_bits == v.key_bits;
        for (int j = 0; j < d; ++j) same = same && hg.cpd[j] == v.cpd[j] && hg.strides[j] == v.strides[j];
        if (!same) fail(SJ_ERR_CUDA, "device and host geometry disagree (internal error)");

        ix.w = v.w;
        ix.eps2 = v.eps2;
        for (int j = 0; j < d; ++j) {
            ix.mins[j] = v.mins[j];
            ix.cpd[j] = v.cpd[j];
            ix.strides[j] = v.strides[j];
        }
        // masks: one bitmap, |g_j| bits per dimension, only when <= 2^30 bits (they never change S);
        // small ones were built by the key pass, larger ones by one more pass over the points
        uint64_t mask_total = 0;
        bool want_masks = o.build_masks != 0;
        for (int j = 0; j < d; ++j) {
            v.mask_offsets[j] = mask_total;
            mask_total += v.cpd[j];
            if (mask_total > (1ull << 30)) want_masks = false;
        }
        v.mask_offsets[d] = mask_total;
        for (int j = 0; j <= d; ++j) ix.mask_off[j] = v.mask_offsets[j];
        // packed per-cell coordinates (c_j at bit cshift[j]) when the widths fit 64 bits
        bool pack_fits = true;
        {
            uint32_t sh = 0;
            for (int j = 0; j < d; ++j) {
                uint32_t b = 0;
                while (b < 64 && ((v.cpd[j] - 1) >> b)) ++b;
                ix.cbits[j] = b;
                ix.cshift[j] = sh;
                sh += b;
            }
            pack_fits = sh <= 64;
        }
        // (the refine decodes a cell's coordinates from its key and tests the small masks directly:
        // no per-cell coordinate / mask arrays -- 24 B per cell less to write and read)
        (void)pack_fits;
        ccoord = nullptr;
        cmask = nullptr;
        const DirPlan dp = plan_dir(v);
        apply_dir_geometry(ix, v, dp);
        // a3 strategy: sparse keys (<= 2 points per top-k prefix on average, P <= 2^22 so the
        // bucket arrays stay L2-sized; measured slower than LSD at P = 11.4 M) -> prefix buckets +
        // per-bucket sort; otherwise stable LSD radix sort.  (Same rule as k_geometry's.)
        const bool use_bucket = allow_bucket && dp.k >= 1 && (double)n <= 2.0 * (double)dp.P &&
                                dp.P <= (1ull << 22) && v.key_bits <= 62 && bucket_items_pack(dp.div, N);
        if (use_bucket != (hg.use_bucket != 0) || dp.P != hg.P || dp.k != hg.k)
            fail(SJ_ERR_CUDA, "device and host directory plans disagree (internal error)");
        uint32_t *masks = nullptr;
        if (want_masks) {
            if (hg.masks_on) {
                masks = small_masks;
            } else {
                const size_t mask_bytes = 4 * ((mask_total + 31) / 32);
                masks = static_cast<uint32_t *>(own(dev_alloc(mask_bytes, s)));
                SJ_CUDA(cudaMemsetAsync(masks, 0, mask_bytes, s));
                ix.mask_off[0] = v.mask_offsets[0];
                ba.masks = masks;
                launch(d, 3, grid, s, ix, ba);
            }
        }
        // are the masks trivial (finish_aux reads aux[4])?  A one-CTA check on the side stream,
        // off the critical path; s joins it before its final copy
        bool mask_check = false;
        // with the speculative estimate, its publishing CTA checks the masks (no side kernel)
        const bool spec_early = v.key_bits <= 62 && o.speculative_estimate;
        if (masks && masks == small_masks && !spec_early) {
            DevIndex mx = ix;
            mx.masks = masks;
            SJ_CUDA(cudaStreamWaitEvent(s_side, cg.c->events[2], 0));
            launch_masks_full(mx, aux + 4, s_side);
            SJ_CUDA(cudaEventRecord(cg.c->events[3], s_side));
            mask_check = true;
        }
        tr.mark("geometry + allocs");
        idx->view = v;
        alloc_dir(idx, dp, s);
        tr.dev("alloc dir", s);
        uint32_t *dir = const_cast<uint32_t *>(idx->dev.dir);

        Scratch<uint32_t> dirhist;
        ix.masks = masks;
        ix.occ = idx->dev.occ;
        ix.occ2 = idx->dev.occ2;
        ix.dir = idx->dev.dir;
        if (use_bucket) {
            // ---- a3, prefix buckets: scatter by top-k prefix, each bucket sorted by (key, id) (=
            // the stable order, R14); the sort also numbers each bucket's cells: pcell = cell index
            // within the bucket, bhist = cells per bucket, whose exclusive scan IS the directory
            bucket_sort_pairs(keys, A, keys_tmp, ids_tmp, N, dp.div, dp.P, bhist, aux + 3, pcell, bhist, s);
            exclusive_scan_u32_consume(bhist, dir, (uint64_t)dp.P + 1, s);    // (leaves bhist zero)
            tr.dev("bucket sort + dir scan", s);
            SJ_CUDA(cudaMemcpyAsync(aux, dir + dp.P, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
            ev.rec(4, s);
            // ---- a4: compaction (cell = directory entry of its prefix + index within the bucket),
            // B, G, SoA gather, occupancy bits
            ba.keys = keys;
            ba.A = A;
            ba.pcell = pcell;
            ba.B = B;
            ba.G = G;
            ba.X = X;
            ba.ccoord = ccoord;
            ba.cmask = cmask;
            ba.ndense = aux + 2;
            ba.dirhist = nullptr;
            ba.bucket_cells = true;
            ba.dir_inv = 1.0 / (double)dp.div;
            ba.occ = const_cast<uint32_t *>(ix.occ);
            launch(d, 2, grid, s, ix, ba);
            tr.dev("compact", s);
        } else {
            // ---- a3: stable LSD radix sort of (key, id) (reading R14)
            bool in_tmp = false;
            radix_sort_pairs(keys, A, keys_tmp, ids_tmp, N, v.key_bits, s, &in_tmp);
            const uint64_t *skeys = in_tmp ? keys_tmp : keys;
            if (in_tmp) SJ_CUDA(cudaMemcpyAsync(A, ids_tmp, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
            ev.rec(4, s);
            tr.mark("sort enqueued");
            if (debug_sync()) { SJ_CUDA(cudaStreamSynchronize(s)); std::fprintf(stderr, "[sj-debug] sort ok\n"); }
            // ---- a4: cell numbering (heads + scan), compaction, SoA gather, directory histogram,
            // occupancy bits.  B and G are sized for the upper bound N cells so no host round trip is
            // needed here; |G| is read back by the single sync of finish_aux.
            k_heads<<<grid, kThreads, 0, s>>>(skeys, N, flags);
            SJ_LAUNCHED();
            if (debug_sync()) { SJ_CUDA(cudaStreamSynchronize(s)); std::fprintf(stderr, "[sj-debug] heads ok\n"); }
            inclusive_scan_u32(flags, pcell, n, s);
            if (debug_sync()) { SJ_CUDA(cudaStreamSynchronize(s)); std::fprintf(stderr, "[sj-debug] scan ok\n"); }
            SJ_CUDA(cudaMemcpyAsync(aux, pcell + (n - 1), sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
            dirhist.p = dalloc<uint32_t>((size_t)dp.P + 1, s);
            dirhist.s = s;
            SJ_CUDA(cudaMemsetAsync(dirhist.p, 0, sizeof(uint32_t) * ((size_t)dp.P + 1), s));
            ba.keys = const_cast<uint64_t *>(skeys);
            ba.A = A;
            ba.pcell = pcell;
            ba.B = B;
            ba.G = G;
            ba.X = X;
            ba.ccoord = ccoord;
            ba.cmask = cmask;
            ba.ndense = aux + 2;
            ba.dirhist = dirhist.p;
            ba.bucket_cells = false;
            ba.dir_inv = 1.0 / (double)dp.div;
            ba.occ = const_cast<uint32_t *>(ix.occ);
            launch(d, 2, grid, s, ix, ba);
            tr.dev("compact", s);
        }
        if (l2p) l2_persist_stop(o.device, s);
        ix.ccoord = ccoord;
        ix.cmask = cmask;
        ev.rec(5, s);
        tr.mark("compaction enqueued");
        if (debug_sync()) { SJ_CUDA(cudaStreamSynchronize(s)); std::fprintf(stderr, "[sj-debug] compaction ok\n"); }

        v.n_cells = n;            // provisional upper bound until finish_aux() reads |G|
        v.B = B;
        v.G = G;
        v.A = A;
        v.pcell = pcell;
        v.X = X;
        v.masks = masks;
        v.dir = ix.dir;
        ix.nG = N;
        ix.B = B;
        ix.G = G;
        ix.A = A;
        ix.pcell = pcell;
        ix.X = X;
        idx->view = v;
        idx->dev = ix;
        // LSD path: the directory from its histogram (the bucket path scanned it before compaction)
        if (dirhist.p) exclusive_scan_u32(dirhist.p, dir, (uint64_t)dp.P + 1, s);
        // a5 for the default join, speculatively, before the final sync: the provisional index
        // bounds cell ranges by N (B carries a sentinel after the last cell) and chooses the search
        // mode from N; the result is kept only if the mode from |G| is the same
        const double pavg = (double)n / (double)dp.P;
        const int prov_mode = dp.k == d ? kSearchDenseRows
                              : (pavg <= 8.0 && (double)dp.div < 4.0e15 ? kSearchCellScan : kSearchRows);
        const bool spec = v.key_bits <= 62 && o.speculative_estimate;
        EstimateShape es_spec;
        Publish pub{};
        char *h_stage = static_cast<char *>(cg.c->h_slots) + kEstOffset;
        const unsigned long long *hbk = reinterpret_cast<const unsigned long long *>(h_stage + kAuxEstOffset);
        if (spec) {
            DevIndex px = ix;
            px.search_mode = prov_mode;
            px.dense_T = 0;
            px.dense_tasks = nullptr;
            px.n_dense_tasks = 0;
            es_spec = estimate_shape(n);
            if (es_spec.nbk > kMaxEstBuckets) fail(SJ_ERR_CUDA, "estimate bucket count out of range (internal error)");
            unsigned long long *dbk = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(aux) + kAuxEstOffset);
            sj_join_opts jo;
            sj_join_opts_default(&jo);
            // the estimate's last CTA publishes aux + the buckets into the mapped staging slot (and
            // the masks-trivial flag into aux[4] first) and rings a doorbell: no D2H copy + sync
            void *dh = nullptr;
            SJ_CUDA(cudaHostGetDevicePointer(&dh, cg.c->h_slots, 0));
            pub.src = reinterpret_cast<unsigned long long *>(aux);
            pub.dst = reinterpret_cast<unsigned long long *>(static_cast<char *>(dh) + kEstOffset);
            pub.words = (uint32_t)((kAuxEstOffset + 8 * es_spec.nbk) / 8);
            pub.zero_src = 0;
            pub.bell = reinterpret_cast<volatile unsigned int *>(static_cast<char *>(dh) + kBellOffset + 64);
            pub.epoch = ++cg.c->doorbell;
            pub.masks_flag = (masks && masks == small_masks) ? aux + 4 : nullptr;
            pub.masks = masks;
            pub.d = d;
            for (int j = 0; j < d; ++j) {
                pub.mask_lo[j] = v.mask_offsets[j] + 1;
                pub.mask_hi[j] = v.mask_offsets[j] + v.cpd[j] - 2;
            }
            launch_estimate(px, o.device, jo, 0, n, es_spec, dbk, s, &pub);
            tr.dev("speculative estimate", s);
        }
        if (mask_check) SJ_CUDA(cudaStreamWaitEvent(s, cg.c->events[3], 0));
        const volatile unsigned int *est_bell =
            pub.src ? reinterpret_cast<const volatile unsigned int *>(static_cast<char *>(cg.c->h_slots) + kBellOffset + 64)
                    : nullptr;
        finish_aux(idx, s, aux, dp, nullptr, false, h_aux, h_stage,
                   kAuxEstOffset + (spec ? 8 * es_spec.nbk : 0), !mask_check && !pub.masks_flag, est_bell,
                   pub.epoch);     // the build's late host sync (or doorbell)
        if (l2p) l2_persist_end(o.device);   // s is synced: demote the input's persisting lines
        scratch.leave_zero = s_h;            // the histogram region is zero again (see BuildScratch)
        cg.idle = true;                      // s synced by finish_aux, the side stream by the geometry event
        {
            sj_index_view &vv = idx->view;
            const uint64_t nGf = vv.n_cells;
            vv.packed = arena;
            vv.off_X = o_X;
            vv.off_A = o_A;
            vv.off_pcell = o_pc;
            vv.off_G = o_G;
            vv.off_masks = (masks == small_masks) ? o_mk : UINT64_MAX;
            vv.off_B = o_B;
            vv.packed_bytes = o_B + 8 * std::min<uint64_t>(nGf + 1, n);
        }
        if (spec && !h_aux[3] && idx->dev.search_mode == prov_mode) {
            idx->spec_est_valid = true;
            idx->spec_shape = es_spec;
            idx->spec_buckets.assign(hbk, hbk + es_spec.nbk);
        }
        ev.rec(6, s);
        tr.dev("finish", s);
        tr.mark("compact+dir+dense (synced)");
        if (tr.on) std::fprintf(stderr, "[sj-trace] aux = %u %u %u %u  bucket=%d P=%llu\n", h_aux[0], h_aux[1], h_aux[2], h_aux[3], (int)use_bucket, (unsigned long long)dp.P);
        for (int i = 0; i < 7; ++i) {
            idx->tev[i] = ev.e[i];
            ev.e[i] = nullptr;
        }
    } catch (...) {
        cudaStreamSynchronize(s);
        if (l2p) {
            l2_persist_stop(o.device, s);
            l2_persist_end(o.device);
        }
        free_index_impl(idx);
        throw;
    }
    if (h_aux[3]) {
        // a prefix bucket held more than the shared-memory sorter takes: rebuild with the LSD sort
        tr.mark("bucket overflow -> LSD rebuild");
        free_index_impl(idx);
        return build_index_impl2(points, n, d, eps, o, false);
    }
    return idx;
}

void free_index_impl(sj_index *idx)
{
    if (!idx) return;
    cudaSetDevice(idx->device);
    for (int i = 0; i < idx->nbufs; ++i) dev_free(idx->bufs[i], nullptr);
    cudaDeviceSynchronize();
    for (int i = 0; i < 2; ++i) zbuf_put(idx->device, idx->zbufs[i], idx->zbytes[i]);   // zeroed + cached
    for (auto &e : idx->tev) event_put(idx->device, e);
    delete idx;
}


sj_index *import_index_impl(const sj_index_view &src, int device, bool borrow)
{
    if (src.d < 2 || src.d > SJ_MAX_DIM) fail(SJ_ERR_DIM, "d must be in [2,6]");
    if (src.n == 0 || src.n >= (1ull << 32) || src.n_cells == 0 || src.n_cells > src.n)
        fail(SJ_ERR_ARG, "inconsistent index view sizes");
    if (!src.B || !src.G || !src.A || !src.pcell || !src.X) fail(SJ_ERR_ARG, "index view has NULL arrays");
    SJ_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    SJ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    sj_index *idx = new sj_index();
    idx->device = device;
    auto own = [&](size_t bytes) { void *p = dev_alloc(bytes, s); idx->bufs[idx->nbufs++] = p; return p; };
    try {
        const uint64_t n = src.n, nG = src.n_cells;
        const int d = src.d;
        sj_index_view v = src;
        v.device = device;
        uint64_t *B;
        uint32_t *G, *A, *pcell, *masks = nullptr;
        double *X;
        if (borrow) {
            B = const_cast<uint64_t *>(src.B);
            G = const_cast<uint32_t *>(src.G);
            A = const_cast<uint32_t *>(src.A);
            pcell = const_cast<uint32_t *>(src.pcell);
            X = const_cast<double *>(src.X);
            if (src.masks && src.mask_offsets[d] > 0) masks = const_cast<uint32_t *>(src.masks);
        } else {
            B = static_cast<uint64_t *>(own(8 * nG));
            G = static_cast<uint32_t *>(own(4 * (nG + 1)));
            A = static_cast<uint32_t *>(own(4 * n));
            pcell = static_cast<uint32_t *>(own(4 * n));
            X = static_cast<double *>(own(8 * n * d));
            SJ_CUDA(cudaMemcpyAsync(B, src.B, 8 * nG, cudaMemcpyDefault, s));
            SJ_CUDA(cudaMemcpyAsync(G, src.G, 4 * (nG + 1), cudaMemcpyDefault, s));
            SJ_CUDA(cudaMemcpyAsync(A, src.A, 4 * n, cudaMemcpyDefault, s));
            SJ_CUDA(cudaMemcpyAsync(pcell, src.pcell, 4 * n, cudaMemcpyDefault, s));
            SJ_CUDA(cudaMemcpyAsync(X, src.X, 8 * n * d, cudaMemcpyDefault, s));
            if (src.masks && src.mask_offsets[d] > 0) {
                const size_t mb = 4 * ((src.mask_offsets[d] + 31) / 32);
                masks = static_cast<uint32_t *>(own(mb));
                SJ_CUDA(cudaMemcpyAsync(masks, src.masks, mb, cudaMemcpyDefault, s));
            }
            v.packed = nullptr;
            v.packed_bytes = 0;
        }
        v.B = B; v.G = G; v.A = A; v.pcell = pcell; v.X = X; v.masks = masks;
        DevIndex ix{};
        ix.d = d;
        ix.n = (uint32_t)n;
        ix.nG = (uint32_t)nG;
        ix.w = v.w;
        ix.eps2 = v.eps2;
        for (int j = 0; j < d; ++j) {
            ix.mins[j] = v.mins[j];
            ix.cpd[j] = v.cpd[j];
            ix.strides[j] = v.strides[j];
        }
        for (int j = 0; j <= d; ++j) ix.mask_off[j] = v.mask_offsets[j];
        ix.B = B; ix.G = G; ix.A = A; ix.pcell = pcell; ix.X = X; ix.masks = masks;
        const DirPlan dp = plan_dir(v);
        apply_dir_geometry(ix, v, dp);
        idx->view = v;
        idx->dev = ix;
        alloc_dir(idx, dp, s);
        uint32_t *aux = static_cast<uint32_t *>(own(4 * kAuxWords));
        const uint32_t hn[kAuxWords] = {(uint32_t)nG, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        SJ_CUDA(cudaMemcpyAsync(aux, hn, sizeof(hn), cudaMemcpyHostToDevice, s));
        // directory histogram and occupancy bits from B (the build fuses these into its compaction)
        Scratch<uint32_t> hist((size_t)dp.P + 1, s);
        SJ_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(uint32_t) * ((size_t)dp.P + 1), s));
        const uint32_t gN = (uint32_t)((nG + kThreads - 1) / kThreads);
        k_dir_hist<<<gN, kThreads, 0, s>>>(B, aux, dp.div, 1.0 / (double)dp.div, hist.p);
        SJ_LAUNCHED();
        if (idx->dev.occ) {
            uint32_t *o1 = const_cast<uint32_t *>(idx->dev.occ), *o2 = const_cast<uint32_t *>(idx->dev.occ2);
            switch (d) {
            case 2: k_occ_import<2><<<gN, kThreads, 0, s>>>(idx->dev, B, aux, o1, o2); break;
            case 3: k_occ_import<3><<<gN, kThreads, 0, s>>>(idx->dev, B, aux, o1, o2); break;
            case 4: k_occ_import<4><<<gN, kThreads, 0, s>>>(idx->dev, B, aux, o1, o2); break;
            case 5: k_occ_import<5><<<gN, kThreads, 0, s>>>(idx->dev, B, aux, o1, o2); break;
            default: k_occ_import<6><<<gN, kThreads, 0, s>>>(idx->dev, B, aux, o1, o2); break;
            }
            SJ_LAUNCHED();
        }
        uint32_t h_aux[kAuxWords];
        finish_aux(idx, s, aux, dp, hist.p, true, h_aux);
    } catch (...) {
        cudaStreamDestroy(s);
        free_index_impl(idx);
        throw;
    }
    cudaStreamDestroy(s);
    return idx;
}

}  // namespace sj
