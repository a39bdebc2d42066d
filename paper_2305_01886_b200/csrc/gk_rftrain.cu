// gk_rftrain.cu -- K5: random-forest training (RandomForestRegressor.fit as
// wrapped by gpukalc_trainer.training._make_model, training.py:73-76).
//
// Reference semantics (scikit-learn):
//  * bootstrap: counts = bincount(RandomState(tree_seed).randint(0, n, n))
//    (SK/ensemble/_forest.py:95-112, 150-156) -- reproduced bit-exactly here
//    with one MT19937 stream per tree (warp-parallel twist) and numpy's masked
//    rejection for bounded integers;
//  * squared-error trees, all features per split, min_samples_split = 2,
//    min_samples_leaf = 1, leaf value = weighted mean.
// Split search is histogram-based over u8 feature bins (quantile edges, one
// bin per distinct value when a feature has <= 256 of them), so trees are not
// identical to sklearn's exact float32 midpoints -- the parity bar for training
// is R^2 / MAPE (BASELINE.json).  Sums of w*y use 64-bit fixed point, so split
// decisions are deterministic despite atomics.
//
// Level-wise growth over a batch of trees; a "task" is one node to split:
//   rows <= 64       -> one warp: sorted keys (<= 32 rows, k5_split_sorted) or
//                       rank-compacted histograms (k5_split_rank)
//   rows <= kMedRows -> one CTA, shared-memory histograms per 16-feature chunk
//   larger           -> row-chunked CTAs accumulate global histograms, then
//                       one CTA per task evaluates (k5_hist_big + k5_eval_big)
#include <algorithm>
#include <cmath>

#include "gk_internal.cuh"

namespace gk {

constexpr int kFC = 16;          // features per histogram chunk
constexpr int kBins = 256;
constexpr int kMedRows = 32768;  // larger nodes use the multi-CTA histogram path
#ifndef GK_BIG_ROWS
#define GK_BIG_ROWS 2048  // rows per CTA of the multi-CTA histograms (GBT 1M x 64: 7.7 -> 5.4 ms/stage vs 32768)
#endif
constexpr int kBigRows = GK_BIG_ROWS;
static_assert(kMedRows % kBigRows == 0, "chunking");

struct RfTrainData {
    const uint8_t *Xb;      // [n][F] bins
    const int64_t *yfp;     // [n] y in fixed point
    const double *y;        // [n]
    const uint32_t *counts; // [n_trees][n] bootstrap counts
    int64_t n;
    int32_t F;
    int32_t rs;             // row-record stride (bytes), rec_stride(F)
};

// Row records.  A node's rows are a contiguous range of records in one of two
// ping-pong buffers, and the partition moves whole records, so every kernel
// reads its node's rows as one contiguous stream: {row id i32, bootstrap
// weight u32, w * y fixed point i64, the row's F bins (padded to 16 B)}.
// Round 2 kept row ids only and gathered the weight, target and bins of every
// row at every level from [n]-sized arrays: three random 32-byte sectors per
// row and feature chunk (ncu, level 7 of config #3: 5.8 GB of DRAM reads per
// level, 67 % of the stall samples waiting on them).
constexpr int kRecHdr = 16;
__host__ __device__ __forceinline__ int rec_stride(int F) { return kRecHdr + ((F + 15) & ~15); }
struct RecView {
    const uint8_t *p;
    __device__ __forceinline__ int32_t row() const { return *reinterpret_cast<const int32_t *>(p); }
    __device__ __forceinline__ uint32_t w() const { return *reinterpret_cast<const uint32_t *>(p + 4); }
    __device__ __forceinline__ int64_t sv() const { return *reinterpret_cast<const int64_t *>(p + 8); }
    __device__ __forceinline__ const uint8_t *bins() const { return p + kRecHdr; }
};
__device__ __forceinline__ RecView rec_at(const uint8_t *buf, int rs, int pos) {
    return RecView{buf + (size_t)pos * rs};
}

struct RfTask {             // one node to split (or one leaf to summarise)
    int32_t tree, begin, end, parity;
};

struct RfSplit {
    int32_t feat, bin, n_left, pad;
    double proxy;
};

// ---------------------------------------------------------------- bootstrap

// One CTA per tree: MT19937 (init_genrand(seed)), tempering, numpy's masked
// rejection for randint(0, n) (mask = 2^bitlen(n-1) - 1, accept v <= n-1),
// counts[v] += 1 for the first n accepted draws.  The whole forest's trees go
// in one launch (a CTA per tree fills the GPU; one warp per tree in batches of
// 16-32 trees left most SMs idle: 0.33 ms per tree).  Per 624-word round: the
// twist in its three dependency phases ([0,227) reads old words, [227,454)
// needs phase-1 results, [454,623) phase-2's, 623 needs the new mt[0]), one
// thread per word and phase; then every thread tempers its word and a
// CTA-wide ballot scan gives each accepted draw its position in the stream.
constexpr int kBootThreads = 640;  // >= 624 words, 20 warps
__global__ void __launch_bounds__(kBootThreads) k5_bootstrap(const uint32_t *__restrict__ seeds,
                                                             int n_trees, int64_t n,
                                                             uint32_t *__restrict__ counts) {
    __shared__ uint32_t mt[624];
    __shared__ int32_t wtot[kBootThreads / 32];
    const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
    const int t = blockIdx.x;
    if (t >= n_trees) return;
    uint32_t *cnt = counts + (size_t)t * n;
    const uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) {
        if (k == 0) cnt[0] = (uint32_t)n;
        return;
    }
    uint32_t mask = rng;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    if (k == 0) {  // init_genrand: a sequential recurrence, 624 steps
        uint32_t v = seeds[t];
        mt[0] = v;
        for (int i = 1; i < 624; i++) {
            v = 1812433253u * (v ^ (v >> 30)) + (uint32_t)i;
            mt[i] = v;
        }
    }
    __syncthreads();
    auto twist = [&](int i) {
        const uint32_t y = (mt[i] & 0x80000000u) | (mt[(i + 1) % 624] & 0x7fffffffu);
        return mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    };
    int64_t accepted = 0;
    while (accepted < n) {
        // phase p: words [lo_p, hi_p); each thread reads before any writes
        {
            const uint32_t v = k < 227 ? twist(k) : 0u;
            __syncthreads();
            if (k < 227) mt[k] = v;
            __syncthreads();
        }
        {
            const uint32_t v = k < 227 ? twist(227 + k) : 0u;
            __syncthreads();
            if (k < 227) mt[227 + k] = v;
            __syncthreads();
        }
        {
            const uint32_t v = k < 169 ? twist(454 + k) : 0u;
            __syncthreads();
            if (k < 169) mt[454 + k] = v;
            __syncthreads();
        }
        if (k == 0) mt[623] = twist(623);
        __syncthreads();
        uint32_t y = k < 624 ? mt[k] : 0u;
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        const uint32_t v = y & mask;
        const bool ok = k < 624 && v <= rng;
        const unsigned bal = __ballot_sync(GK_FULL, ok);
        if (lane == 0) wtot[warp] = __popc(bal);
        __syncthreads();
        int before = __popc(bal & ((1u << lane) - 1u)), total = 0;
#pragma unroll
        for (int w = 0; w < kBootThreads / 32; w++) {
            const int c = wtot[w];
            before += w < warp ? c : 0;
            total += c;
        }
        if (ok && accepted + before < n) atomicAdd(cnt + v, 1u);
        accepted += total;
        __syncthreads();  // wtot / mt reuse
    }
}

// records of the rows with count > 0, per tree, compacted (order within a
// tree is not kept): row id, weight, w * yfp, the row's bins
__global__ void k5_compact(RfTrainData D, int n_trees, const int64_t *__restrict__ tree_base,
                           uint8_t *__restrict__ recs, int32_t *__restrict__ fill) {
    const int t = blockIdx.y;
    const int64_t n = D.n;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t w = i < n ? D.counts[(size_t)t * n + i] : 0u;
    const bool in = w > 0;
    const unsigned bal = __ballot_sync(GK_FULL, in);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(bal) - 1) base = atomicAdd(fill + t, __popc(bal));
    base = __shfl_sync(GK_FULL, base, __ffs(bal) - 1);
    if (!in) return;
    uint8_t *r = recs + (size_t)(tree_base[t] + base + __popc(bal & ((1u << lane) - 1u))) * D.rs;
    const int64_t sv = (int64_t)w * D.yfp[i];
    *reinterpret_cast<int4 *>(r) = make_int4((int32_t)i, (int32_t)w, (int32_t)(uint32_t)sv,
                                             (int32_t)(sv >> 32));
    const uint8_t *xb = D.Xb + (size_t)i * D.F;
    if ((D.F & 15) == 0) {  // rows of Xb are 16-byte aligned
        for (int k = 0; k < D.F; k += 16)
            *reinterpret_cast<uint4 *>(r + kRecHdr + k) = *reinterpret_cast<const uint4 *>(xb + k);
    } else {  // the zero padding is written too (whole 16-byte groups move later)
        for (int k = 0; k < rec_stride(D.F) - kRecHdr; k++) r[kRecHdr + k] = k < D.F ? xb[k] : 0;
    }
}

// ---------------------------------------------------------------- binning

__device__ __forceinline__ uint32_t f2ord(float f) {  // order-preserving float -> uint
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Xb[r][f] = #edges < float32(X[r][f]); per-bin min/max of the float32 values
__global__ void k5_bin(const double *__restrict__ X, int64_t n, int F, int64_t ld,
                       const float *__restrict__ edges, const int32_t *__restrict__ n_edges,
                       uint8_t *__restrict__ Xb, uint32_t *__restrict__ bmin,
                       uint32_t *__restrict__ bmax) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * F) return;
    const int64_t r = i / F;
    const int f = (int)(i % F);
    const float v = (float)X[r * ld + f];  // sklearn fits on float32 X
    const float *e = edges + (size_t)f * (kBins - 1);
    int lo = 0, hi = n_edges[f];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (e[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    Xb[i] = (uint8_t)lo;
    const uint32_t o = f2ord(v);
    atomicMin(bmin + f * kBins + lo, o);
    atomicMax(bmax + f * kBins + lo, o);
}

// ------------------------------------------------------------ split search

struct BestSplit {
    double proxy;
    int feat, bin;
    uint32_t n_left;
};

__device__ __forceinline__ bool better(double p, int f, int b, const BestSplit &o) {
    return p > o.proxy || (p == o.proxy && (f < o.feat || (f == o.feat && b < o.bin)));
}

// Float bound on the MSE proxy.  The exact proxy's two IEEE fp64 divisions
// were the split search's largest instruction share (ncu, level 15 of config
// #3: ~25 % of the warp-per-node kernel's stall samples).  pf = p * 2^-64 to
// within ~1e-6 relative (each operand rounded once, __fdividef <= 2 ulp, both
// terms >= 0; an integer SL != 0 keeps every term >= 2^-96, far from float
// underflow).  A candidate whose pf is below the lane's exact best * (1 -
// 2^-12) can neither beat nor tie it, so it is skipped and the chosen split is
// unchanged; the others take the exact fp64 proxy and the (proxy, feature,
// bin) order as before.
__device__ __forceinline__ float proxy_f(int64_t SL, int64_t SR, uint32_t WL, uint32_t WR) {
    const float a = __ll2float_rn(SL) * 0x1p-32f, b = __ll2float_rn(SR) * 0x1p-32f;
    return __fdividef(a * a, __uint2float_rn(WL)) + __fdividef(b * b, __uint2float_rn(WR));
}
__device__ __forceinline__ float proxy_floor(double best) {
    return best < 0.0 ? -1.0f : __double2float_rd(best * 0x1p-64) * (1.0f - 0x1p-12f);
}
// one candidate: left = (SL, WL, CL) of a node with totals (S, W); exact
// proxy only past the float bound; thr tracks proxy_floor(best.proxy)
__device__ __forceinline__ void consider(int64_t SL, int64_t S, uint32_t WL, uint32_t W,
                                         uint32_t CL, int f, int b, BestSplit &best, float &thr) {
    if (proxy_f(SL, S - SL, WL, W - WL) < thr) return;
    const double SLd = (double)SL, SRd = (double)(S - SL);
    const double p = SLd * SLd / (double)WL + SRd * SRd / (double)(W - WL);
    if (better(p, f, b, best)) {
        best = BestSplit{p, f, b, CL};
        thr = proxy_floor(p);
    }
}

// Evaluate all boundaries of one feature's histogram with one warp:
// left = bins <= b; proxy = S_L^2 / W_L + S_R^2 / W_R (sklearn's MSE proxy).
// The candidates are the non-empty bins (an empty bin repeats the previous
// boundary's split, whose proxy ties and wins by the lower bin: exact).  The
// proxy's two fp64 divisions were a quarter of the split search's
// instructions when every one of a lane's 8 bin slots took them; sparse
// histograms now compact their candidates first.
// A histogram bin as four 32-bit words: row count, bootstrap weight, and the
// fixed-point sum of w * y split into low / high words.  B200 has no native
// 64-bit shared-memory atomic add (ATOMS.CAST.SPIN.64 CAS loops were 60 % of
// the node-split instructions); 32-bit adds are native, and the carry out of
// the low word is recovered from the returned old value -- exact.
template <bool kCnt>
struct BinsT {
    uint32_t *cnt, *wgt, *slo;
    int32_t *shi;
    // (row count << 32 | weight); without a count word (the CTA-per-node and
    // multi-CTA paths) the weight stands in for the count: every row of a
    // node has weight >= 1, so "both sides non-empty" is the same test, and
    // the split's row count comes from the partition's cursor instead
    __device__ __forceinline__ uint64_t cw(int b) const {
        return kCnt ? (((uint64_t)cnt[b] << 32) | wgt[b]) : (((uint64_t)wgt[b] << 32) | wgt[b]);
    }
    __device__ __forceinline__ int64_t sum(int b) const {
        return (int64_t)(((uint64_t)(uint32_t)shi[b] << 32) + slo[b]);
    }
    __device__ __forceinline__ void add(int b, uint32_t w, int64_t sv) const {
        if (kCnt) atomicAdd(cnt + b, 1u);
        atomicAdd(wgt + b, w);
        const uint32_t lo = (uint32_t)sv;
        const uint32_t old = atomicAdd(slo + b, lo);
        atomicAdd(shi + b, (int32_t)(sv >> 32) + (old + lo < old ? 1 : 0));
    }
    __device__ __forceinline__ void clear(int b) const {
        if (kCnt) cnt[b] = 0;
        wgt[b] = 0;
        slo[b] = 0;
        shi[b] = 0;
    }
    __device__ __forceinline__ void set(int b, uint64_t c, int64_t sv) const {
        if (kCnt) cnt[b] = (uint32_t)(c >> 32);
        wgt[b] = (uint32_t)c;
        slo[b] = (uint32_t)sv;
        shi[b] = (int32_t)(sv >> 32);
    }
};
using BinsRef = BinsT<true>;
using Bins3 = BinsT<false>;

struct CandSmem {  // one warp's compacted split candidates (<= 64)
    uint64_t c[64];
    int64_t s[64];
    uint16_t b[64];
};

template <bool kCompact, class Bins>
__device__ __forceinline__ void eval_feature(const Bins &H, int f, int lane, CandSmem *cc,
                                             BestSplit &best) {
    uint64_t c8[8];
    int64_t s8[8];
    uint64_t cacc = 0;
    int64_t sacc = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        cacc += H.cw(lane * 8 + j);
        sacc += H.sum(lane * 8 + j);
        c8[j] = cacc;
        s8[j] = sacc;
    }
    // exclusive warp scan of the per-lane totals
    uint64_t cpre = cacc;
    int64_t spre = sacc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t a = __shfl_up_sync(GK_FULL, cpre, o);
        const int64_t b = __shfl_up_sync(GK_FULL, spre, o);
        if (lane >= o) {
            cpre += a;
            spre += b;
        }
    }
    const uint64_t ctot = __shfl_sync(GK_FULL, cpre, 31);
    const int64_t stot = __shfl_sync(GK_FULL, spre, 31);
    cpre -= cacc;
    spre -= sacc;
    const uint32_t C = (uint32_t)(ctot >> 32), W = (uint32_t)ctot;
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const int b = lane * 8 + j;
        const uint32_t CL = (uint32_t)((cpre + c8[j]) >> 32);
        const bool nonempty = c8[j] != (j ? c8[j - 1] : 0ull);
        if (b < kBins - 1 && nonempty && CL >= 1 && C - CL >= 1) mask |= 1u << j;
    }
    const int n = __popc(mask);
    int off = n;  // inclusive scan of the candidate counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(GK_FULL, off, o);
        if (lane >= o) off += a;
    }
    const int total = __shfl_sync(GK_FULL, off, 31);
    float thr = proxy_floor(best.proxy);
    if (kCompact && total <= 64) {
        // sparse (every node of <= 64 rows; small medium nodes): compact the
        // candidates so each division pair runs once per candidate, <= 2
        // rounds, instead of in all 8 bin slots of the warp
        off -= n;
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (mask >> j & 1u) {
                cc->c[off] = cpre + c8[j];
                cc->s[off] = spre + s8[j];
                cc->b[off] = (uint16_t)(lane * 8 + j);
                off++;
            }
        __syncwarp();
        for (int i = lane; i < total; i += 32) {
            const uint64_t cl = cc->c[i];
            consider(cc->s[i], stot, (uint32_t)cl, W, (uint32_t)(cl >> 32), f, cc->b[i], best, thr);
        }
        __syncwarp();
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (!(mask >> j & 1u)) continue;
            const uint64_t cl = cpre + c8[j];
            consider(spre + s8[j], stot, (uint32_t)cl, W, (uint32_t)(cl >> 32), f, lane * 8 + j,
                     best, thr);
        }
    }
    // folded into this lane's best only: callers reduce the warp once per task
    // (better() is a total order, so the result is the same)
}

__device__ __forceinline__ BestSplit warp_best(BestSplit best) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        BestSplit q;
        q.proxy = __shfl_xor_sync(GK_FULL, best.proxy, o);
        q.feat = __shfl_xor_sync(GK_FULL, best.feat, o);
        q.bin = __shfl_xor_sync(GK_FULL, best.bin, o);
        q.n_left = __shfl_xor_sync(GK_FULL, best.n_left, o);
        if (better(q.proxy, q.feat, q.bin, best)) best = q;
    }
    return best;
}

// parent proxy S^2/W: a split must improve on it (else the node is pure)
__device__ __forceinline__ RfSplit make_split(const BestSplit &b, double parent) {
    RfSplit r;
    const bool ok = b.feat != 0x7fffffff && b.proxy > parent + 1e-12 * fabs(parent);
    r.feat = ok ? b.feat : -1;
    r.bin = ok ? b.bin : 0;
    r.n_left = ok ? (int32_t)b.n_left : 0;
    r.pad = 0;
    r.proxy = ok ? b.proxy : 0.0;
    return r;
}
__device__ __forceinline__ void finish_split(const BestSplit &b, double parent, RfSplit *out) {
    *out = make_split(b, parent);
}

// Partition fused into the warp-per-node split search: the warp that chose the
// split moves its node's records to the other buffer right away (left rows up
// from the node's begin, right rows down from its end, as k5_partition) and
// the split record carries n_left with pad = 1 (the level bookkeeping reads it
// instead of the partition's cursor; k5_partition skips the task).  K rows
// per lane: local row lane + 32 h.  Returns n_left.
template <int K>
__device__ __forceinline__ int warp_partition(const RfTrainData &D, const uint8_t *in_node,
                                              uint8_t *out_node, int m, int lane, int feat,
                                              int bin) {
    const unsigned below = (1u << lane) - 1u;
    int nl = 0, nr = 0;
#pragma unroll
    for (int h = 0; h < K; h++) {
        const int i = lane + 32 * h;
        const bool valid = i < m;
        const uint8_t *src = in_node + (size_t)i * D.rs;
        const bool left = valid && src[kRecHdr + feat] <= bin;
        const unsigned bl = __ballot_sync(GK_FULL, left), br = __ballot_sync(GK_FULL, valid && !left);
        if (valid) {
            const int q = left ? nl + __popc(bl & below) : m - 1 - (nr + __popc(br & below));
            const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
            uint4 *d4 = reinterpret_cast<uint4 *>(out_node + (size_t)q * D.rs);
            for (int k = 0; k < (D.rs >> 4); k++) d4[k] = s4[k];
        }
        nl += __popc(bl);
        nr += __popc(br);
    }
    return nl;
}

// the warp's chosen split: partition (when it splits) and write the record
template <int K>
__device__ __forceinline__ void warp_finish(const RfTrainData &D, const BestSplit &best,
                                            double parent, const uint8_t *in_node,
                                            uint8_t *out_node, int m, int lane, RfSplit *out) {
    RfSplit r = make_split(best, parent);  // warp-uniform (best is the warp's reduction)
    if (r.feat >= 0) {
        r.n_left = warp_partition<K>(D, in_node, out_node, m, lane, r.feat, r.bin);
        r.pad = 1;
    }
    if (lane == 0) *out = r;
}

// CTA-per-node / multi-CTA histograms: three 32-bit words per bin (weight,
// low / high word of the fixed-point sum of w * y; no row count, see BinsT)
struct HistSmem {
    uint32_t wgt[kFC][kBins];  // bootstrap weight
    uint32_t slo[kFC][kBins];  // sum of w * y (fixed point), low word
    int32_t shi[kFC][kBins];   //   high word
    BestSplit best[8];
    double parent;
    __device__ __forceinline__ Bins3 feat(int j) {
        return Bins3{nullptr, wgt[j], slo[j], shi[j]};
    }
};

#ifndef GK_ACC_BIG
#define GK_ACC_BIG 8  // rows per thread in flight, k5_hist_big (config #3: 4 -> 8, 12.1 -> 11.4 ms per 32 trees)
#endif
#ifndef GK_ACC_MED
#define GK_ACC_MED 1  // rows per thread in flight, k5_split_medium (80-register budget)
#endif
// add one task's rows [p0, p1) to the shared histograms of feature chunk fc.
// Per row: the 16 bins in one 16-byte load, then every feature's returning
// low-word atomic is issued before any dependent high-word add -- 16
// independent round trips in flight instead of a return-then-add chain per
// feature (the SASS had one ATOMS latency per feature: issue active 7 %).
template <int kAccRows>
__device__ __forceinline__ void accumulate(HistSmem &H, const RfTrainData &D,
                                           const uint8_t *__restrict__ recs, int p0, int p1,
                                           int fc) {
    const int f0 = fc * kFC, nf = min(kFC, D.F - f0);
    if (nf == kFC) {  // CTA-uniform; records are 16-byte aligned (rec_stride)
        // kAccRows records per thread in flight: all their loads, then the
        // atomics (one dependent chain per kAccRows rows)
        const int step = blockDim.x * kAccRows;
        for (int pb = p0 + threadIdx.x; pb < p1; pb += step) {
            uint4 h[kAccRows], q[kAccRows];
#pragma unroll
            for (int u = 0; u < kAccRows; u++) {
                const int p = pb + u * blockDim.x;
                if (p < p1) {
                    const uint8_t *r = recs + (size_t)p * D.rs;
                    h[u] = *reinterpret_cast<const uint4 *>(r);
                    q[u] = *reinterpret_cast<const uint4 *>(r + kRecHdr + f0);
                }
            }
#pragma unroll
            for (int u = 0; u < kAccRows; u++) {
                if (pb + u * (int)blockDim.x >= p1) continue;
                const uint32_t w = h[u].y, lo = h[u].z;
                const int32_t hi = (int32_t)h[u].w;
                const uint32_t qw[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
                uint32_t old[kFC];
#pragma unroll
                for (int j = 0; j < kFC; j++) {
                    const int b = (qw[j >> 2] >> (8 * (j & 3))) & 0xFF;
                    atomicAdd(&H.wgt[j][b], w);
                    old[j] = atomicAdd(&H.slo[j][b], lo);
                }
#pragma unroll
                for (int j = 0; j < kFC; j++) {
                    const int b = (qw[j >> 2] >> (8 * (j & 3))) & 0xFF;
                    atomicAdd(&H.shi[j][b], hi + (old[j] + lo < old[j] ? 1 : 0));
                }
            }
        }
        return;
    }
    for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const RecView R = rec_at(recs, D.rs, p);
        const uint32_t w = R.w();
        const int64_t sv = R.sv();
        const uint8_t *xb = R.bins() + f0;
        for (int j = 0; j < nf; j++) H.feat(j).add(xb[j], w, sv);
    }
}

__device__ __forceinline__ void zero_hist(HistSmem &H) {
    uint4 *a = reinterpret_cast<uint4 *>(&H.wgt[0][0]);  // the word arrays are contiguous
    for (int i = threadIdx.x; i < 3 * kFC * kBins / 4; i += blockDim.x)
        a[i] = make_uint4(0, 0, 0, 0);
}

// evaluate the kFC features in shared memory; fold into H.best[warp]
__device__ __forceinline__ void eval_chunk(HistSmem &H, int F, int fc, BestSplit &mine) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int j = warp; j < kFC; j += nwarps) {
        const int f = fc * kFC + j;
        if (f >= F) break;
        // measured: compaction costs the CTA-per-node path more than it saves
        eval_feature<false>(H.feat(j), f, lane, nullptr, mine);
    }
}

__device__ __forceinline__ void reduce_best(HistSmem &H, BestSplit mine, RfSplit *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    mine = warp_best(mine);
    if (lane == 0) H.best[warp] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        BestSplit b = H.best[0];
        for (int w = 1; w < nwarps; w++)
            if (better(H.best[w].proxy, H.best[w].feat, H.best[w].bin, b)) b = H.best[w];
        finish_split(b, H.parent, out);
    }
}

__device__ __forceinline__ void parent_proxy(HistSmem &H) {
    // totals from feature 0's histogram (every row lands in exactly one bin)
    if (threadIdx.x < 32) {
        uint64_t c = 0;
        int64_t s = 0;
        const Bins3 f0 = H.feat(0);
        for (int b = threadIdx.x; b < kBins; b += 32) {
            c += f0.cw(b);
            s += f0.sum(b);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            c += __shfl_xor_sync(GK_FULL, c, o);
            s += __shfl_xor_sync(GK_FULL, s, o);
        }
        if (threadIdx.x == 0) {
            const double S = (double)s;
            H.parent = S * S / (double)(uint32_t)c;
        }
    }
}

// Medium tasks of <= kMidRows rows: the CTA's rows are staged once in shared
// memory and each warp owns every 8th feature with its own rank-compacted
// histogram (as the warp-per-node path, k5_split_rank): no block barriers per
// feature chunk, no 64 KB zeroing, and each entry scanned is a present bin.
// Same candidates, proxies and (proxy, feature, bin) order as the 256-bin scan.
#ifndef GK_MID_ROWS
#define GK_MID_ROWS 256  // 0 disables the path (512 measured no faster than the CTA path)
#endif
constexpr int kMidRows = GK_MID_ROWS > 0 ? GK_MID_ROWS : 32;
constexpr int kMidK = kMidRows / 32;  // rows per lane
constexpr int kMidXS = 68;  // staged bin row stride (17 words: lanes' rows on distinct banks)
struct MidSmem {
    uint8_t xb[kMidRows * kMidXS];  // the node's bins (F <= 64)
    uint32_t w[kMidRows];
    int64_t s[kMidRows];
    uint32_t wgt[8][kBins], slo[8][kBins];
    int32_t shi[8][kBins];
    uint16_t cbin[8][kBins];
    uint32_t bmap[8][8], bpre[8][8];
    BestSplit best[8];
    RfSplit split;
    int32_t nl[8], nr[8];  // per-warp left / right counts of the fused partition
    unsigned long long W;
    long long S;
};

__device__ __forceinline__ void split_mid(const RfTrainData &D, const RfTask &T,
                                       const uint8_t *__restrict__ recs,
                                       uint8_t *__restrict__ out_recs, unsigned char *smem,
                                       RfSplit *out) {
    MidSmem &M = *reinterpret_cast<MidSmem *>(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = T.end - T.begin;
    const uint8_t *node = recs + (size_t)T.begin * D.rs;
    if (threadIdx.x == 0) {
        M.W = 0;
        M.S = 0;
    }
    const Bins3 hb{nullptr, M.wgt[warp], M.slo[warp], M.shi[warp]};
#pragma unroll
    for (int j = 0; j < kBins / 32; j++) hb.clear(lane + 32 * j);
    if (lane < 8) M.bmap[warp][lane] = 0u;
    __syncthreads();
    unsigned long long wsum = 0;
    long long ssum = 0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const RecView R = rec_at(node, D.rs, i);
        const uint32_t w = R.w();
        const int64_t sv = R.sv();
        M.w[i] = w;
        M.s[i] = sv;
        wsum += w;
        ssum += sv;
    }
    // stage the node's bins (one contiguous run of records): 4-byte words,
    // 17-word stride in shared memory
    const int fw = (D.F + 3) >> 2;
    for (int q = threadIdx.x; q < m * fw; q += blockDim.x) {
        const int i = q / fw, k = q - i * fw;
        reinterpret_cast<uint32_t *>(M.xb + i * kMidXS)[k] =
            reinterpret_cast<const uint32_t *>(node + (size_t)i * D.rs + kRecHdr)[k];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wsum += __shfl_xor_sync(GK_FULL, wsum, o);
        ssum += __shfl_xor_sync(GK_FULL, ssum, o);
    }
    if (lane == 0) {
        atomicAdd(&M.W, wsum);
        atomicAdd(reinterpret_cast<unsigned long long *>(&M.S), (unsigned long long)ssum);
    }
    __syncthreads();
    BestSplit best{-1.0, 0x7fffffff, 0x7fffffff, 0};
    float thr = proxy_floor(best.proxy);
    for (int f = warp; f < D.F; f += 8) {
        int bin[kMidK];
#pragma unroll
        for (int k = 0; k < kMidK; k++) {
            const int i = lane + 32 * k;
            bin[k] = i < m ? M.xb[i * kMidXS + f] : -1;
            if (bin[k] >= 0) atomicOr(&M.bmap[warp][bin[k] >> 5], 1u << (bin[k] & 31));
        }
        __syncwarp();
        const uint32_t word = lane < 8 ? M.bmap[warp][lane] : 0u;
        int pc = __popc(word);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const int a = __shfl_up_sync(GK_FULL, pc, o);
            if (lane >= o) pc += a;
        }
        const int nd = __shfl_sync(GK_FULL, pc, 7);
        if (lane < 8) M.bpre[warp][lane] = (uint32_t)(pc - __popc(word));
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kMidK; k++) {
            if (bin[k] < 0) continue;
            const int i = lane + 32 * k;
            const int q = bin[k] >> 5;
            const int rk = (int)M.bpre[warp][q] + __popc(M.bmap[warp][q] & ((1u << (bin[k] & 31)) - 1u));
            hb.add(rk, M.w[i], M.s[i]);
            M.cbin[warp][rk] = (uint16_t)bin[k];
        }
        __syncwarp();
        const int kE = (nd + 31) >> 5;  // entries per lane (warp-uniform, <= 8)
        uint64_t c8[8];
        int64_t s8[8];
        uint64_t cacc = 0;
        int64_t sacc = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (j < kE) {
                cacc += hb.cw(lane * kE + j);
                sacc += hb.sum(lane * kE + j);
            }
            c8[j] = cacc;
            s8[j] = sacc;
        }
        uint64_t cpre = cacc;
        int64_t spre = sacc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t a = __shfl_up_sync(GK_FULL, cpre, o);
            const int64_t b = __shfl_up_sync(GK_FULL, spre, o);
            if (lane >= o) {
                cpre += a;
                spre += b;
            }
        }
        const uint64_t ctot = __shfl_sync(GK_FULL, cpre, 31);
        const int64_t stot = __shfl_sync(GK_FULL, spre, 31);
        cpre -= cacc;
        spre -= sacc;
        const uint32_t Wt = (uint32_t)ctot;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int e = lane * kE + j;
            if (j >= kE || e >= nd - 1) break;
            const uint64_t cl = cpre + c8[j];
            consider(spre + s8[j], stot, (uint32_t)cl, Wt, (uint32_t)(cl >> 32), f,
                     M.cbin[warp][e], best, thr);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (j < kE && lane * kE + j < nd) hb.clear(lane * kE + j);
        if (lane < 8) M.bmap[warp][lane] = 0u;
        __syncwarp();
    }
    best = warp_best(best);
    if (lane == 0) M.best[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        BestSplit b = M.best[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)
            if (better(M.best[w].proxy, M.best[w].feat, M.best[w].bin, b)) b = M.best[w];
        const double S = (double)M.S;
        M.split = make_split(b, S * S / (double)M.W);
    }
    __syncthreads();
    // fused partition (as warp_partition, CTA-wide): one row per thread, the
    // bins from the staged tile, positions from per-warp ballot counts
    RfSplit r = M.split;
    if (r.feat >= 0) {
        const int i = threadIdx.x;  // m <= kMidRows == blockDim.x
        const bool valid = i < m;
        const bool left = valid && M.xb[i * kMidXS + r.feat] <= r.bin;
        const unsigned bl = __ballot_sync(GK_FULL, left), br = __ballot_sync(GK_FULL, valid && !left);
        if (lane == 0) {
            M.nl[warp] = __popc(bl);
            M.nr[warp] = __popc(br);
        }
        __syncthreads();
        int bL = 0, bR = 0, nL = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            bL += w < warp ? M.nl[w] : 0;
            bR += w < warp ? M.nr[w] : 0;
            nL += M.nl[w];
        }
        if (valid) {
            const unsigned below = (1u << lane) - 1u;
            const int q = left ? bL + __popc(bl & below) : m - 1 - (bR + __popc(br & below));
            const uint4 *s4 = reinterpret_cast<const uint4 *>(recs + ((size_t)T.begin + i) * D.rs);
            uint4 *d4 = reinterpret_cast<uint4 *>(out_recs + ((size_t)T.begin + q) * D.rs);
            for (int k = 0; k < (D.rs >> 4); k++) d4[k] = s4[k];
        }
        r.n_left = nL;
        r.pad = 1;
    }
    if (threadIdx.x == 0) *out = r;
}

// Medium tasks, one CTA per task, in two kernels (each with its own register
// budget and instruction footprint; both are launched over the whole medium
// list and each CTA whose task belongs to the other kernel exits at once):
//   <= kMidRows rows: k5_split_mid (staged rows, rank-compacted histograms);
//   larger: k5_split_medium (shared-memory histograms per feature chunk).
constexpr int kMedThreads = 256;
#ifndef GK_MID_MINB
#define GK_MID_MINB 4  // resident CTAs per SM of k5_split_mid (~50 KB shared memory each; 4 vs 3: -2 ms per 32 trees)
#endif
static_assert(kMidRows <= kMedThreads, "split_mid partitions one row per thread");
__global__ void __launch_bounds__(kMedThreads, GK_MID_MINB) k5_split_mid(
    RfTrainData D, const RfTask *__restrict__ tasks, const int32_t *__restrict__ task_ids,
    uint8_t *__restrict__ rows0, uint8_t *__restrict__ rows1, RfSplit *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ti = task_ids[blockIdx.x];
    const RfTask T = tasks[ti];
    if (T.end - T.begin > kMidRows) return;  // CTA-uniform: k5_split_medium's task
    split_mid(D, T, T.parity ? rows1 : rows0, T.parity ? rows0 : rows1, smem_raw, out + ti);
}

#ifndef GK_MED_MINB
#define GK_MED_MINB 3  // resident CTAs per SM of k5_split_medium (48 KB histograms each)
#endif
__global__ void __launch_bounds__(kMedThreads, GK_MED_MINB) k5_split_medium(
    RfTrainData D, const RfTask *__restrict__ tasks, const int32_t *__restrict__ task_ids,
    const uint8_t *__restrict__ rows0, const uint8_t *__restrict__ rows1,
    RfSplit *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HistSmem &H = *reinterpret_cast<HistSmem *>(smem_raw);
    const int ti = task_ids[blockIdx.x];
    const RfTask T = tasks[ti];
    if (GK_MID_ROWS > 0 && D.F <= 64 && T.end - T.begin <= kMidRows) return;  // k5_split_mid's
    const uint8_t *rows = T.parity ? rows1 : rows0;
    BestSplit mine{-1.0, 0x7fffffff, 0x7fffffff, 0};
    const int n_fc = (D.F + kFC - 1) / kFC;
    for (int fc = 0; fc < n_fc; fc++) {
        zero_hist(H);
        __syncthreads();
        accumulate<GK_ACC_MED>(H, D, rows, T.begin, T.end, fc);
        __syncthreads();
        if (fc == 0) parent_proxy(H);
        eval_chunk(H, D.F, fc, mine);
        __syncthreads();
    }
    reduce_best(H, mine, out + ti);
}

// Sibling subtraction for big tasks: the two children of a big parent that
// are both big -- the smaller builds its histogram, the larger takes the
// parent's (kept from the previous level) minus the smaller's (exact integer
// sums).  par_slot[task] = the parent's slot in the previous level's
// histogram workspace (-1: none), slot_cur[task] = the task's slot in this
// level's (-1: not big).  Children are adjacent (2 e, 2 e + 1: sibling = task ^ 1).
__device__ __forceinline__ bool derives(const RfTask *__restrict__ tasks,
                                        const int32_t *__restrict__ par_slot,
                                        const int32_t *__restrict__ slot_cur, int ti) {
    if (!par_slot || par_slot[ti] < 0) return false;
    const int tj = ti ^ 1;
    if (slot_cur[tj] < 0) return false;
    const int mi = tasks[ti].end - tasks[ti].begin, mj = tasks[tj].end - tasks[tj].begin;
    return mi > mj || (mi == mj && (ti & 1));
}

// the big list's slots (histogram workspace index) by task
__global__ void k5_big_slots(const int32_t *__restrict__ task_ids, int n_big,
                             int32_t *__restrict__ slot_cur) {
    const int bi = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi < n_big) slot_cur[task_ids[bi]] = bi;
}

// derived histograms: parent - sibling, per (task, 256-bin feature row)
__global__ void k5_hist_derive(const RfTask *__restrict__ tasks, const int32_t *__restrict__ task_ids,
                               const int32_t *__restrict__ par_slot,
                               const int32_t *__restrict__ slot_cur, int F,
                               const uint64_t *__restrict__ prev, uint64_t *__restrict__ cur) {
    const int bi = blockIdx.y;
    const int ti = task_ids[bi];
    if (!derives(tasks, par_slot, slot_cur, ti)) return;
    const size_t row = (size_t)F * kBins * 2;  // interleaved {weight, sum} per bin
    const uint64_t *p = prev + (size_t)par_slot[ti] * row;
    const uint64_t *s = cur + (size_t)slot_cur[ti ^ 1] * row;
    uint64_t *d = cur + (size_t)bi * row;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < row;
         i += (size_t)gridDim.x * blockDim.x)
        d[i] = p[i] - s[i];
}

// big tasks: CTA = (task, row chunk, feature chunk) -> global histograms,
// interleaved {weight, fixed-point sum} per bin
__global__ void __launch_bounds__(256) k5_hist_big(RfTrainData D, const RfTask *__restrict__ tasks,
                                                   const int32_t *__restrict__ task_ids,
                                                   const uint8_t *__restrict__ rows0,
                                                   const uint8_t *__restrict__ rows1,
                                                   const int32_t *__restrict__ par_slot,
                                                   const int32_t *__restrict__ slot_cur,
                                                   uint64_t *__restrict__ gh) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HistSmem &H = *reinterpret_cast<HistSmem *>(smem_raw);
    const int bi = blockIdx.z;           // index among big tasks
    if (derives(tasks, par_slot, slot_cur, task_ids[bi])) return;  // k5_hist_derive fills it
    const RfTask T = tasks[task_ids[bi]];
    const uint8_t *rows = T.parity ? rows1 : rows0;
    const int fc = blockIdx.y;
    const int p0 = T.begin + blockIdx.x * kBigRows;
    if (p0 >= T.end) return;
    const int p1 = min(T.end, p0 + kBigRows);
    zero_hist(H);
    __syncthreads();
    accumulate<GK_ACC_BIG>(H, D, rows, p0, p1, fc);
    __syncthreads();
    const int f0 = fc * kFC, nf = min(kFC, D.F - f0);
    uint64_t *dh = gh + ((size_t)bi * D.F + f0) * kBins * 2;
    for (int i = threadIdx.x; i < nf * kBins; i += blockDim.x) {
        const Bins3 hb = H.feat(i / kBins);
        const int b = i % kBins;
        const uint32_t c = hb.wgt[b];
        if (c) {
            atomicAdd((unsigned long long *)(dh + 2 * i), (unsigned long long)c);
            atomicAdd((unsigned long long *)(dh + 2 * i + 1), (unsigned long long)hb.sum(b));
        }
    }
}

__global__ void __launch_bounds__(256) k5_eval_big(RfTrainData D, const int32_t *__restrict__ task_ids,
                                                   const uint64_t *__restrict__ gh,
                                                   RfSplit *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HistSmem &H = *reinterpret_cast<HistSmem *>(smem_raw);
    const int bi = blockIdx.x;
    BestSplit mine{-1.0, 0x7fffffff, 0x7fffffff, 0};
    const int n_fc = (D.F + kFC - 1) / kFC;
    for (int fc = 0; fc < n_fc; fc++) {
        const int f0 = fc * kFC, nf = min(kFC, D.F - f0);
        const uint64_t *sh = gh + ((size_t)bi * D.F + f0) * kBins * 2;
        for (int i = threadIdx.x; i < kFC * kBins; i += blockDim.x)
            H.feat(i / kBins).set(i % kBins, i < nf * kBins ? sh[2 * i] : 0,
                                  i < nf * kBins ? (int64_t)sh[2 * i + 1] : 0);
        __syncthreads();
        if (fc == 0) parent_proxy(H);
        eval_chunk(H, D.F, fc, mine);
        __syncthreads();
    }
    reduce_best(H, mine, out + task_ids[bi]);
}

// Small nodes (<= kSmallRows = 64 rows): one warp per node, in two kernels by
// node size so that each stays small in the instruction cache.  ncu on level
// 15 of config #3 (973k nodes per 32 trees): the single kernel that held the
// all-pairs, sorted and rank-histogram forms (9.9k SASS instructions, 158 KB)
// spent 67 % of its stall samples on "no instructions".
//   <= 32 rows (k5_split_sorted): lane = feature, sorted keys (split_sorted);
//   33..64 rows (k5_split_rank): rank-compacted per-warp histograms.
// Both loop over the small list (warp-strided) and skip the other kernel's
// nodes.
constexpr int kTiny = 16;
#ifndef GK_SMALL_RPL
#define GK_SMALL_RPL 2  // rows per lane of the warp-per-node path (host SMALL = 32 x this)
#endif
constexpr int kSmallRpl = GK_SMALL_RPL;
constexpr int kSmallRows = 32 * kSmallRpl;  // host forest.SMALL
#ifndef GK_SMALL_MINB
#define GK_SMALL_MINB 6  // resident CTAs per SM of the warp-per-node kernels
#endif
constexpr int kSmallThreads = 128;

template <int N>
__device__ __forceinline__ void sort_keys(uint32_t (&k)[N]) {
#pragma unroll
    for (int size = 2; size <= N; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1)
#pragma unroll
            for (int i = 0; i < N; i++) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const uint32_t a = k[i], b = k[j];
                    const uint32_t lo = min(a, b), hi = max(a, b);
                    k[i] = up ? lo : hi;
                    k[j] = up ? hi : lo;
                }
            }
}

struct SortSmem {        // one warp's node of <= 32 rows
    int64_t s[32];       // fixed-point w * y by local row
    uint32_t w[32];      // bootstrap weight by local row
    uint32_t key[32][32];  // [position][lane]: each lane's sorted keys
};

// Nodes of <= N rows (N = 16 or 32), lane = feature: each lane packs its
// feature's (bin << 8 | row) keys, sorts them with a register bitonic network
// (80 / 240 compare-exchanges), parks them in shared memory and walks them in
// order accumulating the rows' weights and fixed-point sums; each position
// whose bin differs from the next one's is a candidate -- "left = bins <= b"
// for every distinct bin b present but the largest, with the exact integer
// sums the histogram paths form -- so the chosen split is identical to theirs.
template <int N>
__device__ __forceinline__ void split_sorted(const RfTrainData &D, int m, int lane, SortSmem &Z,
                                             uint32_t wv, int64_t sv, const uint8_t *node,
                                             uint8_t *out_node, RfSplit *out) {
    if (lane < m) {
        Z.w[lane] = wv;
        Z.s[lane] = sv;
    }
    uint32_t W = lane < m ? wv : 0u;
    int64_t S = lane < m ? sv : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        W += __shfl_xor_sync(GK_FULL, W, o);
        S += __shfl_xor_sync(GK_FULL, S, o);
    }
    const double parent = (double)S * (double)S / (double)W;
    BestSplit best{-1.0, 0x7fffffff, 0x7fffffff, 0};
    float thr = -1.0f;
    __syncwarp();
#pragma unroll 1
    for (int f0 = 0; f0 < D.F; f0 += 32) {
        const int f = f0 + lane;
        const bool fv = f < D.F;
        uint32_t k[N];
#pragma unroll
        for (int j = 0; j < N; j++) {
            // rows past m sort last (key 0xFFFF.. > any bin << 8 | row); the
            // node's records are contiguous: row j's bin f is one coalesced
            // byte per lane
            k[j] = (j < m && fv) ? ((uint32_t)node[(size_t)j * D.rs + kRecHdr + f] << 8) | (uint32_t)j
                                 : 0xFFFFFFFFu;
        }
        sort_keys<N>(k);
        __syncwarp();  // the previous feature group's reads of Z.key are done
#pragma unroll
        for (int j = 0; j < N; j++) Z.key[j][lane] = k[j];
        __syncwarp();
        if (fv) {
            uint32_t WL = 0, CL = 0;
            int64_t SL = 0;
            uint32_t cur = k[0];
            for (int p = 0; p + 1 < m; p++) {  // the last present row closes no candidate
                const uint32_t nxt = Z.key[p + 1][lane];
                const int idx = (int)(cur & 0xFFu);
                WL += Z.w[idx];
                SL += Z.s[idx];
                CL++;
                const uint32_t b = cur >> 8;
                if ((nxt >> 8) != b && b < (uint32_t)(kBins - 1))
                    consider(SL, S, WL, W, CL, f, (int)b, best, thr);
                cur = nxt;
            }
        }
    }
    best = warp_best(best);
    warp_finish<1>(D, best, parent, node, out_node, m, lane, out);
}

// one kernel per network size (<= 16 rows, 17..32 rows): each keeps one sort
// network in the instruction cache (ncu, level 15: the kernel holding both
// spent 25 % of its stall samples on instruction fetch)
template <int N>
__global__ void __launch_bounds__(kSmallThreads, GK_SMALL_MINB) k5_split_sorted(
    RfTrainData D, const RfTask *__restrict__ tasks, const int32_t *__restrict__ task_ids,
    int n_ids, uint8_t *__restrict__ rows0, uint8_t *__restrict__ rows1,
    RfSplit *__restrict__ out) {
    __shared__ SortSmem Z[kSmallThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = gridDim.x * (kSmallThreads / 32);
    for (int wi = blockIdx.x * (kSmallThreads / 32) + wib; wi < n_ids; wi += nw) {
        const int ti = task_ids[wi];
        const RfTask T = tasks[ti];
        const int m = T.end - T.begin;
        if (m > N || m <= (N == 32 ? kTiny : 0)) continue;  // warp-uniform: another kernel's node
        const uint8_t *node = (T.parity ? rows1 : rows0) + (size_t)T.begin * D.rs;
        uint8_t *out_node = (T.parity ? rows0 : rows1) + (size_t)T.begin * D.rs;
        uint32_t wv = 0u;
        int64_t sv = 0;
        if (lane < m) {
            const uint4 h = *reinterpret_cast<const uint4 *>(node + (size_t)lane * D.rs);
            wv = h.y;
            sv = (int64_t)(((uint64_t)h.w << 32) | h.z);
        }
        split_sorted<N>(D, m, lane, Z[wib], wv, sv, node, out_node, out + ti);
        __syncwarp();  // Z reuse by the warp's next node
    }
}

#ifndef GK_SMALL_RADIX
#define GK_SMALL_RADIX 1  // 33..64 rows: lane-per-feature radix (0: warp-per-feature rank histograms)
#endif
// Nodes of 33..64 rows: lane = feature, as split_sorted, with each lane's
// keys ordered by a two-pass LSD radix sort on the bin's nibbles in shared
// memory ([position][lane] columns, 16-bit keys bin << 8 | row) and the 16
// digit counters packed 8 bits wide in four registers (no shared-memory
// read-modify-write chains).  The warp-per-feature rank histograms it
// replaces spent ~20k warp instructions per node (64 features one after the
// other, 2 rows per lane); here one warp instruction serves 32 features.
// Same candidates (every present bin but the largest, left = bins <= b),
// exact integer sums and proxies, so the chosen split is identical.
struct Cnt16 {  // 16 counters of <= 255, 8 bits each
    uint32_t c[4];
    __device__ __forceinline__ void zero() { c[0] = c[1] = c[2] = c[3] = 0u; }
    __device__ __forceinline__ void inc(uint32_t d) {
        const uint32_t one = 1u << (8 * (d & 3u)), r = d >> 2;
        c[0] += r == 0 ? one : 0u;
        c[1] += r == 1 ? one : 0u;
        c[2] += r == 2 ? one : 0u;
        c[3] += r == 3 ? one : 0u;
    }
    __device__ __forceinline__ uint32_t take(uint32_t d) {  // value, then increment
        const uint32_t r = d >> 2, sh = 8 * (d & 3u);
        const uint32_t w = r == 0 ? c[0] : r == 1 ? c[1] : r == 2 ? c[2] : c[3];
        inc(d);
        return (w >> sh) & 0xFFu;
    }
    __device__ __forceinline__ void excl_prefix() {
        uint32_t run = 0;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const uint32_t w = c[r];
            uint32_t o = 0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                o |= run << (8 * k);
                run += (w >> (8 * k)) & 0xFFu;
            }
            c[r] = o;
        }
    }
};

struct RadixSmem {        // one warp's node of <= 64 rows
    int64_t s[64];        // fixed-point w * y by local row
    uint32_t w[64];       // bootstrap weight by local row
    uint16_t ka[64][32];  // [position][lane] keys (bin << 8 | row)
    uint16_t kb[64][32];  // the radix passes' other buffer
};

__device__ __forceinline__ void split_radix(const RfTrainData &D, int m, int lane, RadixSmem &Z,
                                            const uint8_t *node, uint8_t *out_node,
                                            RfSplit *out) {
    uint32_t W = 0u;
    int64_t S = 0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int i = lane + 32 * h;
        if (i < m) {
            const uint4 hd = *reinterpret_cast<const uint4 *>(node + (size_t)i * D.rs);
            const int64_t sv = (int64_t)(((uint64_t)hd.w << 32) | hd.z);
            Z.w[i] = hd.y;
            Z.s[i] = sv;
            W += hd.y;
            S += sv;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        W += __shfl_xor_sync(GK_FULL, W, o);
        S += __shfl_xor_sync(GK_FULL, S, o);
    }
    __syncwarp();
    const double parent = (double)S * (double)S / (double)W;
    BestSplit best{-1.0, 0x7fffffff, 0x7fffffff, 0};
    float thr = -1.0f;
#pragma unroll 1
    for (int f0 = 0; f0 < D.F; f0 += 32) {
        const int f = f0 + lane;
        const bool fv = f < D.F;
        const uint8_t *col = node + kRecHdr + (fv ? f : 0);
        // keys, and both nibbles' digit counts (each lane owns column `lane`:
        // no cross-lane hazards, no warp syncs between the passes)
        Cnt16 lo, hi;
        lo.zero();
        hi.zero();
#pragma unroll 4
        for (int j = 0; j < m; j++) {
            const uint32_t b = col[(size_t)j * D.rs];
            Z.ka[j][lane] = (uint16_t)(b << 8 | (uint32_t)j);
            lo.inc(b & 15u);
            hi.inc(b >> 4);
        }
        lo.excl_prefix();
        hi.excl_prefix();
#pragma unroll 4
        for (int j = 0; j < m; j++) {  // pass 1: low nibble, ka -> kb (stable)
            const uint32_t k = Z.ka[j][lane];
            Z.kb[lo.take((k >> 8) & 15u)][lane] = (uint16_t)k;
        }
#pragma unroll 4
        for (int j = 0; j < m; j++) {  // pass 2: high nibble, kb -> ka (stable)
            const uint32_t k = Z.kb[j][lane];
            Z.ka[hi.take(k >> 12)][lane] = (uint16_t)k;
        }
        if (fv) {
            uint32_t WL = 0, CL = 0;
            int64_t SL = 0;
            uint32_t cur = Z.ka[0][lane];
            for (int p = 0; p + 1 < m; p++) {  // the last row closes no candidate
                const uint32_t nxt = Z.ka[p + 1][lane];
                const int idx = (int)(cur & 0xFFu);
                WL += Z.w[idx];
                SL += Z.s[idx];
                CL++;
                const uint32_t b = cur >> 8;
                if ((nxt >> 8) != b && b < (uint32_t)(kBins - 1))
                    consider(SL, S, WL, W, CL, f, (int)b, best, thr);
                cur = nxt;
            }
        }
    }
    best = warp_best(best);
    warp_finish<2>(D, best, parent, node, out_node, m, lane, out);
}

__global__ void __launch_bounds__(kSmallThreads, GK_SMALL_MINB) k5_split_radix(
    RfTrainData D, const RfTask *__restrict__ tasks, const int32_t *__restrict__ task_ids,
    int n_ids, uint8_t *__restrict__ rows0, uint8_t *__restrict__ rows1,
    RfSplit *__restrict__ out) {
    static_assert(kSmallRows <= 64, "split_radix: <= 64 rows (8-bit counters, 6-bit rows)");
    __shared__ RadixSmem Z[kSmallThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = gridDim.x * (kSmallThreads / 32);
    for (int wi = blockIdx.x * (kSmallThreads / 32) + wib; wi < n_ids; wi += nw) {
        const int ti = task_ids[wi];
        const RfTask T = tasks[ti];
        const int m = T.end - T.begin;
        if (m <= 32) continue;  // warp-uniform: k5_split_sorted's node
        const uint8_t *node = (T.parity ? rows1 : rows0) + (size_t)T.begin * D.rs;
        uint8_t *out_node = (T.parity ? rows0 : rows1) + (size_t)T.begin * D.rs;
        split_radix(D, m, lane, Z[wib], node, out_node, out + ti);
        __syncwarp();  // Z reuse by the warp's next node
    }
}

// Nodes of 33..64 rows: rank-compacted histograms.  A node of <= 32 * kE rows
// has at most that many distinct bins.  A 256-bit occupancy map gives each
// present bin its rank among them, the three-word bins are indexed by rank,
// and lane l scans entries [l * kE, (l + 1) * kE) -- kE per lane instead of 8,
// every entry non-empty, so entry e is a candidate iff a later entry exists
// (then its bin is < 255 and both sides hold rows): the same candidates,
// proxies and (proxy, feature, bin) order as the 256-bin scan.
__global__ void __launch_bounds__(kSmallThreads, GK_SMALL_MINB) k5_split_rank(
    RfTrainData D, const RfTask *__restrict__ tasks, const int32_t *__restrict__ task_ids,
    int n_ids, uint8_t *__restrict__ rows0, uint8_t *__restrict__ rows1,
    RfSplit *__restrict__ out) {
    constexpr int kE = kSmallRpl;
    constexpr int kN = 32 * kE;
    constexpr int kW = kSmallThreads / 32;
    __shared__ uint32_t cwgt[kW][kN], cslo[kW][kN];
    __shared__ int32_t cshi[kW][kN];
    __shared__ uint16_t cbin[kW][kN];
    __shared__ uint32_t bmap[kW][8], bpre[kW][8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const Bins3 hb{nullptr, cwgt[wib], cslo[wib], cshi[wib]};
    const int nw = gridDim.x * kW;
    for (int wi = blockIdx.x * kW + wib; wi < n_ids; wi += nw) {
        const int ti = task_ids[wi];
        const RfTask T = tasks[ti];
        const int m = T.end - T.begin;
        if (m <= 32) continue;  // warp-uniform: k5_split_sorted's node
        const uint8_t *node = (T.parity ? rows1 : rows0) + (size_t)T.begin * D.rs;
        uint8_t *out_node = (T.parity ? rows0 : rows1) + (size_t)T.begin * D.rs;
        const uint8_t *xb[kSmallRpl];  // this lane's rows' bins (nullptr past m)
        uint32_t w[kSmallRpl];
        int64_t s[kSmallRpl];
        uint32_t W = 0;
        int64_t S = 0;
#pragma unroll
        for (int h = 0; h < kSmallRpl; h++) {
            const int i = lane + 32 * h;
            xb[h] = nullptr;
            w[h] = 0u;
            s[h] = 0;
            if (i < m) {
                const uint8_t *rp = node + (size_t)i * D.rs;
                const uint4 hd = *reinterpret_cast<const uint4 *>(rp);
                xb[h] = rp + kRecHdr;
                w[h] = hd.y;
                s[h] = (int64_t)(((uint64_t)hd.w << 32) | hd.z);
            }
            W += w[h];
            S += s[h];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            W += __shfl_xor_sync(GK_FULL, W, o);
            S += __shfl_xor_sync(GK_FULL, S, o);
        }
        const double parent = (double)S * (double)S / (double)W;
        BestSplit best{-1.0, 0x7fffffff, 0x7fffffff, 0};
        float thr = -1.0f;
#pragma unroll
        for (int j = 0; j < kE; j++) hb.clear(lane * kE + j);
        if (lane < 8) bmap[wib][lane] = 0u;
        __syncwarp();
        for (int f = 0; f < D.F; f++) {
            int bin[kSmallRpl], rk[kSmallRpl];
#pragma unroll
            for (int h = 0; h < kSmallRpl; h++) {
                bin[h] = xb[h] ? xb[h][f] : -1;
                if (bin[h] >= 0) atomicOr(&bmap[wib][bin[h] >> 5], 1u << (bin[h] & 31));
            }
            __syncwarp();
            const uint32_t word = lane < 8 ? bmap[wib][lane] : 0u;
            int pc = __popc(word);
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const int a = __shfl_up_sync(GK_FULL, pc, o);
                if (lane >= o) pc += a;
            }
            const int nd = __shfl_sync(GK_FULL, pc, 7);  // distinct bins
            if (lane < 8) bpre[wib][lane] = (uint32_t)(pc - __popc(word));
            __syncwarp();
#pragma unroll
            for (int h = 0; h < kSmallRpl; h++) {
                rk[h] = -1;
                if (bin[h] >= 0) {
                    const int k = bin[h] >> 5;
                    rk[h] = (int)bpre[wib][k] + __popc(bmap[wib][k] & ((1u << (bin[h] & 31)) - 1u));
                    hb.add(rk[h], w[h], s[h]);
                    cbin[wib][rk[h]] = (uint16_t)bin[h];
                }
            }
            __syncwarp();
            uint64_t c8[kE];
            int64_t s8[kE];
            uint64_t cacc = 0;
            int64_t sacc = 0;
#pragma unroll
            for (int j = 0; j < kE; j++) {
                cacc += hb.cw(lane * kE + j);
                sacc += hb.sum(lane * kE + j);
                c8[j] = cacc;
                s8[j] = sacc;
            }
            uint64_t cpre = cacc;
            int64_t spre = sacc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t a = __shfl_up_sync(GK_FULL, cpre, o);
                const int64_t b = __shfl_up_sync(GK_FULL, spre, o);
                if (lane >= o) {
                    cpre += a;
                    spre += b;
                }
            }
            const uint64_t ctot = __shfl_sync(GK_FULL, cpre, 31);
            const int64_t stot = __shfl_sync(GK_FULL, spre, 31);
            cpre -= cacc;
            spre -= sacc;
            const uint32_t Wt = (uint32_t)ctot;
#pragma unroll
            for (int j = 0; j < kE; j++) {
                const int e = lane * kE + j;
                if (e >= nd - 1) break;
                const uint64_t cl = cpre + c8[j];
                consider(spre + s8[j], stot, (uint32_t)cl, Wt, (uint32_t)(cl >> 32), f,
                         cbin[wib][e], best, thr);
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < kSmallRpl; h++)
                if (rk[h] >= 0) hb.clear(rk[h]);
            if (lane < 8) bmap[wib][lane] = 0u;
            __syncwarp();
        }
        best = warp_best(best);
        warp_finish<kSmallRpl>(D, best, parent, node, out_node, m, lane, out + ti);
    }
}

// ---------------------------------------------------------------- partition

// CTA = (task, 256-position chunk); the records of split tasks move to the
// other buffer: left rows up from `begin`, right rows down from `end` (so no
// row count is needed up front); the final left cursor is the split's n_left,
// read by the next-level bookkeeping (k5_level_emit)
__global__ void __launch_bounds__(256) k5_partition(RfTrainData D, const RfTask *__restrict__ tasks,
                                                    const RfSplit *__restrict__ split,
                                                    const int32_t *__restrict__ task_ids,
                                                    const uint8_t *__restrict__ rows0,
                                                    uint8_t *__restrict__ rows1_out0,
                                                    const uint8_t *__restrict__ rows1,
                                                    uint8_t *__restrict__ rows0_out1,
                                                    int32_t *__restrict__ cursor) {
    const int ti = task_ids[blockIdx.x];  // tasks on x (can exceed 65535), chunks on y
    const RfTask T = tasks[ti];
    if (T.begin + (int)(blockIdx.y * blockDim.x) >= T.end) return;  // whole CTA past the node
    const RfSplit sp = split[ti];
    if (sp.feat < 0 || sp.pad == 1) return;  // kept as a leaf / partitioned by its split search
    const uint8_t *in = T.parity ? rows1 : rows0;
    uint8_t *outp = T.parity ? rows0_out1 : rows1_out0;
    const int p = T.begin + blockIdx.y * blockDim.x + threadIdx.x;
    const bool valid = p < T.end;
    const uint8_t *src = in + (size_t)p * D.rs;
    const bool left = valid && src[kRecHdr + sp.feat] <= sp.bin;
    const bool right = valid && !left;
    const int lane = threadIdx.x & 31;
    const unsigned bl = __ballot_sync(GK_FULL, left), br = __ballot_sync(GK_FULL, right);
    int lb = 0, rb = 0;
    if (lane == 0) {
        if (bl) lb = atomicAdd(cursor + 2 * ti, __popc(bl));
        if (br) rb = atomicAdd(cursor + 2 * ti + 1, __popc(br));
    }
    lb = __shfl_sync(GK_FULL, lb, 0);
    rb = __shfl_sync(GK_FULL, rb, 0);
    const unsigned below = (1u << lane) - 1u;
    if (!valid) return;
    const int q = left ? T.begin + lb + __popc(bl & below) : T.end - 1 - (rb + __popc(br & below));
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(outp + (size_t)q * D.rs);
    for (int k = 0; k < (D.rs >> 4); k++) d4[k] = s4[k];
}

// ---------------------------------------------------------------- next level
//
// Level bookkeeping on the device (it was numpy on the host, ~3/4 of a fit's
// wall time).  Tasks of a level are sorted by tree.  A split task i gets its
// children at 2 * excl[i], 2 * excl[i] + 1 of the next level (excl = number of
// split tasks before i: task order, as the host did) and the BFS ids
// lid = next_id[tree] + 2 * (rank of i among its tree's split tasks), i.e.
// lid_base[tree] + 2 * excl[i] with lid_base = next_id - 2 * (splits of the
// earlier trees).  Children are classified for the next level's split search
// (small / medium / big lists; a child with < 2 rows or at max depth is in no
// list and stays a leaf).  The lists are appended with warp-aggregated
// atomics, so their order varies from run to run; every kernel that reads them
// writes per-task results, so trees do not.
constexpr int kLvlThreads = 256;

enum : int {  // stats[] slots (int32)
    kStNext = 0, kStSmall = 1, kStMed = 2, kStBig = 3, kStMaxMed = 4, kStMaxBig = 5
};

__global__ void __launch_bounds__(kLvlThreads) k5_level_count(const RfTask *__restrict__ tasks,
                                                              const RfSplit *__restrict__ split,
                                                              int n_tasks,
                                                              int32_t *__restrict__ block_cnt,
                                                              int32_t *__restrict__ tree_cnt) {
    const int i = blockIdx.x * kLvlThreads + threadIdx.x;
    const bool s = i < n_tasks && split[i].feat >= 0;
    const int c = __syncthreads_count(s);
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = c;
    const int tree = s ? tasks[i].tree : -1;
    const unsigned act = __ballot_sync(GK_FULL, s);
    if (s) {
        const unsigned peers = __match_any_sync(act, tree);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(tree_cnt + tree, __popc(peers));
    }
}

// one CTA: exclusive scans of the per-block and per-tree split counts
__global__ void __launch_bounds__(1024) k5_level_scan(int32_t *__restrict__ block_cnt, int n_blocks,
                                                      const int32_t *__restrict__ tree_cnt,
                                                      int n_trees, int32_t *__restrict__ next_id,
                                                      int32_t *__restrict__ lid_base,
                                                      int32_t *__restrict__ stats) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto scan = [&](const int32_t *a, int n, auto &&emit) {
        if (threadIdx.x == 0) carry = 0;
        __syncthreads();
        for (int b0 = 0; b0 < n; b0 += 1024) {
            const int i = b0 + threadIdx.x;
            const int32_t v = i < n ? a[i] : 0;
            int32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(GK_FULL, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {
                int32_t w = wsum[lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(GK_FULL, w, o);
                    if (lane >= o) w += y;
                }
                wsum[lane] = w;  // inclusive over warps
            }
            __syncthreads();
            const int32_t excl = carry + (warp ? wsum[warp - 1] : 0) + x - v;
            if (i < n) emit(i, excl, v);
            __syncthreads();
            if (threadIdx.x == 0) carry += wsum[31];
            __syncthreads();
        }
    };
    scan(block_cnt, n_blocks, [&](int i, int32_t excl, int32_t) { block_cnt[i] = excl; });
    if (threadIdx.x == 0) stats[kStNext] = 2 * carry;
    __syncthreads();
    scan(tree_cnt, n_trees, [&](int t, int32_t excl, int32_t v) {
        lid_base[t] = next_id[t] - 2 * excl;
        next_id[t] += 2 * v;
    });
}

__device__ __forceinline__ void append_class(int cls, int k, int32_t *__restrict__ lists, int cap,
                                             int32_t *__restrict__ stats, int size) {
    // warp-aggregated appends: one atomic per (warp, class); every lane calls
#pragma unroll
    for (int c = 0; c < 3; c++) {
        const unsigned m = __ballot_sync(GK_FULL, cls == c);
        if (!m) continue;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(stats + kStSmall + c, __popc(m));
        base = __shfl_sync(GK_FULL, base, leader);
        if (cls == c) lists[c * cap + base + __popc(m & ((1u << lane) - 1u))] = k;
    }
    if (cls == 1) atomicMax(stats + kStMaxMed, size);
    if (cls == 2) atomicMax(stats + kStMaxBig, size);
}

__global__ void __launch_bounds__(kLvlThreads) k5_level_emit(
    const RfTask *__restrict__ tasks, const int32_t *__restrict__ node,
    const RfSplit *__restrict__ split, int n_tasks, const int32_t *__restrict__ block_excl,
    const int32_t *__restrict__ lid_base, const int32_t *__restrict__ cursor, int child_depth,
    int max_depth, int32_t *__restrict__ lid_out, RfTask *__restrict__ tasks_next,
    int32_t *__restrict__ node_next, int32_t *__restrict__ lists, int cap,
    int32_t *__restrict__ stats, const int32_t *__restrict__ slot_cur,
    int32_t *__restrict__ par_slot_next) {
    __shared__ int32_t wsum[kLvlThreads / 32];
    const int i = blockIdx.x * kLvlThreads + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool valid = i < n_tasks;
    const RfSplit sp = valid ? split[i] : RfSplit{-1, 0, 0, 0, 0.0};
    const bool s = sp.feat >= 0;
    const unsigned bal = __ballot_sync(GK_FULL, s);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0;
#pragma unroll
    for (int w = 0; w < kLvlThreads / 32; w++) before += w < warp ? wsum[w] : 0;
    const int excl = block_excl[blockIdx.x] + before + __popc(bal & ((1u << lane) - 1u));
    int cls_l = -1, cls_r = -1, sz_l = 0, sz_r = 0;
    if (s) {
        const RfTask T = tasks[i];
        const int32_t lid = lid_base[T.tree] + 2 * excl;
        lid_out[i] = lid;
        // the partition's final left count (the fused warp / mid partitions
        // leave it in the split record)
        const int n_left = sp.pad == 1 ? sp.n_left : cursor[2 * i];
        const int mid = T.begin + n_left;
        tasks_next[2 * excl] = RfTask{T.tree, T.begin, mid, 1 - T.parity};
        tasks_next[2 * excl + 1] = RfTask{T.tree, mid, T.end, 1 - T.parity};
        node_next[2 * excl] = lid;
        node_next[2 * excl + 1] = lid + 1;
        if (par_slot_next) {  // the children's parent histogram (sibling subtraction)
            const int32_t ps = slot_cur ? slot_cur[i] : -1;
            par_slot_next[2 * excl] = ps;
            par_slot_next[2 * excl + 1] = ps;
        }
        sz_l = n_left;
        sz_r = T.end - mid;
        const bool deep_ok = child_depth < max_depth;
        cls_l = (deep_ok && sz_l >= 2) ? (sz_l > kSmallRows) + (sz_l > kMedRows) : -1;
        cls_r = (deep_ok && sz_r >= 2) ? (sz_r > kSmallRows) + (sz_r > kMedRows) : -1;
    } else if (valid) {
        lid_out[i] = -1;
    }
    append_class(cls_l, 2 * excl, lists, cap, stats, sz_l);
    append_class(cls_r, 2 * excl + 1, lists, cap, stats, sz_r);
}

// ---------------------------------------------------------------- leaf stats

// leaf segments: n, sum w, sum w*y, sum w*y^2 as exact 64-bit fixed-point
// integer sums (row order inside a segment is not deterministic, integer sums
// are).  grid = (leaf, row chunk): a few warps per large leaf accumulate into
// out[] with integer atomics (associative: still exact and deterministic).
// y2fp = y^2 in its own fixed-point scale; out must be zeroed.
__global__ void k5_leaf_stats(RfTrainData D, const int64_t *__restrict__ y2fp,
                              const RfTask *__restrict__ leaves, int n_leaves,
                              const uint8_t *__restrict__ rows0, const uint8_t *__restrict__ rows1,
                              int64_t *__restrict__ out /*[n_leaves][4]*/) {
    const int lane = threadIdx.x & 31;
    const int li = blockIdx.x;
    const RfTask T = leaves[li];
    const uint8_t *rows = T.parity ? rows1 : rows0;
    long long w = 0, sy = 0, sy2 = 0;
    const int stride = gridDim.y * blockDim.x;
    for (int p = T.begin + blockIdx.y * blockDim.x + threadIdx.x; p < T.end; p += stride) {
        const RecView R = rec_at(rows, D.rs, p);
        const long long ww = R.w();
        w += ww;
        sy += R.sv();
        sy2 += ww * y2fp[R.row()];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        w += __shfl_xor_sync(GK_FULL, w, o);
        sy += __shfl_xor_sync(GK_FULL, sy, o);
        sy2 += __shfl_xor_sync(GK_FULL, sy2, o);
    }
    if (lane == 0 && (w | sy | sy2)) {
        atomicAdd((unsigned long long *)&out[4 * li + 1], (unsigned long long)w);
        atomicAdd((unsigned long long *)&out[4 * li + 2], (unsigned long long)sy);
        atomicAdd((unsigned long long *)&out[4 * li + 3], (unsigned long long)sy2);
    }
    if (blockIdx.y == 0 && threadIdx.x == 0) out[4 * li + 0] = T.end - T.begin;
}

// ---------------------------------------------------------- tree assembly
//
// The sklearn-shaped arrays of a batch from its level records (all levels'
// tasks / BFS ids / splits / child ids concatenated in level order; node g of
// the batch = node_base[tree] + BFS id).  Replaces ~100 small torch launches
// per batch (gathers, index_put, where, stack per level).

// split nodes: feature, bin, left child id; per-tree depth = deepest level
// holding a split + 1
__global__ void k5_asm_nodes(const RfTask *__restrict__ tk, const RfSplit *__restrict__ sp,
                             const int32_t *__restrict__ nd, const int32_t *__restrict__ lid,
                             const int32_t *__restrict__ lvl, int n,
                             const int64_t *__restrict__ node_base, int64_t *__restrict__ feat,
                             int64_t *__restrict__ nbin, int64_t *__restrict__ left,
                             unsigned long long *__restrict__ depth) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool split = i < n && sp[i].feat >= 0;
    const unsigned act = __ballot_sync(GK_FULL, split);
    if (!split) return;
    const RfSplit s = sp[i];
    const int t = tk[i].tree;
    const int64_t g = node_base[t] + nd[i];
    feat[g] = s.feat;
    nbin[g] = s.bin;
    left[g] = lid[i];
    // one atomic per (warp, tree): a level's tasks are in tree order, so a
    // warp's split tasks share one or two trees (per-task atomics on 32
    // addresses serialised: 1.3 ms per 32-tree batch)
    const unsigned peers = __match_any_sync(act, t);
    const unsigned dmax = __reduce_max_sync(peers, (unsigned)(lvl[i] + 1));
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicMax(depth + t, (unsigned long long)dmax);
}

// one level bottom-up: every split node's {n, w, w*y, w*y^2} = the sum of its
// two children's (exact integers)
__global__ void k5_asm_up(const RfTask *__restrict__ tk, const RfSplit *__restrict__ sp,
                          const int32_t *__restrict__ nd, const int32_t *__restrict__ lid, int n,
                          const int64_t *__restrict__ node_base, int64_t *__restrict__ ist) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || sp[i].feat < 0) return;
    const int64_t nb = node_base[tk[i].tree];
    const int64_t g = nb + nd[i], c = nb + lid[i];
    const longlong4 a = *reinterpret_cast<const longlong4 *>(ist + 4 * c);
    const longlong4 b = *reinterpret_cast<const longlong4 *>(ist + 4 * (c + 1));
    *reinterpret_cast<longlong4 *>(ist + 4 * g) =
        make_longlong4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// fl [4][N] f64 = {threshold (-2 for leaves), value, impurity, weighted_n},
// it [4][N] i64 = {left, right, feature, n_node_samples}; the same float64
// expressions as the host form (ldexp by a power of two, IEEE division)
__global__ void k5_asm_final(int64_t N, const int64_t *__restrict__ ist,
                             const int64_t *__restrict__ feat, const int64_t *__restrict__ nbin,
                             const int64_t *__restrict__ left, const double *__restrict__ thr,
                             double sc2, double sc3, double *__restrict__ fl,
                             int64_t *__restrict__ it) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N) return;
    const longlong4 v = *reinterpret_cast<const longlong4 *>(ist + 4 * g);
    const int64_t l = left[g], f = feat[g];
    const bool split = l >= 0;
    const double w = (double)v.y;
    const double s2 = __dmul_rn((double)v.z, sc2), s3 = __dmul_rn((double)v.w, sc3);
    const double val = __ddiv_rn(s2, w);
    fl[g] = split ? thr[f * kBins + nbin[g]] : -2.0;
    fl[N + g] = val;
    fl[2 * N + g] = __dsub_rn(__ddiv_rn(s3, w), __dmul_rn(val, val));
    fl[3 * N + g] = w;
    it[g] = l;
    it[N + g] = split ? l + 1 : -1;
    it[2 * N + g] = f;
    it[3 * N + g] = v.x;
}

// ---------------------------------------------------------- gradient boosting

// One boosting update (sklearn GradientBoostingRegressor, squared error): for
// every row of every leaf of the stage's tree, F += leaf_val (= learning_rate *
// leaf mean, computed like sklearn's `learning_rate * value`), then the next
// stage's negative gradient r = y - F in fixed point (yfp = rint(r * 2^shift),
// y2fp = rint(r^2 * 2^shift2), the K5 histogram targets) and max |r| (the
// bits of a non-negative double order like the double) for the next shift.
__global__ void __launch_bounds__(256) k5_gb_step(const RfTask *__restrict__ leaves,
                                                  const double *__restrict__ leaf_val,
                                                  const uint8_t *__restrict__ rows0,
                                                  const uint8_t *__restrict__ rows1, int rs,
                                                  const double *__restrict__ y,
                                                  double *__restrict__ F, int64_t *__restrict__ yfp,
                                                  int64_t *__restrict__ y2fp, int shift, int shift2,
                                                  unsigned long long *__restrict__ absmax) {
    const RfTask T = leaves[blockIdx.x];
    const uint8_t *rows = T.parity ? rows1 : rows0;
    const double v = leaf_val[blockIdx.x];
    double m = 0.0;
    for (int p = T.begin + (int)(blockIdx.y * blockDim.x + threadIdx.x); p < T.end;
         p += (int)(gridDim.y * blockDim.x)) {
        const int32_t r = rec_at(rows, rs, p).row();
        const double f = __dadd_rn(F[r], v);
        F[r] = f;
        const double g = __dsub_rn(y[r], f);
        yfp[r] = __double2ll_rn(ldexp(g, shift));
        y2fp[r] = __double2ll_rn(ldexp(__dmul_rn(g, g), shift2));
        m = fmax(m, fabs(g));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(GK_FULL, m, o));
    // one atomic per CTA (m >= 0: the bit patterns order like the values)
    __shared__ unsigned long long wmax[8];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = (unsigned long long)__double_as_longlong(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long b = wmax[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) b = b > wmax[w] ? b : wmax[w];
        if (b) atomicMax(absmax, b);
    }
}

}  // namespace gk

// ------------------------------------------------------------------ C-ABI

extern "C" {

int gk_rf_bootstrap(const uint32_t *tree_seeds, uint32_t n_trees, int64_t n_rows,
                    uint32_t *counts, void *stream) {
    if (n_rows < 1 || n_rows > 0xffffffffll) {
        gk_set_error("gk_rf_bootstrap: n_rows out of range");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (size_t)n_trees * n_rows, st);
    if (n_trees == 0) return 0;
    gk::k5_bootstrap<<<n_trees, gk::kBootThreads, 0, st>>>(tree_seeds, (int)n_trees, n_rows, counts);
    return gk_check_launch("k5_bootstrap");
}

size_t gk_rf_record_bytes(int32_t n_feat) { return (size_t)gk::rec_stride(n_feat); }

int gk_rf_compact(const uint32_t *counts, uint32_t n_trees, int64_t n_rows, const uint8_t *Xb,
                  int32_t n_feat, const int64_t *yfp, const int64_t *tree_base, void *recs,
                  int32_t *fill, void *stream) {
    const cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(fill, 0, sizeof(int32_t) * n_trees, st);
    if (n_trees == 0 || n_rows <= 0) return 0;
    gk::RfTrainData D{Xb, yfp, nullptr, counts, n_rows, n_feat, gk::rec_stride(n_feat)};
    dim3 grid((unsigned)((n_rows + 255) / 256), n_trees);
    gk::k5_compact<<<grid, 256, 0, st>>>(D, (int)n_trees, tree_base, (uint8_t *)recs, fill);
    return gk_check_launch("k5_compact");
}

int gk_rf_bin(const double *X, int64_t n_rows, int32_t n_feat, int64_t ld, const float *edges,
              const int32_t *n_edges, uint8_t *Xb, uint32_t *bin_min, uint32_t *bin_max,
              void *stream) {
    const cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(bin_min, 0xff, sizeof(uint32_t) * n_feat * gk::kBins, st);
    cudaMemsetAsync(bin_max, 0x00, sizeof(uint32_t) * n_feat * gk::kBins, st);
    const int64_t tot = n_rows * n_feat;
    gk::k5_bin<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(X, n_rows, n_feat, ld, edges,
                                                              n_edges, Xb, bin_min, bin_max);
    return gk_check_launch("k5_bin");
}

// One level of split search + partition for a task list.
//   tasks[n_tasks] (tree, begin, end, parity); small/med/big index lists
//   partition ids: tasks that split after the search (filled by the host)
int gk_rf_split_level(const uint8_t *Xb, const int64_t *yfp, const double *y,
                      const uint32_t *counts, int64_t n_rows, int32_t n_feat,
                      const void *tasks, const int32_t *small_ids, int32_t n_small,
                      const int32_t *med_ids, int32_t n_med, const int32_t *big_ids,
                      int32_t n_big, int32_t big_max_chunks, void *recs0, void *recs1,
                      void *hist_ws, void *split_out, const void *prev_hist_ws,
                      const int32_t *par_slot, int32_t *slot_cur, int32_t n_tasks, void *stream) {
    const cudaStream_t st = (cudaStream_t)stream;
    gk::RfTrainData D{Xb, yfp, y, counts, n_rows, n_feat, gk::rec_stride(n_feat)};
    uint8_t *rows0 = (uint8_t *)recs0, *rows1 = (uint8_t *)recs1;
    const gk::RfTask *T = (const gk::RfTask *)tasks;
    gk::RfSplit *out = (gk::RfSplit *)split_out;
    const size_t smem = sizeof(gk::HistSmem), smem_mid = sizeof(gk::MidSmem);
    static const bool attr = [smem, smem_mid] {  // thread-safe one-time init (concurrent tree batches)
        cudaFuncSetAttribute(gk::k5_split_medium, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(gk::k5_split_medium, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(gk::k5_split_mid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_mid);
        cudaFuncSetAttribute(gk::k5_split_mid, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(gk::k5_hist_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(gk::k5_eval_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return true;
    }();
    (void)attr;
    static const int n_sm = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    if (n_small > 0) {
        // warp-strided over the small list: ~4 waves of resident CTAs
        constexpr int wpb = gk::kSmallThreads / 32;
        const int64_t want = ((int64_t)n_small + wpb - 1) / wpb;
        const int64_t cap = (int64_t)n_sm * GK_SMALL_MINB * 4;
        const unsigned blocks = (unsigned)(want < cap ? want : cap);
        gk::k5_split_sorted<16><<<blocks, gk::kSmallThreads, 0, st>>>(D, T, small_ids, n_small,
                                                                       rows0, rows1, out);
        gk::k5_split_sorted<32><<<blocks, gk::kSmallThreads, 0, st>>>(D, T, small_ids, n_small,
                                                                       rows0, rows1, out);
        if (GK_SMALL_RADIX)
            gk::k5_split_radix<<<blocks, gk::kSmallThreads, 0, st>>>(D, T, small_ids, n_small,
                                                                      rows0, rows1, out);
        else
            gk::k5_split_rank<<<blocks, gk::kSmallThreads, 0, st>>>(D, T, small_ids, n_small,
                                                                     rows0, rows1, out);
    }
    if (n_med > 0) {
        if (GK_MID_ROWS > 0 && n_feat <= 64)
            gk::k5_split_mid<<<n_med, gk::kMedThreads, smem_mid, st>>>(D, T, med_ids, rows0, rows1,
                                                                       out);
        gk::k5_split_medium<<<n_med, gk::kMedThreads, smem, st>>>(D, T, med_ids, rows0, rows1, out);
    }
    // this level's big slots by task (-1: not big), for the sibling
    // subtraction and the next level's parent slots
    if (slot_cur && n_tasks > 0) cudaMemsetAsync(slot_cur, 0xFF, sizeof(int32_t) * (size_t)n_tasks, st);
    if (n_big > 0) {
        uint64_t *gh = (uint64_t *)hist_ws;
        const int32_t *ps = (prev_hist_ws && slot_cur) ? par_slot : nullptr;
        if (slot_cur)
            gk::k5_big_slots<<<(n_big + 255) / 256, 256, 0, st>>>(big_ids, n_big, slot_cur);
        cudaMemsetAsync(hist_ws, 0, 2 * sizeof(uint64_t) * (size_t)n_big * n_feat * gk::kBins, st);
        // the host sizes big_max_chunks in kMedRows units; CTAs take kBigRows
        dim3 grid(big_max_chunks * (gk::kMedRows / gk::kBigRows), (n_feat + gk::kFC - 1) / gk::kFC,
                  n_big);
        gk::k5_hist_big<<<grid, 256, smem, st>>>(D, T, big_ids, rows0, rows1, ps, slot_cur, gh);
        if (ps)
            gk::k5_hist_derive<<<dim3(8, n_big), 256, 0, st>>>(T, big_ids, ps, slot_cur, n_feat,
                                                               (const uint64_t *)prev_hist_ws, gh);
        gk::k5_eval_big<<<n_big, 256, smem, st>>>(D, big_ids, gh, out);
    }
    return gk_check_launch("k5_split_level");
}

size_t gk_rf_hist_bytes(int32_t n_big, int32_t n_feat) {
    return 2 * sizeof(uint64_t) * (size_t)n_big * n_feat * gk::kBins;
}

int gk_rf_partition(const uint8_t *Xb, const int64_t *yfp, const double *y,
                    const uint32_t *counts, int64_t n_rows, int32_t n_feat, const void *tasks,
                    int32_t n_tasks, const void *split, const int32_t *ids, int32_t n_ids,
                    int32_t max_rows, void *recs0, void *recs1, int32_t *cursor,
                    void *stream) {
    if (n_ids <= 0) return 0;
    const cudaStream_t st = (cudaStream_t)stream;
    gk::RfTrainData D{Xb, yfp, y, counts, n_rows, n_feat, gk::rec_stride(n_feat)};
    uint8_t *rows0 = (uint8_t *)recs0, *rows1 = (uint8_t *)recs1;
    cudaMemsetAsync(cursor, 0, sizeof(int32_t) * 2 * (size_t)n_tasks, st);
    const int64_t chunks = ((int64_t)max_rows + 255) / 256;
    if (chunks > 65535) {
        gk_set_error("gk_rf_partition: node of %d rows exceeds the 16.7M-row chunk grid", max_rows);
        return -1;
    }
    dim3 grid((unsigned)n_ids, (unsigned)chunks);
    gk::k5_partition<<<grid, 256, 0, st>>>(D, (const gk::RfTask *)tasks, (const gk::RfSplit *)split,
                                           ids, rows0, rows1, rows1, rows0, cursor);
    return gk_check_launch("k5_partition");
}

// Next level of a tree batch from this level's tasks and splits (device-side
// bookkeeping, see k5_level_emit).  stats[8] (int32): [0] next-level task
// count, [1..3] small / medium / big list lengths, [4] / [5] largest medium /
// big task; lists = 3 regions of list_cap (>= 2 * n_tasks) entries.
size_t gk_rf_level_scratch_bytes(int32_t n_tasks, int32_t n_trees) {
    const size_t nb = ((size_t)n_tasks + gk::kLvlThreads - 1) / gk::kLvlThreads;
    return sizeof(int32_t) * (nb + 2 * (size_t)n_trees + 8);
}

int gk_rf_next_level(const void *tasks, const int32_t *node, const void *split,
                     const int32_t *cursor, int32_t n_tasks, int32_t n_trees, int32_t child_depth,
                     int32_t max_depth, int32_t *next_id, int32_t *lid_out, void *tasks_next,
                     int32_t *node_next, int32_t *lists, int32_t list_cap, int32_t *stats,
                     void *scratch, const int32_t *slot_cur, int32_t *par_slot_next,
                     void *stream) {
    if (n_tasks < 0 || n_trees < 1 || list_cap < 2 * (int64_t)n_tasks) {
        gk_set_error("gk_rf_next_level: bad sizes (n_tasks %d, n_trees %d, list_cap %d)", n_tasks,
                     n_trees, list_cap);
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    const int nb = (n_tasks + gk::kLvlThreads - 1) / gk::kLvlThreads;
    int32_t *block_cnt = (int32_t *)scratch;
    int32_t *tree_cnt = block_cnt + nb;
    int32_t *lid_base = tree_cnt + n_trees;
    cudaMemsetAsync(stats, 0, 8 * sizeof(int32_t), st);
    cudaMemsetAsync(tree_cnt, 0, sizeof(int32_t) * n_trees, st);
    if (nb == 0) return gk_check_launch("k5_next_level");
    const gk::RfTask *T = (const gk::RfTask *)tasks;
    const gk::RfSplit *S = (const gk::RfSplit *)split;
    gk::k5_level_count<<<nb, gk::kLvlThreads, 0, st>>>(T, S, n_tasks, block_cnt, tree_cnt);
    gk::k5_level_scan<<<1, 1024, 0, st>>>(block_cnt, nb, tree_cnt, n_trees, next_id, lid_base, stats);
    gk::k5_level_emit<<<nb, gk::kLvlThreads, 0, st>>>(T, node, S, n_tasks, block_cnt, lid_base,
                                                       cursor, child_depth, max_depth, lid_out,
                                                       (gk::RfTask *)tasks_next, node_next, lists,
                                                       list_cap, stats, slot_cur, par_slot_next);
    return gk_check_launch("k5_next_level");
}

// gk_rf_partition over the three search lists of a level (cursor: 2 * n_tasks,
// zeroed here once); tasks whose search kept them a leaf are skipped
int gk_rf_partition_lists(const uint8_t *Xb, const uint32_t *counts, int64_t n_rows,
                          int32_t n_feat, const void *tasks, int32_t n_tasks, const void *split,
                          const int32_t *small_ids, int32_t n_small, const int32_t *med_ids,
                          int32_t n_med, int32_t max_med, const int32_t *big_ids, int32_t n_big,
                          int32_t max_big, void *recs0, void *recs1, int32_t *cursor,
                          void *stream) {
    const cudaStream_t st = (cudaStream_t)stream;
    gk::RfTrainData D{Xb, nullptr, nullptr, counts, n_rows, n_feat, gk::rec_stride(n_feat)};
    uint8_t *rows0 = (uint8_t *)recs0, *rows1 = (uint8_t *)recs1;
    cudaMemsetAsync(cursor, 0, sizeof(int32_t) * 2 * (size_t)n_tasks, st);
    const int32_t *ids[3] = {small_ids, med_ids, big_ids};
    const int32_t nid[3] = {n_small, n_med, n_big};
    const int32_t mx[3] = {gk::kSmallRows, max_med, max_big};
    for (int c = 1; c < 3; c++) {  // small tasks: partitioned by k5_split_sorted / _rank
        if (nid[c] <= 0) continue;
        const int64_t chunks = ((int64_t)mx[c] + 255) / 256;
        if (chunks < 1 || chunks > 65535) {
            gk_set_error("gk_rf_partition_lists: node of %d rows out of the chunk grid", mx[c]);
            return -1;
        }
        dim3 grid((unsigned)nid[c], (unsigned)chunks);
        gk::k5_partition<<<grid, 256, 0, st>>>(D, (const gk::RfTask *)tasks,
                                               (const gk::RfSplit *)split, ids[c], rows0, rows1,
                                               rows1, rows0, cursor);
    }
    return gk_check_launch("k5_partition_lists");
}

int gk_rf_leaf_stats(const uint32_t *counts, int64_t n_rows, int32_t n_feat, const int64_t *yfp,
                     const int64_t *y2fp, const void *leaves, int32_t n_leaves,
                     const void *recs0, const void *recs1, int64_t *out,
                     int32_t max_leaf_rows, void *stream) {
    if (n_leaves <= 0) return 0;
    const cudaStream_t st = (cudaStream_t)stream;
    gk::RfTrainData D{nullptr, yfp, nullptr, counts, n_rows, n_feat, gk::rec_stride(n_feat)};
    const uint8_t *rows0 = (const uint8_t *)recs0, *rows1 = (const uint8_t *)recs1;
    cudaMemsetAsync(out, 0, sizeof(int64_t) * 4 * (size_t)n_leaves, st);
    // chunks sized by the largest leaf: one 32-lane warp per 256 rows, at most
    // 1024 per leaf and ~2^18 warps per launch (few large leaves -- a boosting
    // stage's 8 -- fill the GPU; a forest batch's ~1M tiny ones take one each)
    int max_rows = 0;
    if (max_leaf_rows > 0) max_rows = max_leaf_rows;
    int64_t chunks = ((int64_t)max_rows + 255) / 256;
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(1024, (1 << 18) / n_leaves));
    if (chunks > cap) chunks = cap;
    if (chunks < 1) chunks = 1;
    gk::k5_leaf_stats<<<dim3((unsigned)n_leaves, (unsigned)chunks), 32, 0, st>>>(
        D, y2fp, (const gk::RfTask *)leaves, n_leaves, rows0, rows1, out);
    return gk_check_launch("k5_leaf_stats");
}

int gk_rf_assemble_nodes(const void *tasks, const void *split, const int32_t *node,
                         const int32_t *lid, const int32_t *level, int32_t n,
                         const int64_t *node_base, int64_t *feat, int64_t *nbin, int64_t *left,
                         int64_t *depth, void *stream) {
    if (n <= 0) return 0;
    gk::k5_asm_nodes<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        (const gk::RfTask *)tasks, (const gk::RfSplit *)split, node, lid, level, n, node_base,
        feat, nbin, left, (unsigned long long *)depth);
    return gk_check_launch("k5_asm_nodes");
}

int gk_rf_assemble_up(const void *tasks, const void *split, const int32_t *node,
                      const int32_t *lid, int32_t n, const int64_t *node_base, int64_t *ist,
                      void *stream) {
    if (n <= 0) return 0;
    gk::k5_asm_up<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        (const gk::RfTask *)tasks, (const gk::RfSplit *)split, node, lid, n, node_base, ist);
    return gk_check_launch("k5_asm_up");
}

int gk_rf_assemble_final(int64_t n_nodes, const int64_t *ist, const int64_t *feat,
                         const int64_t *nbin, const int64_t *left, const double *thr,
                         int32_t shift, int32_t shift2, double *fl, int64_t *it, void *stream) {
    if (n_nodes <= 0) return 0;
    gk::k5_asm_final<<<(unsigned)((n_nodes + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n_nodes, ist, feat, nbin, left, thr, ldexp(1.0, -shift), ldexp(1.0, -shift2), fl, it);
    return gk_check_launch("k5_asm_final");
}

int gk_gb_step(const void *leaves, int32_t n_leaves, const double *leaf_val,
               const void *recs0, const void *recs1, int32_t n_feat, const double *y, double *F,
               int64_t *yfp, int64_t *y2fp, int32_t shift, int32_t shift2,
               uint64_t *absmax, int32_t max_leaf_rows, void *stream) {
    if (n_leaves <= 0) return 0;
    if (shift < -1000 || shift > 1000 || shift2 < -1000 || shift2 > 1000) {
        gk_set_error("gk_gb_step: fixed-point shift out of range");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    // 256 rows per CTA of the largest leaf, at most 1024 CTAs per leaf and
    // ~2^18 CTAs per launch (max_leaf_rows may be a bound: n for a stage of
    // few leaves, whose sizes are not read back)
    int64_t chunks = ((int64_t)max_leaf_rows + 255) / 256;
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(1024, (1 << 18) / n_leaves));
    if (chunks > cap) chunks = cap;
    if (chunks < 1) chunks = 1;
    dim3 grid((unsigned)n_leaves, (unsigned)chunks);
    gk::k5_gb_step<<<grid, 256, 0, st>>>((const gk::RfTask *)leaves, leaf_val,
                                        (const uint8_t *)recs0, (const uint8_t *)recs1,
                                        gk::rec_stride(n_feat), y, F,
                                        yfp, y2fp, shift, shift2,
                                        (unsigned long long *)absmax);
    return gk_check_launch("k5_gb_step");
}

}  // extern "C"
