// gk_walk.cuh -- the ensemble walk shared by K4 (k4_rf_predict) and the fused
// sweep kernel.  Reference: power.py:156-168 -- total = base_score, then for
// every tree in file order walk from the root (x[f] <= threshold -> left) and
// add the leaf.  Here GK_RF_ILP trees are walked in lock-step for max(depth)
// steps (leaves are absorbing: left = self) and their leaves are added in tree
// order, so the fp64 sum is bit-identical to the reference's.
#pragma once

#include "gk_internal.cuh"

#ifndef GK_RF_ILP
#define GK_RF_ILP 8  // trees walked in lock-step per thread (8 measured best on B200)
#endif

namespace gk {

// x: this row's scaled features, feature f at x[f * stride], and x[-stride]
// must hold +inf: a leaf {value, -1, self - 1} then compares +inf <= value
// (false) and steps "right" to itself, so walks absorb without a leaf test.
template <int kIlp, bool kTail>
__device__ __forceinline__ void walk16_group(const gk_ensemble &E, uint32_t t, int nq,
                                             const double *x, int stride, double &total) {
    const gk_node *__restrict__ nodes = E.nodes;
    const gk_node *base[kIlp];
    int32_t idx[kIlp];
    double v[kIlp];
    int d = 0;
#pragma unroll
    for (int q = 0; q < kIlp; q++) {
        const uint32_t tq = t + (!kTail || q < nq ? q : 0);
        base[q] = nodes + __ldg(E.tree_off + tq);
        idx[q] = 0;
        d = max(d, __ldg(E.tree_depth + tq));
    }
    for (int s = 0; s <= d; s++) {
#pragma unroll
        for (int q = 0; q < kIlp; q++) {
            const double2 raw = __ldg(reinterpret_cast<const double2 *>(base[q] + idx[q]));
            const int f = __double2loint(raw.y), l = __double2hiint(raw.y);
            v[q] = raw.x;
            idx[q] = x[f * stride] <= raw.x ? l : l + 1;
        }
    }
#pragma unroll
    for (int q = 0; q < kIlp; q++)
        if (!kTail || q < nq) total = __dadd_rn(total, v[q]);  // tree order
}

// Groups of kIlp trees in lock-step.  A partial last group keeps the lock
// step: its idle slots re-walk the group's first tree (loads in flight, no
// latency chain of their own) and are not added -- tail trees walked one by
// one would serialise max(depth) dependent loads each.
template <int kIlp = GK_RF_ILP>
__device__ __forceinline__ double walk_ensemble(const gk_ensemble &E, const double *x,
                                                int stride) {
    double total = E.base_score;
    uint32_t t = 0;
    for (; t + kIlp <= E.n_trees; t += kIlp) walk16_group<kIlp, false>(E, t, kIlp, x, stride, total);
    if (t < E.n_trees) walk16_group<kIlp, true>(E, t, (int)(E.n_trees - t), x, stride, total);
    return total;
}

// Compact walk over gk_node8 (include/gk.h).  xf: this row's features rounded
// toward -inf to f32 (feature f at xf[f * stride], xf[-stride] = +inf);
// x64(f): the exact scaled fp64 feature, needed only when a == t.  Per visit:
// one 8-byte node load, one 4-byte shared load, two f32 compares -- 12 bytes
// through the L1 data pipe instead of 24.  Loads of the kIlp trees are issued
// together; the rare tie test runs out of line.
template <int kIlp, bool kTail, class X64>
__device__ __forceinline__ void walk8_group(const gk_ensemble &E, uint32_t t, int nq,
                                            const float *xf, int stride, const X64 &x64,
                                            double &total) {
    const uint2 *__restrict__ n8 = reinterpret_cast<const uint2 *>(E.nodes8);
    const uint2 *base[kIlp];
    int32_t idx[kIlp];
    int d = 0;
#pragma unroll
    for (int q = 0; q < kIlp; q++) {  // idle slots (partial group) re-walk tree t
        const uint32_t tq = t + (!kTail || q < nq ? q : 0);
        base[q] = n8 + __ldg(E.tree_off + tq);
        idx[q] = 0;
        d = max(d, __ldg(E.tree_depth + tq));
    }
    for (int s = 0; s < d; s++) {
        uint2 raw[kIlp];
        float a[kIlp];
#pragma unroll
        for (int q = 0; q < kIlp; q++) raw[q] = __ldg(base[q] + idx[q]);
#pragma unroll
        for (int q = 0; q < kIlp; q++) a[q] = xf[((int)raw[q].y >> 24) * stride];  // leaf: +inf slot
        uint32_t tie = 0;
        bool le[kIlp];
#pragma unroll
        for (int q = 0; q < kIlp; q++) {
            const float th = __uint_as_float(raw[q].x);
            le[q] = a[q] < th;
            tie |= (a[q] == th ? 1u : 0u) << q;
        }
        if (__builtin_expect(tie != 0, 0)) {
#pragma unroll
            for (int q = 0; q < kIlp; q++)
                if (tie >> q & 1u)
                    le[q] = x64((int)raw[q].y >> 24) <=
                            __ldg(&E.nodes[(base[q] - n8) + idx[q]].v);
        }
#pragma unroll
        for (int q = 0; q < kIlp; q++) {
            const int r = (int)(raw[q].y & 0xFFFFFFu);
            idx[q] = le[q] ? r - 1 : r;
        }
    }
#pragma unroll
    for (int q = 0; q < kIlp; q++)
        if (!kTail || q < nq) total = __dadd_rn(total, __ldg(&E.nodes[(base[q] - n8) + idx[q]].v));
}

template <int kIlp, class X64>
__device__ __forceinline__ double walk_ensemble8(const gk_ensemble &E, const float *xf, int stride,
                                                 const X64 &x64) {
    double total = E.base_score;
    uint32_t t = 0;
    for (; t + kIlp <= E.n_trees; t += kIlp) walk8_group<kIlp, false>(E, t, kIlp, xf, stride, x64, total);
    if (t < E.n_trees)
        walk8_group<kIlp, true>(E, t, (int)(E.n_trees - t), xf, stride, x64, total);
    return total;
}

// Blocked walk over gk_block2 (include/gk.h): one 256-bit load per tree per
// two levels.  xf: this row's features rounded toward -inf to f32 (feature f
// at xf[f * stride]); x64(f): the exact scaled fp64 feature, needed only when a
// row value and a threshold share one f32 bucket (the tie test runs out of
// line).  kIlp trees advance in lock-step for ceil(max depth / 2) steps; a
// tree that reached its leaf stops loading.  Leaves are added in tree order.
__device__ __forceinline__ void ld_block2(const gk_block2 *p, uint32_t (&w)[8]) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                   "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

// kS64: the feature tile's stride is 64 floats (256 B), so a feature byte
// becomes its byte offset with one PRMT (byte k -> byte 1) instead of a
// shift / mask / multiply-add chain per slot.  kSink: finished trees load a
// shared dummy block instead of a predicated load + zeroed words -- fewer
// instructions and registers for more L1 wavefronts.  Measured on B200: the
// fused sweep (issue-bound with this walk) wants both; K4 on config #4
// (L1-wavefront-bound) loses 10 % with kSink and gains nothing from kS64.
template <int kIlp, bool kTail, bool kS64, bool kSink, bool kLds2, class X64>
__device__ __forceinline__ void walk_b2_group(const gk_ensemble &E, uint32_t t, int nq,
                                              const float *xf, int stride, const X64 &x64,
                                              double &total) {
    // hoisted for the sink form (the fused sweep, where E sits in a dynamically
    // indexed parameter array); K4 keeps re-reading E.blocks -- measured: the
    // hoisted pointer costs K4 5 % on config #4
    const gk_block2 *__restrict__ blocks = E.blocks;
    uint32_t ref[kIlp];
    int d = 0;
#pragma unroll
    for (int q = 0; q < kIlp; q++) {  // idle slots of a partial group start at a leaf
        const bool on = !kTail || q < nq;
        ref[q] = on ? __ldg(E.root + t + q) : GK_LEAF;
        if (on) d = max(d, __ldg(E.tree_depth + t + q));
    }
    const int steps = (d + 1) >> 1;
    for (int s = 0; s < steps; s++) {
        uint32_t w[kIlp][8];
#pragma unroll
        for (int q = 0; q < kIlp; q++) {
            if (kSink) {
                // a finished tree loads block 0 (one shared line; its words are
                // never used) instead of predicating the load and zeroing
                ld_block2(blocks + (ref[q] & GK_LEAF ? 0u : ref[q]), w[q]);
            } else if (!(ref[q] & GK_LEAF)) {
                ld_block2(E.blocks + ref[q], w[q]);
            } else {
#pragma unroll
                for (int k = 0; k < 8; k++) w[q][k] = 0;
            }
        }
        auto feat = [&](uint32_t fw, uint32_t k) {  // feature byte k of fw -> its tile value
            return kS64 ? *reinterpret_cast<const float *>(reinterpret_cast<const char *>(xf) +
                                                           __byte_perm(fw, 0u, 0x4404u | (k << 4)))
                        : xf[((fw >> (8 * k)) & 0xFFu) * stride];
        };
        float a[kIlp][3];
        if (kLds2) {
            // two shared loads per block: the second level's feature after the
            // first decision (each LDS is an L1/TEX data-pipe wavefront, shared
            // with the block loads' lines)
#pragma unroll
            for (int q = 0; q < kIlp; q++) a[q][0] = feat(w[q][3], 0u);
#pragma unroll
            for (int q = 0; q < kIlp; q++)
                a[q][1] = feat(w[q][3], a[q][0] < __uint_as_float(w[q][0]) ? 1u : 2u);
        } else {
#pragma unroll
            for (int q = 0; q < kIlp; q++)
#pragma unroll
                for (int k = 0; k < 3; k++) a[q][k] = feat(w[q][3], (uint32_t)k);
        }
        uint32_t tie = 0;
        uint32_t nref[kIlp];
#pragma unroll
        for (int q = 0; q < kIlp; q++) {
            const float t0 = __uint_as_float(w[q][0]);
            const bool c0 = a[q][0] < t0;
            const float as = kLds2 ? a[q][1] : (c0 ? a[q][1] : a[q][2]);
            const float ts = __uint_as_float(c0 ? w[q][1] : w[q][2]);
            const bool c1 = as < ts;
            tie |= (((a[q][0] == t0) | (as == ts)) && !(ref[q] & GK_LEAF) ? 1u : 0u) << q;
            const uint32_t lo = c1 ? w[q][4] : w[q][5], hi = c1 ? w[q][6] : w[q][7];
            nref[q] = c0 ? lo : hi;
        }
        if (__builtin_expect(tie != 0, 0)) {
#pragma unroll
            for (int q = 0; q < kIlp; q++) {
                if (!(tie >> q & 1u)) continue;
                const double *th = E.thr64 + 3 * (size_t)ref[q];
                const uint32_t fw = w[q][3];
                const bool c0 = x64((int)(fw & 0xFFu)) <= th[0];
                const bool c1 = c0 ? x64((int)((fw >> 8) & 0xFFu)) <= th[1]
                                   : x64((int)((fw >> 16) & 0xFFu)) <= th[2];
                const uint32_t lo = c1 ? w[q][4] : w[q][5], hi = c1 ? w[q][6] : w[q][7];
                nref[q] = c0 ? lo : hi;
            }
        }
#pragma unroll
        for (int q = 0; q < kIlp; q++)
            if (!(ref[q] & GK_LEAF)) ref[q] = nref[q];
    }
#pragma unroll
    for (int q = 0; q < kIlp; q++)
        if (!kTail || q < nq) total = __dadd_rn(total, __ldg(E.leaf_val + (ref[q] & ~GK_LEAF)));
}

// kLds2: two shared feature loads per block instead of three (the second
// after the first decision).  Measured on B200: the fused sweep on config #5
// 127.2 -> 134.3 M points/s (its L1/TEX data pipe also serves the scheduler's
// tables); K4 alone on config #4 82.1 -> 73.8 M rows/s (the dependent load
// lengthens its latency-bound chain) -- so only the sweep uses it.
template <int kIlp, bool kS64 = false, bool kSink = false, bool kLds2 = false, class X64>
__device__ __forceinline__ double walk_ensemble_b2(const gk_ensemble &E, const float *xf, int stride,
                                                   const X64 &x64) {
    double total = E.base_score;
    uint32_t t = 0;
    for (; t + kIlp <= E.n_trees; t += kIlp)
        walk_b2_group<kIlp, false, kS64, kSink, kLds2>(E, t, kIlp, xf, stride, x64, total);
    if (t < E.n_trees)
        walk_b2_group<kIlp, true, kS64, kSink, kLds2>(E, t, (int)(E.n_trees - t), xf, stride, x64,
                                                     total);
    return total;
}

// ---- three-level blocks with 16-bit keys (gk_block3, include/gk.h)
// One 256-bit load per tree per three levels, and the last split level's
// leaves inline (terminal blocks): a depth-16 path is 6 scattered 32-byte
// loads instead of the two-level blocks' 8 + a leaf-value load.  Scattered
// per-lane loads cost one L1/TEX wavefront per distinct 128-byte line
// (tools/ubench/gather.cu: 0.99 per SM-cycle on every load path), so the
// walk's ceiling rises with the lines it avoids.
__device__ __forceinline__ uint32_t key16(double v) {  // include/gk.h gk_block3 keys
    float a = __double2float_rd(v);
    if (a == 0.0f) a = 0.0f;  // -0.0 == +0.0
    const uint32_t u = __float_as_uint(a);
    const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return a != a ? 0xFFFFu : o >> 16;
}

#define GK_B3_INLINE 0x40000000u  // done, value in val[] (terminal block)

// one block step of one tree: the fast decisions (ties flagged), the exact
// redo of a block with a tie out of line
template <class KeyAt, class X64>
__device__ __forceinline__ void b3_step(const gk_ensemble &E, const uint32_t (&w)[8],
                                        uint32_t &ref, double &val, const KeyAt &key,
                                        const X64 &x64) {
    const uint32_t blk = ref;
    const uint32_t f0 = (w[3] >> 16) & 0xFFu, t0 = w[0] & 0xFFFFu;
    const uint32_t a0 = key(f0);
    uint32_t b0 = a0 > t0;
    if (((w[5] >> 16) & 0xFFu) == GK_B3_TERMINAL) {  // node 0 only; leaves inline
        if (__builtin_expect(a0 == t0, 0)) b0 = !(x64((int)f0) <= E.thr64[7 * (size_t)blk]);
        val = __hiloint2double(b0 ? w[7] : w[2], b0 ? w[6] : w[1]);
        ref = GK_LEAF | GK_B3_INLINE;
        return;
    }
    uint32_t tie = a0 == t0;
    // level 1: node 1 + b0; level 2: node 3 + 2 b0 + b1 (halfwords 3..6 and
    // feature bytes 17..20 as one 64-bit / 32-bit funnel each)
    const uint32_t t1 = b0 ? (w[1] & 0xFFFFu) : (w[0] >> 16);
    const uint32_t f1 = b0 ? (w[4] & 0xFFu) : (w[3] >> 24);
    const uint32_t a1 = key(f1);
    uint32_t b1 = a1 > t1;
    tie |= a1 == t1;
    const uint64_t T2 = (uint64_t)(w[1] >> 16) | ((uint64_t)w[2] << 16) |
                        ((uint64_t)(w[3] & 0xFFFFu) << 48);
    const uint32_t F2 = __funnelshift_r(w[4], w[5], 8);
    uint32_t j = 2 * b0 + b1;
    uint32_t t2 = (uint32_t)(T2 >> (16 * j)) & 0xFFFFu, f2 = (F2 >> (8 * j)) & 0xFFu;
    const uint32_t a2 = key(f2);
    uint32_t b2 = a2 > t2;
    tie |= a2 == t2;
    if (__builtin_expect(tie != 0, 0)) {  // exact fp64 tests, in path order
        const double *th = E.thr64 + 7 * (size_t)blk;
        b0 = a0 == t0 ? !(x64((int)f0) <= th[0]) : a0 > t0;
        const uint32_t tt1 = b0 ? (w[1] & 0xFFFFu) : (w[0] >> 16);
        const uint32_t ff1 = b0 ? (w[4] & 0xFFu) : (w[3] >> 24);
        const uint32_t aa1 = key(ff1);
        b1 = aa1 == tt1 ? !(x64((int)ff1) <= th[1 + b0]) : aa1 > tt1;
        j = 2 * b0 + b1;
        t2 = (uint32_t)(T2 >> (16 * j)) & 0xFFFFu;
        f2 = (F2 >> (8 * j)) & 0xFFu;
        const uint32_t aa2 = key(f2);
        b2 = aa2 == t2 ? !(x64((int)f2) <= th[3 + j]) : aa2 > t2;
    }
    const uint32_t s = 4 * b0 + 2 * b1 + b2;
    const uint32_t mask = (w[5] >> 8) & 0xFFu, below = (1u << s) - 1u;
    ref = (mask >> s & 1u) ? (GK_LEAF | (w[7] + __popc(mask & below)))
                           : (w[6] + __popc(~mask & below & 0xFFu));
}

// trees t .. t + nq - 1 (kIlp in lock-step); xk: this row's 16-bit keys,
// feature f at xk[f * stride]
template <int kIlp, bool kTail, class X64>
__device__ __forceinline__ void walk_b3_group(const gk_ensemble &E, uint32_t t, int nq,
                                              const uint16_t *xk, int stride, const X64 &x64,
                                              double &total) {
    const gk_block3 *__restrict__ B = E.blocks3;
    uint32_t ref[kIlp];
    double val[kIlp];
    int d = 0;
#pragma unroll
    for (int q = 0; q < kIlp; q++) {  // idle slots of a partial group start done
        const bool on = !kTail || q < nq;
        ref[q] = on ? __ldg(E.root + t + q) : (GK_LEAF | GK_B3_INLINE);
        val[q] = 0.0;
        if (on) d = max(d, __ldg(E.tree_depth + t + q));
    }
    auto key = [&](uint32_t f) { return (uint32_t)xk[f * stride]; };
    const int steps = d > 0 ? (d - 1) / 3 + 1 : 0;
    for (int st = 0; st < steps; st++) {
        uint32_t w[kIlp][8];
#pragma unroll
        for (int q = 0; q < kIlp; q++)
            if (!(ref[q] & GK_LEAF)) ld_block2(reinterpret_cast<const gk_block2 *>(B + ref[q]), w[q]);
#pragma unroll
        for (int q = 0; q < kIlp; q++)
            if (!(ref[q] & GK_LEAF)) b3_step(E, w[q], ref[q], val[q], key, x64);
    }
#pragma unroll
    for (int q = 0; q < kIlp; q++)
        if (!kTail || q < nq)
            total = __dadd_rn(total, (ref[q] & GK_B3_INLINE)
                                         ? val[q]
                                         : __ldg(E.leaf_val + (ref[q] & ~(GK_LEAF | GK_B3_INLINE))));
}

template <int kIlp, class X64>
__device__ __forceinline__ double walk_ensemble_b3(const gk_ensemble &E, const uint16_t *xk,
                                                   int stride, const X64 &x64) {
    double total = E.base_score;
    uint32_t t = 0;
    for (; t + kIlp <= E.n_trees; t += kIlp)
        walk_b3_group<kIlp, false>(E, t, kIlp, xk, stride, x64, total);
    if (t < E.n_trees) walk_b3_group<kIlp, true>(E, t, (int)(E.n_trees - t), xk, stride, x64, total);
    return total;
}

// power.py:144 -- (v - lo) / (hi - lo), or 0 when hi <= lo
__device__ __forceinline__ double scale_feature(double v, double lo, double hi) {
    return hi > lo ? __ddiv_rn(__dsub_rn(v, lo), __dsub_rn(hi, lo)) : 0.0;
}

}  // namespace gk
