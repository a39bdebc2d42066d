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
template <int kIlp = GK_RF_ILP>
__device__ __forceinline__ double walk_ensemble(const gk_ensemble &E, const double *x,
                                                int stride) {
    const gk_node *__restrict__ nodes = E.nodes;
    double total = E.base_score;
    uint32_t t = 0;
    for (; t + kIlp <= E.n_trees; t += kIlp) {
        const gk_node *base[kIlp];
        int32_t idx[kIlp];
        double v[kIlp];
        int d = 0;
#pragma unroll
        for (int q = 0; q < kIlp; q++) {
            base[q] = nodes + __ldg(E.tree_off + t + q);
            idx[q] = 0;
            d = max(d, __ldg(E.tree_depth + t + q));
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
        for (int q = 0; q < kIlp; q++) total = __dadd_rn(total, v[q]);  // tree order
    }
    for (; t < E.n_trees; t++) {
        const gk_node *b = nodes + E.tree_off[t];
        int32_t i = 0;
        while (true) {
            const double2 raw = __ldg(reinterpret_cast<const double2 *>(b + i));
            const int f = __double2loint(raw.y), l = __double2hiint(raw.y);
            if (f < 0) {
                total = __dadd_rn(total, raw.x);
                break;
            }
            i = x[f * stride] <= raw.x ? l : l + 1;
        }
    }
    return total;
}

// power.py:144 -- (v - lo) / (hi - lo), or 0 when hi <= lo
__device__ __forceinline__ double scale_feature(double v, double lo, double hi) {
    return hi > lo ? __ddiv_rn(__dsub_rn(v, lo), __dsub_rn(hi, lo)) : 0.0;
}

}  // namespace gk
