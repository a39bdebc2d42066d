// gk_internal.cuh -- shared device helpers for libgk (sm_100a).
//
// Every floating-point expression below keeps the reference's evaluation order
// and rounding: the library is compiled with -fmad=false (no FMA contraction;
// SURVEY §7.3.1), int64 -> double conversions are round-to-nearest (Python's
// float(int)), integer true divisions are IEEE double divisions of exactly
// representable operands (Python's int / int).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gk.h"
#include "gk_exp.h"

#define GK_FULL 0xffffffffu

namespace gk {

// per_sm_block_cap (reference scheduler.py:220-237); < 1 means infeasible
__device__ __forceinline__ int64_t block_cap(const gk_arch &A, const gk_config &c) {
    int64_t cap = A.nTh_sm_max / c.tpb;
    if (A.nB_max < cap) cap = A.nB_max;
    if (c.regs > 0) {
        int64_t r = A.reg_b_max / ((int64_t)c.regs * c.tpb);
        if (r < cap) cap = r;
    }
    if (c.shmem > 0) {
        int64_t s = A.shm_b_max / c.shmem;
        if (s < cap) cap = s;
    }
    return cap;
}

// global_mem_latency -> PiecewiseLinearModel.evaluate (profiles.py:58-61, 146-150)
__device__ __forceinline__ double gm_latency(const gk_arch &A, const gk_config &c) {
    double x = (double)((int64_t)c.n_blocks * c.tpb);
    int i = 0;
    while (i < A.n_bp && A.bp[i] <= x) i++;  // bisect_right
    return __dadd_rn(__dmul_rn(A.seg_slope[i], x), A.seg_icpt[i]);
}

// mem_throughput with ExpGrowthModel (profiles.py:76-77, 159-182)
__device__ __forceinline__ double tput(double a, double b, double c, double floor_, double n) {
    double v = __dmul_rn(a, __dsub_rn(b, gk_exp(__dmul_rn(-c, n))));
    return v <= 0.0 ? floor_ : v;
}

__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

__device__ __forceinline__ double shfl_d(double v, int src, int width = 32) {
    return __shfl_sync(GK_FULL, v, src, width);
}
__device__ __forceinline__ double shfl_up_d(double v, int d, int width = 32) {
    return __shfl_up_sync(GK_FULL, v, d, width);
}

}  // namespace gk

// error plumbing shared by the entry points
void gk_set_error(const char *fmt, ...);
int gk_check_launch(const char *what);
