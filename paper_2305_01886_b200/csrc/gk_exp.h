/*
 * gk_exp.h -- bit-exact restatement of the host libm `exp` that the reference's
 * `math.exp` resolves to (glibc 2.39 exp@@GLIBC_2.29, FMA IFUNC variant; the
 * algorithm of sysdeps/ieee754/dbl-64/e_exp.c / ARM optimized-routines).
 *
 * Needed because mem_throughput (reference profiles.py:76-77, 159-182) feeds
 * exp(-c*n) into the contention penalties, which flow into d_total / time_us
 * and the glb_penalty / sh_penalty features -- all required bit-exact.  CUDA's
 * exp is not bit-identical to glibc's (neither is correctly rounded).
 *
 * Host + device: on the host `fma()` is the correctly rounded C99 fma, on the
 * device __fma_rn; every other operation is a separately rounded IEEE op (the
 * library is built with -fmad=false, the host test with -ffp-contract=off).
 */
#pragma once
#include <stdint.h>
#include <string.h>

#include "gk_exp_table.h"

#if defined(__CUDACC__)
#define GK_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#define GK_HD static inline
#endif

GK_HD double gk_asdouble(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}
GK_HD uint64_t gk_asuint64(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}
GK_HD double gk_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

static const uint64_t GK_EXP_TAB[256] = GK_EXP_TAB_INIT;
#if defined(__CUDACC__)
static __constant__ uint64_t gk_exp_tab_dev[256] = GK_EXP_TAB_INIT;
#endif

GK_HD uint64_t gk_exp_tab(int i) {
#if defined(__CUDA_ARCH__)
    return gk_exp_tab_dev[i];
#else
    return GK_EXP_TAB[i];
#endif
}

/* exp(x), identical bits to glibc 2.39's FMA variant for every finite x. */
GK_HD double gk_exp(double x) {
    const double InvLn2N = 0x1.71547652b82fep+7, Shift = 0x1.8p52;
    const double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    uint32_t abstop = (uint32_t)(gk_asuint64(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {                 /* |x| < 2^-54 or |x| >= 512 */
        if ((uint32_t)(abstop - 0x3c9u) >= 0x80000000u) return 1.0 + x;
        if (abstop >= 0x409u) {                     /* |x| >= 1024 */
            if (gk_asuint64(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return (gk_asuint64(x) >> 63) ? 0.0 : gk_asdouble(0x7ff0000000000000ull);
        }
        abstop = 0;                                 /* large |x|: special case below */
    }
    double kd = gk_fma(x, InvLn2N, Shift);
    uint64_t ki = gk_asuint64(kd);
    kd = kd - Shift;
    double r = gk_fma(kd, NegLn2loN, gk_fma(kd, NegLn2hiN, x));
    int idx = (int)(2 * (ki & 127));
    uint64_t top = ki << 45;
    double tail = gk_asdouble(gk_exp_tab(idx));
    uint64_t sbits = gk_exp_tab(idx + 1) + top;
    double r2 = r * r;
    double tmp = gk_fma(r2 * r2, gk_fma(r, C5, C4), gk_fma(gk_fma(r, C3, C2), r2, r + tail));
    if (abstop != 0) {
        double scale = gk_asdouble(sbits);
        return gk_fma(scale, tmp, scale);
    }
    if ((ki & 0x80000000ull) == 0) {                /* k > 0: exponent may overflow */
        double scale = gk_asdouble(sbits - (1009ull << 52));
        return 0x1p1009 * gk_fma(scale, tmp, scale);
    }
    /* k < 0: subnormal range, evaluated without fusion */
    double scale = gk_asdouble(sbits + (1022ull << 52));
    double st = scale * tmp;
    double y = scale + st;
    if (1.0 > y) {
        double hi = y + 1.0;
        double lo = (scale - y) + st;
        y = ((((1.0 - hi) + y) + lo) + hi) - 1.0;
        if (y == 0.0) y = 0.0;
    }
    return y * 0x1p-1022;
}
