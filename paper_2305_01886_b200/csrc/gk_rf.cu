// gk_rf.cu -- K4 (+K6): tree-ensemble inference and the energy epilogue.
//
// Reference: power.py:128-145 (_scaled_input), :148-168 (predict_power),
// :171-181 (predict_energy).  Nothing here is a dense contraction, so no
// tensor cores: the kernel is a gather-bound traversal over 16-byte nodes
// (BFS layout, right = left + 1, so one 16-byte load per visit).
//
// Layout per CTA: a tile of 128 rows is staged into shared memory with a bulk
// async copy (cp.async.bulk, the TMA 1-D path) when the rows are contiguous,
// scaled in place (x = (v - lo) / (hi - lo), or 0 when hi <= lo), then every
// thread walks kIlp trees concurrently for its row.  Leaves are added to the
// running total strictly in tree order, so the fp64 sum is bit-identical to
// the reference's sequential `total += leaf`.
#include <cooperative_groups.h>

#include "gk_internal.cuh"
#include "gk_walk.cuh"

namespace cg = cooperative_groups;

namespace gk {

constexpr int kRfThreads = 128;
// feature limits: the compact layouts' feature byte (gk_block2/3: 0..254;
// gk_node8 builders stop at 126) and the fp64 gk_node path's shared tile
// ((n_feat + 1) x 128 doubles <= 227 KB)
constexpr int kMaxFeatCompact = 255;
constexpr int kMaxFeat64 = 220;       // 128-row tiles
constexpr int kWideRows = 32;
constexpr int kMaxFeatWide = 886;     // 32-row tiles

struct RfArgs {
    gk_ensemble ens[4];        // up to 4 ensembles selected per row by `arch`
    uint32_t n_ens;
    const double *X;
    int64_t ld, n_rows;
    const uint8_t *status;
    const double *time_us;     // optional, indexed like rows
    double *power, *energy;
    // row -> arch map for grids: arch = (row / n_cfg) % n_arch (n_cfg = 0: arch 0)
    uint32_t n_cfg, n_arch;
};

__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gsrc, uint32_t bytes,
                                         uint64_t *bar) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
        "l"(gsrc), "r"(bytes), "r"(b)
        : "memory");
}

// kMaxF: compile-time bound on the feature count for the in-place transpose
// through registers (16 or 32); 0 = no staging, rows read straight from global.
// kT: rows (threads) per CTA -- 128, or 32 for wide tables (the tile is
// (n_feat + 1) x kT doubles)
template <int kMaxF, int kT = kRfThreads>
__global__ void __launch_bounds__(kT) k4_rf_predict(RfArgs R) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    const int64_t row0 = (int64_t)blockIdx.x * kT;
    const int64_t nr = min((int64_t)kT, R.n_rows - row0);
    const uint32_t nf = R.ens[0].n_feat;
    // one tile: row -1 = +inf (leaf slot), rows 0..nf-1 = [feature][thread]; the
    // raw [thread][feature] rows are staged into rows 0.. and transposed in place
    double *xt = reinterpret_cast<double *>(smem_raw) + kT;
    double *xs = xt;

    // ---- stage the row tile (contiguous when ld == n_feat)
    const bool bulk = kMaxF > 0 && (R.ld == (int64_t)nf) && ((nr * nf * 8) % 16 == 0) &&
                      ((reinterpret_cast<uintptr_t>(R.X + row0 * R.ld) & 15) == 0);
    if (kMaxF == 0) {
        // no staging: each thread reads its own row below
    } else if (bulk) {
        const uint32_t bytes = (uint32_t)(nr * nf * 8);
        if (threadIdx.x == 0) {
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
            asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(b));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes)
                         : "memory");
            bulk_g2s(xs, R.X + row0 * R.ld, bytes, &bar);
        }
        __syncthreads();
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n"
            " @!p bra WAIT_%=;\n}\n" ::"r"(b)
            : "memory");
    } else {
        for (int64_t q = threadIdx.x; q < nr * nf; q += kT) {
            const int64_t r = q / nf, f = q % nf;
            xs[r * nf + f] = R.X[(row0 + r) * R.ld + f];
        }
        __syncthreads();
    }
    const int64_t row = row0 + threadIdx.x;
    const bool live = threadIdx.x < nr;
    const uint32_t ai = (live && R.n_cfg) ? (uint32_t)((row / R.n_cfg) % R.n_arch) : 0u;
    const gk_ensemble &E = R.ens[ai < R.n_ens ? ai : 0];
    // scale and transpose to [feature][thread]: the per-visit reads x[f] with a
    // lane-varying f are then bank-conflict-free
    xt[(int)threadIdx.x - kT] = __longlong_as_double(0x7ff0000000000000ll);
    if (kMaxF > 0) {
        double v[kMaxF > 0 ? kMaxF : 1];
#pragma unroll
        for (int f = 0; f < kMaxF; f++)
            v[f] = (live && f < (int)nf) ? xs[threadIdx.x * nf + f] : 0.0;
        __syncthreads();  // every raw row is in registers before the tile is overwritten
#pragma unroll
        for (int f = 0; f < kMaxF; f++)
            if (live && f < (int)nf)
                xt[f * kT + threadIdx.x] = scale_feature(v[f], E.scale_lo[f], E.scale_hi[f]);
    } else if (live) {
        for (uint32_t f = 0; f < nf; f++)
            xt[f * kT + threadIdx.x] =
                scale_feature(R.X[row * R.ld + f], E.scale_lo[f], E.scale_hi[f]);
    }
    if (!live) return;
    const double NaN = __longlong_as_double(0x7ff8000000000000ll);
    if (R.status && R.status[row]) {
        R.power[row] = NaN;
        if (R.energy) R.energy[row] = NaN;
        return;
    }
    const double total = walk_ensemble(E, xt + threadIdx.x, kT);
    R.power[row] = total;
    if (R.energy) R.energy[row] = __dmul_rn(total, R.time_us[row]);
}

#ifndef GK_RF_B2_ILP
#define GK_RF_B2_ILP 10  // config #4: 82 M rows/s (8: 72 M, 4: 52 M, 12: 51 M)
#endif
// K4 over compact layouts (gk_node8 / gk_block2): the CTA's row tile is loaded
// coalesced, scaled, rounded toward -inf to f32 and stored transposed
// [feature][row] (stride kRfThreads: each walk read -- lane-varying feature,
// one row per lane -- hits 32 distinct banks).
// The exact fp64 feature is recomputed from X only for the rare a == t visit.
#ifndef GK_RF_B3_ILP
#define GK_RF_B3_ILP 8  // trees in lock-step per thread, gk_block3 walk
#endif
// kMode 0: gk_node8, 1: gk_block2 (f32 key tile), 2: gk_block3 (16-bit key
// tile, include/gk.h: half the shared memory per row)
template <int kMode>
__device__ __forceinline__ void rf_tile_c(const RfArgs &R, int64_t tile, float *xf_raw) {
    constexpr int S = kRfThreads;
    float *xf = xf_raw + S;  // row -1: the +inf slot of the leaf step
    uint16_t *xk = reinterpret_cast<uint16_t *>(xf_raw);
    const int64_t row0 = tile * kRfThreads;
    const int nr = (int)min((int64_t)kRfThreads, R.n_rows - row0);
    const int nf = (int)R.ens[0].n_feat;
    if (kMode != 2) xf_raw[threadIdx.x] = __int_as_float(0x7f800000);
    for (int q = threadIdx.x; q < nr * nf; q += kRfThreads) {
        const int r = q / nf, f = q - r * nf;
        const int64_t row = row0 + r;
        const uint32_t ai = R.n_cfg ? (uint32_t)((row / R.n_cfg) % R.n_arch) : 0u;
        const gk_ensemble &Er = R.ens[ai < R.n_ens ? ai : 0];
        const double v = scale_feature(R.X[row * R.ld + f], Er.scale_lo[f], Er.scale_hi[f]);
        if (kMode == 2)
            xk[f * S + r] = (uint16_t)key16(v);
        else
            xf[f * S + r] = __double2float_rd(v);
    }
    __syncthreads();
    if ((int)threadIdx.x >= nr) return;
    const int64_t row = row0 + threadIdx.x;
    const uint32_t ai = R.n_cfg ? (uint32_t)((row / R.n_cfg) % R.n_arch) : 0u;
    const gk_ensemble &E = R.ens[ai < R.n_ens ? ai : 0];
    const double NaN = __longlong_as_double(0x7ff8000000000000ll);
    if (R.status && R.status[row]) {
        R.power[row] = NaN;
        if (R.energy) R.energy[row] = NaN;
        return;
    }
    const double *xrow = R.X + row * R.ld;
    auto x64 = [&](int f) { return scale_feature(xrow[f], E.scale_lo[f], E.scale_hi[f]); };
    const double total = kMode == 2 ? walk_ensemble_b3<GK_RF_B3_ILP>(E, xk + threadIdx.x, S, x64)
                       : kMode == 1 ? walk_ensemble_b2<GK_RF_B2_ILP>(E, xf + threadIdx.x, S, x64)
                                    : walk_ensemble8<GK_RF_ILP>(E, xf + threadIdx.x, S, x64);
    R.power[row] = total;
    if (R.energy) R.energy[row] = __dmul_rn(total, R.time_us[row]);
}

template <int kMode>
__global__ void __launch_bounds__(kRfThreads) k4_rf_predict_c(RfArgs R) {
    extern __shared__ __align__(16) float xf_raw[];
    rf_tile_c<kMode>(R, blockIdx.x, xf_raw);
}

// Persistent form for large row tables: every resident CTA takes one tile per
// round and all CTAs cross a grid barrier between rounds, so the whole GPU
// walks the same few trees at any time -- the working set is a handful of
// trees (L2-resident) instead of the entire ensemble (> L2), which turns the
// deep-level node gathers from DRAM into L2 hits.
template <int kMode>
__global__ void __launch_bounds__(kRfThreads) k4_rf_predict_rounds(RfArgs R, int64_t n_tiles) {
    extern __shared__ __align__(16) float xf_raw[];
    cg::grid_group grid = cg::this_grid();
    const int64_t rounds = (n_tiles + gridDim.x - 1) / gridDim.x;
    for (int64_t k = 0; k < rounds; k++) {
        const int64_t tile = k * gridDim.x + blockIdx.x;
        if (tile < n_tiles) rf_tile_c<kMode>(R, tile, xf_raw);
        grid.sync();
    }
}

}  // namespace gk

int gk_launch_rf(const gk_ensemble *ens, uint32_t n_ens, const double *X, int64_t ld,
                 int64_t n_rows, const uint8_t *status, const double *time_us, double *power,
                 double *energy, uint32_t n_cfg, uint32_t n_arch, cudaStream_t st) {
    if (n_rows <= 0) return 0;
    if (n_ens < 1 || n_ens > 4) {
        gk_set_error("gk_rf_predict: 1..4 ensembles per launch (got %u)", n_ens);
        return -1;
    }
    gk::RfArgs R;
    memset(&R, 0, sizeof R);
    const uint32_t nf = ens[0].n_feat;
    for (uint32_t a = 0; a < n_ens; a++) {
        R.ens[a] = ens[a];
        if (ens[a].n_feat != nf) {
            gk_set_error("gk_rf_predict: ensembles of one sweep must share the manifest");
            return -1;
        }
    }
    if (nf < 1 || ld < (int64_t)nf) {
        gk_set_error("gk_rf_predict: n_feat=%u ld=%lld unsupported", nf, (long long)ld);
        return -1;
    }
    R.n_ens = n_ens;
    R.X = X;
    R.ld = ld;
    R.n_rows = n_rows;
    R.status = status;
    R.time_us = time_us;
    R.power = power;
    R.energy = energy;
    R.n_cfg = n_cfg;
    R.n_arch = n_arch ? n_arch : 1;
    bool all_b3 = true, all_blocks = true, all_n8 = true;
    for (uint32_t a = 0; a < n_ens; a++) {
        all_b3 &= ens[a].blocks3 != nullptr;
        all_blocks &= ens[a].blocks != nullptr;
        all_n8 &= ens[a].nodes8 != nullptr;
    }
    if (all_b3 || all_blocks || all_n8) {
        if (nf > (uint32_t)gk::kMaxFeatCompact) {
            gk_set_error("gk_rf_predict: n_feat=%u > %d", nf, gk::kMaxFeatCompact);
            return -1;
        }
        const int mode = all_b3 ? 2 : all_blocks ? 1 : 0;
        const size_t smem8 = mode == 2 ? (size_t)nf * gk::kRfThreads * sizeof(uint16_t)
                                       : ((size_t)nf + 1) * gk::kRfThreads * sizeof(float);
        const auto k8 = mode == 2 ? gk::k4_rf_predict_c<2>
                      : mode == 1 ? gk::k4_rf_predict_c<1> : gk::k4_rf_predict_c<0>;
        if (smem8 > 48 * 1024)
            cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k8, gk::kRfThreads, smem8);
        const size_t need = (smem8 + 1024) * (per_sm > 0 ? per_sm : 1);
        const int carve = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
        cudaFuncSetAttribute(k8, cudaFuncAttributePreferredSharedMemoryCarveout,
                             carve > 100 ? 100 : carve);
        const int64_t tiles = (n_rows + gk::kRfThreads - 1) / gk::kRfThreads;
        // persistent rounds once the table spans several waves of resident CTAs
        int dev = 0, n_sm = 0, coop = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        const auto kp = mode == 2 ? gk::k4_rf_predict_rounds<2>
                      : mode == 1 ? gk::k4_rf_predict_rounds<1> : gk::k4_rf_predict_rounds<0>;
        int per_sm_p = 0;
        if (smem8 > 48 * 1024)
            cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
        cudaFuncSetAttribute(kp, cudaFuncAttributePreferredSharedMemoryCarveout,
                             carve > 100 ? 100 : carve);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_p, kp, gk::kRfThreads, smem8);
        const int64_t resident = (int64_t)per_sm_p * n_sm;
        const char *pe = getenv("GK_RF_ROUNDS");
        const bool rounds_on = (pe ? atoi(pe) != 0 : true) && coop && resident > 0 &&
                               tiles >= 32 * resident;
        if (rounds_on) {
            int64_t nt = tiles;
            void *args[] = {&R, &nt};
            cudaError_t e = cudaLaunchCooperativeKernel((const void *)kp, dim3((unsigned)resident),
                                                        dim3(gk::kRfThreads), args, smem8, st);
            if (e != cudaSuccess) {
                gk_set_error("k4_rf_predict_rounds: %s", cudaGetErrorString(e));
                return -1;
            }
            return gk_check_launch("k4_rf_predict_rounds");
        }
        k8<<<(unsigned)tiles, gk::kRfThreads, smem8, st>>>(R);
        return gk_check_launch(mode == 2 ? "k4_rf_predict_c<blocks3>"
                               : mode == 1 ? "k4_rf_predict_c<blocks>" : "k4_rf_predict_c<nodes8>");
    }
    if (nf > (uint32_t)gk::kMaxFeatWide) {
        gk_set_error("gk_rf_predict: n_feat=%u > %d (fp64 node layout)", nf, gk::kMaxFeatWide);
        return -1;
    }
    const bool wide = nf > (uint32_t)gk::kMaxFeat64;
    const int rows_per_cta = wide ? gk::kWideRows : gk::kRfThreads;
    // one tile: leading +inf row + [feature][thread] (the staged raw rows are
    // transposed in place through registers)
    const size_t smem = ((size_t)nf + 1) * rows_per_cta * sizeof(double);
    const auto kern = wide ? gk::k4_rf_predict<0, gk::kWideRows>
                    : nf <= 16 ? gk::k4_rf_predict<16>
                    : nf <= 32 ? gk::k4_rf_predict<32> : gk::k4_rf_predict<0>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // the node gathers live in L1: give shared memory only what resident CTAs need
    {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, rows_per_cta, smem);
        const size_t need = (smem + 1024) * (per_sm > 0 ? per_sm : 1);
        int carve = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             carve > 100 ? 100 : carve);
    }
    const int64_t blocks = (n_rows + rows_per_cta - 1) / rows_per_cta;
    kern<<<(unsigned)blocks, rows_per_cta, smem, st>>>(R);
    return gk_check_launch("k4_rf_predict");
}
