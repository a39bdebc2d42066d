// gk_sched.cu -- K1 (static segmented counts) and K2/K3 (per-point cycle
// estimator + feature composition) for sm_100a.
//
// K3 design: one warp = 32 points of the SAME kernel, one
// point per lane.  All lanes walk the kernel's token stream in lock-step
// (warp-uniform token loads and loop bounds -- list lengths depend only on the
// token stream), each carrying its own reservation table in shared memory.
// The reference's sequential first-fit (scheduler.py:59-68) is kept exactly:
// spans of every block are sorted (start, end) tuples; while no span of the
// block has negative length the spans are disjoint, hence their ends sorted,
// and the prefix the reference skips with `continue` (ends <= ready) is jumped
// by binary search; otherwise (negative global latency) the
// scan starts at the list head.  insort-right (scheduler.py:70-71) is a
// binary search plus shift.  Latency / unit / gap tables are staged in shared
// memory per CTA; `pipeline * (batches - 1)` is computed once per point.
#include <stdio.h>
#include <stdlib.h>

#include "gk_internal.cuh"
#include "gk_walk.cuh"

namespace gk {

// mem_throughput clamps to tp_floor (profiles.py:173-181, where the reference
// logs a warning per call) counted on the device into the caller's per-grid
// counter (gk_grid.tp_clamps; NULL = not counted): no library-global state, so
// concurrent sweeps on different streams keep separate counts
__device__ __forceinline__ double tput_c(double a, double b, double c, double floor_, double n,
                                         unsigned long long *clamps) {
    const double v = __dmul_rn(a, __dsub_rn(b, gk_exp(__dmul_rn(-c, n))));
    if (v <= 0.0) {
        if (clamps) atomicAdd(clamps, 1ull);
        return floor_;
    }
    return v;
}

constexpr int kWarps = 4;            // warps per CTA (each warp: 32 points of one kernel)
constexpr int kXfStride = 64;        // floats between feature rows of the compact-walk key tile
#ifndef GK_PROBE
#define GK_PROBE 2  // backward probe steps before the binary search for the first live span
#endif
#ifndef GK_SCAN_UNROLL
#define GK_SCAN_UNROLL 4  // spans loaded per first-fit scan iteration (4 measured best)
#endif
#ifndef GK_K23_CARVE
// measured (tools/sweep_variants.sh, B200): 0% carveout (max L1 for the
// reservation tables) beats a carveout sized for more resident CTAs
#define GK_K23_CARVE 0  // >= 0: percent; -1: driver default; -2: just enough for the CTAs
#endif
#ifndef GK_K23_FUSED_CARVE
#define GK_K23_FUSED_CARVE -1  // fused sweep carveout (percent); -1: computed like -2
#endif

// ------------------------------------------------------------------ K1

// One warp per kernel: coalesced token reads, exact integer tallies via warp
// sums, and the per-arch latency sums accumulated in program order (the
// reference's sequential `lat_sums[k] += m * latency`, features.py:161-165).
__global__ void __launch_bounds__(256) k1_static(gk_corpus C, gk_grid G, gk_kstat *__restrict__ ks,
                                                 double *__restrict__ latsum) {
    const int lane = threadIdx.x & 31;
    const uint32_t ki = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ki >= G.n_k) return;
    const gk_kernel K = C.ker[G.kernel_ids[ki]];
    long long cnt[4] = {0, 0, 0, 0}, br = 0, ld = 0, st = 0;
    // per-arch ordered sums, replicated in every lane
    double acc[3 * 4];
#pragma unroll
    for (int j = 0; j < 12; j++) acc[j] = 0.0;
    const uint32_t n_arch = G.n_arch;
    for (uint32_t b = 0; b < K.n_blk; b++) {
        const gk_block B = C.blk[K.blk0 + b];
        const double m = (double)B.mult;
        for (uint32_t i0 = 0; i0 < B.n; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool v = i < B.n;
            uint32_t cls = 0xff, sig = 0;
            if (v) {
                const gk_token T = C.tok[B.tok0 + i];
                cls = T.cls;
                sig = T.sig;
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if ((cls & 3) == (uint32_t)q) cnt[q] += B.mult;
                if (cls & GK_F_BRANCH) br += B.mult;
                if (cls & GK_F_GLOAD) ld += B.mult;
                if (cls & GK_F_GSTORE) st += B.mult;
            }
            const int nvalid = (int)min(32u, B.n - i0);
#pragma unroll
            for (int a = 0; a < 4; a++) {
                if ((uint32_t)a >= n_arch) break;
                double term = 0.0;
                int slot = 3;
                if (v) {
                    const uint32_t c = cls & 3;
                    slot = c == GK_COMPUTE ? 0 : (c == GK_SHARED ? 1 : (c == GK_MISC ? 2 : 3));
                    if (slot < 3) term = __dmul_rn(m, G.lat[(size_t)a * C.n_sig + sig]);
                }
                // ordered accumulation: lane j's term enters after lane j-1's
                for (int j = 0; j < nvalid; j++) {
                    const double tj = shfl_d(term, j);
                    const int sj = __shfl_sync(GK_FULL, slot, j);
#pragma unroll
                    for (int q = 0; q < 3; q++)
                        if (sj == q) acc[a * 3 + q] = __dadd_rn(acc[a * 3 + q], tj);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
#pragma unroll
        for (int j = 0; j < 4; j++) cnt[j] += __shfl_xor_sync(GK_FULL, cnt[j], o);
        br += __shfl_xor_sync(GK_FULL, br, o);
        ld += __shfl_xor_sync(GK_FULL, ld, o);
        st += __shfl_xor_sync(GK_FULL, st, o);
    }
    if (lane == 0) {
        gk_kstat s;
        for (int j = 0; j < 4; j++) s.cnt[j] = cnt[j];
        s.branches = br;
        s.loads = ld;
        s.stores = st;
        s.pad_ = 0;
        ks[ki] = s;
    }
    if (lane < 3 * (int)min(n_arch, 4u)) {
        const int a = lane / 3, j = lane % 3;
        latsum[((size_t)a * G.n_k + ki) * 3 + j] = acc[a * 3 + j];
    }
}

// more than 4 archs: fall back to one thread per (kernel, arch) for the sums
__global__ void k1_latsum_wide(gk_corpus C, gk_grid G, double *__restrict__ latsum) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)G.n_k * G.n_arch) return;
    const uint32_t ki = idx % G.n_k, a = idx / G.n_k;
    if (a < 4) return;
    const gk_kernel K = C.ker[G.kernel_ids[ki]];
    double s[3] = {0.0, 0.0, 0.0};
    for (uint32_t b = 0; b < K.n_blk; b++) {
        const gk_block B = C.blk[K.blk0 + b];
        for (uint32_t i = 0; i < B.n; i++) {
            const gk_token T = C.tok[B.tok0 + i];
            const uint32_t c = T.cls & 3;
            if (c == GK_GLOBAL) continue;
            const int j = c == GK_COMPUTE ? 0 : (c == GK_SHARED ? 1 : 2);
            s[j] = __dadd_rn(s[j], __dmul_rn((double)B.mult, G.lat[(size_t)a * C.n_sig + T.sig]));
        }
    }
    for (int j = 0; j < 3; j++) latsum[((size_t)a * G.n_k + ki) * 3 + j] = s[j];
}

// ------------------------------------------------------------ K2 / K3
//
// Lane-per-point: a warp owns 32 points of ONE kernel (consecutive (arch,
// config) pairs), so every lane walks the same token stream (uniform loads and
// control flow) while carrying its own reservation table.  Per-point tables
// live in shared memory as [row][lane] (conflict-free 8-byte accesses):
//   fin[row]      finish time of instruction `row` of the current block
//   ss/se[row]    sorted (start, end) spans; resource r's list occupies rows
//                 [tok.lst_row, +res_cnt[r]) and holds tok.lst_len spans when
//                 instruction i is scheduled.
// Blocks longer than the shared slab use the same layout in a global scratch
// slab (L1/L2 resident).

struct PointOut {
    uint8_t *status;
    int64_t *si;
    double *sf, *feat;
    const int32_t *sel_idx;
    uint32_t n_sel;
    double *sel;
    double *time_us;   // optional dense time_us column (fused sweep)
    gk_trace trace;
    int has_trace;
};

struct ArchSmem {
    double pipeline;
    double gap[GK_NRES];
    int64_t units[GK_NRES];
};

struct PointScalars {
    int active;
    uint32_t ki, ai, ci;
    size_t p;
    int64_t cap, n_schd, n_sm, waves;
    double gm;
};

// Per-lane constants of one point, selected by the warp-uniform resource id.
struct ResTerms {
    double dt[GK_NRES];   // pipeline * (ceil(n_tw / units_r) - 1)
    double gap[GK_NRES];
    int64_t nb[GK_NRES];
    __device__ __forceinline__ void pick(int r, double &d, double &g, int64_t &n) const {
        switch (r) {  // r is warp-uniform: a jump, not divergence
            case 0: d = dt[0]; g = gap[0]; n = nb[0]; break;
            case 1: d = dt[1]; g = gap[1]; n = nb[1]; break;
            case 2: d = dt[2]; g = gap[2]; n = nb[2]; break;
            case 3: d = dt[3]; g = gap[3]; n = nb[3]; break;
            default: d = dt[4]; g = gap[4]; n = nb[4]; break;
        }
    }
};

struct Slab {       // [row][32] tables of the current block (smem or global)
    double *fin, *ss, *se;
};

#define ROW(a, r) (a)[(size_t)(r) * 32 + lane]

#ifndef GK_DISCARD
#define GK_DISCARD 2  // 0: off; 1: dead tables dropped per work item; 2: span tables per block
#endif
// The per-warp reservation tables are dead once their block is scheduled (the
// next block writes every row it reads: schedule_block starts an empty table,
// as the reference's ReservationTable per block, scheduler.py:137-145), and
// the CFG rows once the item's schedule is composed.  Global stores write
// through to L2; without discards L2 writes the dirty lines back to HBM when
// the ensemble walk streams through it (ncu: 1.97 GB of DRAM writes per
// config-#2 sweep against 16 MB of results).  `discard.global.L2` invalidates
// a 128-byte line without write-back.  Rows are 256 B ([row][32] doubles),
// i.e. two lines each; the warp's lanes split the lines.  Per item (mode 1)
// many lines are already written back when the item ends (-34 % DRAM writes,
// r1); per block (mode 2) they are dropped while still L2-resident.
__device__ __forceinline__ void discard_rows(const double *base, uint32_t rows, int lane) {
#if GK_DISCARD
    const char *p = reinterpret_cast<const char *>(base);
    for (uint32_t q = lane; q < 2 * rows; q += 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + (size_t)q * 128) : "memory");
#endif
}

// schedule_block (scheduler.py:137-185) for this lane's point; returns delay.
__device__ __forceinline__ double schedule_block(const gk_corpus &C, const gk_block &B,
                                                 const ResTerms &RT, const double *lat_a,
                                                 double gm_lat, Slab m, int lane,
                                                 double *tr_start, double *tr_dur,
                                                 double *tr_lat, int64_t *tr_nb) {
    double delay = 0.0;
    bool neg = false;  // a negative-length span exists: ends may be unsorted
    const gk_token *tok = C.tok + B.tok0;
    gk_token Tn = tok[0];  // carried: token i + 1 is loaded once (its pred0 ends i's list)
    for (uint32_t i = 0; i < B.n; i++) {
        const gk_token T = Tn;
        Tn = tok[i + 1];  // the next block's first token or the corpus sentinel
        const uint32_t p1 = Tn.pred0;
        // the resource list's last span, loaded early: the probe's first step
        // and the insertion's first compare read it (70 % of inserts append)
        const uint32_t base = T.lst_row, L = T.lst_len;
        double s_last = 0.0, e_last = 0.0;
        if (L) {
            s_last = ROW(m.ss, base + L - 1);
            e_last = ROW(m.se, base + L - 1);
        }
        double dterm, gap;
        int64_t nb;
        RT.pick(T.res, dterm, gap, nb);
        const double lat = ((T.cls & 3) == GK_GLOBAL) ? gm_lat : lat_a[T.sig];
        const double d = __dadd_rn(lat, dterm);  // lat + pipeline * (nb - 1)
        const double len = __dadd_rn(d, gap);
        double ready = 0.0;  // scheduler.py:166-168
        for (uint32_t q = T.pred0; q < p1; q++) ready = dmax(ready, ROW(m.fin, C.preds[q]));

        // earliest_start (scheduler.py:59-68).  With only non-negative spans
        // the list is disjoint, so its ends are sorted and every span before
        // the first end > ready is skipped by the reference's `continue`.
        // first span with end > ready: probe back from the frontier (ready is
        // usually near it -- measured: 39 % of queries need no span at all),
        // binary search only past GK_PROBE steps
        uint32_t k = 0;
        if (!neg) {
            k = L;
            int steps = 0;
            if (k > 0 && e_last > ready) {
                k--;
                steps++;
                while (k > 0 && steps < GK_PROBE && ROW(m.se, base + k - 1) > ready) {
                    k--;
                    steps++;
                }
            }
            if (k > 0 && steps == GK_PROBE && ROW(m.se, base + k - 1) > ready) {
                uint32_t lo = 0, hi = k - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (ROW(m.se, base + mid) > ready) hi = mid;
                    else lo = mid + 1;
                }
                k = lo;
            }
        }
        double t = ready;
        // the reference's scan from there (2.9 spans on average), GK_SCAN_UNROLL
        // spans per iteration: independent loads, then the sequential decisions
        bool hit = false;
        for (; k < L && !hit; k += GK_SCAN_UNROLL) {
            double s4[GK_SCAN_UNROLL], e4[GK_SCAN_UNROLL];
#pragma unroll
            for (int u = 0; u < GK_SCAN_UNROLL; u++) {
                const bool in = k + u < L;
                s4[u] = in ? ROW(m.ss, base + k + u) : 0.0;
                e4[u] = in ? ROW(m.se, base + k + u) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < GK_SCAN_UNROLL; u++) {
                if (hit || k + u >= L) continue;
                if (e4[u] <= t) continue;
                if (s4[u] >= __dadd_rn(t, len)) {
                    hit = true;
                    continue;
                }
                t = e4[u];
            }
        }
        const double start = t;
        const double fin = __dadd_rn(start, d);
        const double end = __dadd_rn(fin, gap);  // (start + d) + gap
        neg |= end < start;
        // insort-right on (start, end) tuples (scheduler.py:70-71): one
        // insertion-sort step from the back (70 % of inserts append)
        uint32_t q = L;
        if (q > 0 && (start < s_last || (start == s_last && end < e_last))) {
            ROW(m.ss, base + q) = s_last;
            ROW(m.se, base + q) = e_last;
            q--;
            while (q > 0) {
                const double s = ROW(m.ss, base + q - 1), e = ROW(m.se, base + q - 1);
                if (!(start < s || (start == s && end < e))) break;
                ROW(m.ss, base + q) = s;
                ROW(m.se, base + q) = e;
                q--;
            }
        }
        ROW(m.ss, base + q) = start;
        ROW(m.se, base + q) = end;
        ROW(m.fin, i) = fin;
        delay = dmax(delay, fin);  // scheduler.py:184
        if (tr_start) {
            tr_start[i] = start;
            tr_dur[i] = d;
            tr_lat[i] = lat;
            tr_nb[i] = nb;
        }
    }
    return delay;
}

// Returns time_us when the point is fully valid (status OK), else NaN.  In the
// fused sweep, `xw` (this lane's column of the warp's feature tile, stride 32)
// receives the manifest features already scaled by ensemble `E` (power.py:144).
__device__ __forceinline__ double finish_point(const gk_corpus &C, const gk_grid &G,
                                               const gk_kstat *__restrict__ ks,
                                               const double *__restrict__ latsum,
                                               const gk_kernel &K, const PointScalars &P,
                                               double cfg_delay, const PointOut &O,
                                               double *xw = nullptr,
                                               const gk_ensemble *E = nullptr,
                                               float *xf = nullptr) {
    const gk_arch &A = G.arch[P.ai];
    const gk_config c = G.cfg[P.ci];
    const gk_kstat S = ks[P.ki];
    const int64_t tpb = c.tpb, nB = c.n_blocks, tt = nB * tpb, waves = P.waves;
    const double gm = P.gm;
    // schedule_kernel tail (scheduler.py:338-363)
    const double d_kernel = __dmul_rn((double)waves, cfg_delay);
    const int64_t n_gm = waves * S.cnt[GK_GLOBAL], n_shm = waves * S.cnt[GK_SHARED];
    const double x = (double)tt;
    const double overhead = __dmul_rn(__dadd_rn(__dmul_rn(A.ov_slope, x), A.ov_icpt), A.nu_gpu);
    const double lsu = (double)A.units[GK_LSU];
    double gm_pen = 0.0, sm_pen = 0.0, cm_pen = 0.0;
    if (n_gm != 0) {
        const double tp = tput_c(A.tpg_a, A.tpg_b, A.tpg_c, A.tp_floor, (double)n_gm, G.tp_clamps);
        gm_pen = __dmul_rn(__dmul_rn(__ddiv_rn(x, lsu), __ddiv_rn((double)A.access_gm_sz, tp)),
                           (double)n_gm);
        const double lines = __ddiv_rn((double)(waves * A.L2_sz), (double)A.access_sz);
        cm_pen = __dmul_rn(__ddiv_rn((double)(tt * n_gm), lines), gm);
    }
    if (n_shm != 0) {
        const double tp = tput_c(A.tps_a, A.tps_b, A.tps_c, A.tp_floor, (double)n_shm, G.tp_clamps);
        sm_pen = __dmul_rn(__dmul_rn(__ddiv_rn(x, (double)(A.units[GK_LSU] * A.nSM)),
                                     __ddiv_rn((double)A.access_shm_sz, tp)),
                           (double)n_shm);
    }
    const double d_total =
        __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d_kernel, overhead), gm_pen), sm_pen), cm_pen);

    // theoretical_occupancy (features.py:123-138)
    const int64_t wpb = (tpb + A.Sz_w - 1) / A.Sz_w;
    int64_t ob = A.wSM_max / wpb;
    if (A.nB_max < ob) ob = A.nB_max;
    if (c.regs > 0) {
        const int64_t r = A.reg_b_max / ((int64_t)c.regs * tpb);
        if (r < ob) ob = r;
    }
    if (c.shmem > 0) {
        const int64_t s = A.shm_b_max / c.shmem;
        if (s < ob) ob = s;
    }
    const int status = ob < 1 ? GK_INFEASIBLE_OCCUPANCY : GK_OK;
    const size_t p = P.p;
    if (O.status) O.status[p] = (uint8_t)status;
    if (O.si) {
        int64_t *si = O.si + p * GK_NSI;
        si[GK_SI_THREADS_SCHED] = P.n_schd;
        si[GK_SI_THREADS_PER_SM] = P.n_sm;
        si[GK_SI_BLOCKS_PER_SM] = P.cap;
        si[GK_SI_WAVES] = waves;
        si[GK_SI_N_GLOBAL] = n_gm;
        si[GK_SI_N_SHARED] = n_shm;
    }
    if (O.sf) {
        double *sf = O.sf + p * GK_NSF;
        sf[GK_SF_GM_LATENCY] = gm;
        sf[GK_SF_D_KERNEL] = d_kernel;
        sf[GK_SF_OVERHEAD] = overhead;
        sf[GK_SF_GM_PENALTY] = gm_pen;
        sf[GK_SF_SM_PENALTY] = sm_pen;
        sf[GK_SF_CM_PENALTY] = cm_pen;
        sf[GK_SF_D_TOTAL] = d_total;
        sf[GK_SF_TIME_US] = __ddiv_rn(d_total, A.nu_gpu);
        sf[GK_SF_CFG_DELAY] = cfg_delay;
    }
    const double time_us = __ddiv_rn(d_total, A.nu_gpu);
    if (O.time_us) O.time_us[p] = time_us;
    const double NaN = __longlong_as_double(0x7ff8000000000000ll);
    if (!O.feat && !O.sel && !xw) return status == GK_OK ? time_us : NaN;
    if (status != GK_OK) {
        if (O.feat)
            for (int j = 0; j < GK_NFEAT; j++) O.feat[p * GK_NFEAT + j] = NaN;
        if (O.sel)
            for (uint32_t j = 0; j < O.n_sel; j++) O.sel[p * O.n_sel + j] = NaN;
        return NaN;
    }
    // extract_features (features.py:149-247)
    const double *ls = latsum + ((size_t)P.ai * G.n_k + P.ki) * 3;
    double glob_sum = 0.0;  // GLOBAL latency terms replayed in program order
    for (uint32_t b = 0; b < K.n_blk; b++) {
        const gk_block &B = C.blk[K.blk0 + b];
        const double term = __dmul_rn((double)B.mult, gm);
        for (uint32_t j = 0; j < B.n_glob; j++) glob_sum = __dadd_rn(glob_sum, term);
    }
    const double wv = (double)waves;
    const double comp_sm = (double)(waves * S.cnt[GK_COMPUTE]);
    const double glob_sm = (double)(waves * S.cnt[GK_GLOBAL]);
    const double shar_sm = (double)(waves * S.cnt[GK_SHARED]);
    const double misc_sm = (double)(waves * S.cnt[GK_MISC]);
    const double comp_lat = __dmul_rn(wv, ls[0]), shar_lat = __dmul_rn(wv, ls[1]);
    const double misc_lat = __dmul_rn(wv, ls[2]), glob_lat = __dmul_rn(wv, glob_sum);
    const double total_inst = __dadd_rn(__dadd_rn(__dadd_rn(comp_sm, glob_sm), shar_sm), misc_sm);
    double cache_pen = 0.0, glb_pen = 0.0, sh_pen = 0.0;
    if (glob_sm > 0) {
        const double lines = __ddiv_rn((double)(waves * A.L2_sz), (double)A.access_sz);
        cache_pen = __dmul_rn(__ddiv_rn(__dmul_rn(x, glob_sm), lines), gm);
        glb_pen = __dmul_rn(
            __dmul_rn(__ddiv_rn(x, lsu),
                      __ddiv_rn((double)A.access_sz,
                                tput_c(A.tpg_a, A.tpg_b, A.tpg_c, A.tp_floor, glob_sm, G.tp_clamps))),
            glob_sm);
    }
    if (shar_sm > 0) {
        sh_pen = __dmul_rn(
            __dmul_rn(__ddiv_rn(x, (double)(A.units[GK_LSU] * A.nSM)),
                      __ddiv_rn((double)A.access_sz,
                                tput_c(A.tps_a, A.tps_b, A.tps_c, A.tp_floor, shar_sm, G.tp_clamps))),
            shar_sm);
    }
    // features on demand (no 32-double array: keeps register pressure down)
    auto feature = [&](int q) -> double {
        switch (q) {
            case 0: return comp_sm != 0 ? __ddiv_rn(comp_lat, comp_sm) : 0.0;
            case 1: return glob_sm != 0 ? __ddiv_rn(glob_lat, glob_sm) : 0.0;
            case 2: return misc_sm != 0 ? __ddiv_rn(misc_lat, misc_sm) : 0.0;
            case 3: return shar_sm != 0 ? __ddiv_rn(shar_lat, shar_sm) : 0.0;
            case 4: return (double)S.branches;
            case 5: return (double)S.cnt[GK_COMPUTE];
            case 6: return comp_sm;
            case 7: return comp_lat;
            case 8: return (double)S.cnt[GK_GLOBAL];
            case 9: return glob_sm;
            case 10: return glob_lat;
            case 11: return (double)(waves * S.loads);
            case 12: return (double)(waves * S.stores);
            case 13: return (double)S.cnt[GK_MISC];
            case 14: return misc_sm;
            case 15: return misc_lat;
            case 16: return (double)S.cnt[GK_SHARED];
            case 17: return shar_sm;
            case 18: return shar_lat;
            case 19: return (double)(nB < A.nSM ? nB : A.nSM);
            case 20: return (double)((P.n_sm + A.Sz_w - 1) / A.Sz_w);
            case 21: return wv;
            case 22: return x;
            case 23:
                return __dmul_rn(__ddiv_rn(x, (double)(A.nWS * A.Sz_w)),
                                 __ddiv_rn(total_inst, (double)A.nDU));
            case 24: return cache_pen;
            case 25: return glb_pen;
            case 26: return sh_pen;
            case 27: return __ddiv_rn((double)(ob * wpb), (double)A.wSM_max);
            case 28: return (double)c.regs;
            case 29: return (double)c.shmem;
            case 30: return (double)tpb;
            default: return (double)nB;
        }
    };
    if (O.feat) {
        double *o = O.feat + p * GK_NFEAT;
        for (int j = 0; j < GK_NFEAT; j++) o[j] = feature(j);
    }
    if (O.sel) {
        double *o = O.sel + p * O.n_sel;
        for (uint32_t j = 0; j < O.n_sel; j++) o[j] = feature(O.sel_idx[j]);
    }
    if (xw)
        for (uint32_t j = 0; j < O.n_sel; j++) {
            const double v = scale_feature(feature(O.sel_idx[j]), E->scale_lo[j], E->scale_hi[j]);
            xw[(size_t)j * 32] = v;
            if (xf) xf[(size_t)j * kXfStride] = __double2float_rd(v);  // compact-walk key
        }
    return time_us;
}


// Fused sweep (K2/K3 -> K4 -> K6 in one kernel): after a warp's 32 points are
// scheduled and their features composed, the same lanes walk their arch's
// ensemble.  Warps in the latency-bound scheduling phase and warps in the
// L1-bound walk phase then share each SM.
struct FusedArgs {
    gk_ensemble ens[4];
    uint32_t n_ens;
    int compact;  // walk a compact layout when the ensemble has one (default; GK_FUSED_COMPACT=0: 16-byte nodes)
    double *power, *energy;
};

// Persistent warps over work items (kernel, up to 32 consecutive (arch, config) pairs).
#ifndef GK_K23_MINB
#define GK_K23_MINB 4  // cycle-only sweep (c2): 2.60 ms at 4 (3: 2.82, 5: 2.67, 6: 2.77, 7: 2.82)
#endif
#ifndef GK_FUSED_MINB
#define GK_FUSED_MINB 8  // blocked walk, c2: 6.22 ms at 8 (7: 6.35, 9: 6.40, 10: 8.3); 16-byte nodes preferred 7
#endif
#ifndef GK_FUSED_ILP
#define GK_FUSED_ILP 8  // trees walked in lock-step inside the fused sweep (8 measured best)
#endif
#ifndef GK_FUSED_B2_SINK
#define GK_FUSED_B2_SINK 1
#endif
#ifndef GK_FUSED_B2_LDS2
#define GK_FUSED_B2_LDS2 1  // 2 shared feature loads per block (gk_walk.cuh): c5 127.2 -> 134.3 M points/s
#endif
#ifndef GK_FUSED_B2_ILP
#define GK_FUSED_B2_ILP 5  // blocked walk: trees in lock-step (each step = 2 levels); c2 at MINB 8: 6.22 ms (4: 6.40, 6: 6.49)
#endif
template <bool kFused>
__global__ void __launch_bounds__(kWarps * 32, kFused ? GK_FUSED_MINB : GK_K23_MINB) k23_schedule(
    gk_corpus C, gk_grid G, const gk_kstat *__restrict__ ks, const double *__restrict__ latsum,
    PointOut O, uint64_t n_items, uint32_t items_per_kernel, uint32_t ns,
    double *__restrict__ gscratch, uint32_t g_rows, uint32_t max_blk,
    unsigned long long *__restrict__ queue, FusedArgs F) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t n_arch = G.n_arch, n_sig = C.n_sig;
    ArchSmem *arch_s = reinterpret_cast<ArchSmem *>(smem_raw);
    double *lat_s = reinterpret_cast<double *>(arch_s + n_arch);
    double *slab_base = lat_s + (size_t)n_arch * n_sig;
    for (uint32_t t = threadIdx.x; t < n_arch; t += blockDim.x) {
        const gk_arch &A = G.arch[t];
        arch_s[t].pipeline = A.pipeline;
        for (int r = 0; r < GK_NRES; r++) {
            arch_s[t].gap[r] = A.gap[r];
            arch_s[t].units[r] = A.units[r];
        }
    }
    for (uint32_t t = threadIdx.x; t < n_arch * n_sig; t += blockDim.x) lat_s[t] = G.lat[t];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Slab smem_slab;
    smem_slab.fin = slab_base + (size_t)warp * 3 * ns * 32;
    smem_slab.ss = smem_slab.fin + (size_t)ns * 32;
    smem_slab.se = smem_slab.ss + (size_t)ns * 32;
    const uint64_t gwarp = (uint64_t)blockIdx.x * kWarps + warp;
    const uint64_t n_warps = (uint64_t)gridDim.x * kWarps;
    const size_t gslab = (3 * (size_t)g_rows + 2 * (size_t)max_blk) * 32;
    double *my_g = gscratch + gwarp * gslab;
    Slab glob_slab;
    glob_slab.fin = my_g;
    glob_slab.ss = my_g + (size_t)g_rows * 32;
    glob_slab.se = my_g + 2 * (size_t)g_rows * 32;
    double *blk_delay = my_g + 3 * (size_t)g_rows * 32;   // [max_blk][32]
    double *blk_finish = blk_delay + (size_t)max_blk * 32;
    const uint32_t P_k = n_arch * G.n_cfg;
    const double NaN = __longlong_as_double(0x7ff8000000000000ll);
    // fused: per-warp [n_sel][32] tile of scaled manifest features after the slabs
    // (row 0 of each warp's tile is the +inf leaf slot; features start at row 1)
    double *xw = slab_base + (size_t)kWarps * 3 * ns * 32 + (size_t)warp * (O.n_sel + 1) * 32 +
                 32 + lane;
    // fused: f32 keys for the compact walk after the fp64 tiles (only allocated
    // when the fused walk uses a compact layout, F.compact), a warp pair's
    // tiles interleaved as [n_sel + 1][64] so the row stride is 256 B (the
    // blocked walk's PRMT feature offsets)
    float *xf = (kFused && F.compact)
                    ? reinterpret_cast<float *>(slab_base + (size_t)kWarps * 3 * ns * 32 +
                                                (size_t)kWarps * (O.n_sel + 1) * 32) +
                          (size_t)(warp >> 1) * (O.n_sel + 1) * 64 + 64 + (warp & 1) * 32 + lane
                    : nullptr;
    if (kFused) {
        xw[-32] = __longlong_as_double(0x7ff0000000000000ll);
        if (xf) xf[-kXfStride] = __int_as_float(0x7f800000);
    }

    // dynamic work queue (items differ widely in cost; G.order puts the most
    // expensive kernels first so the tail is short)
    (void)n_warps;
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(queue, 1ull);
    item = __shfl_sync(GK_FULL, item, 0);
    for (; item < n_items;) {
        const uint32_t kr = (uint32_t)(item / items_per_kernel);
        const uint32_t ki = G.order ? G.order[kr] : kr;
        const uint32_t j0 = (uint32_t)(item % items_per_kernel) * 32;
        PointScalars P;
        P.active = j0 + lane < P_k;
        const uint32_t j = P.active ? j0 + lane : j0;
        P.ki = ki;
        P.ai = j / G.n_cfg;
        P.ci = j % G.n_cfg;
        P.p = (size_t)ki * P_k + j;
        const gk_kernel K = C.ker[G.kernel_ids[ki]];
        const gk_arch &A = G.arch[P.ai];
        const ArchSmem &AS = arch_s[P.ai];
        const gk_config cfg = G.cfg[P.ci];
        P.cap = block_cap(A, cfg);
        const bool feasible = P.cap >= 1;
        const int64_t tpb = cfg.tpb;
        P.n_schd = ((int64_t)cfg.n_blocks + A.nSM - 1) / A.nSM * tpb;
        P.n_sm = feasible ? P.cap * tpb : tpb;
        P.waves = (P.n_schd + P.n_sm - 1) / P.n_sm;
        P.gm = gm_latency(A, cfg);
        int64_t n_tw = P.n_sm;  // schedule_block / schedule_cfg faces override these
        if (G.n_tw_override && G.n_tw_override[P.ci] > 0) n_tw = G.n_tw_override[P.ci];
        if (G.gm_override && !isnan(G.gm_override[P.ci])) P.gm = G.gm_override[P.ci];
        ResTerms RT;
#pragma unroll
        for (int r = 0; r < GK_NRES; r++) {
            const int64_t u = AS.units[r];
            RT.nb[r] = (n_tw + u - 1) / u;  // batches, types.py:150-152
            RT.dt[r] = __dmul_rn(AS.pipeline, (double)(RT.nb[r] - 1));
            RT.gap[r] = AS.gap[r];
        }
        const double *lat_a = lat_s + (size_t)P.ai * n_sig;
        const bool write_trace = O.has_trace && P.active && feasible;

        for (uint32_t b = 0; b < K.n_blk; b++) {  // scheduler.py:203-205
            const gk_block B = C.blk[K.blk0 + b];
            const Slab m = B.n <= ns ? smem_slab : glob_slab;
            const size_t trow = P.p * K.n_tok + (B.tok0 - K.tok0);
            const double dl = schedule_block(
                C, B, RT, lat_a, P.gm, m, lane, write_trace ? O.trace.start + trow : nullptr,
                write_trace ? O.trace.duration + trow : nullptr,
                write_trace ? O.trace.latency + trow : nullptr,
                write_trace ? O.trace.n_batches + trow : nullptr);
            ROW(blk_delay, b) = dl;
#if GK_DISCARD == 2
            if (B.n > ns) {  // the block's tables are dead: drop them while L2-resident
                __syncwarp();
                discard_rows(glob_slab.fin, B.n, lane);
                discard_rows(glob_slab.ss, B.n, lane);
                discard_rows(glob_slab.se, B.n, lane);
                __syncwarp();  // ordered before the next block's writes to these lines
            }
#endif
        }
        // schedule_cfg composition (scheduler.py:206-211)
        const uint32_t *topo = C.topo + K.topo0;
        for (uint32_t q = 0; q < K.n_blk; q++) {
            const uint32_t i = topo[q];
            const gk_block &B = C.blk[K.blk0 + i];
            double d_in = 0.0;  // max(..., default=0.0)
            for (uint32_t u = 0; u < B.n_fpred; u++) {
                const double f = ROW(blk_finish, C.fpreds[B.fpred0 + u]);
                d_in = u == 0 ? f : dmax(d_in, f);
            }
            ROW(blk_finish, i) = __dadd_rn(d_in, __dmul_rn(ROW(blk_delay, i), (double)B.mult));
        }
        double cfg_delay = 0.0;
        bool first = true;
        for (uint32_t b = 0; b < K.n_blk; b++) {
            if (!C.blk[K.blk0 + b].is_exit) continue;
            const double f = ROW(blk_finish, b);
            if (first || f > cfg_delay) cfg_delay = f;
            first = false;
        }
        if (write_trace) {
            for (uint32_t b = 0; b < K.n_blk; b++) {
                O.trace.blk_delay[P.p * K.n_blk + b] = ROW(blk_delay, b);
                O.trace.blk_finish[P.p * K.n_blk + b] = ROW(blk_finish, b);
            }
        }
        // the item's tables are dead: drop them from L2 before the walk streams
        // the ensemble through it (only the global slab; rows actually used)
        __syncwarp();
        if (GK_DISCARD == 1 && K.max_n > ns) {
            const uint32_t used = min(K.max_n, g_rows);
            discard_rows(glob_slab.fin, used, lane);
            discard_rows(glob_slab.ss, used, lane);
            discard_rows(glob_slab.se, used, lane);
        }
        discard_rows(blk_delay, K.n_blk, lane);
        discard_rows(blk_finish, K.n_blk, lane);
        double t_ok = NaN;  // time_us of a fully valid point, else NaN
        const gk_ensemble *Ep = kFused ? &F.ens[P.ai < F.n_ens ? P.ai : 0] : nullptr;
        if (P.active) {
            if (feasible) {
                t_ok = finish_point(C, G, ks, latsum, K, P, cfg_delay, O, kFused ? xw : nullptr, Ep,
                                    xf);
            } else {
                if (O.status) O.status[P.p] = GK_INFEASIBLE_LAUNCH;
                if (O.si)
                    for (int q = 0; q < GK_NSI; q++) O.si[P.p * GK_NSI + q] = 0;
                if (O.sf)
                    for (int q = 0; q < GK_NSF; q++) O.sf[P.p * GK_NSF + q] = NaN;
                if (O.time_us) O.time_us[P.p] = NaN;
                if (O.feat)
                    for (int q = 0; q < GK_NFEAT; q++) O.feat[P.p * GK_NFEAT + q] = NaN;
                if (O.sel)
                    for (uint32_t q = 0; q < O.n_sel; q++) O.sel[P.p * O.n_sel + q] = NaN;
            }
        }
        if constexpr (kFused) {  // K4 + K6 for this lane's point
            if (P.active) {
                double pw = NaN, en = NaN;
                if (!isnan(t_ok)) {
                    auto x64 = [&](int f) { return xw[f * 32]; };
                    // measured on B200 (c2): the blocked walk (half the L1
                    // wavefronts of the 16-byte nodes, more instructions) wins
                    // once its loads are unpredicated (sink) and its feature
                    // offsets are one PRMT: 6.36 vs 6.44 ms; nodes8 loses
                    pw = F.compact && Ep->blocks
                             ? walk_ensemble_b2<GK_FUSED_B2_ILP, true, GK_FUSED_B2_SINK, GK_FUSED_B2_LDS2>(*Ep, xf, kXfStride, x64)
                         : F.compact && Ep->nodes8 ? walk_ensemble8<GK_FUSED_ILP>(*Ep, xf, kXfStride, x64)
                                                   : walk_ensemble<GK_FUSED_ILP>(*Ep, xw, 32);
                    en = __dmul_rn(pw, t_ok);
                }
                F.power[P.p] = pw;
                F.energy[P.p] = en;
            }
        }
        __syncwarp();
        if (lane == 0) item = atomicAdd(queue, 1ull);
        item = __shfl_sync(GK_FULL, item, 0);
    }
}

}  // namespace gk

// ------------------------------------------------------------- host side

namespace {
int g_sm_count = 0;
int sm_count() {
    if (!g_sm_count) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (g_sm_count <= 0) g_sm_count = 148;
    }
    return g_sm_count;
}
// per-lane shared-memory rows (instructions per block held on chip); GK_SMEM_ROWS tunes it
uint32_t smem_rows_cap() {
    static uint32_t v = 0;
    if (!v) {
        const char *e = getenv("GK_SMEM_ROWS");
        // measured on B200: L1-backed tables at 24 warps/SM beat a shared slab at
        // lower occupancy (profiles/README.md); 0 = all tables in the L1 scratch
        v = e ? (uint32_t)atoi(e) + 1 : 1;  // stored +1 so that 0 rows is representable
        if (v > 257) v = 257;
    }
    return v - 1;
}
constexpr int kMaxCtaPerSm = 16;
}  // namespace

int gk_launch_static(const gk_corpus *C, const gk_grid *G, gk_kstat *ks, double *latsum,
                     cudaStream_t st) {
    if (G->n_k == 0) return 0;
    const unsigned blocks = (G->n_k * 32 + 255) / 256;
    gk::k1_static<<<blocks, 256, 0, st>>>(*C, *G, ks, latsum);
    if (G->n_arch > 4) {
        const size_t n = (size_t)G->n_k * G->n_arch;
        gk::k1_latsum_wide<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*C, *G, latsum);
    }
    return gk_check_launch("k1_static");
}

static uint32_t smem_rows(uint32_t max_n) {
    const uint32_t cap = smem_rows_cap();
    return max_n < cap ? max_n : cap;
}
static uint32_t global_rows(uint32_t max_n) {
    return max_n > smem_rows_cap() ? (max_n ? max_n : 1) : 1;
}

size_t gk_sched_scratch_bytes(const gk_grid *G, uint32_t max_n, uint32_t max_blk) {
    (void)G;
    const size_t warps = (size_t)sm_count() * kMaxCtaPerSm * gk::kWarps;
    const size_t slab = (3 * (size_t)global_rows(max_n) + 2 * (size_t)max_blk) * 32;
    return warps * slab * sizeof(double) + 256;  // + the work-queue counter
}

template <bool kFused>
static int launch_sched(const gk_corpus *C, const gk_grid *G, const gk_kstat *ks,
                        const double *latsum, uint8_t *status, int64_t *si, double *sf,
                        double *feat, const int32_t *sel_idx, uint32_t n_sel, double *sel,
                        double *time_us, const gk_trace *trace, uint32_t max_n, uint32_t max_blk,
                        double *gscratch, const gk::FusedArgs &F, cudaStream_t st) {
    const auto kern = gk::k23_schedule<kFused>;
    const uint64_t P_k = (uint64_t)G->n_arch * G->n_cfg;
    if (G->n_k == 0 || P_k == 0) return 0;
    const uint32_t ipk = (uint32_t)((P_k + 31) / 32);
    const uint64_t n_items = (uint64_t)G->n_k * ipk;
    gk::PointOut O;
    O.status = status;
    O.si = si;
    O.sf = sf;
    O.feat = feat;
    O.sel_idx = sel_idx;
    O.n_sel = n_sel;
    O.sel = sel;
    O.time_us = time_us;
    O.has_trace = trace != nullptr && trace->start != nullptr;
    if (O.has_trace) O.trace = *trace;
    else memset(&O.trace, 0, sizeof O.trace);
    const uint32_t ns = smem_rows(max_n);
    const size_t smem = G->n_arch * (sizeof(gk::ArchSmem) + (size_t)C->n_sig * sizeof(double)) +
                        (size_t)gk::kWarps * 3 * ns * 32 * sizeof(double) +
                        (kFused ? (size_t)gk::kWarps * (n_sel + 1) * 32 *
                                      (sizeof(double) + (F.compact ? sizeof(float) : 0))
                                : 0);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    // the reservation tables that do not fit the shared slab live in L1: prefer L1
    // (a 0% carveout caps resident CTAs at 5/SM even for ~1 KB of tables: ask
    // for just enough shared memory for the register-limited CTA count)
    {
        const size_t per_sm_bytes = (smem + 1024) * 8;
        int carve = (int)((per_sm_bytes * 100 + 228 * 1024 - 1) / (228 * 1024));
        if (carve > 100) carve = 100;
        const int computed = carve;
        if (GK_K23_CARVE >= 0) carve = GK_K23_CARVE;
        // the fused kernel needs shared memory for its feature tiles
        if (kFused) carve = GK_K23_FUSED_CARVE >= 0 ? GK_K23_FUSED_CARVE : computed;
        if (GK_K23_CARVE != -1 || kFused)
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, gk::kWarps * 32, smem);
    if (per_sm < 1) {
        gk_set_error("k23_schedule: %zu B shared memory per CTA does not fit", smem);
        return -1;
    }
    if (per_sm > kMaxCtaPerSm) per_sm = kMaxCtaPerSm;
    uint64_t grid = (uint64_t)sm_count() * per_sm;
    const uint64_t need = (n_items + gk::kWarps - 1) / gk::kWarps;
    if (grid > need) grid = need;
    // work-queue counter lives past the per-warp slabs
    const size_t warps_cap = (size_t)sm_count() * kMaxCtaPerSm * gk::kWarps;
    unsigned long long *queue = reinterpret_cast<unsigned long long *>(
        gscratch + warps_cap * (3 * (size_t)global_rows(max_n) + 2 * (size_t)max_blk) * 32);
    cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st);
    kern<<<(unsigned)grid, gk::kWarps * 32, smem, st>>>(*C, *G, ks, latsum, O, n_items, ipk, ns,
                                                         gscratch, global_rows(max_n), max_blk,
                                                         queue, F);
    return gk_check_launch(kFused ? "k23_schedule<fused>" : "k23_schedule");
}

int gk_launch_sched(const gk_corpus *C, const gk_grid *G, const gk_kstat *ks, const double *latsum,
                    uint8_t *status, int64_t *si, double *sf, double *feat, const int32_t *sel_idx,
                    uint32_t n_sel, double *sel, double *time_us, const gk_trace *trace,
                    uint32_t max_n, uint32_t max_blk, double *gscratch, cudaStream_t st) {
    gk::FusedArgs F;
    memset(&F, 0, sizeof F);
    return launch_sched<false>(C, G, ks, latsum, status, si, sf, feat, sel_idx, n_sel, sel,
                               time_us, trace, max_n, max_blk, gscratch, F, st);
}

// fused sweep: schedule + features + ensemble walk + energy in one kernel
int gk_launch_sweep_fused(const gk_corpus *C, const gk_grid *G, const gk_kstat *ks,
                          const double *latsum, const gk_ensemble *ens, uint32_t n_ens,
                          const int32_t *sel_idx, uint32_t n_sel, uint8_t *status,
                          double *time_us, double *power, double *energy, uint32_t max_n,
                          uint32_t max_blk, double *gscratch, cudaStream_t st) {
    if (n_ens < 1 || n_ens > 4 || n_sel < 1 || n_sel > 64) {
        gk_set_error("fused sweep: 1..4 ensembles and 1..64 manifest features");
        return -1;
    }
    gk::FusedArgs F;
    memset(&F, 0, sizeof F);
    for (uint32_t a = 0; a < n_ens; a++) {
        if (ens[a].n_feat != n_sel) {
            gk_set_error("fused sweep: ensemble %u has %u features, manifest has %u", a,
                         ens[a].n_feat, n_sel);
            return -1;
        }
        F.ens[a] = ens[a];
    }
    F.n_ens = n_ens;
    {
        const char *e = getenv("GK_FUSED_COMPACT");
        F.compact = e ? atoi(e) != 0 : 1;
    }
    F.power = power;
    F.energy = energy;
    return launch_sched<true>(C, G, ks, latsum, status, nullptr, nullptr, nullptr, sel_idx, n_sel,
                              nullptr, time_us, nullptr, max_n, max_blk, gscratch, F, st);
}
