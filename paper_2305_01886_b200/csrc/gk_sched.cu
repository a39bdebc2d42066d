// gk_sched.cu -- K1 (static segmented counts) and K2/K3 (per-point cycle
// estimator + feature composition) for sm_100a.
//
// K3 design: one warp = 4 points of the SAME kernel (4
// segments x 8 lanes).  All segments walk the kernel's token stream in
// lock-step (warp-uniform control flow; the per-resource span-list lengths
// depend only on the token stream), while each segment carries its own
// reservation table.  The reference's sequential first-fit scan
// (scheduler.py:59-68) is evaluated exactly with a segmented prefix-max over
// the (start, end)-sorted span list: t_k = max(ready, e_0..e_{k-1}); the
// answer is t_k at the first k with e_k > t_k and s_k >= t_k + length, else
// the running max -- valid for negative-length spans too.
// insort (scheduler.py:70-71) becomes a segmented ballot count + shift.
// Span lists live in shared memory (spilling to a global scratch slot for
// blocks longer than kSmemInstr); latency / unit / gap tables are staged in
// shared memory per CTA.
#include <stdio.h>

#include "gk_internal.cuh"

namespace gk {

constexpr int kSeg = 8;              // lanes per point
constexpr int kPts = 32 / kSeg;      // points per warp
constexpr int kWarps = 8;            // warps per CTA
constexpr int kSmemInstr = 48;       // per-point span/fin capacity in shared memory

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

// shared-memory staging of the per-arch tables
struct ArchSmem {
    double pipeline;
    double gap[GK_NRES];
    int64_t units[GK_NRES];
};

// One segment's reservation table + per-instruction finish times.
struct SegMem {
    double *fin;   // [cap]
    double *ss;    // span starts [cap], resource r at [res_off[r], +res_cnt[r])
    double *se;    // span ends
};

// Schedule one basic block for the 4 points of this warp.  Returns the block
// delay of this lane's point (segment-uniform).  scheduler.py:137-185.
__device__ __forceinline__ double schedule_block(
    const gk_corpus &C, const gk_block &B, const ArchSmem *__restrict__ arch_s,
    const double *__restrict__ lat_s, uint32_t n_sig, int ai, int64_t n_tw, double gm_lat,
    SegMem mem, int sl, unsigned seg_mask, int seg_shift, double *tr_start, double *tr_dur,
    double *tr_lat, int64_t *tr_nb, bool write_trace) {
    const ArchSmem &A = arch_s[ai];
    uint32_t res_off[GK_NRES], res_len[GK_NRES];
    {
        uint32_t o = 0;
#pragma unroll
        for (int r = 0; r < GK_NRES; r++) {
            res_off[r] = o;
            res_len[r] = 0;
            o += B.res_cnt[r];
        }
    }
    double delay = 0.0;
    const gk_token *tok = C.tok + B.tok0;
    for (uint32_t i = 0; i < B.n; i++) {
        const gk_token T = tok[i];
        const uint32_t next_pred = tok[i + 1].pred0;
        const int r = T.res;
        const double lat = ((T.cls & 3) == GK_GLOBAL) ? gm_lat : lat_s[ai * n_sig + T.sig];
        const int64_t units = A.units[r];
        const int64_t nb = (n_tw + units - 1) / units;  // types.py:150-152
        const double d = __dadd_rn(lat, __dmul_rn(A.pipeline, (double)(nb - 1)));
        const double gap = A.gap[r];
        const double len = __dadd_rn(d, gap);
        // ready = max(0, finish of DFG producers)   scheduler.py:166-168
        double ready = 0.0;
        for (uint32_t q = T.pred0; q < next_pred; q++) ready = dmax(ready, mem.fin[C.preds[q]]);

        // ---- earliest_start: segmented prefix-max scan over sorted spans
        const uint32_t L = res_len[r];
        const uint32_t base = res_off[r];
        double carry = ready, start = 0.0;
        bool found = false;
        for (uint32_t c0 = 0; c0 < L; c0 += kSeg) {
            const uint32_t k = c0 + sl;
            const bool valid = k < L;
            const double s = valid ? mem.ss[base + k] : 0.0;
            const double e = valid ? mem.se[base + k] : -__longlong_as_double(0x7ff0000000000000ll);
            double pm = e;  // inclusive prefix max of ends inside the chunk
#pragma unroll
            for (int off = 1; off < kSeg; off <<= 1) {
                const double o = shfl_up_d(pm, off, kSeg);
                if (sl >= off) pm = dmax(pm, o);
            }
            double ex = shfl_up_d(pm, 1, kSeg);
            const double tk = sl == 0 ? carry : dmax(carry, ex);
            const bool hit = valid && !found && (e > tk) && (s >= __dadd_rn(tk, len));
            const unsigned bal = (__ballot_sync(GK_FULL, hit) >> seg_shift) & 0xffu;
            const double tsel = shfl_d(tk, bal ? __ffs(bal) - 1 : 0, kSeg);
            const double cmax = shfl_d(pm, kSeg - 1, kSeg);
            if (!found) {
                if (bal) {
                    start = tsel;
                    found = true;
                } else {
                    carry = dmax(carry, cmax);
                }
            }
            if (__all_sync(GK_FULL, found)) break;
        }
        if (!found) start = carry;
        const double fin = __dadd_rn(start, d);
        const double end = __dadd_rn(fin, gap);  // (start + d) + gap, scheduler.py:171

        // ---- insort-right: pos = #elements <= (start, end)
        uint32_t pos = 0;
        for (uint32_t c0 = 0; c0 < L; c0 += kSeg) {
            const uint32_t k = c0 + sl;
            const bool valid = k < L;
            bool le = false;
            if (valid) {
                const double s = mem.ss[base + k], e = mem.se[base + k];
                le = !(start < s || (start == s && end < e));
            }
            const unsigned bal = (__ballot_sync(GK_FULL, le) >> seg_shift) & 0xffu;
            pos += __popc(bal);
            // sorted list: once a chunk is not all-le for every segment, stop
            const bool seg_done = __popc(bal) < min((uint32_t)kSeg, L - c0);
            if (__all_sync(GK_FULL, seg_done)) break;
        }
        // shift elements [pos, L) up by one, last chunk first
        if (L > 0) {
            for (int c0 = (int)((L - 1) / kSeg) * kSeg; c0 >= 0; c0 -= kSeg) {
                const uint32_t k = (uint32_t)c0 + sl;
                const bool mv = k < L && k >= pos;
                double s = 0.0, e = 0.0;
                if (mv) {
                    s = mem.ss[base + k];
                    e = mem.se[base + k];
                }
                __syncwarp();
                if (mv) {
                    mem.ss[base + k + 1] = s;
                    mem.se[base + k + 1] = e;
                }
                __syncwarp();
                if (!__any_sync(GK_FULL, pos < (uint32_t)c0)) break;
            }
        }
        if (sl == 0) {
            mem.ss[base + pos] = start;
            mem.se[base + pos] = end;
            mem.fin[i] = fin;
            if (write_trace) {
                tr_start[i] = start;
                tr_dur[i] = d;
                tr_lat[i] = lat;
                tr_nb[i] = nb;
            }
        }
        __syncwarp();
        res_len[r] = L + 1;
        delay = dmax(delay, fin);  // scheduler.py:184
    }
    (void)seg_mask;
    return delay;
}

struct PointScalars {
    int active;
    uint32_t ki, ai, ci;
    size_t p;
    int64_t cap, n_schd, n_sm, waves;
    double gm;
};

__device__ __forceinline__ void finish_point(const gk_corpus &C, const gk_grid &G,
                                             const gk_kstat *__restrict__ ks,
                                             const double *__restrict__ latsum,
                                             const gk_kernel &K, const PointScalars &P,
                                             double cfg_delay, const PointOut &O) {
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
        const double tp = tput(A.tpg_a, A.tpg_b, A.tpg_c, A.tp_floor, (double)n_gm);
        gm_pen = __dmul_rn(__dmul_rn(__ddiv_rn(x, lsu), __ddiv_rn((double)A.access_gm_sz, tp)),
                           (double)n_gm);
        const double lines = __ddiv_rn((double)(waves * A.L2_sz), (double)A.access_sz);
        cm_pen = __dmul_rn(__ddiv_rn((double)(tt * n_gm), lines), gm);
    }
    if (n_shm != 0) {
        const double tp = tput(A.tps_a, A.tps_b, A.tps_c, A.tp_floor, (double)n_shm);
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
    if (O.time_us) O.time_us[p] = __ddiv_rn(d_total, A.nu_gpu);
    if (!O.feat && !O.sel) return;
    const double NaN = __longlong_as_double(0x7ff8000000000000ll);
    if (status != GK_OK) {
        if (O.feat)
            for (int j = 0; j < GK_NFEAT; j++) O.feat[p * GK_NFEAT + j] = NaN;
        if (O.sel)
            for (uint32_t j = 0; j < O.n_sel; j++) O.sel[p * O.n_sel + j] = NaN;
        return;
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
                                tput(A.tpg_a, A.tpg_b, A.tpg_c, A.tp_floor, glob_sm))),
            glob_sm);
    }
    if (shar_sm > 0) {
        sh_pen = __dmul_rn(
            __dmul_rn(__ddiv_rn(x, (double)(A.units[GK_LSU] * A.nSM)),
                      __ddiv_rn((double)A.access_sz,
                                tput(A.tps_a, A.tps_b, A.tps_c, A.tp_floor, shar_sm))),
            shar_sm);
    }
    double f[GK_NFEAT];
    f[0] = comp_sm != 0 ? __ddiv_rn(comp_lat, comp_sm) : 0.0;
    f[1] = glob_sm != 0 ? __ddiv_rn(glob_lat, glob_sm) : 0.0;
    f[2] = misc_sm != 0 ? __ddiv_rn(misc_lat, misc_sm) : 0.0;
    f[3] = shar_sm != 0 ? __ddiv_rn(shar_lat, shar_sm) : 0.0;
    f[4] = (double)S.branches;
    f[5] = (double)S.cnt[GK_COMPUTE];
    f[6] = comp_sm;
    f[7] = comp_lat;
    f[8] = (double)S.cnt[GK_GLOBAL];
    f[9] = glob_sm;
    f[10] = glob_lat;
    f[11] = (double)(waves * S.loads);
    f[12] = (double)(waves * S.stores);
    f[13] = (double)S.cnt[GK_MISC];
    f[14] = misc_sm;
    f[15] = misc_lat;
    f[16] = (double)S.cnt[GK_SHARED];
    f[17] = shar_sm;
    f[18] = shar_lat;
    f[19] = (double)(nB < A.nSM ? nB : A.nSM);
    f[20] = (double)((P.n_sm + A.Sz_w - 1) / A.Sz_w);
    f[21] = wv;
    f[22] = x;
    f[23] = __dmul_rn(__ddiv_rn(x, (double)(A.nWS * A.Sz_w)), __ddiv_rn(total_inst, (double)A.nDU));
    f[24] = cache_pen;
    f[25] = glb_pen;
    f[26] = sh_pen;
    f[27] = __ddiv_rn((double)(ob * wpb), (double)A.wSM_max);
    f[28] = (double)c.regs;
    f[29] = (double)c.shmem;
    f[30] = (double)tpb;
    f[31] = (double)nB;
    if (O.feat) {
        double *o = O.feat + p * GK_NFEAT;
#pragma unroll
        for (int j = 0; j < GK_NFEAT; j++) o[j] = f[j];
    }
    if (O.sel) {
        double *o = O.sel + p * O.n_sel;
        for (uint32_t j = 0; j < O.n_sel; j++) {
            const int fi = O.sel_idx[j];
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < GK_NFEAT; q++) v = q == fi ? f[q] : v;
            o[j] = v;
        }
    }
}

// Persistent warps over work items (kernel, 4 consecutive (arch, config) pairs).
__global__ void __launch_bounds__(kWarps * 32) k23_schedule(
    gk_corpus C, gk_grid G, const gk_kstat *__restrict__ ks, const double *__restrict__ latsum,
    PointOut O, uint64_t n_items, uint32_t items_per_kernel, uint32_t smem_cap,
    double *__restrict__ gscratch, uint32_t gscratch_instr, uint32_t max_blk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t n_arch = G.n_arch, n_sig = C.n_sig;
    ArchSmem *arch_s = reinterpret_cast<ArchSmem *>(smem_raw);
    double *lat_s = reinterpret_cast<double *>(arch_s + n_arch);
    double *seg_base = lat_s + (size_t)n_arch * n_sig;
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
    const int seg = lane / kSeg, sl = lane % kSeg, seg_shift = seg * kSeg;
    const unsigned seg_mask = 0xffu << seg_shift;
    // this segment's shared-memory slab: fin | ss | se, smem_cap entries each
    double *my_smem = seg_base + ((size_t)(warp * kPts + seg)) * 3 * smem_cap;
    const uint64_t gwarp = ((uint64_t)blockIdx.x * kWarps + warp);
    const uint64_t n_warps = (uint64_t)gridDim.x * kWarps;
    // global slab: [3 * gscratch_instr] spans + [2 * max_blk] block delay/finish
    const size_t gslab = 3 * (size_t)gscratch_instr + 2 * (size_t)max_blk;
    double *my_g = gscratch + (gwarp * kPts + seg) * gslab;
    double *blk_delay = my_g + 3 * (size_t)gscratch_instr;
    double *blk_finish = blk_delay + max_blk;
    const uint32_t P_k = n_arch * G.n_cfg;

    for (uint64_t item = gwarp; item < n_items; item += n_warps) {
        const uint32_t ki = (uint32_t)(item / items_per_kernel);
        const uint32_t j = (uint32_t)(item % items_per_kernel) * kPts + seg;
        PointScalars P;
        P.active = j < P_k;
        const uint32_t jj = P.active ? j : (uint32_t)(item % items_per_kernel) * kPts;
        P.ki = ki;
        P.ai = jj / G.n_cfg;
        P.ci = jj % G.n_cfg;
        P.p = (size_t)ki * P_k + jj;
        const gk_kernel K = C.ker[G.kernel_ids[ki]];
        const gk_arch &A = G.arch[P.ai];
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

        const bool write_trace = O.has_trace && P.active && feasible;
        // schedule every block (scheduler.py:203-205)
        for (uint32_t b = 0; b < K.n_blk; b++) {
            const gk_block B = C.blk[K.blk0 + b];
            SegMem mem;
            if (B.n <= smem_cap) {
                mem.fin = my_smem;
                mem.ss = my_smem + smem_cap;
                mem.se = my_smem + 2 * smem_cap;
            } else {
                mem.fin = my_g;
                mem.ss = my_g + gscratch_instr;
                mem.se = my_g + 2 * (size_t)gscratch_instr;
            }
            const size_t t0 = B.tok0 - K.tok0;
            const size_t trow = P.p * K.n_tok + t0;
            const double dl = schedule_block(
                C, B, arch_s, lat_s, n_sig, (int)P.ai, n_tw, P.gm, mem, sl, seg_mask, seg_shift,
                write_trace ? O.trace.start + trow : nullptr,
                write_trace ? O.trace.duration + trow : nullptr,
                write_trace ? O.trace.latency + trow : nullptr,
                write_trace ? O.trace.n_batches + trow : nullptr, write_trace);
            if (sl == 0) blk_delay[b] = dl;
        }
        __syncwarp();
        if (sl == 0 && P.active) {
            // schedule_cfg composition (scheduler.py:206-211)
            const uint32_t *topo = C.topo + K.topo0;
            for (uint32_t q = 0; q < K.n_blk; q++) {
                const uint32_t i = topo[q];
                const gk_block &B = C.blk[K.blk0 + i];
                double d_in = 0.0;
                for (uint32_t u = 0; u < B.n_fpred; u++) {
                    const double f = blk_finish[C.fpreds[B.fpred0 + u]];
                    d_in = u == 0 ? f : dmax(d_in, f);
                }
                blk_finish[i] = __dadd_rn(d_in, __dmul_rn(blk_delay[i], (double)B.mult));
            }
            double cfg_delay = 0.0;
            bool first = true;
            for (uint32_t b = 0; b < K.n_blk; b++) {
                if (!C.blk[K.blk0 + b].is_exit) continue;
                if (first || blk_finish[b] > cfg_delay) cfg_delay = blk_finish[b];
                first = false;
            }
            if (write_trace) {
                for (uint32_t b = 0; b < K.n_blk; b++) {
                    O.trace.blk_delay[P.p * K.n_blk + b] = blk_delay[b];
                    O.trace.blk_finish[P.p * K.n_blk + b] = blk_finish[b];
                }
            }
            if (feasible) {
                finish_point(C, G, ks, latsum, K, P, cfg_delay, O);
            } else {
                const double NaN = __longlong_as_double(0x7ff8000000000000ll);
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
        __syncwarp();
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

size_t gk_sched_scratch_bytes(const gk_grid *G, uint32_t max_n, uint32_t max_blk) {
    (void)G;
    const size_t warps = (size_t)sm_count() * 8 * gk::kWarps;  // upper bound of resident warps
    const size_t slab = 3 * (size_t)max_n + 2 * (size_t)max_blk;
    return warps * gk::kPts * slab * sizeof(double);
}

int gk_launch_sched(const gk_corpus *C, const gk_grid *G, const gk_kstat *ks, const double *latsum,
                    uint8_t *status, int64_t *si, double *sf, double *feat, const int32_t *sel_idx,
                    uint32_t n_sel, double *sel, double *time_us, const gk_trace *trace,
                    uint32_t max_n, uint32_t max_blk, double *gscratch, cudaStream_t st) {
    const uint64_t P_k = (uint64_t)G->n_arch * G->n_cfg;
    if (G->n_k == 0 || P_k == 0) return 0;
    const uint32_t ipk = (uint32_t)((P_k + gk::kPts - 1) / gk::kPts);
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
    const uint32_t smem_cap = max_n < (uint32_t)gk::kSmemInstr ? (max_n ? max_n : 1) : gk::kSmemInstr;
    const size_t smem = G->n_arch * (sizeof(gk::ArchSmem) + (size_t)C->n_sig * sizeof(double)) +
                        (size_t)gk::kWarps * gk::kPts * 3 * smem_cap * sizeof(double);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(gk::k23_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gk::k23_schedule, gk::kWarps * 32, smem);
    if (per_sm < 1) {
        gk_set_error("k23_schedule: %zu B shared memory per CTA does not fit", smem);
        return -1;
    }
    if (per_sm > 8) per_sm = 8;
    uint64_t grid = (uint64_t)sm_count() * per_sm;
    const uint64_t need = (n_items + gk::kWarps - 1) / gk::kWarps;
    if (grid > need) grid = need;
    gk::k23_schedule<<<(unsigned)grid, gk::kWarps * 32, smem, st>>>(
        *C, *G, ks, latsum, O, n_items, ipk, smem_cap, gscratch, max_n, max_blk);
    return gk_check_launch("k23_schedule");
}
