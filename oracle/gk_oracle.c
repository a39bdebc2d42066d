/*
 * gk_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * algorithm (gpukalc, arXiv 2305.01886) over the packed records of
 * include/gk.h.  Used by tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline leg as the CHECKER; never linked into or called by the product path.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py) and against the reference's own known-answer
 * values (worked example, vecadd, nn_euclid, energy cells).
 *
 * The restatement is deliberately literal: sorted reservation spans with
 * insort-right insertion and a linear first-fit scan (scheduler.py:53-71),
 * sequential fp64 sums in program order, glibc `exp` (the same libm entry
 * point Python's math.exp calls).  Build with -ffp-contract=off so no FMA
 * contraction changes a rounding.
 */
#include "../include/gk.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

enum { GK_NEGATIVE_COUNT = 3 };

/* Minimal static-chunk parallel-for over [0, n) with pthreads (CPU baseline
 * uses every host core; n_threads <= 1 runs inline). */
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } range_job;

static void *range_tramp(void *a) {
    range_job *j = (range_job *)a;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static void parallel_for(int64_t n, int n_threads, range_fn fn, void *ctx) {
    if (n_threads <= 1 || n < 2 * n_threads) {
        fn(ctx, 0, n);
        return;
    }
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    range_job jobs[256];
    for (int t = 0; t < n_threads; t++) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].lo = n * t / n_threads;
        jobs[t].hi = n * (t + 1) / n_threads;
        pthread_create(&th[t], NULL, range_tramp, &jobs[t]);
    }
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- helpers */

/* scheduler.py:220-237 per_sm_block_cap; returns cap (may be < 1). */
static int64_t block_cap(const gk_arch *A, const gk_config *c) {
    int64_t cap = A->nTh_sm_max / c->tpb;
    if (A->nB_max < cap) cap = A->nB_max;
    if (c->regs > 0) {
        int64_t r = A->reg_b_max / ((int64_t)c->regs * c->tpb);
        if (r < cap) cap = r;
    }
    if (c->shmem > 0) {
        int64_t s = A->shm_b_max / c->shmem;
        if (s < cap) cap = s;
    }
    return cap;
}

/* profiles.py:58-61 PiecewiseLinearModel.evaluate via global_mem_latency (:146-150) */
static double gm_latency(const gk_arch *A, const gk_config *c) {
    double x = (double)((int64_t)c->n_blocks * c->tpb);
    int i = 0;
    while (i < A->n_bp && A->bp[i] <= x) i++; /* bisect_right */
    return A->seg_slope[i] * x + A->seg_icpt[i];
}

/* profiles.py:159-182 mem_throughput, with ExpGrowthModel (:76-77) */
static double tput(double a, double b, double c, double floor_, double n) {
    double v = a * (b - exp(-c * n));
    return v <= 0 ? floor_ : v;
}

/* ------------------------------------------------------------------- K1 */

int gko_static_features(const gk_corpus *C, const gk_grid *G, gk_kstat *ks, double *latsum) {
    for (uint32_t ki = 0; ki < G->n_k; ki++) {
        const gk_kernel *K = &C->ker[G->kernel_ids[ki]];
        gk_kstat s;
        memset(&s, 0, sizeof s);
        for (uint32_t a = 0; a < G->n_arch; a++)
            for (int j = 0; j < 3; j++) latsum[((size_t)a * G->n_k + ki) * 3 + j] = 0.0;
        /* features.py:161-172: blocks in index order, instructions in order */
        for (uint32_t b = 0; b < K->n_blk; b++) {
            const gk_block *B = &C->blk[K->blk0 + b];
            int64_t m = B->mult;
            for (uint32_t i = 0; i < B->n; i++) {
                const gk_token *T = &C->tok[B->tok0 + i];
                int cls = T->cls & 3;
                s.cnt[cls] += m;
                if (T->cls & GK_F_BRANCH) s.branches += m;
                if (T->cls & GK_F_GLOAD) s.loads += m;
                if (T->cls & GK_F_GSTORE) s.stores += m;
                if (cls == GK_GLOBAL) continue; /* point-dependent, replayed per point */
                int j = cls == GK_COMPUTE ? 0 : (cls == GK_SHARED ? 1 : 2);
                for (uint32_t a = 0; a < G->n_arch; a++) {
                    double lat = G->lat[(size_t)a * C->n_sig + T->sig];
                    latsum[((size_t)a * G->n_k + ki) * 3 + j] += (double)m * lat;
                }
            }
        }
        ks[ki] = s;
    }
    return 0;
}

/* ------------------------------------------------------------ scheduler */

typedef struct { double s, e; } span;

/* scheduler.py:59-68 ReservationTable.earliest_start */
static double earliest_start(const span *sp, int n, double ready, double length) {
    double t = ready;
    for (int k = 0; k < n; k++) {
        if (sp[k].e <= t) continue;
        if (sp[k].s >= t + length) break;
        t = sp[k].e;
    }
    return t;
}

/* scheduler.py:70-71 reserve = bisect.insort (right) on (start, end) tuples */
static void insort(span *sp, int *n, double s, double e) {
    int pos = *n;
    for (int k = 0; k < *n; k++) {
        if (s < sp[k].s || (s == sp[k].s && e < sp[k].e)) { pos = k; break; }
    }
    memmove(&sp[pos + 1], &sp[pos], (size_t)(*n - pos) * sizeof(span));
    sp[pos].s = s;
    sp[pos].e = e;
    (*n)++;
}

/* scheduler.py:137-185 schedule_block; returns the block delay */
static double schedule_block(const gk_corpus *C, const gk_block *B, const gk_arch *A,
                             const double *lat_a, int64_t n_tw, double gm_lat,
                             span *spans, double *fin, double *tr_start, double *tr_dur,
                             double *tr_lat, int64_t *tr_nb) {
    span *res_sp[GK_NRES];
    int res_n[GK_NRES];
    uint32_t off = 0;
    for (int r = 0; r < GK_NRES; r++) {
        res_sp[r] = spans + off;
        res_n[r] = 0;
        off += B->res_cnt[r];
    }
    double delay = 0.0;
    for (uint32_t i = 0; i < B->n; i++) {
        const gk_token *T = &C->tok[B->tok0 + i];
        int res = T->res;
        double lat = ((T->cls & 3) == GK_GLOBAL) ? gm_lat : lat_a[T->sig];
        int64_t nb = (n_tw + A->units[res] - 1) / A->units[res];   /* types.py:150-152 */
        double d = lat + A->pipeline * (double)(nb - 1);
        double ready = 0.0;
        for (uint32_t q = T->pred0; q < T[1].pred0; q++) {
            double f = fin[C->preds[q]];
            if (f > ready) ready = f;
        }
        double gap = A->gap[res];
        double start = earliest_start(res_sp[res], res_n[res], ready, d + gap);
        insort(res_sp[res], &res_n[res], start, (start + d) + gap);
        fin[i] = start + d;
        if (start + d > delay) delay = start + d;
        if (tr_start) {
            tr_start[i] = start;
            tr_dur[i] = d;
            tr_lat[i] = lat;
            tr_nb[i] = nb;
        }
    }
    return delay;
}

/* One point: schedule_kernel (scheduler.py:325-363) + extract_features
 * (features.py:149-247).  Returns status. */
static int one_point(const gk_corpus *C, const gk_grid *G, const gk_kstat *ks,
                     const double *latsum, uint32_t ki, uint32_t ai, uint32_t ci,
                     int64_t *si, double *sf, double *feat, span *spans, double *fin,
                     double *blk_delay, double *blk_finish, const gk_trace *tr, size_t p) {
    const gk_kernel *K = &C->ker[G->kernel_ids[ki]];
    const gk_arch *A = &G->arch[ai];
    const gk_config *c = &G->cfg[ci];
    const double *lat_a = G->lat + (size_t)ai * C->n_sig;
    const gk_kstat *S = &ks[ki];

    int64_t cap = block_cap(A, c);
    if (cap < 1) return GK_INFEASIBLE_LAUNCH;
    int64_t tpb = c->tpb, nB = c->n_blocks;
    int64_t n_schd = (nB + A->nSM - 1) / A->nSM * tpb;           /* scheduler.py:249 */
    int64_t n_sm = cap * tpb;                                      /* :250 */
    int64_t waves = (n_schd + n_sm - 1) / n_sm;                    /* :251 */
    double gm = gm_latency(A, c);
    /* block/CFG-level faces: explicit n_tw / gm_latency (scheduler.py:137, 188) */
    int64_t n_tw = n_sm;
    if (G->n_tw_override && G->n_tw_override[ci] > 0) n_tw = G->n_tw_override[ci];
    if (G->gm_override && !isnan(G->gm_override[ci])) gm = G->gm_override[ci];
    int64_t tt = nB * tpb;

    /* schedule_cfg (scheduler.py:188-217) */
    for (uint32_t b = 0; b < K->n_blk; b++) {
        const gk_block *B = &C->blk[K->blk0 + b];
        size_t t0 = B->tok0 - K->tok0;
        int has_tr = tr && tr->start;
        blk_delay[b] = schedule_block(
            C, B, A, lat_a, n_tw, gm, spans, fin,
            has_tr ? tr->start + p * K->n_tok + t0 : NULL,
            has_tr ? tr->duration + p * K->n_tok + t0 : NULL,
            has_tr ? tr->latency + p * K->n_tok + t0 : NULL,
            has_tr ? tr->n_batches + p * K->n_tok + t0 : NULL);
    }
    for (uint32_t q = 0; q < K->n_blk; q++) {
        uint32_t i = C->topo[K->topo0 + q];
        const gk_block *B = &C->blk[K->blk0 + i];
        /* max(..., default=0.0): the default applies only with no predecessor */
        double d_in = 0.0;
        for (uint32_t j = 0; j < B->n_fpred; j++) {
            double f = blk_finish[C->fpreds[B->fpred0 + j]];
            if (j == 0 || f > d_in) d_in = f;
        }
        blk_finish[i] = d_in + blk_delay[i] * (double)B->mult;
    }
    double cfg_delay = 0.0;
    int first = 1;
    for (uint32_t b = 0; b < K->n_blk; b++) {
        if (!C->blk[K->blk0 + b].is_exit) continue;
        if (first || blk_finish[b] > cfg_delay) cfg_delay = blk_finish[b];
        first = 0;
    }
    if (tr && tr->blk_delay) {
        memcpy(tr->blk_delay + p * K->n_blk, blk_delay, K->n_blk * sizeof(double));
        memcpy(tr->blk_finish + p * K->n_blk, blk_finish, K->n_blk * sizeof(double));
    }

    double d_kernel = (double)waves * cfg_delay;
    int64_t n_gm = waves * S->cnt[GK_GLOBAL], n_shm = waves * S->cnt[GK_SHARED];
    if (n_gm < 0 || n_shm < 0) return GK_NEGATIVE_COUNT;
    double x = (double)tt;
    double overhead = (A->ov_slope * x + A->ov_icpt) * A->nu_gpu;  /* profiles.py:138-156 */
    double lsu = (double)A->units[GK_LSU];
    double gm_pen = 0.0, sm_pen = 0.0, cm_pen = 0.0;
    if (n_gm != 0) {                                               /* scheduler.py:269-282 */
        double tp = tput(A->tpg_a, A->tpg_b, A->tpg_c, A->tp_floor, (double)n_gm);
        gm_pen = ((double)tt / lsu) * ((double)A->access_gm_sz / tp) * (double)n_gm;
        double lines = (double)(waves * A->L2_sz) / (double)A->access_sz; /* :321 */
        cm_pen = (double)(tt * n_gm) / lines * gm;                        /* :322 */
    }
    if (n_shm != 0) {                                              /* :285-298 */
        double tp = tput(A->tps_a, A->tps_b, A->tps_c, A->tp_floor, (double)n_shm);
        sm_pen = ((double)tt / (double)(A->units[GK_LSU] * A->nSM)) *
                 ((double)A->access_shm_sz / tp) * (double)n_shm;
    }
    double d_total = (((d_kernel + overhead) + gm_pen) + sm_pen) + cm_pen; /* :123-131 */

    /* features.py:123-138 theoretical_occupancy */
    int64_t wpb = (tpb + A->Sz_w - 1) / A->Sz_w;
    int64_t ob = A->wSM_max / wpb;
    if (A->nB_max < ob) ob = A->nB_max;
    if (c->regs > 0) {
        int64_t r = A->reg_b_max / ((int64_t)c->regs * tpb);
        if (r < ob) ob = r;
    }
    if (c->shmem > 0) {
        int64_t s = A->shm_b_max / c->shmem;
        if (s < ob) ob = s;
    }
    int status = ob < 1 ? GK_INFEASIBLE_OCCUPANCY : GK_OK;

    if (si) {
        si[GK_SI_THREADS_SCHED] = n_schd;
        si[GK_SI_THREADS_PER_SM] = n_sm;
        si[GK_SI_BLOCKS_PER_SM] = cap;
        si[GK_SI_WAVES] = waves;
        si[GK_SI_N_GLOBAL] = n_gm;
        si[GK_SI_N_SHARED] = n_shm;
    }
    if (sf) {
        sf[GK_SF_GM_LATENCY] = gm;
        sf[GK_SF_D_KERNEL] = d_kernel;
        sf[GK_SF_OVERHEAD] = overhead;
        sf[GK_SF_GM_PENALTY] = gm_pen;
        sf[GK_SF_SM_PENALTY] = sm_pen;
        sf[GK_SF_CM_PENALTY] = cm_pen;
        sf[GK_SF_D_TOTAL] = d_total;
        sf[GK_SF_TIME_US] = d_total / A->nu_gpu;                   /* profiles.py:142-143 */
        sf[GK_SF_CFG_DELAY] = cfg_delay;
    }
    if (!feat || status != GK_OK) return status;

    /* extract_features (features.py:149-247) */
    const double *ls = latsum + ((size_t)ai * G->n_k + ki) * 3;
    double glob_sum = 0.0;        /* features.py:165 GLOBAL terms, program order */
    for (uint32_t b = 0; b < K->n_blk; b++) {
        const gk_block *B = &C->blk[K->blk0 + b];
        double term = (double)B->mult * gm;
        for (uint32_t j = 0; j < B->n_glob; j++) glob_sum += term;
    }
    double wv = (double)waves;
    double comp_sm = (double)(waves * S->cnt[GK_COMPUTE]);
    double glob_sm = (double)(waves * S->cnt[GK_GLOBAL]);
    double shar_sm = (double)(waves * S->cnt[GK_SHARED]);
    double misc_sm = (double)(waves * S->cnt[GK_MISC]);
    double comp_lat = wv * ls[0], shar_lat = wv * ls[1], misc_lat = wv * ls[2];
    double glob_lat = wv * glob_sum;
    double total_inst = ((comp_sm + glob_sm) + shar_sm) + misc_sm;
    double cache_pen = 0.0, glb_pen = 0.0, sh_pen = 0.0;
    if (glob_sm > 0) {
        double lines = (double)(waves * A->L2_sz) / (double)A->access_sz;
        cache_pen = ((double)tt * glob_sm) / lines * gm;
        glb_pen = ((double)tt / lsu) *
                  ((double)A->access_sz / tput(A->tpg_a, A->tpg_b, A->tpg_c, A->tp_floor, glob_sm)) *
                  glob_sm;
    }
    if (shar_sm > 0) {
        sh_pen = ((double)tt / (double)(A->units[GK_LSU] * A->nSM)) *
                 ((double)A->access_sz / tput(A->tps_a, A->tps_b, A->tps_c, A->tp_floor, shar_sm)) *
                 shar_sm;
    }
    double *f = feat;
    f[0] = comp_sm != 0 ? comp_lat / comp_sm : 0.0;     /* avg_comp_lat */
    f[1] = glob_sm != 0 ? glob_lat / glob_sm : 0.0;     /* avg_glob_lat */
    f[2] = misc_sm != 0 ? misc_lat / misc_sm : 0.0;     /* avg_misc_lat */
    f[3] = shar_sm != 0 ? shar_lat / shar_sm : 0.0;     /* avg_shar_lat */
    f[4] = (double)S->branches;
    f[5] = (double)S->cnt[GK_COMPUTE];
    f[6] = comp_sm;
    f[7] = comp_lat;
    f[8] = (double)S->cnt[GK_GLOBAL];
    f[9] = glob_sm;
    f[10] = glob_lat;
    f[11] = (double)(waves * S->loads);
    f[12] = (double)(waves * S->stores);
    f[13] = (double)S->cnt[GK_MISC];
    f[14] = misc_sm;
    f[15] = misc_lat;
    f[16] = (double)S->cnt[GK_SHARED];
    f[17] = shar_sm;
    f[18] = shar_lat;
    f[19] = (double)(nB < A->nSM ? nB : A->nSM);
    f[20] = (double)((n_sm + A->Sz_w - 1) / A->Sz_w);
    f[21] = wv;
    f[22] = (double)tt;
    f[23] = ((double)tt / (double)(A->nWS * A->Sz_w)) * (total_inst / (double)A->nDU);
    f[24] = cache_pen;
    f[25] = glb_pen;
    f[26] = sh_pen;
    f[27] = (double)(ob * wpb) / (double)A->wSM_max;
    f[28] = (double)c->regs;
    f[29] = (double)c->shmem;
    f[30] = (double)tpb;
    f[31] = (double)nB;
    return GK_OK;
}

typedef struct {
    const gk_corpus *C; const gk_grid *G; const gk_kstat *ks; const double *latsum;
    uint8_t *status; int64_t *si; double *sf; double *feat; const int32_t *sel_idx;
    uint32_t n_sel; double *sel; const gk_trace *tr; uint32_t max_n, max_blk;
} sf_ctx;

static void sf_range(void *vctx, int64_t lo, int64_t hi) {
    sf_ctx *X = (sf_ctx *)vctx;
    const gk_grid *G = X->G;
    span *spans = (span *)malloc(sizeof(span) * X->max_n);
    double *fin = (double *)malloc(sizeof(double) * X->max_n);
    double *bd = (double *)malloc(sizeof(double) * X->max_blk);
    double *bf = (double *)malloc(sizeof(double) * X->max_blk);
    double fbuf[GK_NFEAT];
    for (int64_t pl = lo; pl < hi; pl++) {
        size_t p = (size_t)pl;
        uint32_t ci = p % G->n_cfg, ai = (p / G->n_cfg) % G->n_arch,
                 ki = p / ((size_t)G->n_cfg * G->n_arch);
        int64_t sib[GK_NSI];
        double sfb[GK_NSF];
        int st = one_point(X->C, G, X->ks, X->latsum, ki, ai, ci, sib, sfb,
                           (X->feat || X->sel) ? fbuf : NULL, spans, fin, bd, bf, X->tr, p);
        if (X->status) X->status[p] = (uint8_t)st;
        int sched_ok = (st == GK_OK || st == GK_INFEASIBLE_OCCUPANCY);
        if (X->si) for (int j = 0; j < GK_NSI; j++) X->si[p * GK_NSI + j] = sched_ok ? sib[j] : 0;
        if (X->sf) for (int j = 0; j < GK_NSF; j++) X->sf[p * GK_NSF + j] = sched_ok ? sfb[j] : NAN;
        if (X->feat)
            for (int j = 0; j < GK_NFEAT; j++) X->feat[p * GK_NFEAT + j] = st == GK_OK ? fbuf[j] : NAN;
        if (X->sel)
            for (uint32_t j = 0; j < X->n_sel; j++)
                X->sel[p * X->n_sel + j] = st == GK_OK ? fbuf[X->sel_idx[j]] : NAN;
    }
    free(spans); free(fin); free(bd); free(bf);
}

int gko_schedule_features(const gk_corpus *C, const gk_grid *G, const gk_kstat *ks,
                          const double *latsum, uint8_t *status, int64_t *si, double *sf,
                          double *feat, const int32_t *sel_idx, uint32_t n_sel, double *sel,
                          const gk_trace *tr, int n_threads) {
    sf_ctx X = {C, G, ks, latsum, status, si, sf, feat, sel_idx, n_sel, sel, tr, 1, 1};
    for (uint32_t ki = 0; ki < G->n_k; ki++) {
        const gk_kernel *K = &C->ker[G->kernel_ids[ki]];
        if (K->max_n > X.max_n) X.max_n = K->max_n;
        if (K->n_blk > X.max_blk) X.max_blk = K->n_blk;
    }
    int64_t n_points = (int64_t)G->n_k * G->n_arch * G->n_cfg;
    parallel_for(n_points, (tr && tr->start) ? 1 : n_threads, sf_range, &X);
    return 0;
}

/* ------------------------------------------------------------ ensemble */

/* power.py:128-168 _scaled_input + predict_power over a flattened ensemble */
typedef struct {
    const gk_ensemble *E; const double *X; int64_t ld; const uint8_t *status;
    const double *time_us; double *power; double *energy;
} rf_ctx;

static void rf_range(void *vctx, int64_t lo, int64_t hi) {
    rf_ctx *R = (rf_ctx *)vctx;
    const gk_ensemble *E = R->E;
    double x[1024];
    for (int64_t r = lo; r < hi; r++) {
        if (R->status && R->status[r]) {
            R->power[r] = NAN;
            if (R->energy) R->energy[r] = NAN;
            continue;
        }
        const double *v = R->X + r * R->ld;
        for (uint32_t j = 0; j < E->n_feat; j++) {
            double lo_ = E->scale_lo[j], hi_ = E->scale_hi[j];
            x[j] = hi_ > lo_ ? (v[j] - lo_) / (hi_ - lo_) : 0.0;
        }
        double total = E->base_score;
        for (uint32_t t = 0; t < E->n_trees; t++) {
            const gk_node *N = E->nodes + E->tree_off[t];
            int32_t i = 0;
            while (N[i].feature >= 0) i = x[N[i].feature] <= N[i].v ? N[i].left : N[i].left + 1;
            total += N[i].v;
        }
        R->power[r] = total;
        if (R->energy) R->energy[r] = total * R->time_us[r];
    }
}

/* power.py:128-168 _scaled_input + predict_power over a flattened ensemble */
int gko_rf_predict(const gk_ensemble *E, const double *X, int64_t ld, int64_t n_rows,
                   const uint8_t *status, const double *time_us, double *power,
                   double *energy, int n_threads) {
    if (E->n_feat > 1024) return -1;
    rf_ctx R = {E, X, ld, status, time_us, power, energy};
    parallel_for(n_rows, n_threads, rf_range, &R);
    return 0;
}

/* ------------------------------------------------ RF bootstrap (sklearn) */

/* MT19937 (numpy legacy RandomState) -- SK/ensemble/_forest.py:95-112 draws
 * randint(0, n, n) from RandomState(tree_seed); randint uses masked rejection
 * on 32-bit outputs (numpy random/_bounded_integers, legacy path). */
typedef struct { uint32_t mt[624]; int i; } mt19937;

static void mt_seed(mt19937 *m, uint32_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 624; i++)
        m->mt[i] = 1812433253u * (m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) + (uint32_t)i;
    m->i = 624;
}

static uint32_t mt_next(mt19937 *m) {
    if (m->i >= 624) {
        for (int k = 0; k < 624; k++) {
            uint32_t y = (m->mt[k] & 0x80000000u) | (m->mt[(k + 1) % 624] & 0x7fffffffu);
            m->mt[k] = m->mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        m->i = 0;
    }
    uint32_t y = m->mt[m->i++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* counts[n] = bincount(RandomState(seed).randint(0, n, n)) */
int gko_bootstrap_counts(uint32_t seed, int64_t n, uint8_t *counts) {
    mt19937 m;
    mt_seed(&m, seed);
    uint32_t rng = (uint32_t)(n - 1), mask = rng;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    memset(counts, 0, (size_t)n);
    for (int64_t k = 0; k < n; k++) {
        uint32_t v;
        do { v = mt_next(&m) & mask; } while (v > rng);
        counts[v]++;
    }
    return 0;
}

int gko_abi_version(void) { return GK_ABI_VERSION; }
