// gk_api.cu -- the C-ABI of libgk (declared in include/gk.h).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "gk_internal.cuh"

static thread_local char g_err[512] = "";

void gk_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int gk_check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        gk_set_error("%s: %s", what, cudaGetErrorString(e));
        return -2;
    }
    return 0;
}

// defined in gk_sched.cu / gk_rf.cu
int gk_launch_static(const gk_corpus *, const gk_grid *, gk_kstat *, double *, cudaStream_t);
size_t gk_sched_scratch_bytes(const gk_grid *, uint32_t, uint32_t);
int gk_launch_sched(const gk_corpus *, const gk_grid *, const gk_kstat *, const double *, uint8_t *,
                    int64_t *, double *, double *, const int32_t *, uint32_t, double *, double *,
                    const gk_trace *, uint32_t, uint32_t, double *, cudaStream_t);
int gk_launch_rf(const gk_ensemble *, uint32_t, const double *, int64_t, int64_t, const uint8_t *,
                 const double *, double *, double *, uint32_t, uint32_t, cudaStream_t);
int gk_launch_sweep_fused(const gk_corpus *, const gk_grid *, const gk_kstat *, const double *,
                          const gk_ensemble *, uint32_t, const int32_t *, uint32_t, uint8_t *,
                          double *, double *, double *, uint32_t, uint32_t, double *,
                          cudaStream_t);

// GK_SWEEP_FUSED=0 selects the two-kernel sweep (K3 then K4) for A/B measurements
static bool sweep_fused() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("GK_SWEEP_FUSED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

namespace {

// optional per-stage timing of the fused sweep (profiling aid; synchronises)
bool g_stage_timing = false;
cudaEvent_t g_ev[4] = {nullptr, nullptr, nullptr, nullptr};

void stage_mark(int i, cudaStream_t st) {
    if (!g_stage_timing) return;
    if (!g_ev[i]) cudaEventCreate(&g_ev[i]);
    cudaEventRecord(g_ev[i], st);
}

int check_grid(const gk_corpus *C, const gk_grid *G) {
    if (!C || !G) {
        gk_set_error("null corpus or grid");
        return -1;
    }
    if (G->n_arch == 0 || G->n_cfg == 0) {
        gk_set_error("grid needs at least one arch and one config");
        return -1;
    }
    return 0;
}

}  // namespace

extern "C" {

int gk_abi_version(void) { return GK_ABI_VERSION; }

int gk_set_stage_timing(int on) {
    g_stage_timing = on != 0;
    return 0;
}

int gk_get_stage_ms(float *out3) {
    if (!g_ev[3]) {
        gk_set_error("no timed sweep recorded");
        return -1;
    }
    if (cudaEventSynchronize(g_ev[3]) != cudaSuccess) return -2;
    for (int i = 0; i < 3; i++) cudaEventElapsedTime(&out3[i], g_ev[i], g_ev[i + 1]);
    return 0;
}

const char *gk_last_error(void) { return g_err; }

int gk_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

int gk_static_features(const gk_corpus *corpus, const gk_grid *grid, gk_kstat *out_kstat,
                       double *out_latsum, void *stream) {
    if (int rc = check_grid(corpus, grid)) return rc;
    return gk_launch_static(corpus, grid, out_kstat, out_latsum, (cudaStream_t)stream);
}

int gk_schedule_features(const gk_corpus *corpus, const gk_grid *grid, const gk_kstat *kstat,
                         const double *latsum, uint8_t *out_status, int64_t *out_si,
                         double *out_sf, double *out_feat, const int32_t *sel_idx, uint32_t n_sel,
                         double *out_sel, const gk_trace *trace, void *stream) {
    if (int rc = check_grid(corpus, grid)) return rc;
    if (trace && trace->start && grid->n_k != 1) {
        gk_set_error("per-instruction trace needs a single-kernel grid");
        return -1;
    }
    if (out_sel && (!sel_idx || n_sel == 0)) {
        gk_set_error("out_sel given without sel_idx");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    const uint32_t max_n = corpus->max_n ? corpus->max_n : 1;
    const uint32_t max_blk = corpus->max_blk ? corpus->max_blk : 1;
    // stream-ordered scratch from the device's default pool: reentrant per
    // stream; the pool keeps freed memory (release threshold raised once per
    // device) so repeated calls do not map / unmap ~1 GB each time
    {
        static std::once_flag once[64];
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 0 && dev < 64)
            std::call_once(once[dev], [dev] {
                cudaMemPool_t pool;
                if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                    uint64_t keep = UINT64_MAX;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
                }
            });
    }
    void *ws = nullptr;
    const size_t bytes = gk_sched_scratch_bytes(grid, max_n, max_blk);
    cudaError_t e = cudaMallocAsync(&ws, bytes, st);
    if (e != cudaSuccess) {
        gk_set_error("scratch allocation of %zu B: %s", bytes, cudaGetErrorString(e));
        return -2;
    }
    const int rc = gk_launch_sched(corpus, grid, kstat, latsum, out_status, out_si, out_sf,
                                   out_feat, sel_idx, n_sel, out_sel, nullptr, trace, max_n,
                                   max_blk, (double *)ws, st);
    cudaFreeAsync(ws, st);
    return rc;
}

int gk_rf_predict(const gk_ensemble *ens, const double *X, int64_t ld, int64_t n_rows,
                  const uint8_t *status, const double *time_us, double *out_power,
                  double *out_energy, void *stream) {
    if (n_rows < 0) {
        gk_set_error("gk_rf_predict: n_rows=%lld", (long long)n_rows);
        return -1;
    }
    if (!ens || ((!X || !out_power) && n_rows > 0)) {  // an empty batch may carry null buffers
        gk_set_error("gk_rf_predict: null argument");
        return -1;
    }
    if (out_energy && !time_us) {
        gk_set_error("gk_rf_predict: energy requested without time_us");
        return -1;
    }
    return gk_launch_rf(ens, 1, X, ld, n_rows, status, time_us, out_power, out_energy, 0, 1,
                        (cudaStream_t)stream);
}

size_t gk_sweep_workspace_bytes(const gk_corpus *corpus, const gk_grid *grid, uint32_t n_sel) {
    const size_t n_points = (size_t)grid->n_k * grid->n_arch * grid->n_cfg;
    size_t b = 0;
    b += ((sizeof(gk_kstat) * grid->n_k + 255) / 256) * 256;
    b += ((sizeof(double) * 3 * grid->n_k * grid->n_arch + 255) / 256) * 256;
    // the two-kernel form stages the manifest features of every point; the
    // fused sweep keeps them on chip (config #5 full: 92 GB not allocated)
    if (!sweep_fused()) b += ((sizeof(double) * n_points * n_sel + 255) / 256) * 256;
    // the per-warp reservation-table slabs + work-queue counter: owned by the
    // caller's workspace, so concurrent sweeps on different streams never share
    const uint32_t max_n = corpus && corpus->max_n ? corpus->max_n : 1;
    const uint32_t max_blk = corpus && corpus->max_blk ? corpus->max_blk : 1;
    b += ((gk_sched_scratch_bytes(grid, max_n, max_blk) + 255) / 256) * 256;
    return b;
}

int gk_predict_energy_sweep(const gk_corpus *corpus, const gk_grid *grid,
                            const gk_ensemble *ens_host, const int32_t *sel_idx, uint32_t n_sel,
                            void *work, uint8_t *out_status, double *out_time_us,
                            double *out_power, double *out_energy, void *stream) {
    if (int rc = check_grid(corpus, grid)) return rc;
    if (!ens_host || !sel_idx || !n_sel || !work || !out_status || !out_time_us || !out_power ||
        !out_energy) {
        gk_set_error("gk_predict_energy_sweep: null argument");
        return -1;
    }
    if (grid->n_arch > 4) {
        gk_set_error("gk_predict_energy_sweep: at most 4 archs per sweep");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    char *w = (char *)work;
    gk_kstat *ks = (gk_kstat *)w;
    w += ((sizeof(gk_kstat) * grid->n_k + 255) / 256) * 256;
    double *latsum = (double *)w;
    w += ((sizeof(double) * 3 * grid->n_k * grid->n_arch + 255) / 256) * 256;
    double *sel = (double *)w;
    const size_t n_points = (size_t)grid->n_k * grid->n_arch * grid->n_cfg;
    stage_mark(0, st);
    if (int rc = gk_launch_static(corpus, grid, ks, latsum, st)) return rc;
    stage_mark(1, st);
    const uint32_t max_n = corpus->max_n ? corpus->max_n : 1;
    const uint32_t max_blk = corpus->max_blk ? corpus->max_blk : 1;
    if (!sweep_fused()) w += ((sizeof(double) * n_points * n_sel + 255) / 256) * 256;
    void *ws = w;  // scratch slabs inside the caller's workspace (gk_sweep_workspace_bytes)
    if (sweep_fused()) {
        // one kernel: schedule + features + ensemble walk + energy per warp of points
        if (int rc = gk_launch_sweep_fused(corpus, grid, ks, latsum, ens_host, grid->n_arch,
                                           sel_idx, n_sel, out_status, out_time_us, out_power,
                                           out_energy, max_n, max_blk, (double *)ws, st))
            return rc;
        stage_mark(2, st);
        stage_mark(3, st);
        return 0;
    }
    if (int rc = gk_launch_sched(corpus, grid, ks, latsum, out_status, nullptr, nullptr, nullptr,
                                 sel_idx, n_sel, sel, out_time_us, nullptr, max_n, max_blk,
                                 (double *)ws, st))
        return rc;
    stage_mark(2, st);
    const int rc = gk_launch_rf(ens_host, grid->n_arch, sel, n_sel, (int64_t)n_points, out_status,
                                out_time_us, out_power, out_energy, grid->n_cfg, grid->n_arch, st);
    stage_mark(3, st);
    return rc;
}

}  // extern "C"
