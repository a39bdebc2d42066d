// gk_corr.cu -- correlation pruning statistics on the GPU.
//
// Reference: gpukalc_trainer/dataset.py:138-193 (prune_correlated,
// prune_two_stage) computes DataFrame.corr("pearson") and
// DataFrame.corr("kendall"); pandas' Kendall is scipy.stats.kendalltau per
// column pair (tau-b): with x = the lower-index column, y = the other,
//   dis  = pairs ordered one way by x and the other by y (strictly),
//   xtie, ytie = sum over tie groups of t (t - 1) / 2, ntie = joint ties,
//   tau = (tot - xtie - ytie + ntie - 2 dis) / sqrt(tot - xtie) / sqrt(tot - ytie).
// Every count is an exact integer here, so tau is bit-identical to scipy's.
//
// Kernels:
//   * dense ranks per column: radix sort of (order-preserving key, row), tie
//     groups by value equality (-0.0 == 0.0), xtie by run lengths;
//   * per batch of pairs: one radix sort of (pair | rank_x | rank_y) keys, joint
//     ties from equal-key runs, then discordant pairs = strict inversions of
//     rank_y in that order, counted by an MSD bit split: at bit b, inside each
//     group of equal higher bits, every 0 inherits the count of 1s before it
//     (a segmented scan), then the group is stably split 0s-then-1s;
//   * Pearson: deterministic two-pass co-moments (fixed-order reductions).
#include <cub/cub.cuh>

#include "gk_internal.cuh"

namespace gk {

struct SegScan {  // segmented inclusive scan element: segment start + running count
    uint32_t flag, start, count;
};
struct SegOp {
    __device__ __forceinline__ SegScan operator()(const SegScan &a, const SegScan &b) const {
        return b.flag ? b : SegScan{a.flag, a.start, a.count + b.count};
    }
};

__device__ __forceinline__ uint64_t order_key(double v) {
    uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_col_keys(const double *__restrict__ X, int64_t n, int64_t ld, int col,
                           uint64_t *__restrict__ key, uint32_t *__restrict__ row) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = order_key(X[i * ld + col]);
    row[i] = (uint32_t)i;
}

// run heads by VALUE equality (the sort key distinguishes -0.0 from 0.0)
__global__ void k_col_heads(const double *__restrict__ X, int64_t n, int64_t ld, int col,
                            const uint32_t *__restrict__ row, SegScan *__restrict__ s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool head = i == 0 || X[(int64_t)row[i] * ld + col] != X[(int64_t)row[i - 1] * ld + col];
    s[i] = SegScan{head ? 1u : 0u, (uint32_t)i, head ? 1u : 0u};
}

// rank = number of heads so far - 1; ties: sum over runs of (i - run start)
__global__ void k_col_ranks(const SegScan *__restrict__ inc, const uint32_t *__restrict__ heads,
                            int64_t n, const uint32_t *__restrict__ row, uint32_t *__restrict__ rank,
                            unsigned long long *__restrict__ tie) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long t = 0;
    if (i < n) {
        rank[row[i]] = heads[i] - 1;
        t = (unsigned long long)(i - inc[i].start);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(GK_FULL, t, o);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(tie, t);
}

__global__ void k_pair_keys(const uint32_t *__restrict__ rank, int64_t n,
                            const int32_t *__restrict__ pa, const int32_t *__restrict__ pb, int P,
                            int bb, int bab, uint64_t *__restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)P * n) return;
    const int p = (int)(i / n);
    const int64_t r = i - (int64_t)p * n;
    key[i] = ((uint64_t)p << bab) | ((uint64_t)rank[(int64_t)pa[p] * n + r] << bb) |
             (uint64_t)rank[(int64_t)pb[p] * n + r];
}

// joint ties (equal full keys) + the rank_y sequence for the inversion levels
__global__ void k_pair_heads(const uint64_t *__restrict__ key, int64_t n, int64_t N, int bb,
                             SegScan *__restrict__ s, uint32_t *__restrict__ y) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const bool head = (i % n) == 0 || key[i] != key[i - 1];
    s[i] = SegScan{head ? 1u : 0u, (uint32_t)i, 0u};
    y[i] = (uint32_t)(key[i] & ((1ull << bb) - 1));
}

__device__ __forceinline__ void add_per_pair(unsigned long long v, int p,
                                             unsigned long long *__restrict__ out) {
    // warp-aggregated when the warp's lanes belong to one pair (the common case)
    const int p0 = __shfl_sync(GK_FULL, p, 0);
    if (__all_sync(GK_FULL, p == p0)) {
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(GK_FULL, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + p0, v);
    } else if (v) {
        atomicAdd(out + p, v);
    }
}

__global__ void k_pair_ntie(const SegScan *__restrict__ inc, int64_t n, int64_t N,
                            unsigned long long *__restrict__ ntie) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < N;
    const unsigned long long v = live ? (unsigned long long)(i - inc[i].start) : 0ull;
    add_per_pair(v, live ? (int)(i / n) : -1, ntie);
}

__global__ void k_lvl_in(const uint32_t *__restrict__ y, int64_t n, int64_t N, int b,
                         SegScan *__restrict__ s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t v = y[i];
    const bool head = (i % n) == 0 || (v >> (b + 1)) != (y[i - 1] >> (b + 1));
    s[i] = SegScan{head ? 1u : 0u, (uint32_t)i, (v >> b) & 1u};
}

__global__ void k_lvl_tot(const uint32_t *__restrict__ y, const SegScan *__restrict__ inc, int64_t n,
                          int64_t N, int b, uint32_t *__restrict__ ones_tot,
                          uint32_t *__restrict__ seg_len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const bool last = i + 1 == N || ((i + 1) % n) == 0 || (y[i + 1] >> (b + 1)) != (y[i] >> (b + 1));
    if (last) {
        const uint32_t st = inc[i].start;
        ones_tot[st] = inc[i].count;
        seg_len[st] = (uint32_t)(i - st + 1);
    }
}

__global__ void k_lvl_split(const uint32_t *__restrict__ y, const SegScan *__restrict__ inc,
                            int64_t n, int64_t N, int b, const uint32_t *__restrict__ ones_tot,
                            const uint32_t *__restrict__ seg_len, uint32_t *__restrict__ y_out,
                            unsigned long long *__restrict__ dis) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < N;
    unsigned long long v = 0;
    if (live) {
        const uint32_t yi = y[i], bit = (yi >> b) & 1u;
        const SegScan s = inc[i];
        const uint32_t before = s.count - bit;  // 1s earlier in the group
        const uint32_t st = s.start;
        const uint32_t zeros = seg_len[st] - ones_tot[st];
        const uint32_t pos = bit ? st + zeros + before : st + ((uint32_t)i - st - before);
        y_out[pos] = yi;
        if (!bit) v = before;  // each earlier 1 with the same higher bits is an inversion
    }
    add_per_pair(v, live ? (int)(i / n) : -1, dis);
}

// ----------------------------------------------------------------- Pearson

constexpr int kPR = 256;  // rows per block slice

// column sums over row slices (fixed order inside a slice)
__global__ void k_col_partial(const double *__restrict__ X, int64_t n, int64_t ld, int K,
                              const double *__restrict__ mean, double *__restrict__ part) {
    // grid.x = slices; threads = columns pairs handled below: here one thread per column
    const int64_t r0 = (int64_t)blockIdx.x * kPR;
    const int64_t r1 = min(n, r0 + kPR);
    for (int c = threadIdx.x; c < K; c += blockDim.x) {
        double s = 0.0;
        const double m = mean ? mean[c] : 0.0;
        for (int64_t r = r0; r < r1; r++) s = __dadd_rn(s, __dsub_rn(X[r * ld + c], m));
        part[(int64_t)blockIdx.x * K + c] = s;
    }
}

// co-moment partials: thread t of the block owns pairs (a, b) with a <= b, t + k * blockDim
__global__ void k_comoment_partial(const double *__restrict__ X, int64_t n, int64_t ld, int K,
                                   const double *__restrict__ mean, double *__restrict__ part) {
    extern __shared__ double tile[];  // [kPR][K] centred values
    const int64_t r0 = (int64_t)blockIdx.x * kPR;
    const int rows = (int)min((int64_t)kPR, n - r0);
    for (int q = threadIdx.x; q < rows * K; q += blockDim.x) {
        const int r = q / K, c = q - r * K;
        tile[q] = __dsub_rn(X[(r0 + r) * ld + c], mean[c]);
    }
    __syncthreads();
    const int npairs = K * (K + 1) / 2;
    for (int pi = threadIdx.x; pi < npairs; pi += blockDim.x) {
        // pair index -> (a, b), a <= b, row-major over the upper triangle
        int a = 0, rem = pi;
        while (rem >= K - a) {
            rem -= K - a;
            a++;
        }
        const int b = a + rem;
        double s = 0.0;
        for (int r = 0; r < rows; r++) s = __dadd_rn(s, __dmul_rn(tile[r * K + a], tile[r * K + b]));
        part[(int64_t)blockIdx.x * npairs + pi] = s;
    }
}

// sum the slice partials in slice order (deterministic)
__global__ void k_reduce_slices(const double *__restrict__ part, int64_t slices, int width,
                                double *__restrict__ out, double scale) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= width) return;
    double s = 0.0;
    for (int64_t k = 0; k < slices; k++) s = __dadd_rn(s, part[k * width + j]);
    out[j] = scale != 0.0 ? __ddiv_rn(s, scale) : s;
}

}  // namespace gk

// ------------------------------------------------------------------ C-ABI

namespace gk {
__global__ void k_flags(const SegScan *__restrict__ s, int64_t n, uint32_t *__restrict__ f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = s[i].flag;
}
}  // namespace gk

namespace {
inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }
int bits_for(uint32_t u) {  // bits to hold 0 .. u - 1 (>= 1)
    int b = 1;
    while (b < 32 && (1ull << b) < (uint64_t)u) b++;
    return b;
}
struct Carve {
    char *w;
    void *take(size_t b) {
        void *p = w;
        w += (b + 255) / 256 * 256;
        return p;
    }
};
size_t cub_tmp(int64_t N) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)N);
    cub::DeviceRadixSort::SortKeys(nullptr, c, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)N);
    a = std::max(a, c);
    cub::DeviceScan::InclusiveScan(nullptr, b, (gk::SegScan *)nullptr, (gk::SegScan *)nullptr,
                                   gk::SegOp{}, (int)N);
    a = std::max(a, b);
    cub::DeviceScan::InclusiveSum(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr, (int)N);
    return std::max(a, b) + 256;
}
}  // namespace

extern "C" {

size_t gk_corr_ranks_workspace(int64_t n) {
    if (n < 1) return 1024;
    return (size_t)n * (8 + 8 + 4 + 4 + 12 + 12 + 4 + 4) + 8 * 256 + cub_tmp(n) + 1024;
}

// Dense ranks of every column (ranks[c * n + row], device), unique counts and
// sum over tie groups of t (t - 1) / 2 per column (device arrays).  X is
// [n][ld] row-major on the device, finite values.
int gk_corr_ranks(const double *X, int64_t n, int32_t K, int64_t ld, uint32_t *ranks,
                  uint32_t *n_unique, int64_t *ties, void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || n >= (1ll << 31) || K < 1) {
        gk_set_error("gk_corr_ranks: bad shape");
        return -1;
    }
    if (ws_bytes < gk_corr_ranks_workspace(n)) {
        gk_set_error("gk_corr_ranks: workspace too small");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    Carve cv{(char *)ws};
    uint64_t *k0 = (uint64_t *)cv.take(8 * n), *k1 = (uint64_t *)cv.take(8 * n);
    uint32_t *r0 = (uint32_t *)cv.take(4 * n), *r1 = (uint32_t *)cv.take(4 * n);
    gk::SegScan *s_in = (gk::SegScan *)cv.take(12 * n), *s_out = (gk::SegScan *)cv.take(12 * n);
    uint32_t *fl = (uint32_t *)cv.take(4 * n), *hs = (uint32_t *)cv.take(4 * n);
    void *tmp = cv.w;
    const size_t tmp_b = ws_bytes - (size_t)(cv.w - (char *)ws);
    cudaMemsetAsync(ties, 0, sizeof(int64_t) * K, st);
    for (int c = 0; c < K; c++) {
        gk::k_col_keys<<<nblk(n), 256, 0, st>>>(X, n, ld, c, k0, r0);
        size_t tb = tmp_b;
        cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, r0, r1, (int)n, 0, 64, st);
        gk::k_col_heads<<<nblk(n), 256, 0, st>>>(X, n, ld, c, r1, s_in);
        tb = tmp_b;
        cub::DeviceScan::InclusiveScan(tmp, tb, s_in, s_out, gk::SegOp{}, (int)n, st);
        gk::k_flags<<<nblk(n), 256, 0, st>>>(s_in, n, fl);
        tb = tmp_b;
        cub::DeviceScan::InclusiveSum(tmp, tb, fl, hs, (int)n, st);
        gk::k_col_ranks<<<nblk(n), 256, 0, st>>>(s_out, hs, n, r1, ranks + (int64_t)c * n,
                                                 (unsigned long long *)(ties + c));
        cudaMemcpyAsync(n_unique + c, hs + n - 1, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    }
    return gk_check_launch("gk_corr_ranks");
}

size_t gk_corr_kendall_workspace(int64_t n, int32_t max_pairs) {
    const int64_t N = n * (int64_t)max_pairs;
    if (N < 1) return 1024;
    return (size_t)N * (8 + 8 + 12 + 12 + 4 + 4 + 4 + 4) + 8 * 256 + cub_tmp(N) + 1024;
}

// Kendall counts for P column pairs (pa[p] < pb[p] by convention: x = pa, y =
// pb): dis[p] = strictly discordant pairs, ntie[p] = joint ties (device int64
// arrays, overwritten).  ranks / n_unique from gk_corr_ranks; pa / pb host
// arrays (to size the keys) and their device copies pa_d / pb_d.
int gk_corr_kendall(const uint32_t *ranks, int64_t n, int32_t K, const uint32_t *n_unique_host,
                    const int32_t *pa, const int32_t *pb, const int32_t *pa_d, const int32_t *pb_d,
                    int32_t P, int64_t *dis, int64_t *ntie, void *ws, size_t ws_bytes,
                    void *stream) {
    const int64_t N = n * (int64_t)P;
    if (P < 1 || n < 2) return 0;
    if (N >= (1ll << 31)) {
        gk_set_error("gk_corr_kendall: %d pairs x %lld rows exceed one batch", P, (long long)n);
        return -1;
    }
    if (ws_bytes < gk_corr_kendall_workspace(n, P)) {
        gk_set_error("gk_corr_kendall: workspace too small");
        return -1;
    }
    int ba = 1, bb = 1;
    for (int p = 0; p < P; p++) {
        if (pa[p] < 0 || pa[p] >= K || pb[p] < 0 || pb[p] >= K) {
            gk_set_error("gk_corr_kendall: column index out of range");
            return -1;
        }
        ba = std::max(ba, bits_for(n_unique_host[pa[p]]));
        bb = std::max(bb, bits_for(n_unique_host[pb[p]]));
    }
    const int bp = bits_for((uint32_t)P);
    if (ba + bb + bp > 64) {
        gk_set_error("gk_corr_kendall: keys need %d bits", ba + bb + bp);
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    Carve cv{(char *)ws};
    uint64_t *k0 = (uint64_t *)cv.take(8 * N), *k1 = (uint64_t *)cv.take(8 * N);
    gk::SegScan *s_in = (gk::SegScan *)cv.take(12 * N), *s_out = (gk::SegScan *)cv.take(12 * N);
    uint32_t *y0 = (uint32_t *)cv.take(4 * N), *y1 = (uint32_t *)cv.take(4 * N);
    uint32_t *ones = (uint32_t *)cv.take(4 * N), *len = (uint32_t *)cv.take(4 * N);
    void *tmp = cv.w;
    const size_t tmp_b = ws_bytes - (size_t)(cv.w - (char *)ws);
    cudaMemsetAsync(dis, 0, sizeof(int64_t) * P, st);
    cudaMemsetAsync(ntie, 0, sizeof(int64_t) * P, st);
    gk::k_pair_keys<<<nblk(N), 256, 0, st>>>(ranks, n, pa_d, pb_d, P, bb, ba + bb, k0);
    size_t tb = tmp_b;
    cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, (int)N, 0, ba + bb + bp, st);
    gk::k_pair_heads<<<nblk(N), 256, 0, st>>>(k1, n, N, bb, s_in, y0);
    tb = tmp_b;
    cub::DeviceScan::InclusiveScan(tmp, tb, s_in, s_out, gk::SegOp{}, (int)N, st);
    gk::k_pair_ntie<<<nblk(N), 256, 0, st>>>(s_out, n, N, (unsigned long long *)ntie);
    for (int b = bb - 1; b >= 0; b--) {
        gk::k_lvl_in<<<nblk(N), 256, 0, st>>>(y0, n, N, b, s_in);
        tb = tmp_b;
        cub::DeviceScan::InclusiveScan(tmp, tb, s_in, s_out, gk::SegOp{}, (int)N, st);
        gk::k_lvl_tot<<<nblk(N), 256, 0, st>>>(y0, s_out, n, N, b, ones, len);
        gk::k_lvl_split<<<nblk(N), 256, 0, st>>>(y0, s_out, n, N, b, ones, len, y1,
                                                  (unsigned long long *)dis);
        std::swap(y0, y1);
    }
    return gk_check_launch("gk_corr_kendall");
}

size_t gk_corr_pearson_workspace(int64_t n, int32_t K) {
    const int64_t slices = (n + gk::kPR - 1) / gk::kPR;
    const int64_t np = (int64_t)K * (K + 1) / 2;
    return (size_t)(slices * std::max<int64_t>(np, K) + np + 2 * K) * 8 + 4096;
}

// Centred co-moments C[a][b] (a <= b, upper triangle, row-major) and the column
// means, by deterministic two-pass fixed-order reductions (device arrays).
int gk_corr_pearson(const double *X, int64_t n, int32_t K, int64_t ld, double *mean,
                    double *comoment, void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || K < 1 || K > 256) {
        gk_set_error("gk_corr_pearson: bad shape");
        return -1;
    }
    if (ws_bytes < gk_corr_pearson_workspace(n, K)) {
        gk_set_error("gk_corr_pearson: workspace too small");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    const int64_t slices = (n + gk::kPR - 1) / gk::kPR;
    const int np = K * (K + 1) / 2;
    double *part = (double *)ws;
    gk::k_col_partial<<<(unsigned)slices, 64, 0, st>>>(X, n, ld, K, nullptr, part);
    gk::k_reduce_slices<<<(K + 127) / 128, 128, 0, st>>>(part, slices, K, mean, (double)n);
    const size_t smem = (size_t)gk::kPR * K * sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(gk::k_comoment_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    gk::k_comoment_partial<<<(unsigned)slices, 256, smem, st>>>(X, n, ld, K, mean, part);
    gk::k_reduce_slices<<<(np + 127) / 128, 128, 0, st>>>(part, slices, np, comoment, 0.0);
    return gk_check_launch("gk_corr_pearson");
}

}  // extern "C"
