/*
 * gk.h -- C-ABI of libgk (sm_100a) for the batched energy-prediction hot path of
 * arXiv 2305.01886 (reference package `gpukalc` / `gpukalc-trainer`).
 *
 * The reference has no FFI: its boundary is the Python API.  Each entry point
 * below replaces the per-point Python call named in its comment; the Python
 * host package (paper_2305_01886_b200) binds these through ctypes and keeps the
 * reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - all pointers are DEVICE pointers unless the name ends in `_host`; the
 *     caller owns every buffer, the library only borrows them;
 *   - `stream` is a cudaStream_t passed as void*; calls are asynchronous and
 *     never synchronise unless documented;
 *   - return 0 on success, <0 on argument / CUDA error; gk_last_error() gives
 *     the message (thread-local);
 *   - per-point failures do not abort a batch: they are written to a status
 *     byte (GK_OK, GK_INFEASIBLE_LAUNCH, GK_INFEASIBLE_OCCUPANCY).
 */
#ifndef GK_H
#define GK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_ABI_VERSION 5

/* resource / class codes (reference ptx/types.py:12-24) */
enum { GK_SP = 0, GK_SFU = 1, GK_DPU = 2, GK_LSU = 3, GK_WS = 4, GK_NRES = 5 };
enum { GK_COMPUTE = 0, GK_GLOBAL = 1, GK_SHARED = 2, GK_MISC = 3, GK_NCLASS = 4 };
/* token flag bits (in gk_token.cls above the 2 class bits) */
#define GK_F_BRANCH 0x04u /* is_branch (classify.py:102-104)            */
#define GK_F_GLOAD  0x08u /* GLOBAL and root in {ld, ldu} (features.py:168-170) */
#define GK_F_GSTORE 0x10u /* GLOBAL and root == st       (features.py:171-172) */

/* per-point status */
enum { GK_OK = 0, GK_INFEASIBLE_LAUNCH = 1, GK_INFEASIBLE_OCCUPANCY = 2 };

#define GK_MAX_BP 8   /* piecewise global-latency breakpoints per arch */
#define GK_NFEAT 32   /* FEATURE_ORDER length (features.py:21-54)      */

/* One PTX instruction, program order (16 B).  The DFG predecessors of token i
 * are preds[tok[i].pred0 .. tok[i+1].pred0) (block-local producer indices);
 * the token array carries one sentinel entry at the end.  lst_row / lst_len
 * place the instruction's reservation span: its resource's span list occupies
 * rows [lst_row, lst_row + res_cnt[res]) of the block's span table and
 * lst_len same-resource instructions precede it in the block. */
typedef struct {
    uint8_t  res;     /* GK_SP..GK_WS                                  */
    uint8_t  cls;     /* class code (bits 0-1) | GK_F_* flags           */
    uint16_t sig;     /* latency signature id -> gk_arch-major lat table */
    uint32_t pred0;   /* offset into preds[]                            */
    uint16_t lst_row; /* first row of this resource's list in the block */
    uint16_t lst_len; /* earlier same-resource instructions in the block */
    uint32_t pad_;
} gk_token;

/* One basic block (40 B). */
typedef struct {
    int64_t  mult;          /* loop multiplier (types.py:109-124)                */
    uint32_t tok0;          /* first token (global index)                        */
    uint32_t n;             /* instructions                                      */
    uint32_t fpred0;        /* forward CFG predecessors: fpreds[fpred0 .. +n_fpred] */
    uint16_t n_fpred;
    uint16_t n_glob;        /* GLOBAL-class instructions in the block            */
    uint16_t res_cnt[GK_NRES]; /* instructions per resource                      */
    uint8_t  is_exit;       /* no forward out-edge (types.py:79-82)              */
    uint8_t  pad_;
} gk_block;

/* One kernel (32 B).  Blocks are contiguous in the block table and their tokens
 * contiguous in the token table. */
typedef struct {
    uint32_t blk0, n_blk;   /* block range                                        */
    uint32_t topo0;         /* topo[topo0 .. +n_blk]: Kahn order (types.py:87-107) */
    uint32_t max_n;         /* largest block (instructions)                       */
    uint32_t tok0, n_tok;   /* token range                                        */
    uint32_t pad_[2];
} gk_kernel;

/* A packed corpus: every array lives on the device (or host for the oracle). */
typedef struct {
    const gk_token  *tok;    /* n_tok + 1 (sentinel)     */
    const uint16_t  *preds;  /* DFG producer lists       */
    const gk_block  *blk;    /* n_blk                    */
    const uint32_t  *fpreds; /* forward CFG preds (kernel-local block ids) */
    const uint32_t  *topo;   /* kernel-local block ids   */
    const gk_kernel *ker;    /* n_ker                    */
    uint32_t n_tok, n_blk, n_ker, n_sig;
    uint32_t max_n;          /* largest block over all kernels (instructions) */
    uint32_t max_blk;        /* most blocks in one kernel                     */
} gk_corpus;

/* Launch configuration (scheduler.py:31-50). */
typedef struct { int32_t n_blocks, tpb, regs, shmem; } gk_config;

/* Architecture record (profiles.py:104-135), one per arch. */
typedef struct {
    int64_t units[GK_NRES];
    double  gap[GK_NRES];
    double  pipeline;
    int64_t nSM, L2_sz, nTh_sm_max, reg_b_max, shm_b_max, nB_max, wSM_max, Sz_w;
    int64_t access_sz, access_gm_sz, access_shm_sz, nWS, nDU;
    double  nu_gpu;
    double  tpg_a, tpg_b, tpg_c, tps_a, tps_b, tps_c, tp_floor;
    double  ov_slope, ov_icpt;
    int32_t n_bp, pad_;
    double  bp[GK_MAX_BP];
    double  seg_slope[GK_MAX_BP + 1], seg_icpt[GK_MAX_BP + 1];
} gk_arch;

/* Static per-kernel tallies (K1; features.py:157-172, scheduler.py:255-266). */
typedef struct {
    int64_t cnt[GK_NCLASS];   /* sum of multipliers per class       */
    int64_t branches, loads, stores, pad_;
} gk_kstat;

/* Indices into the int64 / f64 per-point schedule outputs (KernelSchedule,
 * scheduler.py:105-134). */
enum { GK_SI_THREADS_SCHED = 0, GK_SI_THREADS_PER_SM, GK_SI_BLOCKS_PER_SM, GK_SI_WAVES,
       GK_SI_N_GLOBAL, GK_SI_N_SHARED, GK_NSI };
enum { GK_SF_GM_LATENCY = 0, GK_SF_D_KERNEL, GK_SF_OVERHEAD, GK_SF_GM_PENALTY,
       GK_SF_SM_PENALTY, GK_SF_CM_PENALTY, GK_SF_D_TOTAL, GK_SF_TIME_US, GK_SF_CFG_DELAY,
       GK_NSF };

/* Optional per-instruction schedule (the --trace rows, scheduler.py:74-102).
 * Only valid for grids over ONE kernel; arrays are [n_points][n_tok_kernel]
 * and [n_points][n_blk_kernel]. */
typedef struct {
    double  *start, *duration, *latency;
    int64_t *n_batches;
    double  *blk_delay, *blk_finish;
} gk_trace;

/* Point grid: kernels x archs x configs, point p = (ki*n_arch + ai)*n_cfg + ci. */
typedef struct {
    const uint32_t  *kernel_ids;  /* n_k indices into the corpus            */
    const gk_config *cfg;         /* n_cfg                                  */
    const gk_arch   *arch;        /* n_arch records                         */
    const double    *lat;         /* [n_arch][n_sig] signature latencies     */
    /* optional per-config overrides (NULL = none) for the block/CFG-level faces
     * schedule_block / schedule_cfg (scheduler.py:137, 188), which take n_tw
     * and gm_latency directly: n_tw_override[c] > 0 replaces cap*tpb,
     * a non-NaN gm_override[c] replaces the piecewise global latency. */
    const int64_t   *n_tw_override;
    const double    *gm_override;
    /* optional processing order of the grid's kernels (n_k entries, a
     * permutation of 0..n_k-1; NULL = 0..n_k-1).  Outputs stay indexed by
     * point; the order only balances the device's dynamic work queue
     * (largest kernels first). */
    const uint32_t  *order;
    /* optional device counter (NULL = none): mem_throughput clamps to tp_floor
     * (profiles.py:173-181, where the reference logs a warning per clamped
     * call) are atomically added here.  Per grid, so concurrent sweeps on
     * different streams keep separate counts (no library-global state). */
    unsigned long long *tp_clamps;
    uint32_t n_k, n_cfg, n_arch, pad_;
} gk_grid;

/* Flattened tree ensemble (power.py:22-33).  Node = 16 B: for a split,
 * {threshold, feature, left} with right = left + 1; for a leaf,
 * {value, -1, self - 1} -- the walk reads feature -1 as +inf, +inf <= value is
 * false, so the step goes "right" to the leaf itself: a fixed number of descent
 * steps absorbs at the leaf without a leaf test.  Child indices are tree-local;
 * trees are contiguous from tree_off[t]; tree_depth[t] is the depth of tree t. */
typedef struct { double v; int32_t feature; int32_t left; } gk_node;

/* Compact 8-byte walk node (optional), same index space as gk_node:
 *   t    = f32 bits of round-toward-(-inf)(threshold); 0 for a leaf
 *   meta = feature << 24 | right  (feature 0..126; 0xFF = leaf, right = self)
 * Decision: a = round-down-f32(x) vs t as for gk_block2 below; the exact tie
 * test reads nodes[i].v; a leaf's feature byte selects the +inf slot in front
 * of the feature tile, so the walk absorbs at leaves (value in nodes[i].v). */
typedef struct { uint32_t t; uint32_t meta; } gk_node8;

/* Two-level walk block (32 B, optional; one 256-bit load per lane per step).
 * A block is a depth-2 subtree: slot 0 (its root, an internal node at even
 * depth), slots 1 / 2 (the root's left / right child) and the four exits
 * below them (exit 2k + c = child c of slot 1 + k).
 *   t[s]  f32 bits of round-toward-(-inf)(threshold of slot s)
 *   f     feature of slot s in byte s
 *   e[j]  next block id, or GK_LEAF | leaf id (leaf_val index)
 * A slot that is a leaf has both of its exits = that leaf (its t / f are 0).
 * Decision at a slot: a = round-down-f32(x[f]); a < t -> left, a > t -> right,
 * a == t (x and the threshold share one f32 bucket) -> the exact fp64 test
 * x <= thr64[3 * block + slot].  This equals `x <= threshold` for every x
 * (NaN and +-inf included), so power stays bit-identical (power.py:156-168). */
#define GK_LEAF 0x80000000u
typedef struct { uint32_t t[3]; uint32_t f; uint32_t e[4]; } gk_block2;

/* Three-level walk block (32 B, optional; one 256-bit load per lane per three
 * levels).  Keys: k(v) = the top 16 bits of the order-preserving bits of
 * round-toward-(-inf)-f32(v), -0.0 taken as +0.0, NaN -> 0xFFFF (a NaN
 * threshold -> 0: x <= NaN is false for every x).  Decision
 * at a node: a = k(x[f]) vs t = k(threshold); a < t -> left, a > t -> right,
 * a == t -> the exact fp64 test x <= thr64[7 * block + node] (equals `x <=
 * threshold` for every x incl. NaN, +-inf, -0.0).  Blocks sit at depths 0, 3,
 * 6, ... of a tree (ids level by level in (parent, slot) order), of two kinds
 * (type = byte 22):
 *   type 0, a 3-level subtree: nodes 0..6 (node k's children 2k+1, 2k+2),
 *     w[0..3] = 16-bit keys t[0..6] (t[k] at halfword k), features f[0..6]
 *     at bytes 14..20, leaf mask at byte 21 (bit s: exit slot s is a leaf),
 *     w[6] = first child block id, w[7] = first leaf id; exit slot s = 4 b0 +
 *     2 b1 + b2 (b = went right) is leaf_base + #leaf slots below s or
 *     block_base + #block slots below s.  A leaf inside the subtree is padded
 *     (its nodes route anywhere, all of its slots name that leaf).
 *   type 1, terminal (a node whose children are both leaves): its key and
 *     feature where type 0 keeps node 0's (halfword 0, byte 14), the left /
 *     right leaf values (f64) in w[1..2] / w[6..7].
 * Leaf ids (leaf_val index) stay below 2^30. */
typedef struct { uint32_t w[8]; } gk_block3;
#define GK_B3_TERMINAL 1u

typedef struct {
    const gk_node *nodes;
    const int64_t *tree_off;    /* n_trees                        */
    const int32_t *tree_depth;  /* n_trees                        */
    const double  *scale_lo;    /* n_feat  (power.py:128-145)     */
    const double  *scale_hi;
    double   base_score;
    uint32_t n_trees, n_feat, max_depth;
    /* optional compact forms of the same trees; the walk uses blocks if set,
     * else nodes8 if set, else the 16-byte nodes */
    const gk_node8  *nodes8;    /* per node                                 */
    const gk_block2 *blocks;    /* n_blocks                                 */
    const double    *thr64;     /* 3 per block: exact thresholds (tie test)  */
    const double    *leaf_val;  /* per leaf id                               */
    const uint32_t  *root;      /* n_trees: root block id or GK_LEAF | leaf  */
    /* gk_block3 form (thr64 then 7 per block, leaf_val / root its own); the
     * walks use it when set */
    const gk_block3 *blocks3;
} gk_ensemble;

/* ------------------------------------------------------------------------ */

int         gk_abi_version(void);
const char *gk_last_error(void);
int         gk_device_sm_count(void);

/* K1 -- static segmented counts per kernel and per (arch, kernel) sequential
 * latency sums of the non-global classes.  Replaces the config-independent
 * half of extract_features (features.py:155-172) and static_mem_counts
 * (scheduler.py:255-266).  out_latsum is [n_arch][n_k][3] (Compute, Shared,
 * Misc), out_kstat is [n_k]. */
int gk_static_features(const gk_corpus *corpus, const gk_grid *grid,
                       gk_kstat *out_kstat, double *out_latsum, void *stream);

/* K2+K3 -- per-point schedule and features.  Replaces schedule_kernel
 * (scheduler.py:325-363) and extract_features (features.py:149-247) per
 * point.  Any output pointer may be NULL.
 *   out_status  [n_points] u8
 *   out_si      [n_points][GK_NSI] int64, out_sf [n_points][GK_NSF] f64
 *   out_feat    [n_points][GK_NFEAT] f64 in FEATURE_ORDER
 *   out_sel     [n_points][n_sel] f64: the features listed in sel_idx (manifest
 *               order for a power model), raw (unscaled)
 *   trace       per-instruction rows (single-kernel grids only), may be NULL
 * kstat/latsum come from gk_static_features on the same grid. */
int gk_schedule_features(const gk_corpus *corpus, const gk_grid *grid,
                         const gk_kstat *kstat, const double *latsum,
                         uint8_t *out_status, int64_t *out_si, double *out_sf,
                         double *out_feat, const int32_t *sel_idx, uint32_t n_sel,
                         double *out_sel, const gk_trace *trace, void *stream);

/* K4 (+K6) -- ensemble inference over raw feature rows X[n_rows][ld] (first
 * n_feat columns, manifest order), scaled per power.py:128-145, trees summed in
 * file order onto base_score (power.py:148-168).  If time_us != NULL also
 * writes energy = power * time_us (power.py:171-181, fp64 product).
 * Rows whose status byte (optional) is nonzero get NaN.  n_rows = 0 is a
 * valid empty batch (buffers may then be NULL).  n_feat <= 255 for the
 * compact layouts (nodes8 / blocks / blocks3), <= 886 for the fp64 nodes
 * (32-row tiles above 220 features). */
int gk_rf_predict(const gk_ensemble *ens, const double *X, int64_t ld, int64_t n_rows,
                  const uint8_t *status, const double *time_us,
                  double *out_power, double *out_energy, void *stream);

/* Fused sweep: K1 -> K2/K3 -> K4 -> K6 for a whole grid with one ensemble per
 * arch (ens_host[n_arch], a HOST array of descriptors whose pointers are device
 * pointers; all ensembles share the manifest sel_idx[n_sel], a device array).
 * Writes status / time_us / power_w / energy_uj per point.  `work` must hold
 * gk_sweep_workspace_bytes() bytes of device memory. */
size_t gk_sweep_workspace_bytes(const gk_corpus *corpus, const gk_grid *grid, uint32_t n_sel);
int gk_predict_energy_sweep(const gk_corpus *corpus, const gk_grid *grid,
                            const gk_ensemble *ens_host, const int32_t *sel_idx,
                            uint32_t n_sel, void *work, uint8_t *out_status,
                            double *out_time_us, double *out_power, double *out_energy,
                            void *stream);

/* Profiling aid: when enabled, gk_predict_energy_sweep records CUDA events
 * between its K1 / K2+K3 / K4 launches; gk_get_stage_ms waits for the last
 * sweep and returns the three stage durations in ms. */
/* ---- K5: random-forest training (replaces RandomForestRegressor.fit as built by
 * gpukalc_trainer.training._make_model, training.py:73-76; sklearn internals
 * SK/ensemble/_forest.py:95-175, SK/tree/_splitter.pyx).  Host driver:
 * paper_2305_01886_b200/forest.py.  Task / split records:
 *   task  = {int32 tree, begin, end, parity}   (row segment in rows0/rows1)
 *   split = {int32 feat (-1: leaf), bin, n_left, pad; double proxy} */

/* counts[t][i] = bincount(RandomState(tree_seeds[t]).randint(0, n, n))[i] */
int gk_rf_bootstrap(const uint32_t *tree_seeds, uint32_t n_trees, int64_t n_rows,
                    uint32_t *counts, void *stream);
/* Row records (gk_rftrain.cu): a node's rows are a contiguous run of
 * gk_rf_record_bytes(n_feat)-byte records {row id i32, bootstrap weight u32,
 * weight * yfp i64, the row's n_feat bins (zero-padded to 16 B)} in one of two
 * ping-pong buffers (recs0 / recs1); the partition moves whole records. */
size_t gk_rf_record_bytes(int32_t n_feat);
/* recs[tree_base[t] ..] = the records of the rows i with counts[t][i] > 0
 * (fill[t] = how many; order within a tree unspecified); Xb [n_rows][n_feat]
 * bins, yfp [n_rows] fixed-point targets */
int gk_rf_compact(const uint32_t *counts, uint32_t n_trees, int64_t n_rows, const uint8_t *Xb,
                  int32_t n_feat, const int64_t *yfp, const int64_t *tree_base, void *recs,
                  int32_t *fill, void *stream);
/* Xb[i][f] = #{edges[f][j] < float32(X[i][f])}; per-bin min/max (order-mapped) */
int gk_rf_bin(const double *X, int64_t n_rows, int32_t n_feat, int64_t ld, const float *edges,
              const int32_t *n_edges, uint8_t *Xb, uint32_t *bin_min, uint32_t *bin_max,
              void *stream);
/* best split of every task (small / medium / big index lists).  Tasks of <= 256
 * rows are partitioned by their split search (records moved to the other
 * buffer): their split record has pad = 1 and n_left = the left row count;
 * for the others (pad = 0) n_left is NOT filled -- gk_rf_partition_lists moves
 * their records and its cursor gives the left row count.  Big tasks keep
 * their histograms in hist_ws (gk_rf_hist_bytes; interleaved {weight, sum}
 * per bin, slot = position in big_ids); slot_cur[n_tasks] receives each
 * task's slot (-1: not big).  Sibling subtraction (optional: prev_hist_ws /
 * par_slot non-null, par_slot from gk_rf_next_level): of two big siblings
 * the smaller is built, the larger = the parent's histogram (prev_hist_ws at
 * par_slot) - the smaller's. */
int gk_rf_split_level(const uint8_t *Xb, const int64_t *yfp, const double *y,
                      const uint32_t *counts, int64_t n_rows, int32_t n_feat,
                      const void *tasks, const int32_t *small_ids, int32_t n_small,
                      const int32_t *med_ids, int32_t n_med, const int32_t *big_ids,
                      int32_t n_big, int32_t big_max_chunks, void *recs0, void *recs1,
                      void *hist_ws, void *split_out, const void *prev_hist_ws,
                      const int32_t *par_slot, int32_t *slot_cur, int32_t n_tasks, void *stream);
size_t gk_rf_hist_bytes(int32_t n_big, int32_t n_feat);
/* move each split task's records to the other buffer: left rows up from begin,
 * right rows down from end; cursor[2*i] ends as task i's left row count (n_left) */
int gk_rf_partition(const uint8_t *Xb, const int64_t *yfp, const double *y,
                    const uint32_t *counts, int64_t n_rows, int32_t n_feat, const void *tasks,
                    int32_t n_tasks, const void *split, const int32_t *ids, int32_t n_ids,
                    int32_t max_rows, void *recs0, void *recs1, int32_t *cursor,
                    void *stream);
/* The level loop's bookkeeping on the device (replaces the per-level host
 * bookkeeping of the tree builder; sklearn's BestFirst/DepthFirst builders,
 * SK/tree/_tree.pyx, grow node by node).  From one level's tasks (sorted by
 * tree), node ids, splits and the partition's cursors (cursor[2*i] = split
 * task i's left row count, after gk_rf_partition_lists): split task i gets
 * children at 2*excl[i] and
 * 2*excl[i]+1 of tasks_next / node_next (excl = split tasks before i) with BFS
 * ids lid = next_id[tree] + 2*(rank among the tree's split tasks), written to
 * lid_out[i] (-1 when task i is a leaf); next_id advances; children with >= 2
 * rows below max_depth are appended to lists[0 / 1 / 2 x list_cap] (small /
 * medium / big search lists, any order).  stats (int32[8], device): next-level
 * task count, the three list lengths, largest medium / big child.  scratch:
 * gk_rf_level_scratch_bytes. */
size_t gk_rf_level_scratch_bytes(int32_t n_tasks, int32_t n_trees);
/* slot_cur (this level's big slots from gk_rf_split_level, or NULL) and
 * par_slot_next (2 * n_tasks, or NULL): each child's parent histogram slot */
int gk_rf_next_level(const void *tasks, const int32_t *node, const void *split,
                     const int32_t *cursor, int32_t n_tasks, int32_t n_trees, int32_t child_depth,
                     int32_t max_depth, int32_t *next_id, int32_t *lid_out, void *tasks_next,
                     int32_t *node_next, int32_t *lists, int32_t list_cap, int32_t *stats,
                     void *scratch, const int32_t *slot_cur, int32_t *par_slot_next,
                     void *stream);
/* gk_rf_partition over a level's three search lists (searched tasks that stayed
 * leaves are skipped); cursor: 2 * n_tasks int32, zeroed here */
int gk_rf_partition_lists(const uint8_t *Xb, const uint32_t *counts, int64_t n_rows,
                          int32_t n_feat, const void *tasks, int32_t n_tasks, const void *split,
                          const int32_t *small_ids, int32_t n_small, const int32_t *med_ids,
                          int32_t n_med, int32_t max_med, const int32_t *big_ids, int32_t n_big,
                          int32_t max_big, void *recs0, void *recs1, int32_t *cursor,
                          void *stream);
/* per leaf segment: int64 {n, sum w, sum w*yfp, sum w*y2fp} (exact fixed-point
 * sums); max_leaf_rows (the largest segment) sizes the row-chunk grid */
int gk_rf_leaf_stats(const uint32_t *counts, int64_t n_rows, int32_t n_feat, const int64_t *yfp,
                     const int64_t *y2fp, const void *leaves, int32_t n_leaves,
                     const void *recs0, const void *recs1, int64_t *out,
                     int32_t max_leaf_rows, void *stream);

/* Tree assembly of a batch from its level records (tasks / splits / BFS ids
 * `node` / child ids `lid` (-1 for leaves) / level of every task, all levels
 * concatenated; node g = node_base[tree] + BFS id):
 *  nodes: split nodes' feat / nbin / left (tree-local left child id) and
 *         depth[tree] = max(level of a split + 1) (int64, zeroed by the caller);
 *  up:    one level, children before parents: ist[g] (int64 {n, w, w*yfp,
 *         w*y2fp}) of every split node = ist[left] + ist[left + 1];
 *  final: fl [4][N] f64 {threshold (-2 leaf), value, impurity, weighted_n}
 *         and it [4][N] i64 {left, right (-1 leaf), feature, n_node_samples}
 *         with thr [F][256] the bins' midpoint thresholds. */
int gk_rf_assemble_nodes(const void *tasks, const void *split, const int32_t *node,
                         const int32_t *lid, const int32_t *level, int32_t n,
                         const int64_t *node_base, int64_t *feat, int64_t *nbin, int64_t *left,
                         int64_t *depth, void *stream);
int gk_rf_assemble_up(const void *tasks, const void *split, const int32_t *node,
                      const int32_t *lid, int32_t n, const int64_t *node_base, int64_t *ist,
                      void *stream);
int gk_rf_assemble_final(int64_t n_nodes, const int64_t *ist, const int64_t *feat,
                         const int64_t *nbin, const int64_t *left, const double *thr,
                         int32_t shift, int32_t shift2, double *fl, int64_t *it, void *stream);

/* One gradient-boosting update (sklearn GradientBoostingRegressor, squared
 * error; reference training.py:67-72 via _make_model("gradient_boosted")):
 * rows of leaf k (tasks as for gk_rf_leaf_stats) get F += leaf_val[k]
 * (learning_rate * leaf mean), then yfp / y2fp = the next stage's residual
 * y - F (and its square) in fixed point 2^shift / 2^shift2, and *absmax =
 * max(*absmax, max |y - F|) as the bit pattern of a non-negative double. */
int gk_gb_step(const void *leaves, int32_t n_leaves, const double *leaf_val,
               const void *recs0, const void *recs1, int32_t n_feat, const double *y, double *F,
               int64_t *yfp, int64_t *y2fp, int32_t shift, int32_t shift2,
               uint64_t *absmax, int32_t max_leaf_rows, void *stream);

/* ---- correlation pruning statistics (gk_corr.cu) -------
 * Reference: gpukalc_trainer/dataset.py:138-193 -> DataFrame.corr("pearson")
 * and DataFrame.corr("kendall") (scipy.stats.kendalltau tau-b per pair).
 * X is [n][ld] row-major fp64 on the device, finite values.  Workspaces are
 * caller-allocated device memory of the *_workspace() size. */
size_t gk_corr_ranks_workspace(int64_t n);
/* dense ranks (ranks[c * n + row]), unique counts and tie sums per column */
int gk_corr_ranks(const double *X, int64_t n, int32_t K, int64_t ld, uint32_t *ranks,
                  uint32_t *n_unique, int64_t *ties, void *ws, size_t ws_bytes, void *stream);
size_t gk_corr_kendall_workspace(int64_t n, int32_t max_pairs);
/* per pair p (x = column pa[p], y = column pb[p]): strictly discordant pairs
 * and joint ties -- the exact integers of scipy's tau-b */
int gk_corr_kendall(const uint32_t *ranks, int64_t n, int32_t K, const uint32_t *n_unique_host,
                    const int32_t *pa, const int32_t *pb, const int32_t *pa_d, const int32_t *pb_d,
                    int32_t P, int64_t *dis, int64_t *ntie, void *ws, size_t ws_bytes,
                    void *stream);
size_t gk_corr_pearson_workspace(int64_t n, int32_t K);
/* column means and centred co-moments (upper triangle, row-major), fixed-order sums */
int gk_corr_pearson(const double *X, int64_t n, int32_t K, int64_t ld, double *mean,
                    double *comoment, void *ws, size_t ws_bytes, void *stream);

int gk_set_stage_timing(int on);
int gk_get_stage_ms(float *out3);

#ifdef __cplusplus
}
#endif
#endif /* GK_H */
