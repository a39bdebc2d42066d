/*
 * gk_ptx.h -- C-ABI of libgkhost: the native PTX front-end.
 *
 * Host-only (no CUDA): tokenises PTX text, classifies opcodes, splits basic
 * blocks, builds the CFG and the per-block def-use DAG, and packs the kernels
 * straight into the device records of gk.h (gk_token / gk_block / gk_kernel),
 * in parallel over kernels.  It replaces, for a whole corpus at once:
 *
 *   parse_ptx(text, kernel_name, loop_counts=...)   reference ptx/parser.py:156-257
 *     _strip_comments / _extract_body               parser.py:34-62
 *     parse_instruction                             parser.py:86-139
 *     build_dfg                                     parser.py:142-153
 *   classify / is_branch                            reference ptx/classify.py:68-104
 *   KernelGraph.topo_order / loop_multipliers /
 *     exit_blocks / forward_preds                   reference ptx/types.py:79-124
 *   + the host packer (paper_2305_01886_b200/pack.py CorpusBuilder)
 *
 * The output is byte-identical to pack_corpus([parse_ptx(...) ...]) in kernel
 * order, including the latency-signature table (ids in first-seen order).
 *
 * Errors follow the reference's sequential loop: the FIRST failing kernel (in
 * input order) is reported with the reference's exception kind and message;
 * unknown-opcode warnings (classify.py:98) are reported per kernel so the
 * caller can log those the sequential loop would have logged.
 */
#ifndef GK_PTX_H
#define GK_PTX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_PTX_ABI_VERSION 1

/* error kinds (gk_ptx_error) */
enum {
    GK_PTX_OK = 0,
    GK_PTX_PARSE_ERROR = 1,    /* PtxParseError (errors.py:8-18); line >= 1 when known */
    GK_PTX_SCHEDULE_ERROR = 2, /* ScheduleError (types.py:117-121, pack.py)            */
    GK_PTX_VALUE_ERROR = 3,    /* ValueError("substring not found"): .entry without '{' */
    GK_PTX_UNSUPPORTED = 4     /* non-ASCII text: the caller must use parse_ptx        */
};

/* Sizes of a packed result (all element counts). */
typedef struct {
    uint64_t n_tok;     /* tokens (the token array holds n_tok + 1 with the sentinel) */
    uint64_t n_preds;   /* DFG producer entries (u16)                                  */
    uint64_t n_blk;
    uint64_t n_fpreds;  /* forward CFG predecessor entries (u32)                       */
    uint64_t n_topo;
    uint64_t n_ker;
    uint64_t n_sig;
    uint64_t n_warn;    /* unknown-opcode warnings, all kernels                        */
} gk_ptx_sizes;

/*
 * Parse + pack n kernels.  Item i is the .entry named
 *   names[name_off[i] .. name_off[i+1])
 * inside the text blob[text_begin[i] .. text_end[i]) (items may share a text),
 * with loop trip counts labels[label_off[j] .. label_off[j+1]) -> loop_count[j]
 * for j in [loop_off[i], loop_off[i+1]).
 * `table` is the opcode table in the line format written by
 * paper_2305_01886_b200/ptx_native.py (`opcode_table_text`); `strict` raises on
 * unknown opcodes instead of warning.  n_threads <= 0: all hardware threads.
 * Returns an opaque handle (NULL only on allocation failure / bad table).
 */
void *gk_ptx_pack(const char *blob, const int64_t *text_begin, const int64_t *text_end,
                  const char *names, const int64_t *name_off,
                  const int64_t *loop_off, const char *labels, const int64_t *label_off,
                  const int64_t *loop_count, uint64_t n, const char *table, int strict,
                  int n_threads);

/* First failing kernel: returns its error kind (GK_PTX_OK if none) and fills
 * *kernel, *line (-1 when the message carries no line) and msg (NUL-terminated,
 * truncated to cap). */
int gk_ptx_error(const void *h, uint64_t *kernel, int64_t *line, char *msg, size_t cap);

void gk_ptx_sizes_of(const void *h, gk_ptx_sizes *out);

/* Copy the packed arrays (host memory, caller-allocated to gk_ptx_sizes):
 * tok = gk_token[n_tok + 1] (sentinel pred0 = n_preds), preds = u16[n_preds],
 * blk = gk_block[n_blk], fpreds = u32[n_fpreds], topo = u32[n_topo],
 * ker = gk_kernel[n_ker].  Only valid when gk_ptx_error() == GK_PTX_OK. */
int gk_ptx_copy(const void *h, void *tok, uint16_t *preds, void *blk, uint32_t *fpreds,
                uint32_t *topo, void *ker);

/* Signature i = (class code, root, kind) with kind 'f', 's' or 0 (None);
 * root is NUL-terminated into root_buf (cap bytes).  Returns the root length. */
int gk_ptx_sig(const void *h, uint64_t i, int *cls, char *root_buf, size_t cap, int *kind);

/* Warning w: kernel index and the unknown opcode (NUL-terminated). */
int gk_ptx_warning(const void *h, uint64_t w, uint64_t *kernel, char *buf, size_t cap);

void gk_ptx_free(void *h);
int gk_ptx_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GK_PTX_H */
