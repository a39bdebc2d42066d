/*
 * gk_ensio.h -- C-ABI of libgkhost's ensemble I/O: the
 * portable tree-ensemble JSON document (reference power.py:73-125 reads it,
 * gpukalc_trainer/export.py:53-83,150-175 writes it) parsed straight into the
 * flat device layout, in parallel over trees.
 *
 *   gk_ens_parse   replaces  json.loads + load_ensemble (power.py:73-125,
 *                            incl. _validate_tree :36-70) + this package's
 *                            ensemble.flatten (BFS renumbering)
 *
 * The native loader accepts exactly the documents the reference accepts with
 * the same meaning; anything it does not model (a validation error, booleans,
 * integers beyond 2^53, unknown node keys, malformed JSON) makes it return
 * status GK_ENS_NEEDS_REFERENCE_PATH, and the caller runs the Python loader,
 * which raises the reference's exception with its message (or loads the
 * unusual document the slow way).
 */
#ifndef GK_ENSIO_H
#define GK_ENSIO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GK_ENS_OK = 0, GK_ENS_NEEDS_REFERENCE_PATH = 1 };

/* node kinds in the original-order arrays */
#define GK_ENS_LEAF 0x01u       /* {"value": v}                      */
#define GK_ENS_VALUE_INT 0x02u  /* value / threshold was a JSON int */

typedef struct {
    uint64_t n_trees, n_nodes, n_feat, manifest_bytes;
    uint32_t max_depth, pad_;
    double base_score;
} gk_ens_sizes;

/* Parse + validate + flatten a document.  *status = GK_ENS_OK or
 * GK_ENS_NEEDS_REFERENCE_PATH (why: a short reason, NUL-terminated).  Returns a
 * handle (free with gk_ens_free) or NULL on allocation failure. */
void *gk_ens_parse(const char *text, size_t len, int n_threads, int *status, char *why,
                   size_t cap);

void gk_ens_sizes_of(const void *h, gk_ens_sizes *out);

/* Copy out (host memory, caller-allocated to gk_ens_sizes):
 *   nodes      gk_node[n_nodes] (include/gk.h), each tree breadth-first
 *              (right = left + 1, leaf = {value, -1, self - 1})
 *   tree_off   int64[n_trees], tree_depth int32[n_trees]
 *   scale_lo / scale_hi / gains  double[n_feat]
 *   manifest   the feature names, UTF-8, concatenated; manifest_off int64[n_feat + 1]
 * and, optionally (any may be NULL), the nodes in their ORIGINAL document order
 * (for materialising the reference's node dicts): orig_feature int32,
 * orig_value double (threshold or leaf value), orig_left / orig_right int32,
 * orig_kind uint8 (GK_ENS_* bits). */
int gk_ens_copy(const void *h, void *nodes, int64_t *tree_off, int32_t *tree_depth,
                double *scale_lo, double *scale_hi, double *gains, char *manifest,
                int64_t *manifest_off, int32_t *orig_feature, double *orig_value,
                int32_t *orig_left, int32_t *orig_right, uint8_t *orig_kind);

void gk_ens_free(void *h);

/*
 * The exporter's document text (reference gpukalc_trainer/export.py:53-83,
 * :150-175 writes json.dumps(ensemble_document(result), indent=2) + "\n"),
 * formatted natively, trees in parallel, byte-identical to CPython's json
 * module (shortest round-trip float repr, ensure_ascii escapes, NaN /
 * Infinity literals).  Trees are given in document node order: node i of tree
 * t is index node_off[t] + i; a leaf has is_leaf[i] = 1 and its (already
 * scaled) value in val[i]; a split has feature / threshold (val) / left /
 * right.  indent >= 0 as json.dumps(indent=...); indent < 0: compact
 * (separators ", " and ": ").  On success *out is a malloc'd buffer of *len
 * bytes (free with gk_ens_buf_free); returns 0, or -1 on allocation failure.
 */
int gk_ens_write(int64_t schema_version, double base_score, const char *manifest,
                 const int64_t *manifest_off, uint64_t n_feat, const double *scale_lo,
                 const double *scale_hi, const double *gains, uint64_t n_trees,
                 const int64_t *node_off, const uint8_t *is_leaf, const int32_t *feature,
                 const double *val, const int32_t *left, const int32_t *right, int indent,
                 int n_threads, char **out, size_t *len);
void gk_ens_buf_free(char *buf);

/* CPython's repr(float) of each input, space-separated (test hook). */
int gk_ens_float_repr(const double *x, uint64_t n, char **out, size_t *len);

#ifdef __cplusplus
}
#endif
#endif /* GK_ENSIO_H */
