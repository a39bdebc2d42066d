/*
 * gk_featio.h -- C-ABI of libgkhost's feature-CSV I/O: the
 * table the `gpukalc features` command writes and the trainer reads.
 *
 *   gk_featcsv_write  replaces  features_to_csv (reference features.py:250-261):
 *                               csv.writer(lineterminator="\n"), header
 *                               "kernel" + names, one row per point, every
 *                               value format(v, ".17g")
 *   gk_featcsv_parse  replaces  features_from_csv (features.py:264-272):
 *                               csv.DictReader, "kernel" kept as text, every
 *                               other field float(v)
 *
 * Rows are formatted / parsed in parallel (n_threads <= 0: all host threads).
 * The writer is byte-identical to the reference for every double (NaN of
 * either sign prints "nan") and every kernel name (QUOTE_MINIMAL: a name
 * holding ',', '"', '\r' or '\n' is quoted, '"' doubled).  The parser accepts
 * the plain dialect the writer produces -- fields matching
 * [+-]?(d+[.d*]|.d+)([eE][+-]?d+)? or [+-]?(nan|inf|infinity) (any case),
 * quoted kernel names, "\n" or "\r\n" line ends -- and returns
 * GK_FEATCSV_NEEDS_REFERENCE_PATH for anything else (blank lines, ragged rows,
 * duplicate columns, whitespace or '_' inside numbers, a bare '\r', ...): the
 * caller then runs the Python parser, which reproduces the reference's result
 * or exception on it.
 */
#ifndef GK_FEATIO_H
#define GK_FEATIO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GK_FEATCSV_OK = 0, GK_FEATCSV_NEEDS_REFERENCE_PATH = 1 };

/* names: n_cols column names (UTF-8, concatenated, names_off[n_cols + 1]);
 * kernels: n_rows kernel ids (concatenated, kernels_off[n_rows + 1]);
 * value (r, j) = feat[r * ld + cols[j]].  On success *out is a malloc'd buffer
 * of *len bytes (free with gk_featcsv_buf_free); returns 0, or -1 on
 * allocation failure. */
int gk_featcsv_write(const char *names, const int64_t *names_off, int32_t n_cols,
                     const char *kernels, const int64_t *kernels_off, const double *feat,
                     int64_t n_rows, int64_t ld, const int32_t *cols, int n_threads, char **out,
                     size_t *len);
void gk_featcsv_buf_free(char *buf);

typedef struct {
    int64_t n_rows;        /* data rows                                          */
    int32_t n_cols;        /* header columns                                     */
    int32_t kernel_col;    /* index of the "kernel" column, -1 if none           */
    int64_t names_bytes;   /* header names, concatenated                         */
    int64_t kernel_bytes;  /* kernel ids (unquoted), concatenated                */
} gk_featcsv_sizes;

/* Parse a CSV text.  *status = GK_FEATCSV_OK or
 * GK_FEATCSV_NEEDS_REFERENCE_PATH (why: a short reason).  Returns a handle
 * (free with gk_featcsv_free) or NULL on allocation failure. */
void *gk_featcsv_parse(const char *text, size_t len, int n_threads, int *status, char *why,
                       size_t cap);
void gk_featcsv_sizes_of(const void *h, gk_featcsv_sizes *out);
/* names / names_off[n_cols + 1]; kernels / kernels_off[n_rows + 1] (may be
 * NULL when kernel_col < 0); values [n_rows, n_cols] row-major float64, the
 * kernel column's entries left 0. */
int gk_featcsv_copy(const void *h, char *names, int64_t *names_off, char *kernels,
                    int64_t *kernels_off, double *values);
void gk_featcsv_free(void *h);

#ifdef __cplusplus
}
#endif

#endif /* GK_FEATIO_H */
