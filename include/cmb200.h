/*
 * libcmb200 -- C ABI of the B200-native cross-map hot path.
 *
 * The reference (`crossmap`, /root/reference/pkg) is pure Python with no FFI;
 * each entry point below replaces one hot function of that package and is
 * bound from Python with ctypes.  Plain pointers and
 * sizes only; every host buffer is caller-owned, read or written during the
 * call and never retained.  Calls block until results are in the caller's
 * buffers.  Calls on one device are serialised internally; calls on
 * different devices may run concurrently from different host threads.
 *
 * Arrays are row-major.  "len" is a series length in samples.  Returns 0 on
 * success or a negative CMB_ERR_* code; cmb_last_error() then holds a
 * one-line, thread-local message.
 */
#ifndef CMB200_H
#define CMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMB_OK 0
#define CMB_ERR_PARAM (-1)       /* -> ParameterError      (errors.py:8)  */
#define CMB_ERR_TOO_SHORT (-2)   /* -> SeriesTooShortError (errors.py:12) */
#define CMB_ERR_ZERO_VAR (-3)    /* -> ZeroVarianceError   (errors.py:16) */
#define CMB_ERR_CUDA (-10)       /* -> DeviceError (CrossmapError subclass) */
#define CMB_ERR_NCCL (-11)
#define CMB_ERR_UNSUPPORTED (-12)

/* rho layouts for cmb_xmap* */
#define CMB_LAYOUT_LIB_MAJOR 0    /* rho[lib * N + tgt]  (SkillMatrix.rho, ccm.py:56-83) */
#define CMB_LAYOUT_TGT_MAJOR 1    /* rho[tgt * N + lib]  (native kernel layout) */

/* Library version, lockstep with the Python package __version__ (0.1.0 -> 100). */
int cmb_version(void);
/* Message for the most recent failing call on this thread. */
const char* cmb_last_error(void);
/* Number of visible CUDA devices. */
int cmb_device_count(int* n);
/* Diagnostics since the last call (then reset): out[0] kNN rows re-selected
 * by the exact fp64 fallback, out[1] rows checked, out[2] kernel launches
 * issued by the library (host-side count), out[3..] reserved.              */
int cmb_diagnostics(int dev, int64_t* out, int n);
/* Release every device buffer held by the library. */
int cmb_shutdown(void);

/* ---- kNN stage (knn.py) -------------------------------------------------- */

/* pairwise_distances (knn.py:97-128): D[n][n] squared distances between all
 * delay vectors, n = len - (E-1)*tau, float64, reference operation order.   */
int cmb_pairwise_distances(int dev, const double* x, int64_t len, int E, int tau,
                           double* D_out);

/* partial_sort_topk (knn.py:144-177): per row the k smallest entries of
 * D[n][n] over columns j != i, ascending, ties to the smaller column.       */
int cmb_partial_sort_topk(int dev, const double* D, int64_t n, int k,
                          double* d_out, int64_t* idx_out);

/* normalize_to_weights (knn.py:180-202): sq[n][k] ascending squared
 * distances -> simplex weights.                                             */
int cmb_normalize_weights(int dev, const double* sq, int64_t n, int k, double* w_out);

/* build_knn_table (knn.py:205-217): fused embedding + distance + exact
 * top-k + weights, the n x n matrix never materialised.  n = len-(E-1)*tau.
 * d_out (nullable) receives the selected squared distances.                 */
int cmb_knn_table(int dev, const double* x, int64_t len, int E, int tau, int k,
                  int64_t* idx_out, double* w_out, double* d_out);

/* ---- prediction stage (prediction.py) ------------------------------------ */

/* PearsonAggregate.from_arrays (prediction.py:45-55):
 * agg_out = {count, mean_a, mean_b, m2_a, m2_b, comoment}.                  */
int cmb_pearson(int dev, const double* a, const double* b, int64_t n, double* agg_out);

/* lookup_batch (prediction.py:122-161): targets Y[M][len] through one table
 * (idx[n][k], w[n][k], sample offset (E-1)*tau).  rho_out[M] (NaN when
 * undefined), pred_out[M][n] (nullable).                                    */
int cmb_lookup(int dev, const int64_t* idx, const double* w, int64_t n, int k, int offset,
               const double* Y, int64_t len, int64_t M, double* rho_out, double* pred_out);

/* simplex_self_predict (prediction.py:164-182). NaN if undefined.           */
int cmb_simplex(int dev, const double* x, int64_t len, int E, int tau, int Tp, double* rho_out);

/* _self_skill_curve + optimal_embedding (prediction.py:197-262), batched over
 * N series X[N][len].  rho_out[N][E_max] (NaN undefined); estar_out[N]
 * (0 = undefined: constant series or an undefined curve point).            */
int cmb_edim(int dev, const double* X, int64_t N, int64_t len, int E_max, int tau, int Tp,
             double* rho_out, int32_t* estar_out);

/* ---- all-to-all cross map (ccm.py:94-151) -------------------------------- */

/* rho over every ordered (library, target) pair; the library is embedded at
 * the target's E (estar[tgt]); Tp = 0 lookup; estar[i] == 0 marks series i
 * undefined (its row and column are NaN).  X[N][len] float32 samples.
 * stats_out (nullable, 8 doubles): seconds {tables, lookup, total},
 * tables_built, distinct_E, pairs, fixup items (library, target block pairs
 * recomputed in fp64 by the lookup), 0.                                     */
int cmb_xmap(int dev, const float* X, int64_t N, int64_t len, const int32_t* estar, int tau,
             float* rho_out, int layout, double* stats_out);

/* cmb_xmap for float64 series X[N][len] (the reference's own dtype, series.py:25):
 * staged in float64 on the device; the fp32 sweep runs on the series minus
 * their fp64 means (so large offsets keep their digits), kNN certification is
 * bounded against the float64 values and uncertified rows are re-selected
 * exactly in float64 (weights then from the float64 distances).            */
int cmb_xmap64(int dev, const double* X, int64_t N, int64_t len, const int32_t* estar, int tau,
               float* rho_out, int layout, double* stats_out);

/* cmb_xmap64 plus materialised predictions (lookup_batch(want_predictions=True)
 * inside ccm_pairwise, prediction.py:145-153, ccm.py:148-149) for P caller-given
 * (pair_lib[p], pair_tgt[p]) pairs, from the same tables and targets as rho:
 * pred_out[p * len + t] for the n_E = len - (E*(tgt)-1)*tau embedded points,
 * NaN after them and for pairs with an undefined series.                    */
int cmb_xmap_predict(int dev, const double* X, int64_t N, int64_t len, const int32_t* estar, int tau,
                     const int32_t* pair_lib, const int32_t* pair_tgt, int64_t P, float* rho_out, int layout,
                     float* pred_out, double* stats_out);

/* Device-resident shard of cmb_xmap for the multi-GPU driver: X_dev[N][ld]
 * (float32, on `dev`), libraries [lib_begin, lib_end); writes
 * rhoT_dev[tgt * ldr + (lib - lib_begin)] (target-major).  `stream` is a
 * cudaStream_t (NULL = the library's stream); the call returns after the
 * work completes.                                                           */
int cmb_xmap_dev(int dev, const float* X_dev, int64_t N, int64_t len, int64_t ld,
                 const int32_t* estar, int tau, int64_t lib_begin, int64_t lib_end,
                 float* rhoT_dev, int64_t ldr, void* stream, double* stats_out);

/* ---- multi-GPU cross map (shards ccm.py:131-149 by library) -- */
/* NCCL is loaded at run time (libnccl.so.2); without it these return CMB_ERR_NCCL.
 * Every rank computes the rho rows of its contiguous library block [lo, hi)
 * (sizes differ by at most one) for all targets; the only collectives are the
 * broadcast of X from rank 0 and the gather of the library-major row blocks
 * to rank 0 (grouped ncclSend / ncclRecv).  rho is bitwise identical for any
 * rank count.  stats_out (nullable, 8 doubles): tables, lookup, total seconds,
 * tables_built, distinct_E, pairs, fixup items, broadcast + gather seconds.   */

/* 128-byte ncclUniqueId for a one-process-per-GPU job (rank 0 creates it and
 * hands it to the others, e.g. over torch.distributed's store).             */
int cmb_nccl_unique_id(void* id_out);
/* Communicator of this process's device `dev` as rank `rank` of `nranks`.    */
int cmb_nccl_init_rank(int dev, const void* id, int nranks, int rank);
/* Ranks in the communicator of `dev`, this process's rank, NCCL version.     */
int cmb_nccl_info(int dev, int* nranks, int* rank, int* version);
int cmb_nccl_destroy(int dev);
/* One rank of the sharded cross map: X_dev[N][len] float32 on `dev`, valid on
 * rank 0 (broadcast in place); estar[N] host on every rank; rank 0 receives
 * rho_dev[lib * N + tgt] (library-major, device, N x N), other ranks pass NULL.
 * `stream` (cudaStream_t, NULL = the library's); returns when done.          */
int cmb_xmap_rank(int dev, float* X_dev, int64_t N, int64_t len, const int32_t* estar, int tau,
                  float* rho_dev, void* stream, double* stats_out);
/* The same job from one process: devs[0..ndev) (ncclCommInitAll, one host
 * thread per device), host X[N][len] float32, host rho_out[lib * N + tgt].   */
int cmb_xmap_multi(const int* devs, int ndev, const float* X, int64_t N, int64_t len,
                   const int32_t* estar, int tau, float* rho_out, double* stats_out);

/* Device-resident edim: X_dev[N][ld] float32; rho_dev[N][E_max] float64,
 * estar_dev[N] int32.                                                       */
int cmb_edim_dev(int dev, const float* X_dev, int64_t N, int64_t len, int64_t ld, int E_max,
                 int tau, int Tp, double* rho_dev, int32_t* estar_dev, void* stream);

/* ---- convergence sweep (no reference implementation) ------- */

/* Library-size convergence sweep at one embedding dimension E (semantics of
 * oracle/crossmap_oracle.py: ccm_convergence; parity unpinned -- the
 * reference has none).  Series X[N][len]; pairs (lib_ids[p], tgt_ids[p]).
 * For library size sizes[s] (E + 2 <= sizes[s] <= n_E) and sample q, the
 * sorted embedded-point indices pts[off_s + q*sizes[s] ..] (off_s = sum of
 * samples * sizes[s'] over s' < s) form the library: every embedded point is
 * matched to its E + 1 nearest sampled points (self excluded), every target
 * predicted at every point (Tp = 0), skill by Pearson.
 * rho_out[P][n_sizes][samples] (NaN undefined).                             */
int cmb_ccm_convergence(int dev, const double* X, int64_t N, int64_t len, int E, int tau,
                        const int32_t* lib_ids, const int32_t* tgt_ids, int64_t P,
                        const int32_t* sizes, int n_sizes, int samples, const int32_t* pts,
                        double* rho_out);

/* ---- data formats either side of the path ---------- */

/* write_skill_matrix (pkg/src/crossmap/io.py:70-78), the cell rows: text of
 * rows [row0, row0 + nrows) of an n x n skill matrix -- per row the
 * pre-rendered CSV name field names[name_off[r] .. name_off[r+1]) (name_off
 * holds n + 1 entries), then for each cell ',' and f"{v:.6f}" of the float64
 * value (float32 input is widened exactly) or "NA" when not finite, then
 * "\r\n" (csv.writer's terminator) -- formatted on the GPU, byte-identical
 * to the reference.  rho points to row row0 (row-major, leading dimension ld),
 * in device memory when rho_on_device, else host memory; is_f32 selects float.
 * Text goes to out (host, capacity out_cap bytes), its length to *out_len;
 * CMB_ERR_PARAM if it does not fit or a finite |v| >= 1e9 (skill is in
 * [-1, 1]).                                                                  */
int cmb_format_skill_csv(int dev, const void* rho, int rho_on_device, int is_f32, int64_t n,
                         int64_t ld, int64_t row0, int64_t nrows, const char* names,
                         const int64_t* name_off, char* out, int64_t out_cap, int64_t* out_len);

/* load_csv / read_skill_matrix (io.py:25-61, 81-110) input side, host only (no
 * device needed).  The grammar is the reference's: Python's csv module (excel
 * dialect, non-strict: quoting with '""' escapes, records ending at \n, \r\n
 * or \r outside quotes, a blank line = a record with no cells) and float() per
 * cell (ASCII blanks, sign, '_' between digits, exponent, inf/nan), correctly
 * rounded.  Status codes: */
#define CMB_CSV_OK 0
#define CMB_CSV_EMPTY 1          /* no record at all                      -> "empty file"            */
#define CMB_CSV_WIDTH 2          /* err[3] cells in record err[1]          -> "row r has n cells ..." */
#define CMB_CSV_NOT_NUMERIC 3    /* load_csv cell err[2] of record err[1]  -> "not numeric: ..."      */
#define CMB_CSV_NON_FINITE 4     /* load_csv inf/nan cell                  -> "non-finite value ..."  */
#define CMB_CSV_BAD_CELL 5       /* read_skill_matrix cell (or a value past the n x n matrix)         */
#define CMB_CSV_FIELD_LIMIT 6    /* a field over 131,072 characters        -> csv.Error               */
#define CMB_CSV_CAPACITY 7       /* a caller buffer is too small / bad arguments                      */

/* First record (the header): its unquoted cells go to text[spans[2c] ..
 * spans[2c] + spans[2c+1]), *ncells cells; *body_off = offset of the next record. */
int cmb_csv_header(const char* buf, int64_t len, char* text, int64_t text_cap, int64_t* spans,
                   int64_t max_cells, int64_t* ncells, int64_t* body_off);

/* The records after the header.  mode 0 (load_csv): ncols numeric finite cells
 * per record -> out[row][ncols].  mode 1 (read_skill_matrix): a label cell then
 * ncols cells, "NA" = NaN; labels of rows < cap_rows go to labels/label_spans,
 * later rows are only counted.  *nrows = records read.  Cells with non-ASCII
 * bytes are left NaN and listed as (row, col, offset, length) in defer[]
 * (*ndefer), their unquoted text in defer_text: the caller converts them with
 * float() (which accepts Unicode digits).  On a non-zero
 * status err = {status, record (0 = first after the header), column, cells of
 * the record, length of the cell text copied to err_text}.                  */
int cmb_csv_body(const char* buf, int64_t len, int mode, int64_t ncols, double* out, int64_t cap_rows,
                 int64_t* nrows, char* labels, int64_t labels_cap, int64_t* label_spans, int64_t* defer,
                 int64_t defer_cap, char* defer_text, int64_t defer_text_cap, int64_t* ndefer, char* err_text,
                 int64_t err_cap, int64_t* err);

#ifdef __cplusplus
}
#endif

#endif /* CMB200_H */
