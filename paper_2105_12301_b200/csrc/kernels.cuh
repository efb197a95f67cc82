// Kernel argument blocks and launchers shared by the C-ABI layer.
#pragma once

#include "cmb_common.cuh"

namespace cmb {

// host-side count of kernel launches issued by the library (diagnostics[2])
void count_launch(int n = 1);

enum KnnMode { KNN_TABLE = 0, KNN_EDIM = 1, KNN_RAW = 2 };

struct KnnArgs {
  const float* x32;         // series-major samples [*][ld] (sweep)
  const double* x64;        // same samples in float64 [*][ld] (exact re-rank, predictions)
  int64_t ld;
  const int32_t* lib_rows;  // series row of each library slot (nullable = identity)
  int nlib;
  int L;                    // library length: T (cross map) or T - Tp (self prediction)
  int tau;
  int e_hi;                 // largest E swept
  uint32_t need;            // bit E-1 set when dimension E is emitted
  int mode;                 // KnnMode
  int k_raw;                // KNN_RAW: neighbour count (else E + 1)
  int rows_per_block;
  int nrb;                  // row blocks per library
  const float* err_m;       // per series row: max |x32 - x64| (nullable = 0)
  // KNN_TABLE: per E base pointer of [nlib][n_E][rec_bytes(E+1)]
  uint8_t* tab[CMB_SWEEP_MAX_E + 1];
  // KNN_EDIM
  int Tp;
  double* part;             // [nlib][nrb][e_hi][5] shifted moments
  int* last_change;         // [nlib] last index where the series changes value
  double* mean;             // [nlib] series mean (Pearson shift)
  // KNN_RAW (single E = e_hi)
  int64_t* raw_idx;
  double* raw_w;
  double* raw_d;
  unsigned long long* diag; // [0] exact fallbacks, [1] rows checked
  int x64_smem;             // set by the launcher: stage the float64 series in shared memory
};

int sweep_width(int e_hi);
cudaError_t launch_knn_sweep(const KnnArgs& a, cudaStream_t st);
cudaError_t launch_edim_finalize(const double* part, const int* last_change, int nlib, int nrb,
                                 int e_hi, int L, int tau, int Tp, double* rho, int32_t* estar,
                                 const int32_t* valid, cudaStream_t st);

// ------------------------------------------------------------------ K3 lookup
#define CMB_MAX_GROUPS 32

struct LookupArgs {
  const float* Y;            // [T][ldy] time-major targets, grouped by E, centred
  int64_t ldy;
  int T;
  int tau;
  int ngroups;
  int g_E[CMB_MAX_GROUPS];   // dimension of each group
  int g_blk0[CMB_MAX_GROUPS];// first 32-target block of each group
  int g_nblk[CMB_MAX_GROUPS];// blocks per group
  int64_t g_item0[CMB_MAX_GROUPS + 1];
  const int32_t* slot_tgt;   // [slots] rho row (target id) or -1 for padding
  const double* obs_s;       // [slots] sum of the centred observed segment
  const double* obs_ss;      // [slots] sum of squares
  const uint8_t* obs_const;  // [slots] 1 when the observed segment is constant
  const uint8_t* tab[CMB_SWEEP_MAX_E + 1];  // per E: [nlib][n_E][rec]
  int nlib;                  // libraries in this chunk
  const int64_t* lib_col;    // [nlib] rho column of each chunk library
  int LS;                    // libraries per work item
  int n_lsub;
  int64_t n_items;
  int* counter;              // work-item counter, zero before launch
  float* rhoT;               // rho_T[tgt * ldr + col]
  int64_t ldr;
  int stage_bytes;           // per-warp table staging slot
  int h16;                   // 16-bit targets, 64 per block, two per lane: 1 fp16, 2 q16 fixed point
  // rotated-lane lookup (lookup.cu rot_library_group; resident fp32 targets):
  // a (library, target block) with a pair whose prediction variance is
  // ill-conditioned in the unshifted fp32 sums is queued here as (library in
  // chunk, first slot of the block) and recomputed in fp64 by lookup_fixup_kernel
  int rot;
  int warps;                 // CTA warps of this launch (0 = kLookupWarps; 12 / 8: rot2 class kernels)
  int tmajor;                // non-resident: work items target-block-major (CMB_LOOKUP_TMAJOR=0: library-major)
  double fix_ratio;          // queue when m2p <= fix_ratio * sum p^2
  int2* fix;
  int* fix_count;
  int fix_cap;
};

constexpr int kLookupWarps = 16;
// CTA warps of the non-resident (long-series) lookup: up to 170 registers per
// thread (the kernel needs 140: no spills, unlike 16 warps at 128) and smaller
// staging rings than 16 warps, so more of the SM's L1 caches target rows
// (K3-L2; 12 warps 4% faster than 8)
#ifndef CMB_NR_WARPS
#define CMB_NR_WARPS 12
#endif
constexpr int kNonResWarps = CMB_NR_WARPS;
// stage size that selects the non-resident (targets in L2) lookup variant
constexpr int kNonResidentStage = 4096 + 16;
int lookup_stage_bytes(int T, int max_rec_bytes, int warps = kLookupWarps);
// two-target rotated path feasible for k at this stage size
bool lookup_rot2_fits(int stage_bytes, int k);
// k <= 3 through the 12-warp two-target path too (else the 16-warp library pairs)
constexpr bool kSmallKRot2 = true;
// CTA warps per neighbour-count class of the resident fp32 lookup.  Fewer warps
// leave larger stage slots, so the two-target path (8 records of two libraries
// per slot) fits for larger k, and more registers per thread.  A/B at full
// size on one box (lookup seconds): every k in one 16-warp kernel 4.705, every
// k with 12 warps 4.543, with 8 4.462; classes 16 (k <= 3) / 12 (4..16) / 8
// (17..24) 4.126; k <= 3 also with 12 warps (two-target path) 3.974.
constexpr int lookup_class_warps(int k) {
  return k <= 3 ? (kSmallKRot2 ? 12 : 16) : (k <= 16 ? 12 : (k <= 24 ? 8 : 16));
}
cudaError_t launch_lookup_xmap(const LookupArgs& a, int grid, cudaStream_t st);
// per-instantiation launchers (lookup*.cu; smem = dynamic shared bytes)
cudaError_t launch_lookup_resident16(const LookupArgs& a, int grid, int smem, cudaStream_t st);
// k ranges of the 16-warp resident kernel's instantiation units
constexpr int lookup_r16_range(int k) { return k <= 3 ? 0 : (k <= 12 ? 1 : (k <= 20 ? 2 : 3)); }
cudaError_t launch_lookup_r16_2_3(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_r16_4_12(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_r16_13_20(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_r16_21_31(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_nonresident(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_h16(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_w12(const LookupArgs& a, int grid, int smem, cudaStream_t st);
cudaError_t launch_lookup_w8(const LookupArgs& a, int grid, int smem, cudaStream_t st);
// predictions of (library, target) pairs from the chunk's tables: pairs[q] =
// (library list index, target slot, E, output row), libraries [c0, c0 + nlib);
// pred[row][t] = sum w y (centred fp32 targets) + shift[slot]
cudaError_t launch_predict_pairs(const LookupArgs& a, const int4* pairs, int64_t npairs, int64_t c0,
                                 const double* shift, float* pred, int64_t ldp, cudaStream_t st);
// exact fp64 completion of the pairs the rotated lookup queued in a.fix
cudaError_t launch_lookup_fixup(const LookupArgs& a, cudaStream_t st);

// ------------------------------------------------------------------ helpers (utils.cu)
cudaError_t launch_series_stats(const float* x32, int64_t N, int64_t T, int64_t ld, double* mean,
                                cudaStream_t st);
cudaError_t launch_promote(const float* x32, int64_t N, int64_t T, int64_t ld, double* x64,
                           cudaStream_t st);
cudaError_t launch_demote(const double* x64, int64_t N, int64_t T, float* x32, float* err_m,
                          cudaStream_t st);
cudaError_t launch_demote_center(const double* x64, int64_t N, int64_t T, float* x32, float* err_m,
                                 double* mu, cudaStream_t st);
// shift[slot] = mean[tgt] + (mu ? mu[tgt] : 0) of each slot's target (0 for padding)
cudaError_t launch_slot_shift(const double* mean, const double* mu, const int32_t* slot_tgt, int64_t slots,
                              double* shift, cudaStream_t st);
cudaError_t launch_build_targets(const float* x32, int64_t ld, const double* mean,
                                 const int32_t* slot_tgt, int64_t slots, int T, float* Y,
                                 int64_t ldy, cudaStream_t st);
cudaError_t launch_obs_moments(const float* Y, int64_t ldy, int T, int tau, const int32_t* slot_E,
                               int64_t slots, double* s, double* ss, uint8_t* cst, cudaStream_t st);
cudaError_t launch_fill_nan(float* p, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st);
// *dst = *src by one thread (dst: mapped page-locked host memory)
cudaError_t launch_copy_count(const int* src, int* dst, cudaStream_t st);
cudaError_t launch_targets_to_half(const float* Y, int64_t ldy, int T, int tau, const int32_t* slot_E,
                                   int64_t slots, void* Yh, double* s, double* ss, uint8_t* cst,
                                   int mode, cudaStream_t st);
cudaError_t launch_pairwise(const double* x, int n, int E, int tau, double* D, cudaStream_t st);
cudaError_t launch_topk_rows(const double* D, int n, int k, double* d_out, int64_t* i_out,
                             cudaStream_t st);
cudaError_t launch_weights(const double* sq, int64_t n, int k, double* w, int* flags,
                           cudaStream_t st);
cudaError_t launch_pearson(const double* a, const double* b, int64_t n, double* agg,
                           cudaStream_t st);
cudaError_t launch_lookup64(const int64_t* idx, const double* w, int64_t n, int k, int offset,
                            const double* Y, int64_t len, int64_t M, double* pred,
                            double* rho, cudaStream_t st);
cudaError_t launch_restricted_records(const double* X, int64_t len, const int32_t* libs, int n, int E,
                                      int tau, const int32_t* pts, const int64_t* size_off,
                                      const int32_t* sizes, int n_sizes, int samples, int64_t chunk0,
                                      int64_t n_pseudo, uint8_t* tab, cudaStream_t st);

cudaError_t launch_transpose_f32(const float* src, int64_t rows, int64_t cols, int64_t lds,
                                 float* dst, int64_t ldd, cudaStream_t st);

// ------------------------------------------------------------------ data formats (io.cu)
cudaError_t format_skill_rows(const void* rho_dev, bool f32, int64_t n, int64_t ld, int64_t row0,
                              int64_t nrows, const char* names_dev, const int64_t* name_off_dev,
                              int64_t* row_len_dev, int64_t* row_off_dev, int64_t* row_off_host,
                              int* range_err_dev, bool* out_of_range, char* out_dev, int64_t out_cap,
                              int64_t* out_len, cudaStream_t st);
// host CSV reader (io.cu): status codes of csv_header / csv_body (CMB_CSV_* in cmb200.h)
enum CsvStatus { CSV_OK = 0, CSV_EMPTY = 1, CSV_WIDTH = 2, CSV_NOT_NUMERIC = 3, CSV_NON_FINITE = 4,
                 CSV_BAD_CELL = 5, CSV_FIELD_LIMIT = 6, CSV_CAPACITY = 7 };
int csv_header(const char* buf, int64_t len, char* text, int64_t text_cap, int64_t* spans, int64_t max_cells,
               int64_t* ncells, int64_t* body_off);
int csv_body(const char* buf, int64_t len, int mode, int64_t ncols, double* out, int64_t cap_rows, int64_t* nrows,
             char* labels, int64_t labels_cap, int64_t* label_spans, int64_t* defer, int64_t defer_cap,
             char* defer_text, int64_t defer_text_cap, int64_t* ndefer, char* err_text, int64_t err_cap,
             int64_t* err);

}  // namespace cmb
