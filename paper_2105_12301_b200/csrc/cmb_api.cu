// extern "C" boundary of libcmb200: validation, device contexts, staging of
// host buffers, and the cross-map driver that sequences the kernels.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace cmb {

// ---------------------------------------------------------------- errors
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  set_error("CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file,
            line, what);
  return CMB_ERR_CUDA;
}

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }

// ---------------------------------------------------------------- device context
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~DevBuf() {}
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max(bytes, (size_t)256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

enum BufId {
  B_X64, B_X32, B_ERR, B_MEAN, B_Y, B_SLOT_TGT, B_SLOT_E, B_OBS_S, B_OBS_SS, B_OBS_C, B_LIBROWS,
  B_LIBCOL, B_TAB, B_COUNTER, B_RHOT, B_RHO, B_PART, B_LAST, B_LMEAN, B_A, B_B, B_C, B_D, B_E,
  B_DIAG, B_EST, B_FMT_RHO, B_FMT_NAMES, B_FMT_OFF, B_FMT_LEN, B_FMT_ROWOFF, B_FMT_OUT, B_YH, B_FIX, B_SLAB, B_MU, B_PAIRS, B_SHIFT, B_PRED, B_NBUF
};

// page-locked host buffer (the pageable-output bounce slabs of xmap_host)
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

// events destroyed on every exit path (early returns leaked them)
struct EventSet {
  std::vector<cudaEvent_t> v;
  cudaError_t make(cudaEvent_t* e, unsigned flags) {
    cudaError_t r = cudaEventCreateWithFlags(e, flags);
    if (r == cudaSuccess) v.push_back(*e);
    return r;
  }
  ~EventSet() {
    for (auto e : v) cudaEventDestroy(e);
  }
};

struct Ctx {
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // D2H overlap of the host-buffer cross map
  std::mutex mu;
  DevBuf buf[B_NBUF];
  HostBuf bounce[2];
  ncclComm_t comm = nullptr;  // cmb_nccl_init_rank / cmb_xmap_multi
  int nranks = 1, rank = 0;
  // mapped page-locked word: per-chunk counters read back by a one-thread
  // kernel, not a DMA copy, which would queue behind the chunk's rho D2H
  int* cnt_host = nullptr;
  int* cnt_dev = nullptr;
  bool ready = false;
};

static std::mutex g_ctx_mu;
static std::vector<std::unique_ptr<Ctx>> g_ctx;

static int get_ctx(int dev, Ctx** out) {
  int n = 0;
  CMB_CUDA(cudaGetDeviceCount(&n));
  if (dev < 0 || dev >= n) {
    set_error("device %d not available (%d visible)", dev, n);
    return CMB_ERR_PARAM;
  }
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if ((int)g_ctx.size() < n) g_ctx.resize(n);
  if (!g_ctx[dev]) g_ctx[dev].reset(new Ctx());
  Ctx* c = g_ctx[dev].get();
  if (!c->ready) {
    CMB_CUDA(cudaSetDevice(dev));
    CMB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CMB_CUDA(c->buf[B_DIAG].ensure(8 * sizeof(unsigned long long)));
    CMB_CUDA(cudaMemset(c->buf[B_DIAG].p, 0, 8 * sizeof(unsigned long long)));
    c->dev = dev;
    c->ready = true;
  }
  *out = c;
  return CMB_OK;
}

#define CMB_CTX(dev)                                  \
  Ctx* ctx = nullptr;                                 \
  {                                                   \
    int _r = get_ctx((dev), &ctx);                    \
    if (_r) return _r;                                \
  }                                                   \
  std::lock_guard<std::mutex> _lock(ctx->mu);         \
  CMB_CUDA(cudaSetDevice(ctx->dev));                  \
  cudaStream_t st = ctx->stream;

#define CMB_TRY(call)               \
  do {                              \
    int _r = (call);                \
    if (_r) return _r;              \
  } while (0)

static int too_short(int64_t len, int E, int tau, int64_t n) {
  set_error("series of length %lld yields %lld embedded points for E=%d, tau=%d; neighbor search needs at least %d",
            (long long)len, (long long)n, E, tau, E + 2);
  return CMB_ERR_TOO_SHORT;
}

// valid_count (series.py:84-98)
static int check_valid_count(int64_t len, int E, int tau) {
  if (len < 1) {
    set_error("a series needs at least one observation");
    return CMB_ERR_TOO_SHORT;
  }
  const int64_t n = len - (int64_t)(E - 1) * tau;
  if (n < E + 2) return too_short(len, E, tau, n);
  return CMB_OK;
}

static int check_spec(int E, int tau) {
  CMB_PARAM(tau >= 1, "lag must be >= 1, got %d", tau);
  CMB_PARAM(E >= 1, "embedding dimension must be >= 1, got %d", E);
  return CMB_OK;
}

// ---------------------------------------------------------------- kNN (RAW) via the sweep
static int knn_raw(Ctx* ctx, cudaStream_t st, const double* x_dev, const float* x32_dev,
                   const float* err_dev, int64_t len, int E, int tau, int k, int64_t* idx_dev,
                   double* w_dev, double* d_dev) {
  KnnArgs a;
  memset(&a, 0, sizeof(a));
  a.x32 = x32_dev;
  a.x64 = x_dev;
  a.ld = len;
  a.nlib = 1;
  a.L = (int)len;
  a.tau = tau;
  a.e_hi = E;
  a.need = 1u << (E - 1);
  a.mode = KNN_RAW;
  a.k_raw = k;
  a.rows_per_block = 128;
  a.nrb = (int)((len + 127) / 128);
  a.err_m = err_dev;
  a.raw_idx = idx_dev;
  a.raw_w = w_dev;
  a.raw_d = d_dev;
  a.diag = ctx->buf[B_DIAG].as<unsigned long long>();
  CMB_CUDA(launch_knn_sweep(a, st));
  return CMB_OK;
}

// upload a float64 series batch and derive its float32 copy + rounding error
static int stage_series64(Ctx* ctx, cudaStream_t st, const double* X, int64_t N, int64_t len) {
  CMB_CUDA(ctx->buf[B_X64].ensure(sizeof(double) * N * len));
  CMB_CUDA(ctx->buf[B_X32].ensure(sizeof(float) * N * len + 256));
  CMB_CUDA(ctx->buf[B_ERR].ensure(sizeof(float) * N));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_X64].p, X, sizeof(double) * N * len, cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_demote(ctx->buf[B_X64].as<double>(), N, len, ctx->buf[B_X32].as<float>(),
                         ctx->buf[B_ERR].as<float>(), st));
  return CMB_OK;
}

// ---------------------------------------------------------------- self-prediction sweep (EDIM)
static int edim_core(Ctx* ctx, cudaStream_t st, const float* x32, const double* x64,
                     const float* err, int64_t N, int64_t len, int64_t ld, int E_hi, uint32_t need,
                     int tau, int Tp, double* rho_dev, int32_t* estar_dev) {
  const int L = (int)(len - Tp);
  const int rpb = 128;
  const int nrb = (L + rpb - 1) / rpb;
  // batch libraries to bound the partial-moment buffer (~256 MB)
  int64_t batch = std::max<int64_t>(1, (256ll << 20) / ((int64_t)nrb * E_hi * 5 * 8));
  batch = std::min<int64_t>(batch, N);
  CMB_CUDA(ctx->buf[B_PART].ensure(sizeof(double) * batch * nrb * E_hi * 5));
  CMB_CUDA(ctx->buf[B_LAST].ensure(sizeof(int) * batch));
  CMB_CUDA(ctx->buf[B_LMEAN].ensure(sizeof(double) * batch));
  for (int64_t b0 = 0; b0 < N; b0 += batch) {
    const int64_t nb = std::min(batch, N - b0);
    KnnArgs a;
    memset(&a, 0, sizeof(a));
    a.x32 = x32 + b0 * ld;
    a.x64 = x64 + b0 * ld;
    a.ld = ld;
    a.nlib = (int)nb;
    a.L = L;
    a.tau = tau;
    a.e_hi = E_hi;
    a.need = need;
    a.mode = KNN_EDIM;
    a.rows_per_block = rpb;
    a.nrb = nrb;
    a.err_m = err ? err + b0 : nullptr;
    a.Tp = Tp;
    a.part = ctx->buf[B_PART].as<double>();
    a.last_change = ctx->buf[B_LAST].as<int>();
    a.mean = ctx->buf[B_LMEAN].as<double>();
    a.diag = ctx->buf[B_DIAG].as<unsigned long long>();
    CMB_CUDA(launch_knn_sweep(a, st));
    CMB_CUDA(launch_edim_finalize(a.part, a.last_change, (int)nb, nrb, E_hi, L, tau, Tp,
                                  rho_dev + b0 * E_hi, estar_dev ? estar_dev + b0 : nullptr,
                                  nullptr, st));
  }
  return CMB_OK;
}

// ---------------------------------------------------------------- cross-map driver
struct XmapStats {
  double t_tables = 0, t_lookup = 0, t_total = 0;
  double tables = 0, distinct = 0, pairs = 0;
  double fixups = 0;  // pairs finished by the exact fp64 fixup of the rotated lookup
};

// capacity of the rotated lookup's fixup queue per library chunk
constexpr int kFixCap = 1 << 22;

// on_chunk(col_lo, col_hi): called after the lookup of each library chunk has
// been enqueued on st, with the rho_T column range that is final once st reaches
// that point (the host-buffer entry point overlaps its D2H copy with later chunks)
using ChunkFn = std::function<int(int64_t, int64_t)>;

// Materialised predictions requested with a cross map: pairs (lib[p], tgt[p]),
// p < P, into pred_dev[p][ldp] (NaN past n_E and for undefined pairs); mu: per
// series the fp64 mean removed before the fp32 sweep (cmb_xmap64), or null.
struct PredReq {
  const int32_t* lib = nullptr;
  const int32_t* tgt = nullptr;
  int64_t P = 0;
  float* pred_dev = nullptr;
  int64_t ldp = 0;
  const double* mu = nullptr;
};

// X: float32 samples [N][ld] on the device.  x64_in (nullable): the caller's
// float64 series [N][ld] when X was derived from them (cmb_xmap64: X centred,
// err_in = per-series certification perturbation); otherwise X is promoted.
static int xmap_core(Ctx* ctx, cudaStream_t st, const float* X, int64_t N, int64_t T, int64_t ld,
                     const int32_t* estar, int tau, int64_t lib_begin, int64_t lib_end, float* rhoT,
                     int64_t ldr, XmapStats* stats, const ChunkFn& on_chunk = nullptr,
                     const double* x64_in = nullptr, const float* err_in = nullptr,
                     const PredReq* preds = nullptr) {
  CMB_PARAM(tau >= 1, "tau must be >= 1, got %d", tau);
  CMB_PARAM(lib_begin >= 0 && lib_begin <= lib_end && lib_end <= N, "bad library range [%lld, %lld)",
            (long long)lib_begin, (long long)lib_end);
  CMB_PARAM(T <= 65535, "series length %lld exceeds the 16-bit table format", (long long)T);
  // ---- group targets by E* (ccm.py:123-127)
  std::vector<std::vector<int>> by_e(CMB_SWEEP_MAX_E + 1);
  for (int64_t t = 0; t < N; ++t) {
    const int e = estar[t];
    if (e == 0) continue;
    CMB_PARAM(e >= 1 && e <= CMB_SWEEP_MAX_E, "dimension %d outside [1, %d]", e, CMB_SWEEP_MAX_E);
    by_e[e].push_back((int)t);
  }
  std::vector<int32_t> slot_tgt, slot_E;
  LookupArgs la;
  memset(&la, 0, sizeof(la));
  uint32_t need = 0;
  int e_hi = 0, max_rec = 0;
  // opt-in fp16 target blocks (64 targets per block, lookup.cu warp_libraries_h16)
  const char* h16_env = getenv("CMB_LOOKUP_FP16");
  // (CMB_LOOKUP_FP16=2: 16-bit fixed point instead of fp16, same layout)
  const int h16_mode = h16_env && (h16_env[0] == '1' || h16_env[0] == '2') ? h16_env[0] - '0' : 0;
  const bool want_h16 = h16_mode != 0;
  const int blk_sz = want_h16 ? 64 : 32;
  for (int e = 1; e <= CMB_SWEEP_MAX_E; ++e) {
    if (by_e[e].empty()) continue;
    CMB_TRY(check_valid_count(T, e, tau));
    const int g = la.ngroups++;
    la.g_E[g] = e;
    la.g_blk0[g] = (int)(slot_tgt.size() / 32);
    const size_t padded = (by_e[e].size() + blk_sz - 1) / blk_sz * blk_sz;
    la.g_nblk[g] = (int)(padded / 32);
    for (size_t q = 0; q < padded; ++q) {
      slot_tgt.push_back(q < by_e[e].size() ? by_e[e][q] : -1);
      slot_E.push_back(e);
    }
    need |= 1u << (e - 1);
    e_hi = e;
    max_rec = std::max(max_rec, rec_bytes(e + 1));
  }
  std::vector<int32_t> lib_rows;
  std::vector<int64_t> lib_col;
  for (int64_t l = lib_begin; l < lib_end; ++l)
    if (estar[l] != 0) {
      lib_rows.push_back((int32_t)l);
      lib_col.push_back(l - lib_begin);
    }
  const int64_t ncols = lib_end - lib_begin;
  CMB_CUDA(launch_fill_nan(rhoT, N, ncols, ldr, st));
  if (la.ngroups == 0 || lib_rows.empty()) {
    if (on_chunk) CMB_TRY(on_chunk(0, ncols));
    return CMB_OK;
  }
  const int stage = lookup_stage_bytes((int)T, max_rec);

  // ---- requested predictions: (library list index, target slot, E, output row),
  //      sorted by library so each chunk's pairs are one contiguous range
  std::vector<int4> pairs;
  if (preds && preds->P > 0) {
    std::vector<int> lib_index(N, -1), tgt_slot(N, -1);
    for (size_t q = 0; q < lib_rows.size(); ++q) lib_index[lib_rows[q]] = (int)q;
    for (size_t q = 0; q < slot_tgt.size(); ++q)
      if (slot_tgt[q] >= 0) tgt_slot[slot_tgt[q]] = (int)q;
    for (int64_t q = 0; q < preds->P; ++q) {
      const int l = preds->lib[q], t = preds->tgt[q];
      CMB_PARAM(l >= 0 && l < N && t >= 0 && t < N, "prediction pair %lld out of range", (long long)q);
      if (lib_index[l] < 0 || tgt_slot[t] < 0) continue;  // undefined pair: its row stays NaN
      pairs.push_back(make_int4(lib_index[l], tgt_slot[t], estar[t], (int)q));
    }
    std::stable_sort(pairs.begin(), pairs.end(), [](const int4& a, const int4& b) { return a.x < b.x; });
    CMB_CUDA(launch_fill_nan(preds->pred_dev, preds->P, preds->ldp, preds->ldp, st));
  }

  // ---- device staging
  const int64_t slots = (int64_t)slot_tgt.size();
  const int64_t ldy = slots;
  CMB_CUDA(ctx->buf[B_SLOT_TGT].ensure(4 * slots));
  CMB_CUDA(ctx->buf[B_SLOT_E].ensure(4 * slots));
  CMB_CUDA(ctx->buf[B_OBS_S].ensure(8 * slots));
  CMB_CUDA(ctx->buf[B_OBS_SS].ensure(8 * slots));
  CMB_CUDA(ctx->buf[B_OBS_C].ensure(slots));
  CMB_CUDA(ctx->buf[B_Y].ensure(sizeof(float) * T * ldy));
  CMB_CUDA(ctx->buf[B_MEAN].ensure(8 * N));
  if (!x64_in) CMB_CUDA(ctx->buf[B_X64].ensure(sizeof(double) * N * ld));
  CMB_CUDA(ctx->buf[B_LIBROWS].ensure(4 * lib_rows.size()));
  CMB_CUDA(ctx->buf[B_LIBCOL].ensure(8 * lib_col.size()));
  CMB_CUDA(ctx->buf[B_COUNTER].ensure(16));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_SLOT_TGT].p, slot_tgt.data(), 4 * slots, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_SLOT_E].p, slot_E.data(), 4 * slots, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_LIBROWS].p, lib_rows.data(), 4 * lib_rows.size(), cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_LIBCOL].p, lib_col.data(), 8 * lib_col.size(), cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_series_stats(X, N, T, ld, ctx->buf[B_MEAN].as<double>(), st));
  CMB_CUDA(launch_build_targets(X, ld, ctx->buf[B_MEAN].as<double>(), ctx->buf[B_SLOT_TGT].as<int32_t>(),
                                slots, (int)T, ctx->buf[B_Y].as<float>(), ldy, st));
  const bool h16 = want_h16 && stage != kNonResidentStage;
  la.tmajor = !(getenv("CMB_LOOKUP_TMAJOR") && getenv("CMB_LOOKUP_TMAJOR")[0] == '0');
  if (h16) {
    for (int g = 0; g < la.ngroups; ++g) {  // blocks of 64 slots
      la.g_blk0[g] /= 2;
      la.g_nblk[g] /= 2;
    }
    CMB_CUDA(ctx->buf[B_YH].ensure(2 * T * ldy));
    CMB_CUDA(launch_targets_to_half(ctx->buf[B_Y].as<float>(), ldy, (int)T, tau, ctx->buf[B_SLOT_E].as<int32_t>(),
                                    slots, ctx->buf[B_YH].p, ctx->buf[B_OBS_S].as<double>(),
                                    ctx->buf[B_OBS_SS].as<double>(), ctx->buf[B_OBS_C].as<uint8_t>(), h16_mode, st));
  } else {
    CMB_CUDA(launch_obs_moments(ctx->buf[B_Y].as<float>(), ldy, (int)T, tau, ctx->buf[B_SLOT_E].as<int32_t>(),
                                slots, ctx->buf[B_OBS_S].as<double>(), ctx->buf[B_OBS_SS].as<double>(),
                                ctx->buf[B_OBS_C].as<uint8_t>(), st));
  }
  if (!pairs.empty()) {
    CMB_CUDA(ctx->buf[B_PAIRS].ensure(sizeof(int4) * pairs.size()));
    CMB_CUDA(ctx->buf[B_SHIFT].ensure(sizeof(double) * slots));
    CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_PAIRS].p, pairs.data(), sizeof(int4) * pairs.size(), cudaMemcpyHostToDevice, st));
    CMB_CUDA(launch_slot_shift(ctx->buf[B_MEAN].as<double>(), preds->mu, ctx->buf[B_SLOT_TGT].as<int32_t>(), slots,
                               ctx->buf[B_SHIFT].as<double>(), st));
  }
  const double* x64 = x64_in;
  if (!x64) {
    CMB_CUDA(launch_promote(X, N, T, ld, ctx->buf[B_X64].as<double>(), st));
    x64 = ctx->buf[B_X64].as<double>();
  }

  // ---- library chunks: tables for every needed E, then the lookup
  size_t per_lib = 0;
  size_t tab_off[CMB_SWEEP_MAX_E + 2] = {0};
  for (int g = 0; g < la.ngroups; ++g) {
    const int e = la.g_E[g];
    per_lib += rec_lib_stride(e + 1, T - (int64_t)(e - 1) * tau);
  }
  const int LS = 4 * kLookupWarps;  // four libraries per warp per work item
  const size_t budget = (size_t)6 << 30;
  int64_t C = (int64_t)(budget / std::max<size_t>(per_lib, 1));
  C = std::max<int64_t>(LS, C / LS * LS);
  C = std::min<int64_t>(C, ((int64_t)lib_rows.size() + LS - 1) / LS * LS);
  CMB_CUDA(ctx->buf[B_TAB].ensure(per_lib * C + 256));
  {
    size_t o = 0;
    for (int g = 0; g < la.ngroups; ++g) {
      const int e = la.g_E[g];
      tab_off[e] = o;
      o += (size_t)C * rec_lib_stride(e + 1, T - (int64_t)(e - 1) * tau);
    }
  }

  const char* rot_env = getenv("CMB_LOOKUP_ROT");
  const char* fix_env = getenv("CMB_FIX_RATIO");
  const char* split_env = getenv("CMB_LOOKUP_SPLIT");  // 0: every k in one 16-warp launch
  CMB_CUDA(ctx->buf[B_FIX].ensure(16 + sizeof(int2) * (size_t)kFixCap));
  if (!ctx->cnt_host) {
    CMB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->cnt_host), 64, cudaHostAllocMapped));
    CMB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->cnt_dev), ctx->cnt_host, 0));
  }
  int64_t fixups = 0;
  EventSet evs;
  cudaEvent_t ev[3];
  for (auto& e : ev) CMB_CUDA(evs.make(&e, 0));
  float ms_tab = 0, ms_look = 0;
  const int rpb = 128;
  for (int64_t c0 = 0; c0 < (int64_t)lib_rows.size(); c0 += C) {
    const int64_t nc = std::min<int64_t>(C, (int64_t)lib_rows.size() - c0);
    KnnArgs a;
    memset(&a, 0, sizeof(a));
    a.x32 = X;
    a.x64 = x64;
    a.ld = ld;
    a.err_m = err_in;
    a.lib_rows = ctx->buf[B_LIBROWS].as<int32_t>() + c0;
    a.nlib = (int)nc;
    a.L = (int)T;
    a.tau = tau;
    a.e_hi = e_hi;
    a.need = need;
    a.mode = KNN_TABLE;
    a.rows_per_block = rpb;
    a.nrb = (int)((T + rpb - 1) / rpb);
    for (int g = 0; g < la.ngroups; ++g) a.tab[la.g_E[g]] = ctx->buf[B_TAB].as<uint8_t>() + tab_off[la.g_E[g]];
    a.diag = ctx->buf[B_DIAG].as<unsigned long long>();
    CMB_CUDA(cudaEventRecord(ev[0], st));
    CMB_CUDA(launch_knn_sweep(a, st));
    CMB_CUDA(cudaEventRecord(ev[1], st));

    la.Y = h16 ? reinterpret_cast<const float*>(ctx->buf[B_YH].p) : ctx->buf[B_Y].as<float>();
    la.h16 = h16 ? h16_mode : 0;
    la.ldy = ldy;
    la.T = (int)T;
    la.tau = tau;
    la.slot_tgt = ctx->buf[B_SLOT_TGT].as<int32_t>();
    la.obs_s = ctx->buf[B_OBS_S].as<double>();
    la.obs_ss = ctx->buf[B_OBS_SS].as<double>();
    la.obs_const = ctx->buf[B_OBS_C].as<uint8_t>();
    for (int g = 0; g < la.ngroups; ++g) la.tab[la.g_E[g]] = a.tab[la.g_E[g]];
    la.nlib = (int)nc;
    la.lib_col = ctx->buf[B_LIBCOL].as<int64_t>() + c0;
    la.LS = LS;
    la.n_lsub = (int)((nc + LS - 1) / LS);
    int64_t items = 0;
    for (int g = 0; g < la.ngroups; ++g) {
      la.g_item0[g] = items;
      items += (int64_t)la.n_lsub * la.g_nblk[g];
    }
    la.g_item0[la.ngroups] = items;
    la.n_items = items;
    la.counter = ctx->buf[B_COUNTER].as<int>();
    la.rhoT = rhoT;
    la.ldr = ldr;
    la.stage_bytes = stage;
    // rotated-lane lookup (lookup.cu rot_library_group) unless CMB_LOOKUP_ROT=0;
    // its ill-conditioned pairs are finished in fp64 by the fixup kernel
    la.rot = h16 ? 0 : (rot_env ? atoi(rot_env) : 2);
    la.fix = reinterpret_cast<int2*>(ctx->buf[B_FIX].as<uint8_t>() + 16);
    la.fix_count = ctx->buf[B_FIX].as<int>();
    la.fix_cap = kFixCap;
    la.fix_ratio = fix_env ? atof(fix_env) : 0.0625;
    la.warps = 0;
    CMB_CUDA(cudaMemsetAsync(la.fix_count, 0, sizeof(int), st));
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->dev);
    // one launch per warp-count class (lookup_class_warps): the groups of a
    // class, their own work items and stage size; a class whose two-target
    // stage does not fit (long series) goes to the 16-warp launch
    auto launch_all = [&](bool split) -> int {
      // classes 0-3: 16-warp launches per k range (lookup_r16_range, one
      // instantiation unit each); 4 / 5: the 12- / 8-warp two-target kernels
      constexpr int NC = 6;
      LookupArgs cls[NC];
      const int cw[NC] = {kLookupWarps, kLookupWarps, kLookupWarps, kLookupWarps, 12, 8};
      for (int c = 0; c < NC; ++c) {
        cls[c] = la;
        cls[c].ngroups = 0;
        cls[c].warps = c < 4 ? 0 : cw[c];
      }
      int mrec[NC] = {0, 0, 0, 0, 0, 0};
      const bool resident = stage != kNonResidentStage;
      for (int g = 0; g < la.ngroups; ++g) {
        const int k = la.g_E[g] + 1;
        // the non-resident and 16-bit kernels cover every k in one launch
        int c = (resident && !h16) ? lookup_r16_range(k) : 0;
        if (split && resident && !h16 && la.rot == 2) {
          const int w = lookup_class_warps(k);
          const int cand = w == 12 ? 4 : (w == 8 ? 5 : -1);
          if (cand > 0 && lookup_rot2_fits(lookup_stage_bytes((int)T, rec_bytes(k), w), k)) c = cand;
        }
        const int q = cls[c].ngroups++;
        cls[c].g_E[q] = la.g_E[g];
        cls[c].g_blk0[q] = la.g_blk0[g];
        cls[c].g_nblk[q] = la.g_nblk[g];
        mrec[c] = std::max(mrec[c], rec_bytes(k));
      }
      for (int c = 0; c < NC; ++c) {
        LookupArgs& L = cls[c];
        if (L.ngroups == 0) continue;
        L.LS = 4 * cw[c];
        L.n_lsub = (int)((nc + L.LS - 1) / L.LS);
        int64_t it = 0;
        for (int g = 0; g < L.ngroups; ++g) {
          L.g_item0[g] = it;
          it += (int64_t)L.n_lsub * L.g_nblk[g];
        }
        L.g_item0[L.ngroups] = it;
        L.n_items = it;
        L.stage_bytes = c < 4 ? stage : lookup_stage_bytes((int)T, mrec[c], cw[c]);
        CMB_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(int), st));
        CMB_CUDA(launch_lookup_xmap(L, (int)std::min<int64_t>(it, dev_sms), st));
      }
      return CMB_OK;
    };
    const bool split = !(split_env && split_env[0] == '0');
    CMB_TRY(launch_all(split));
    if (la.rot) {
      CMB_CUDA(launch_lookup_fixup(la, st));
      CMB_CUDA(launch_copy_count(la.fix_count, ctx->cnt_dev, st));
    }
    if (!pairs.empty()) {
      const auto lo_it = std::lower_bound(pairs.begin(), pairs.end(), (int)c0,
                                          [](const int4& a, int v) { return a.x < v; });
      const auto hi_it = std::lower_bound(pairs.begin(), pairs.end(), (int)(c0 + nc),
                                          [](const int4& a, int v) { return a.x < v; });
      CMB_CUDA(launch_predict_pairs(la, ctx->buf[B_PAIRS].as<int4>() + (lo_it - pairs.begin()), hi_it - lo_it, c0,
                                    ctx->buf[B_SHIFT].as<double>(), preds->pred_dev, preds->ldp, st));
    }
    if (on_chunk) {
      // columns [first column of this chunk (0 for the first), first column of the next chunk)
      const int64_t col_lo = (c0 == 0) ? 0 : lib_rows[c0] - lib_begin;
      const int64_t col_hi = (c0 + nc < (int64_t)lib_rows.size()) ? lib_rows[c0 + nc] - lib_begin : ncols;
      CMB_TRY(on_chunk(col_lo, col_hi));
    }
    CMB_CUDA(cudaEventRecord(ev[2], st));
    CMB_CUDA(cudaEventSynchronize(ev[2]));
    if (la.rot) {
      // written by launch_copy_count before ev[2]: no DMA copy, which would wait
      // behind the previous chunks' rho copies on the D2H engine (host-buffer
      // cross map) and leave the GPU idle until it returns
      const int nfix = *reinterpret_cast<volatile int*>(ctx->cnt_host);
      fixups += nfix;
      if (nfix > kFixCap) {
        // more ill-conditioned pairs than the queue holds (a pathological chunk):
        // redo the chunk with the shifted-moment lookup, which needs no fixups
        la.rot = 0;
        CMB_TRY(launch_all(false));
        CMB_CUDA(cudaEventRecord(ev[2], st));
        CMB_CUDA(cudaEventSynchronize(ev[2]));
      }
    }
    float a_ms = 0, b_ms = 0;
    CMB_CUDA(cudaEventElapsedTime(&a_ms, ev[0], ev[1]));
    CMB_CUDA(cudaEventElapsedTime(&b_ms, ev[1], ev[2]));
    ms_tab += a_ms;
    ms_look += b_ms;
  }
  if (stats) {
    stats->t_tables = ms_tab * 1e-3;
    stats->t_lookup = ms_look * 1e-3;
    stats->tables = (double)lib_rows.size() * la.ngroups;
    stats->distinct = la.ngroups;
    int64_t tg = 0;
    for (int g = 0; g < la.ngroups; ++g) tg += (int64_t)by_e[la.g_E[g]].size();
    stats->pairs = (double)lib_rows.size() * (double)tg;
    stats->fixups = (double)fixups;
  }
  return CMB_OK;
}

static void nccl_destroy(ncclComm_t c);  // NCCL section below

}  // namespace cmb

using namespace cmb;

// =====================================================================================
extern "C" {

int cmb_version(void) { return 100; }

const char* cmb_last_error(void) { return g_err; }

int cmb_device_count(int* n) {
  CMB_CUDA(cudaGetDeviceCount(n));
  return CMB_OK;
}

int cmb_diagnostics(int dev, int64_t* out, int n) {
  CMB_CTX(dev);
  unsigned long long h[8];
  CMB_CUDA(cudaMemcpyAsync(h, ctx->buf[B_DIAG].p, sizeof(h), cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaMemsetAsync(ctx->buf[B_DIAG].p, 0, sizeof(h), st));
  CMB_CUDA(cudaStreamSynchronize(st));
  h[7] = h[2];
  h[2] = (unsigned long long)g_launches.exchange(0);
  for (int q = 0; q < n && q < 8; ++q) out[q] = (int64_t)h[q];
  return CMB_OK;
}

int cmb_shutdown(void) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (auto& c : g_ctx) {
    if (!c) continue;
    std::lock_guard<std::mutex> l(c->mu);
    cudaSetDevice(c->dev);
    for (auto& b : c->buf) b.release();
    for (auto& b : c->bounce) b.release();
    if (c->cnt_host) cudaFreeHost(c->cnt_host);
    c->cnt_host = c->cnt_dev = nullptr;
    if (c->comm) nccl_destroy(c->comm);
    c->comm = nullptr;
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    c->stream = nullptr;
    c->copy_stream = nullptr;
    c->ready = false;
  }
  g_ctx.clear();
  return CMB_OK;
}

int cmb_pairwise_distances(int dev, const double* x, int64_t len, int E, int tau, double* D_out) {
  CMB_TRY(check_spec(E, tau));
  const int64_t n = len - (int64_t)(E - 1) * tau;
  if (n < 2) {
    set_error("series of length %lld yields %lld embedded points for E=%d, tau=%d; pairwise distances need at least 2",
              (long long)len, (long long)n, E, tau);
    return CMB_ERR_TOO_SHORT;
  }
  CMB_CTX(dev);
  CMB_CUDA(ctx->buf[B_A].ensure(8 * len));
  CMB_CUDA(ctx->buf[B_B].ensure(8 * n * n));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_A].p, x, 8 * len, cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_pairwise(ctx->buf[B_A].as<double>(), (int)n, E, tau, ctx->buf[B_B].as<double>(), st));
  CMB_CUDA(cudaMemcpyAsync(D_out, ctx->buf[B_B].p, 8 * n * n, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_partial_sort_topk(int dev, const double* D, int64_t n, int k, double* d_out, int64_t* idx_out) {
  CMB_PARAM(k >= 1 && k <= n - 1, "neighbor count must lie in [1, %lld], got %d", (long long)(n - 1), k);
  CMB_PARAM(n <= 16384, "partial_sort_topk supports n <= 16384, got %lld", (long long)n);
  CMB_CTX(dev);
  CMB_CUDA(ctx->buf[B_A].ensure(8 * n * n));
  CMB_CUDA(ctx->buf[B_B].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_C].ensure(8 * n * k));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_A].p, D, 8 * n * n, cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_topk_rows(ctx->buf[B_A].as<double>(), (int)n, k, ctx->buf[B_B].as<double>(),
                            ctx->buf[B_C].as<int64_t>(), st));
  CMB_CUDA(cudaMemcpyAsync(d_out, ctx->buf[B_B].p, 8 * n * k, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaMemcpyAsync(idx_out, ctx->buf[B_C].p, 8 * n * k, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_normalize_weights(int dev, const double* sq, int64_t n, int k, double* w_out) {
  CMB_PARAM(k >= 1 && n >= 0, "expected an n x k distance array, got (%lld, %d)", (long long)n, k);
  if (n == 0) return CMB_OK;
  CMB_CTX(dev);
  CMB_CUDA(ctx->buf[B_A].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_B].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_C].ensure(16));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_A].p, sq, 8 * n * k, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemsetAsync(ctx->buf[B_C].p, 0, 4, st));
  CMB_CUDA(launch_weights(ctx->buf[B_A].as<double>(), n, k, ctx->buf[B_B].as<double>(), ctx->buf[B_C].as<int>(), st));
  int flags = 0;
  CMB_CUDA(cudaMemcpyAsync(&flags, ctx->buf[B_C].p, 4, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaMemcpyAsync(w_out, ctx->buf[B_B].p, 8 * n * k, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  CMB_PARAM(!(flags & 1), "squared distances must be >= 0");
  CMB_PARAM(!(flags & 2), "distance rows must be ascending");
  return CMB_OK;
}

int cmb_knn_table(int dev, const double* x, int64_t len, int E, int tau, int k, int64_t* idx_out,
                  double* w_out, double* d_out) {
  CMB_TRY(check_spec(E, tau));
  CMB_TRY(check_valid_count(len, E, tau));
  const int64_t n = len - (int64_t)(E - 1) * tau;
  CMB_PARAM(k >= 1 && k <= n - 1, "neighbor count must lie in [1, %lld], got %d", (long long)(n - 1), k);
  CMB_CTX(dev);
  CMB_TRY(stage_series64(ctx, st, x, 1, len));
  CMB_CUDA(ctx->buf[B_A].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_B].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_C].ensure(8 * n * k));
  if (E <= CMB_SWEEP_MAX_E && k + 1 <= 32) {
    CMB_TRY(knn_raw(ctx, st, ctx->buf[B_X64].as<double>(), ctx->buf[B_X32].as<float>(),
                    ctx->buf[B_ERR].as<float>(), len, E, tau, k, ctx->buf[B_A].as<int64_t>(),
                    ctx->buf[B_B].as<double>(), ctx->buf[B_C].as<double>()));
  } else {
    // wide k: materialised distances + per-row sort + weights (same semantics)
    CMB_PARAM(n <= 16384, "k > 31 tables support n <= 16384, got %lld", (long long)n);
    CMB_CUDA(ctx->buf[B_D].ensure(8 * n * n));
    CMB_CUDA(ctx->buf[B_E].ensure(16));
    CMB_CUDA(launch_pairwise(ctx->buf[B_X64].as<double>(), (int)n, E, tau, ctx->buf[B_D].as<double>(), st));
    CMB_CUDA(launch_topk_rows(ctx->buf[B_D].as<double>(), (int)n, k, ctx->buf[B_C].as<double>(),
                              ctx->buf[B_A].as<int64_t>(), st));
    CMB_CUDA(cudaMemsetAsync(ctx->buf[B_E].p, 0, 4, st));
    CMB_CUDA(launch_weights(ctx->buf[B_C].as<double>(), n, k, ctx->buf[B_B].as<double>(), ctx->buf[B_E].as<int>(), st));
  }
  CMB_CUDA(cudaMemcpyAsync(idx_out, ctx->buf[B_A].p, 8 * n * k, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaMemcpyAsync(w_out, ctx->buf[B_B].p, 8 * n * k, cudaMemcpyDeviceToHost, st));
  if (d_out) CMB_CUDA(cudaMemcpyAsync(d_out, ctx->buf[B_C].p, 8 * n * k, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_pearson(int dev, const double* a, const double* b, int64_t n, double* agg_out) {
  CMB_PARAM(n >= 0, "negative length");
  if (n == 0) {
    for (int q = 0; q < 6; ++q) agg_out[q] = 0.0;
    return CMB_OK;
  }
  CMB_CTX(dev);
  CMB_CUDA(ctx->buf[B_A].ensure(8 * n));
  CMB_CUDA(ctx->buf[B_B].ensure(8 * n));
  CMB_CUDA(ctx->buf[B_C].ensure(64));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_A].p, a, 8 * n, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_B].p, b, 8 * n, cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_pearson(ctx->buf[B_A].as<double>(), ctx->buf[B_B].as<double>(), n, ctx->buf[B_C].as<double>(), st));
  CMB_CUDA(cudaMemcpyAsync(agg_out, ctx->buf[B_C].p, 48, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_lookup(int dev, const int64_t* idx, const double* w, int64_t n, int k, int offset,
               const double* Y, int64_t len, int64_t M, double* rho_out, double* pred_out) {
  CMB_PARAM(n >= 1 && k >= 1 && offset >= 0, "bad table shape (%lld, %d)", (long long)n, k);
  CMB_PARAM(len >= n + offset, "target has %lld samples; table needs at least %lld", (long long)len,
            (long long)(n + offset));
  if (M == 0) return CMB_OK;
  CMB_CTX(dev);
  CMB_CUDA(ctx->buf[B_A].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_B].ensure(8 * n * k));
  CMB_CUDA(ctx->buf[B_C].ensure(8 * M * len));
  CMB_CUDA(ctx->buf[B_D].ensure(8 * M * n));
  CMB_CUDA(ctx->buf[B_E].ensure(8 * M));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_A].p, idx, 8 * n * k, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_B].p, w, 8 * n * k, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_C].p, Y, 8 * M * len, cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_lookup64(ctx->buf[B_A].as<int64_t>(), ctx->buf[B_B].as<double>(), n, k, offset,
                           ctx->buf[B_C].as<double>(), len, M, ctx->buf[B_D].as<double>(),
                           ctx->buf[B_E].as<double>(), st));
  CMB_CUDA(cudaMemcpyAsync(rho_out, ctx->buf[B_E].p, 8 * M, cudaMemcpyDeviceToHost, st));
  if (pred_out) CMB_CUDA(cudaMemcpyAsync(pred_out, ctx->buf[B_D].p, 8 * M * n, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_simplex(int dev, const double* x, int64_t len, int E, int tau, int Tp, double* rho_out) {
  CMB_TRY(check_spec(E, tau));
  CMB_PARAM(Tp >= 1, "prediction horizon must be >= 1, got %d", Tp);
  if (len <= Tp) {
    set_error("series of length %lld cannot support horizon %d", (long long)len, Tp);
    return CMB_ERR_TOO_SHORT;
  }
  CMB_TRY(check_valid_count(len - Tp, E, tau));
  CMB_PARAM(E <= CMB_SWEEP_MAX_E, "embedding dimension %d exceeds the supported %d", E, CMB_SWEEP_MAX_E);
  CMB_CTX(dev);
  CMB_TRY(stage_series64(ctx, st, x, 1, len));
  CMB_CUDA(ctx->buf[B_RHO].ensure(8 * E));
  CMB_TRY(edim_core(ctx, st, ctx->buf[B_X32].as<float>(), ctx->buf[B_X64].as<double>(),
                    ctx->buf[B_ERR].as<float>(), 1, len, len, E, 1u << (E - 1), tau, Tp,
                    ctx->buf[B_RHO].as<double>(), nullptr));
  std::vector<double> r(E);
  CMB_CUDA(cudaMemcpyAsync(r.data(), ctx->buf[B_RHO].p, 8 * E, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  *rho_out = r[E - 1];
  return CMB_OK;
}

int cmb_edim(int dev, const double* X, int64_t N, int64_t len, int E_max, int tau, int Tp,
             double* rho_out, int32_t* estar_out) {
  CMB_PARAM(E_max >= 1, "dimension bound must be >= 1, got %d", E_max);
  CMB_PARAM(Tp >= 1, "prediction horizon must be >= 1, got %d", Tp);
  CMB_PARAM(tau >= 1, "lag must be >= 1, got %d", tau);
  CMB_PARAM(E_max <= CMB_SWEEP_MAX_E, "dimension bound %d exceeds the supported %d", E_max, CMB_SWEEP_MAX_E);
  if (len <= Tp) {
    set_error("series of length %lld cannot support horizon %d", (long long)len, Tp);
    return CMB_ERR_TOO_SHORT;
  }
  CMB_TRY(check_valid_count(len - Tp, E_max, tau));
  if (N == 0) return CMB_OK;
  CMB_CTX(dev);
  CMB_TRY(stage_series64(ctx, st, X, N, len));
  CMB_CUDA(ctx->buf[B_RHO].ensure(8 * N * E_max));
  CMB_CUDA(ctx->buf[B_EST].ensure(4 * N));
  const uint32_t need = (E_max >= 32) ? 0xffffffffu : ((1u << E_max) - 1);
  CMB_TRY(edim_core(ctx, st, ctx->buf[B_X32].as<float>(), ctx->buf[B_X64].as<double>(),
                    ctx->buf[B_ERR].as<float>(), N, len, len, E_max, need, tau, Tp,
                    ctx->buf[B_RHO].as<double>(), ctx->buf[B_EST].as<int32_t>()));
  CMB_CUDA(cudaMemcpyAsync(rho_out, ctx->buf[B_RHO].p, 8 * N * E_max, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaMemcpyAsync(estar_out, ctx->buf[B_EST].p, 4 * N, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_edim_dev(int dev, const float* X_dev, int64_t N, int64_t len, int64_t ld, int E_max, int tau,
                 int Tp, double* rho_dev, int32_t* estar_dev, void* stream) {
  CMB_PARAM(E_max >= 1 && E_max <= CMB_SWEEP_MAX_E, "dimension bound %d outside [1, %d]", E_max, CMB_SWEEP_MAX_E);
  CMB_PARAM(Tp >= 1 && tau >= 1, "bad Tp/tau");
  if (len <= Tp) {
    set_error("series of length %lld cannot support horizon %d", (long long)len, Tp);
    return CMB_ERR_TOO_SHORT;
  }
  CMB_TRY(check_valid_count(len - Tp, E_max, tau));
  CMB_CTX(dev);
  if (stream) st = (cudaStream_t)stream;
  CMB_CUDA(ctx->buf[B_X64].ensure(sizeof(double) * N * ld));
  CMB_CUDA(launch_promote(X_dev, N, len, ld, ctx->buf[B_X64].as<double>(), st));
  const uint32_t need = (E_max >= 32) ? 0xffffffffu : ((1u << E_max) - 1);
  CMB_TRY(edim_core(ctx, st, X_dev, ctx->buf[B_X64].as<double>(), nullptr, N, len, ld, E_max, need,
                    tau, Tp, rho_dev, estar_dev));
  CMB_CUDA(cudaStreamSynchronize(st));
  return CMB_OK;
}

int cmb_xmap_dev(int dev, const float* X_dev, int64_t N, int64_t len, int64_t ld, const int32_t* estar,
                 int tau, int64_t lib_begin, int64_t lib_end, float* rhoT_dev, int64_t ldr, void* stream,
                 double* stats_out) {
  CMB_CTX(dev);
  if (stream) st = (cudaStream_t)stream;
  XmapStats s;
  cudaEvent_t e0, e1;
  CMB_CUDA(cudaEventCreate(&e0));
  CMB_CUDA(cudaEventCreate(&e1));
  CMB_CUDA(cudaEventRecord(e0, st));
  CMB_TRY(xmap_core(ctx, st, X_dev, N, len, ld, estar, tau, lib_begin, lib_end, rhoT_dev, ldr, &s));
  CMB_CUDA(cudaEventRecord(e1, st));
  CMB_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (stats_out) {
    const double v[8] = {s.t_tables, s.t_lookup, ms * 1e-3, s.tables, s.distinct, s.pairs, s.fixups, 0};
    memcpy(stats_out, v, sizeof(v));
  }
  return CMB_OK;
}

}  // extern "C"

namespace cmb {

// Host-buffer cross map behind cmb_xmap / cmb_xmap64.  Target-major output is
// copied back per library chunk on a second stream while later chunks compute:
// straight into rho_out when it is page-locked, else through two pinned
// bounce slabs (a device-to-pageable copy would block the host and serialise
// the chunks).
constexpr int kDrainThreads = 8;  // host threads copying a bounce slab into pageable output

static int xmap_host(Ctx* ctx, cudaStream_t st, const void* X, bool f64, int64_t N, int64_t len,
                     const int32_t* estar, int tau, float* rho_out, int layout, double* stats_out,
                     const int32_t* pair_lib = nullptr, const int32_t* pair_tgt = nullptr, int64_t P = 0,
                     float* pred_out = nullptr) {
  const int64_t ldr = (N + 3) / 4 * 4;
  CMB_CUDA(ctx->buf[B_X32].ensure(sizeof(float) * N * len + 256));
  CMB_CUDA(ctx->buf[B_RHOT].ensure(sizeof(float) * N * ldr));
  EventSet evs;
  cudaEvent_t e0, e1;
  CMB_CUDA(evs.make(&e0, 0));
  CMB_CUDA(evs.make(&e1, 0));
  CMB_CUDA(cudaEventRecord(e0, st));
  const double* x64 = nullptr;
  const float* err = nullptr;
  if (f64) {
    CMB_CUDA(ctx->buf[B_X64].ensure(sizeof(double) * N * len));
    CMB_CUDA(ctx->buf[B_ERR].ensure(sizeof(float) * N));
    CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_X64].p, X, sizeof(double) * N * len, cudaMemcpyHostToDevice, st));
    CMB_CUDA(ctx->buf[B_MU].ensure(sizeof(double) * N));
    CMB_CUDA(launch_demote_center(ctx->buf[B_X64].as<double>(), N, len, ctx->buf[B_X32].as<float>(),
                                  ctx->buf[B_ERR].as<float>(), ctx->buf[B_MU].as<double>(), st));
    x64 = ctx->buf[B_X64].as<double>();
    err = ctx->buf[B_ERR].as<float>();
  } else {
    CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_X32].p, X, sizeof(float) * N * len, cudaMemcpyHostToDevice, st));
  }
  XmapStats s;
  PredReq pr;
  if (P > 0) {
    pr.lib = pair_lib;
    pr.tgt = pair_tgt;
    pr.P = P;
    pr.ldp = len;
    CMB_CUDA(ctx->buf[B_PRED].ensure(sizeof(float) * (size_t)P * len));
    pr.pred_dev = ctx->buf[B_PRED].as<float>();
    CMB_CUDA(launch_fill_nan(pr.pred_dev, P, len, len, st));
    pr.mu = f64 ? ctx->buf[B_MU].as<double>() : nullptr;
  }
  const PredReq* prp = P > 0 ? &pr : nullptr;
  if (layout == CMB_LAYOUT_TGT_MAJOR) {
    if (!ctx->copy_stream) CMB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    cudaPointerAttributes attr;
    const bool pinned = cudaPointerGetAttributes(&attr, rho_out) == cudaSuccess &&
                        attr.type != cudaMemoryTypeUnregistered;
    cudaGetLastError();
    const float* rt = ctx->buf[B_RHOT].as<float>();
    // pageable output: chunk slabs go device -> pinned bounce (async) -> rho_out
    // (host memcpy of chunk c while chunk c + 1 computes)
    struct Pending { int64_t lo = 0, hi = 0; float* slab = nullptr; cudaEvent_t ev = nullptr; };
    Pending pend;
    int slot = 0;
    // pageable output: its pages are first touched (faulted and zeroed by the
    // OS, ~1 s for the 11 GB of config 3) by host threads while the first chunk
    // computes, not inside the drains; joined before the first drain writes
    std::vector<std::thread> touch;
    if (!pinned) {
      const size_t bytes = sizeof(float) * (size_t)N * (size_t)N;
      const size_t page = 4096;
      for (int t = 0; t < kDrainThreads; ++t)
        touch.emplace_back([=]() {
          volatile char* b = reinterpret_cast<volatile char*>(rho_out);
          for (size_t o = bytes * t / kDrainThreads / page * page; o < bytes * (t + 1) / kDrainThreads; o += page) b[o] = 0;
        });
    }
    auto join_touch = [&]() {
      for (auto& th : touch) th.join();
      touch.clear();
    };
    auto drain = [&]() -> int {
      join_touch();
      if (!pend.slab) return CMB_OK;
      const auto t0 = std::chrono::steady_clock::now();
      CMB_CUDA(cudaEventSynchronize(pend.ev));
      const auto t1 = std::chrono::steady_clock::now();
      const int64_t w = pend.hi - pend.lo;
      // row copies split over host threads (first touch of the caller's pages
      // and the strided memcpy are both host-bound)
      const float* slab = pend.slab;
      const int64_t lo = pend.lo;
      auto rows = [&](int64_t r0, int64_t r1) {
        for (int64_t r = r0; r < r1; ++r) memcpy(rho_out + r * N + lo, slab + r * w, sizeof(float) * w);
      };
      const int nt = (int)std::min<int64_t>(kDrainThreads, std::max<int64_t>(1, N / 1024));
      std::vector<std::thread> pool;
      for (int t = 1; t < nt; ++t) pool.emplace_back(rows, N * t / nt, N * (t + 1) / nt);
      rows(0, N / nt);
      for (auto& th : pool) th.join();
      pend.slab = nullptr;
      if (getenv("CMB_TRACE"))
        fprintf(stderr, "cmb_xmap trace: drain cols %lld: wait %.1f ms, memcpy %.1f ms\n", (long long)w,
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
      return CMB_OK;
    };
    auto on_chunk = [&](int64_t lo, int64_t hi) -> int {
      if (hi <= lo) return CMB_OK;
      cudaEvent_t ev;
      CMB_CUDA(evs.make(&ev, cudaEventDisableTiming));
      CMB_CUDA(cudaEventRecord(ev, st));
      CMB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev, 0));
      if (pinned) {
        CMB_CUDA(cudaMemcpy2DAsync(rho_out + lo, sizeof(float) * N, rt + lo, sizeof(float) * ldr,
                                   sizeof(float) * (hi - lo), N, cudaMemcpyDeviceToHost, ctx->copy_stream));
        return CMB_OK;
      }
      CMB_TRY(drain());  // the previous chunk's slab (its copy was queued one chunk ago)
      const size_t need = sizeof(float) * (size_t)N * (size_t)(hi - lo);
      CMB_CUDA(ctx->bounce[slot].ensure(need));
      float* slab = reinterpret_cast<float*>(ctx->bounce[slot].p);
      CMB_CUDA(cudaMemcpy2DAsync(slab, sizeof(float) * (hi - lo), rt + lo, sizeof(float) * ldr,
                                 sizeof(float) * (hi - lo), N, cudaMemcpyDeviceToHost, ctx->copy_stream));
      cudaEvent_t cev;
      CMB_CUDA(evs.make(&cev, cudaEventDisableTiming));
      CMB_CUDA(cudaEventRecord(cev, ctx->copy_stream));
      pend.lo = lo;
      pend.hi = hi;
      pend.slab = slab;
      pend.ev = cev;
      slot ^= 1;
      return CMB_OK;
    };
    const auto t_core0 = std::chrono::steady_clock::now();
    const int rc = xmap_core(ctx, st, ctx->buf[B_X32].as<float>(), N, len, len, estar, tau, 0, N,
                             ctx->buf[B_RHOT].as<float>(), ldr, &s, on_chunk, x64, err, prp);
    join_touch();  // (an early error return from xmap_core skips the drains)
    const auto t_core1 = std::chrono::steady_clock::now();
    cudaEvent_t copied;
    CMB_CUDA(evs.make(&copied, cudaEventDisableTiming));
    CMB_CUDA(cudaEventRecord(copied, ctx->copy_stream));
    CMB_CUDA(cudaStreamWaitEvent(st, copied, 0));
    CMB_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    if (getenv("CMB_TRACE")) {
      const auto t_copy = std::chrono::steady_clock::now();
      const auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      fprintf(stderr, "cmb_xmap trace: core %.1f ms (tables %.1f + lookup %.1f), copy tail %.1f ms\n",
              ms(t_core0, t_core1), s.t_tables * 1e3, s.t_lookup * 1e3, ms(t_core1, t_copy));
    }
    if (rc) return rc;
    const auto t_drain0 = std::chrono::steady_clock::now();
    CMB_TRY(drain());
    if (getenv("CMB_TRACE"))
      fprintf(stderr, "cmb_xmap trace: pageable=%d last drain %.1f ms\n", (int)!pinned,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_drain0).count());
  } else {
    CMB_TRY(xmap_core(ctx, st, ctx->buf[B_X32].as<float>(), N, len, len, estar, tau, 0, N,
                      ctx->buf[B_RHOT].as<float>(), ldr, &s, nullptr, x64, err, prp));
    CMB_CUDA(ctx->buf[B_RHO].ensure(sizeof(float) * N * ldr));
    CMB_CUDA(launch_transpose_f32(ctx->buf[B_RHOT].as<float>(), N, N, ldr, ctx->buf[B_RHO].as<float>(), ldr, st));
    CMB_CUDA(cudaMemcpy2DAsync(rho_out, sizeof(float) * N, ctx->buf[B_RHO].p, sizeof(float) * ldr,
                               sizeof(float) * N, N, cudaMemcpyDeviceToHost, st));
  }
  if (P > 0)
    CMB_CUDA(cudaMemcpyAsync(pred_out, pr.pred_dev, sizeof(float) * (size_t)P * len, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaEventRecord(e1, st));
  CMB_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (stats_out) {
    const double v[8] = {s.t_tables, s.t_lookup, ms * 1e-3, s.tables, s.distinct, s.pairs, s.fixups, 0};
    memcpy(stats_out, v, sizeof(v));
  }
  return CMB_OK;
}

}  // namespace cmb

extern "C" {

int cmb_xmap(int dev, const float* X, int64_t N, int64_t len, const int32_t* estar, int tau,
             float* rho_out, int layout, double* stats_out) {
  CMB_PARAM(layout == CMB_LAYOUT_LIB_MAJOR || layout == CMB_LAYOUT_TGT_MAJOR, "bad layout %d", layout);
  CMB_PARAM(N >= 1 && len >= 1, "empty dataset");
  CMB_CTX(dev);
  return xmap_host(ctx, st, X, false, N, len, estar, tau, rho_out, layout, stats_out);
}

int cmb_xmap_predict(int dev, const double* X, int64_t N, int64_t len, const int32_t* estar, int tau,
                     const int32_t* pair_lib, const int32_t* pair_tgt, int64_t P, float* rho_out, int layout,
                     float* pred_out, double* stats_out) {
  CMB_PARAM(layout == CMB_LAYOUT_LIB_MAJOR || layout == CMB_LAYOUT_TGT_MAJOR, "bad layout %d", layout);
  CMB_PARAM(N >= 1 && len >= 1, "empty dataset");
  CMB_PARAM(P >= 0 && (P == 0 || (pair_lib && pair_tgt && pred_out)), "bad prediction pairs");
  CMB_CTX(dev);
  return xmap_host(ctx, st, X, true, N, len, estar, tau, rho_out, layout, stats_out, pair_lib, pair_tgt, P, pred_out);
}

int cmb_xmap64(int dev, const double* X, int64_t N, int64_t len, const int32_t* estar, int tau,
               float* rho_out, int layout, double* stats_out) {
  CMB_PARAM(layout == CMB_LAYOUT_LIB_MAJOR || layout == CMB_LAYOUT_TGT_MAJOR, "bad layout %d", layout);
  CMB_PARAM(N >= 1 && len >= 1, "empty dataset");
  CMB_CTX(dev);
  return xmap_host(ctx, st, X, true, N, len, estar, tau, rho_out, layout, stats_out);
}

}  // extern "C"

// ---------------------------------------------------------------- NCCL (multi-GPU)
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy PyTorch already
// loaded when there is one, else the system's), so the library has no link-time
// NCCL dependency and never mixes two NCCL versions in one process.
namespace cmb {

struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommCount) commCount = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclGetVersion) getVersion = nullptr;
};

static std::mutex g_nccl_mu;
static NcclApi g_nccl;

static NcclApi* nccl_api() {
  std::lock_guard<std::mutex> g(g_nccl_mu);
  if (!g_nccl.tried) {
    g_nccl.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_nccl.why = dlerror() ? dlerror() : "libnccl.so.2 not found";
    } else {
      bool all = true;
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        if (!fp) all = false;
      };
      sym(g_nccl.getUniqueId, "ncclGetUniqueId");
      sym(g_nccl.commInitRank, "ncclCommInitRank");
      sym(g_nccl.commInitAll, "ncclCommInitAll");
      sym(g_nccl.commDestroy, "ncclCommDestroy");
      sym(g_nccl.commCount, "ncclCommCount");
      sym(g_nccl.broadcast, "ncclBroadcast");
      sym(g_nccl.send, "ncclSend");
      sym(g_nccl.recv, "ncclRecv");
      sym(g_nccl.groupStart, "ncclGroupStart");
      sym(g_nccl.groupEnd, "ncclGroupEnd");
      sym(g_nccl.errorString, "ncclGetErrorString");
      sym(g_nccl.getVersion, "ncclGetVersion");
      g_nccl.ok = all;
      if (!all) g_nccl.why = "libnccl.so.2 lacks a required symbol";
    }
  }
  return &g_nccl;
}

static void nccl_destroy(ncclComm_t c) {
  if (nccl_api()->ok) nccl_api()->commDestroy(c);
}

#define CMB_NCCL(call)                                                                        \
  do {                                                                                        \
    ncclResult_t _r = (call);                                                                 \
    if (_r != ncclSuccess) {                                                                  \
      ::cmb::set_error("NCCL error %d (%s) in %s", (int)_r, nccl_api()->errorString(_r), #call); \
      return CMB_ERR_NCCL;                                                                    \
    }                                                                                         \
  } while (0)

static int need_nccl() {
  NcclApi* api = nccl_api();
  if (!api->ok) {
    set_error("NCCL unavailable: %s", api->why.c_str());
    return CMB_ERR_NCCL;
  }
  return CMB_OK;
}

// contiguous library block of rank r (sizes differ by at most one; distributed.py shard_bounds)
static void shard_bounds(int64_t n, int world, int r, int64_t* lo, int64_t* hi) {
  const int64_t base = n / world, extra = n % world;
  *lo = r * base + std::min<int64_t>(r, extra);
  *hi = *lo + base + (r < extra ? 1 : 0);
}

// One rank's part of the sharded cross map (the caller holds ctx->mu, device set):
// broadcast X from rank 0, rho of libraries [lo, hi) for every target
// (xmap_core), the shard transposed to library-major rows, and the rows gathered
// to rank 0 into rho_lm[N][N] (library-major, device, rank 0 only) with grouped
// send/recv.  Per-pair arithmetic does not depend on the rank count, so rho is
// bitwise identical for any G.  stats: {tables, lookup, total, tables_built,
// distinct_E, pairs, fixups, broadcast + gather seconds}.
static int xmap_rank_core(Ctx* ctx, cudaStream_t st, float* X_dev, int64_t N, int64_t len,
                          const int32_t* estar, int tau, float* rho_lm, double* stats_out) {
  NcclApi* api = nccl_api();
  const int G = ctx->nranks, r = ctx->rank;
  EventSet evs;
  cudaEvent_t e0, e1, e2, e3;
  CMB_CUDA(evs.make(&e0, 0));
  CMB_CUDA(evs.make(&e1, 0));
  CMB_CUDA(evs.make(&e2, 0));
  CMB_CUDA(evs.make(&e3, 0));
  CMB_CUDA(cudaEventRecord(e0, st));
  CMB_NCCL(api->broadcast(X_dev, X_dev, (size_t)(N * len), ncclFloat, 0, ctx->comm, st));
  CMB_CUDA(cudaEventRecord(e1, st));
  int64_t lo, hi;
  shard_bounds(N, G, r, &lo, &hi);
  const int64_t w = hi - lo, ldr = std::max<int64_t>(4, (w + 3) / 4 * 4);
  CMB_CUDA(ctx->buf[B_RHOT].ensure(sizeof(float) * (size_t)N * ldr + 16));
  XmapStats s;
  CMB_TRY(xmap_core(ctx, st, X_dev, N, len, len, estar, tau, lo, hi, ctx->buf[B_RHOT].as<float>(), ldr, &s));
  CMB_CUDA(cudaEventRecord(e2, st));
  // library-major rows of the shard: straight into the result on rank 0
  float* mine = rho_lm;
  if (r != 0) {
    CMB_CUDA(ctx->buf[B_SLAB].ensure(sizeof(float) * (size_t)std::max<int64_t>(w, 1) * N));
    mine = ctx->buf[B_SLAB].as<float>();
  }
  if (w > 0)
    CMB_CUDA(launch_transpose_f32(ctx->buf[B_RHOT].as<float>(), N, w, ldr, r == 0 ? mine + lo * N : mine, N, st));
  CMB_NCCL(api->groupStart());
  if (r == 0) {
    for (int g = 1; g < G; ++g) {
      int64_t glo, ghi;
      shard_bounds(N, G, g, &glo, &ghi);
      if (ghi > glo) CMB_NCCL(api->recv(rho_lm + glo * N, (size_t)((ghi - glo) * N), ncclFloat, g, ctx->comm, st));
    }
  } else if (w > 0) {
    CMB_NCCL(api->send(mine, (size_t)(w * N), ncclFloat, 0, ctx->comm, st));
  }
  CMB_NCCL(api->groupEnd());
  CMB_CUDA(cudaEventRecord(e3, st));
  CMB_CUDA(cudaEventSynchronize(e3));
  float ms_b = 0, ms_g = 0, ms_t = 0;
  cudaEventElapsedTime(&ms_b, e0, e1);
  cudaEventElapsedTime(&ms_g, e2, e3);
  cudaEventElapsedTime(&ms_t, e0, e3);
  if (stats_out) {
    const double v[8] = {s.t_tables, s.t_lookup, ms_t * 1e-3, s.tables, s.distinct, s.pairs, s.fixups,
                         (ms_b + ms_g) * 1e-3};
    memcpy(stats_out, v, sizeof(v));
  }
  return CMB_OK;
}

}  // namespace cmb

extern "C" {

int cmb_nccl_unique_id(void* id_out) {
  CMB_TRY(need_nccl());
  ncclUniqueId id;
  CMB_NCCL(nccl_api()->getUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return CMB_OK;
}

int cmb_nccl_init_rank(int dev, const void* id, int nranks, int rank) {
  CMB_PARAM(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d of %d", rank, nranks);
  CMB_TRY(need_nccl());
  CMB_CTX(dev);
  (void)st;
  NcclApi* api = nccl_api();
  if (ctx->comm) {
    api->commDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  CMB_NCCL(api->commInitRank(&ctx->comm, nranks, uid, rank));
  ctx->nranks = nranks;
  ctx->rank = rank;
  return CMB_OK;
}

int cmb_nccl_info(int dev, int* nranks, int* rank, int* version) {
  CMB_TRY(need_nccl());
  CMB_CTX(dev);
  (void)st;
  CMB_PARAM(ctx->comm != nullptr, "device %d has no NCCL communicator", dev);
  CMB_NCCL(nccl_api()->commCount(ctx->comm, nranks));
  *rank = ctx->rank;
  CMB_NCCL(nccl_api()->getVersion(version));
  return CMB_OK;
}

int cmb_nccl_destroy(int dev) {
  CMB_CTX(dev);
  (void)st;
  if (ctx->comm) nccl_api()->commDestroy(ctx->comm);
  ctx->comm = nullptr;
  ctx->nranks = 1;
  ctx->rank = 0;
  return CMB_OK;
}

int cmb_xmap_rank(int dev, float* X_dev, int64_t N, int64_t len, const int32_t* estar, int tau, float* rho_dev,
                  void* stream, double* stats_out) {
  CMB_PARAM(N >= 1 && len >= 1, "empty dataset");
  CMB_TRY(need_nccl());
  CMB_CTX(dev);
  CMB_PARAM(ctx->comm != nullptr, "device %d has no NCCL communicator (cmb_nccl_init_rank)", dev);
  CMB_PARAM(ctx->rank != 0 || rho_dev != nullptr, "rank 0 needs the result buffer");
  cudaStream_t use = stream ? reinterpret_cast<cudaStream_t>(stream) : st;
  return xmap_rank_core(ctx, use, X_dev, N, len, estar, tau, rho_dev, stats_out);
}

int cmb_xmap_multi(const int* devs, int ndev, const float* X, int64_t N, int64_t len, const int32_t* estar,
                   int tau, float* rho_out, double* stats_out) {
  CMB_PARAM(ndev >= 1 && devs, "no devices");
  CMB_PARAM(N >= 1 && len >= 1, "empty dataset");
  CMB_TRY(need_nccl());
  NcclApi* api = nccl_api();
  std::vector<Ctx*> ctxs(ndev);
  for (int g = 0; g < ndev; ++g) CMB_TRY(get_ctx(devs[g], &ctxs[g]));
  std::vector<ncclComm_t> comms(ndev);
  CMB_NCCL(api->commInitAll(comms.data(), ndev, devs));
  std::vector<int> rc(ndev, CMB_OK);
  std::vector<std::string> msg(ndev);
  std::vector<double> st0(8, 0.0);
  // one host thread per device, each the rank body of a one-process-per-GPU job
  auto body = [&](int g) {
    Ctx* ctx = ctxs[g];
    std::lock_guard<std::mutex> lock(ctx->mu);
    int r = CMB_OK;
    do {
      if (cudaSetDevice(ctx->dev) != cudaSuccess) { r = cuda_fail(cudaGetLastError(), "cudaSetDevice", __FILE__, __LINE__); break; }
      ncclComm_t keep = ctx->comm;
      const int keep_n = ctx->nranks, keep_r = ctx->rank;
      ctx->comm = comms[g];
      ctx->nranks = ndev;
      ctx->rank = g;
      float* rho_full = nullptr;
      if (ctx->buf[B_X32].ensure(sizeof(float) * N * len + 256) != cudaSuccess ||
          (g == 0 && ctx->buf[B_RHO].ensure(sizeof(float) * (size_t)N * N) != cudaSuccess)) {
        set_error("out of device memory for the sharded cross map");
        r = CMB_ERR_CUDA;
      } else {
        if (g == 0) {
          rho_full = ctx->buf[B_RHO].as<float>();
          if (cudaMemcpyAsync(ctx->buf[B_X32].p, X, sizeof(float) * N * len, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
            r = cuda_fail(cudaGetLastError(), "H2D X", __FILE__, __LINE__);
        }
        if (r == CMB_OK)
          r = xmap_rank_core(ctx, ctx->stream, ctx->buf[B_X32].as<float>(), N, len, estar, tau, rho_full,
                             g == 0 ? st0.data() : nullptr);
        if (r == CMB_OK && g == 0 &&
            cudaMemcpy(rho_out, rho_full, sizeof(float) * (size_t)N * N, cudaMemcpyDeviceToHost) != cudaSuccess)
          r = cuda_fail(cudaGetLastError(), "D2H rho", __FILE__, __LINE__);
      }
      ctx->comm = keep;
      ctx->nranks = keep_n;
      ctx->rank = keep_r;
    } while (0);
    rc[g] = r;
    if (r) msg[g] = cmb_last_error();
  };
  std::vector<std::thread> th;
  for (int g = 0; g < ndev; ++g) th.emplace_back(body, g);
  for (auto& t : th) t.join();
  for (auto c : comms) api->commDestroy(c);
  for (int g = 0; g < ndev; ++g)
    if (rc[g]) {
      set_error("device %d: %s", devs[g], msg[g].c_str());
      return rc[g];
    }
  if (stats_out) memcpy(stats_out, st0.data(), 8 * sizeof(double));
  return CMB_OK;
}

int cmb_ccm_convergence(int dev, const double* X, int64_t N, int64_t len, int E, int tau,
                        const int32_t* lib_ids, const int32_t* tgt_ids, int64_t P,
                        const int32_t* sizes, int n_sizes, int samples, const int32_t* pts,
                        double* rho_out) {
  CMB_TRY(check_spec(E, tau));
  CMB_TRY(check_valid_count(len, E, tau));
  CMB_PARAM(N >= 1 && P >= 0 && n_sizes >= 0 && samples >= 1, "bad sweep shape");
  const int64_t n = len - (int64_t)(E - 1) * tau;
  const int k = E + 1;
  CMB_PARAM(k <= 31, "embedding dimension %d too large for the convergence sweep", E);
  int64_t total_pts = 0;
  std::vector<int64_t> size_off(n_sizes + 1, 0);
  for (int s = 0; s < n_sizes; ++s) {
    CMB_PARAM(sizes[s] >= E + 2 && sizes[s] <= n,
              "library size %d outside [%d, %lld] (k = E + 1 neighbours excluding the point itself)",
              sizes[s], E + 2, (long long)n);
    size_off[s] = total_pts;
    total_pts += (int64_t)sizes[s] * samples;
  }
  size_off[n_sizes] = total_pts;
  for (int64_t q = 0; q < total_pts; ++q)
    CMB_PARAM(pts[q] >= 0 && pts[q] < n, "library point %d outside [0, %lld)", pts[q], (long long)n);
  for (int64_t p = 0; p < P; ++p)
    CMB_PARAM(lib_ids[p] >= 0 && lib_ids[p] < N && tgt_ids[p] >= 0 && tgt_ids[p] < N, "bad pair %lld",
              (long long)p);
  if (P == 0 || n_sizes == 0) return CMB_OK;
  CMB_PARAM(len <= 65535, "series length %lld exceeds the 16-bit table format", (long long)len);
  CMB_CTX(dev);
  // distinct libraries and targets of the pair list
  std::vector<int32_t> libs, tgts;
  std::vector<int> lib_ix(N, -1), tgt_ix(N, -1);
  for (int64_t p = 0; p < P; ++p) {
    if (lib_ix[lib_ids[p]] < 0) { lib_ix[lib_ids[p]] = (int)libs.size(); libs.push_back(lib_ids[p]); }
    if (tgt_ix[tgt_ids[p]] < 0) { tgt_ix[tgt_ids[p]] = (int)tgts.size(); tgts.push_back(tgt_ids[p]); }
  }
  const int64_t NL = (int64_t)libs.size(), NT = (int64_t)tgts.size();
  const int64_t PL = NL * n_sizes * samples;  // pseudo-libraries (library, size, sample)
  // targets: one E group padded to 32-slot blocks, slot -> target row of the output chunk
  const int64_t slots = (NT + 31) / 32 * 32;
  std::vector<int32_t> slot_series(slots, -1), slot_row(slots, -1), slot_E(slots, 0);
  for (int64_t t = 0; t < NT; ++t) { slot_series[t] = tgts[t]; slot_row[t] = (int32_t)t; slot_E[t] = E; }
  // device staging: X (fp64 for the exact tables, fp32 for the targets), samples, targets
  CMB_CUDA(ctx->buf[B_X64].ensure(sizeof(double) * N * len));
  CMB_CUDA(ctx->buf[B_X32].ensure(sizeof(float) * N * len + 256));
  CMB_CUDA(ctx->buf[B_ERR].ensure(sizeof(float) * N));
  CMB_CUDA(ctx->buf[B_A].ensure(sizeof(int32_t) * total_pts + 16));
  CMB_CUDA(ctx->buf[B_B].ensure(sizeof(int64_t) * (n_sizes + 1) + sizeof(int32_t) * n_sizes + 16));
  CMB_CUDA(ctx->buf[B_LIBROWS].ensure(sizeof(int32_t) * NL));
  CMB_CUDA(ctx->buf[B_SLOT_TGT].ensure(4 * slots));
  CMB_CUDA(ctx->buf[B_SLOT_E].ensure(4 * slots));
  CMB_CUDA(ctx->buf[B_OBS_S].ensure(8 * slots));
  CMB_CUDA(ctx->buf[B_OBS_SS].ensure(8 * slots));
  CMB_CUDA(ctx->buf[B_OBS_C].ensure(slots));
  CMB_CUDA(ctx->buf[B_Y].ensure(sizeof(float) * len * slots));
  CMB_CUDA(ctx->buf[B_MEAN].ensure(8 * N));
  CMB_CUDA(ctx->buf[B_COUNTER].ensure(16));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_X64].p, X, sizeof(double) * N * len, cudaMemcpyHostToDevice, st));
  CMB_CUDA(launch_demote(ctx->buf[B_X64].as<double>(), N, len, ctx->buf[B_X32].as<float>(),
                         ctx->buf[B_ERR].as<float>(), st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_A].p, pts, sizeof(int32_t) * total_pts, cudaMemcpyHostToDevice, st));
  int64_t* d_size_off = ctx->buf[B_B].as<int64_t>();
  int32_t* d_sizes = reinterpret_cast<int32_t*>(d_size_off + n_sizes + 1);
  CMB_CUDA(cudaMemcpyAsync(d_size_off, size_off.data(), sizeof(int64_t) * (n_sizes + 1), cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(d_sizes, sizes, sizeof(int32_t) * n_sizes, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_LIBROWS].p, libs.data(), sizeof(int32_t) * NL, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_SLOT_TGT].p, slot_series.data(), 4 * slots, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_SLOT_E].p, slot_E.data(), 4 * slots, cudaMemcpyHostToDevice, st));
  const float* x32 = ctx->buf[B_X32].as<float>();
  CMB_CUDA(launch_series_stats(x32, N, len, len, ctx->buf[B_MEAN].as<double>(), st));
  CMB_CUDA(launch_build_targets(x32, len, ctx->buf[B_MEAN].as<double>(), ctx->buf[B_SLOT_TGT].as<int32_t>(),
                                slots, (int)len, ctx->buf[B_Y].as<float>(), slots, st));
  CMB_CUDA(launch_obs_moments(ctx->buf[B_Y].as<float>(), slots, (int)len, tau, ctx->buf[B_SLOT_E].as<int32_t>(),
                              slots, ctx->buf[B_OBS_S].as<double>(), ctx->buf[B_OBS_SS].as<double>(),
                              ctx->buf[B_OBS_C].as<uint8_t>(), st));
  // the lookup writes rho_T[row][column]: slot rows are output rows
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_SLOT_TGT].p, slot_row.data(), 4 * slots, cudaMemcpyHostToDevice, st));
  // chunks of pseudo-libraries: tables (<= ~4 GB) and their rho_T columns
  const size_t stride = rec_lib_stride(k, n);
  const int LS = 4 * kLookupWarps;  // four libraries per warp per work item
  int64_t C = std::max<int64_t>(LS, (int64_t)(((size_t)4 << 30) / stride) / LS * LS);
  C = std::min<int64_t>(C, (PL + LS - 1) / LS * LS);
  const int64_t ldr = (C + 3) / 4 * 4;
  CMB_CUDA(ctx->buf[B_TAB].ensure(stride * C + 256));
  CMB_CUDA(ctx->buf[B_RHOT].ensure(sizeof(float) * slots * ldr));
  CMB_CUDA(ctx->buf[B_LIBCOL].ensure(sizeof(int64_t) * C));
  std::vector<int64_t> cols(C);
  for (int64_t c = 0; c < C; ++c) cols[c] = c;
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_LIBCOL].p, cols.data(), sizeof(int64_t) * C, cudaMemcpyHostToDevice, st));
  const int stage = lookup_stage_bytes((int)len, rec_bytes(k));
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->dev);
  // requested pairs by library index, for the scatter
  std::vector<std::vector<std::pair<int64_t, int>>> by_lib(NL);
  for (int64_t p = 0; p < P; ++p) by_lib[lib_ix[lib_ids[p]]].push_back({p, tgt_ix[tgt_ids[p]]});
  std::vector<float> chunk_rho;
  for (int64_t c0 = 0; c0 < PL; c0 += C) {
    const int64_t nc = std::min<int64_t>(C, PL - c0);
    CMB_CUDA(launch_fill_nan(ctx->buf[B_RHOT].as<float>(), slots, nc, ldr, st));
    CMB_CUDA(launch_restricted_records(ctx->buf[B_X64].as<double>(), len, ctx->buf[B_LIBROWS].as<int32_t>(),
                                       (int)n, E, tau, ctx->buf[B_A].as<int32_t>(), d_size_off, d_sizes,
                                       n_sizes, samples, c0, nc, ctx->buf[B_TAB].as<uint8_t>(), st));
    LookupArgs la;
    memset(&la, 0, sizeof(la));
    la.Y = ctx->buf[B_Y].as<float>();
    la.ldy = slots;
    la.T = (int)len;
    la.tau = tau;
    la.ngroups = 1;
    la.g_E[0] = E;
    la.g_blk0[0] = 0;
    la.g_nblk[0] = (int)(slots / 32);
    la.slot_tgt = ctx->buf[B_SLOT_TGT].as<int32_t>();
    la.obs_s = ctx->buf[B_OBS_S].as<double>();
    la.obs_ss = ctx->buf[B_OBS_SS].as<double>();
    la.obs_const = ctx->buf[B_OBS_C].as<uint8_t>();
    la.tab[E] = ctx->buf[B_TAB].as<uint8_t>();
    la.nlib = (int)nc;
    la.lib_col = ctx->buf[B_LIBCOL].as<int64_t>();
    la.LS = LS;
    la.n_lsub = (int)((nc + LS - 1) / LS);
    la.g_item0[0] = 0;
    la.n_items = (int64_t)la.n_lsub * la.g_nblk[0];
    la.g_item0[1] = la.n_items;
    la.counter = ctx->buf[B_COUNTER].as<int>();
    la.rhoT = ctx->buf[B_RHOT].as<float>();
    la.ldr = ldr;
    la.stage_bytes = stage;
    la.tmajor = 1;
    CMB_CUDA(cudaMemsetAsync(la.counter, 0, sizeof(int), st));
    CMB_CUDA(launch_lookup_xmap(la, (int)std::min<int64_t>(la.n_items, dev_sms), st));
    chunk_rho.resize((size_t)NT * ldr);
    CMB_CUDA(cudaMemcpy2DAsync(chunk_rho.data(), sizeof(float) * ldr, ctx->buf[B_RHOT].p, sizeof(float) * ldr,
                               sizeof(float) * nc, NT, cudaMemcpyDeviceToHost, st));
    CMB_CUDA(cudaStreamSynchronize(st));
    // scatter: pseudo-library pl = (li * n_sizes + s) * samples + q
    const int64_t ls0 = c0 / samples, ls1 = (c0 + nc + samples - 1) / samples;
    for (int64_t ls = ls0; ls < ls1; ++ls) {
      const int64_t li = ls / n_sizes;
      const int s = (int)(ls % n_sizes);
      for (const auto& pr : by_lib[li])
        for (int q = 0; q < samples; ++q) {
          const int64_t pl = ls * samples + q;
          if (pl < c0 || pl >= c0 + nc) continue;
          const float v = chunk_rho[(size_t)pr.second * ldr + (pl - c0)];
          rho_out[((size_t)pr.first * n_sizes + s) * samples + q] = (double)v;
        }
    }
  }
  return CMB_OK;
}

// ---------------------------------------------------------------- data formats
int cmb_format_skill_csv(int dev, const void* rho, int rho_on_device, int is_f32, int64_t n,
                         int64_t ld, int64_t row0, int64_t nrows, const char* names,
                         const int64_t* name_off, char* out, int64_t out_cap, int64_t* out_len) {
  CMB_PARAM(n >= 1 && ld >= n && row0 >= 0 && nrows >= 0 && row0 + nrows <= n, "bad skill-matrix block");
  CMB_PARAM(rho && names && name_off && out && out_len, "null buffer");
  CMB_CTX(dev);
  const size_t esz = is_f32 ? 4 : 8;
  const void* src = rho;
  if (!rho_on_device && nrows > 0) {
    CMB_CUDA(ctx->buf[B_FMT_RHO].ensure(esz * nrows * ld));
    CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_FMT_RHO].p, rho, esz * ((nrows - 1) * ld + n), cudaMemcpyHostToDevice, st));
    src = ctx->buf[B_FMT_RHO].p;
  }
  const int64_t nbytes = name_off[n];
  CMB_CUDA(ctx->buf[B_FMT_NAMES].ensure(nbytes + 1));
  CMB_CUDA(ctx->buf[B_FMT_OFF].ensure(8 * (n + 1)));
  CMB_CUDA(ctx->buf[B_FMT_LEN].ensure(8 * (nrows + 1) + 8));
  CMB_CUDA(ctx->buf[B_FMT_ROWOFF].ensure(8 * (nrows + 1)));
  CMB_CUDA(ctx->buf[B_FMT_OUT].ensure(out_cap + 1));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_FMT_NAMES].p, names, nbytes, cudaMemcpyHostToDevice, st));
  CMB_CUDA(cudaMemcpyAsync(ctx->buf[B_FMT_OFF].p, name_off, 8 * (n + 1), cudaMemcpyHostToDevice, st));
  std::vector<int64_t> row_off(nrows + 1);
  bool oor = false;
  int64_t len = 0;
  int64_t* lens = ctx->buf[B_FMT_LEN].as<int64_t>();
  CMB_CUDA(format_skill_rows(src, is_f32 != 0, n, ld, row0, nrows, ctx->buf[B_FMT_NAMES].as<char>(),
                             ctx->buf[B_FMT_OFF].as<int64_t>(), lens, ctx->buf[B_FMT_ROWOFF].as<int64_t>(),
                             row_off.data(), reinterpret_cast<int*>(lens + nrows + 1), &oor,
                             ctx->buf[B_FMT_OUT].as<char>(), out_cap, &len, st));
  CMB_PARAM(!oor, "skill value outside the formatter's range (|v| >= 1e9)");
  CMB_PARAM(len <= out_cap, "text of %lld bytes exceeds the %lld-byte buffer", (long long)len, (long long)out_cap);
  CMB_CUDA(cudaMemcpyAsync(out, ctx->buf[B_FMT_OUT].p, len, cudaMemcpyDeviceToHost, st));
  CMB_CUDA(cudaStreamSynchronize(st));
  *out_len = len;
  return CMB_OK;
}

int cmb_csv_header(const char* buf, int64_t len, char* text, int64_t text_cap, int64_t* spans, int64_t max_cells,
                   int64_t* ncells, int64_t* body_off) {
  if (!buf || len < 0 || !text || !spans || !ncells || !body_off) return CSV_CAPACITY;
  return csv_header(buf, len, text, text_cap, spans, max_cells, ncells, body_off);
}

int cmb_csv_body(const char* buf, int64_t len, int mode, int64_t ncols, double* out, int64_t cap_rows,
                 int64_t* nrows, char* labels, int64_t labels_cap, int64_t* label_spans, int64_t* defer,
                 int64_t defer_cap, char* defer_text, int64_t defer_text_cap, int64_t* ndefer, char* err_text,
                 int64_t err_cap, int64_t* err) {
  if (!buf || len < 0 || (mode != 0 && mode != 1) || ncols < (mode == 1 ? 1 : 0) || !out || !nrows || !ndefer || !err ||
      (mode == 1 && (!labels || !label_spans)))
    return CSV_CAPACITY;
  return csv_body(buf, len, mode, ncols, out, cap_rows, nrows, labels, labels_cap, label_spans, defer, defer_cap,
                  defer_text, defer_text_cap, ndefer, err_text, err_cap, err);
}

}  // extern "C"
