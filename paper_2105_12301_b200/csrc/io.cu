// Data formats either side of the cross-map path:
//
//   * skill-matrix CSV text on the GPU -- write_skill_matrix (reference
//     pkg/src/crossmap/io.py:70-78): one row per library, "name,c0,c1,...\r\n"
//     with each cell f"{v:.6f}" of the float64 value, or "NA" when it is not
//     finite.  Rows are formatted where rho lives (device buffers from the
//     cross map, or host arrays staged in batches) and only text leaves the GPU.
//   * numeric CSV parsing on the host -- load_csv / read_skill_matrix
//     (io.py:25-61, 81-110): std::from_chars is correctly rounded like Python's
//     float(); the Python layer keeps the reference's validation and messages
//     and falls back to the csv module for anything this grammar does not cover
//     (quotes, '_' digit separators).
//
// Exactness of the formatter: |v| = m 2^e exactly (m < 2^53); the printed
// integer N = round_half_even(|v| 10^6) is computed in 128-bit integer
// arithmetic from m 10^6 (< 2^73), so the text equals CPython's correctly
// rounded "%.6f" (including "-0.000000" for negative values that round to 0).
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <charconv>
#include <cstring>
#include <vector>

namespace cmb {

namespace {

constexpr double kFmtMax = 1e9;  // device formatting range; larger values take the host path

__device__ __forceinline__ unsigned long long round6(double a) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
  const int ex = (int)((bits >> 52) & 0x7ff);
  const unsigned long long mant = bits & ((1ull << 52) - 1);
  unsigned long long m;
  int e;
  if (ex == 0) { m = mant; e = -1074; } else { m = mant | (1ull << 52); e = ex - 1075; }
  const unsigned __int128 P = (unsigned __int128)m * 1000000u;
  if (e >= 0) return (unsigned long long)(P << e);  // a < 1e9: no overflow
  const int q = -e;
  if (q >= 128) return 0ull;  // P < 2^73
  const unsigned __int128 N = P >> q;
  const unsigned __int128 rem = P - (N << q);
  const unsigned __int128 half = (unsigned __int128)1 << (q - 1);
  unsigned long long n = (unsigned long long)N;
  if (rem > half || (rem == half && (n & 1ull))) ++n;
  return n;
}

__device__ __forceinline__ int n_digits(unsigned long long v) {
  int d = 1;
  while (v >= 10ull) { v /= 10ull; ++d; }
  return d;
}

// length of the cell text (without separator)
__device__ __forceinline__ int cell_len(double v) {
  if (!isfinite(v)) return 2;
  const unsigned long long n = round6(fabs(v));
  return (signbit(v) ? 1 : 0) + n_digits(n / 1000000ull) + 7;
}

__device__ __forceinline__ int cell_write(double v, char* o) {
  if (!isfinite(v)) { o[0] = 'N'; o[1] = 'A'; return 2; }
  int p = 0;
  if (signbit(v)) o[p++] = '-';
  const unsigned long long n = round6(fabs(v));
  unsigned long long ip = n / 1000000ull;
  unsigned frac = (unsigned)(n - ip * 1000000ull);
  const int nd = n_digits(ip);
  for (int q = nd - 1; q >= 0; --q) { o[p + q] = (char)('0' + (int)(ip % 10ull)); ip /= 10ull; }
  p += nd;
  o[p++] = '.';
  for (int q = 5; q >= 0; --q) { o[p + q] = (char)('0' + (int)(frac % 10u)); frac /= 10u; }
  return p + 6;
}

template <typename F>
__device__ __forceinline__ double cell_value(const F* row, int64_t c) { return (double)row[c]; }

// Per row: bytes of "name,c0,...,c_{n-1}\r\n".
template <typename F>
__global__ void row_len_kernel(const F* __restrict__ rho, int64_t n, int64_t ld,
                               const int64_t* __restrict__ name_off, int64_t row0,
                               int64_t* __restrict__ row_len, int* __restrict__ range_err) {
  const int64_t r = blockIdx.x;
  const F* row = rho + r * ld;
  long long s = 0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
    const double v = cell_value(row, c);
    if (isfinite(v) && fabs(v) >= kFmtMax) *range_err = 1;
    s += 1 + cell_len(v);
  }
  __shared__ long long part[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(CMB_FULL, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += part[q];
    row_len[r] = t + (name_off[row0 + r + 1] - name_off[row0 + r]) + 2;
  }
}

// Per row: the text at out + row_off[r]; each thread formats a contiguous
// range of cells at its block-scanned offset.
template <typename F>
__global__ void row_write_kernel(const F* __restrict__ rho, int64_t n, int64_t ld,
                                 const char* __restrict__ names, const int64_t* __restrict__ name_off,
                                 int64_t row0, const int64_t* __restrict__ row_off, char* __restrict__ out) {
  const int64_t r = blockIdx.x;
  const F* row = rho + r * ld;
  char* o = out + row_off[r];
  const int64_t nb = name_off[row0 + r], ne = name_off[row0 + r + 1];
  for (int64_t q = threadIdx.x; q < ne - nb; q += blockDim.x) o[q] = names[nb + q];
  o += ne - nb;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = min(n, (int64_t)threadIdx.x * per), c1 = min(n, c0 + per);
  long long len = 0;
  for (int64_t c = c0; c < c1; ++c) len += 1 + cell_len(cell_value(row, c));
  // block exclusive scan of len
  __shared__ long long wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl = len;
  for (int d = 1; d < 32; d <<= 1) {
    const long long u = __shfl_up_sync(CMB_FULL, incl, d);
    if (lane >= d) incl += u;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    long long v = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0;
    for (int d = 1; d < 32; d <<= 1) {
      const long long u = __shfl_up_sync(CMB_FULL, v, d);
      if (lane >= d) v += u;
    }
    if (lane < (int)(blockDim.x >> 5)) wsum[lane] = v;
  }
  __syncthreads();
  const long long before = (wid > 0 ? wsum[wid - 1] : 0) + incl - len;
  char* p = o + before;
  for (int64_t c = c0; c < c1; ++c) {
    *p++ = ',';
    p += cell_write(cell_value(row, c), p);
  }
  if (threadIdx.x == blockDim.x - 1) {
    char* end = o + wsum[(blockDim.x >> 5) - 1];
    end[0] = '\r';
    end[1] = '\n';
  }
}

}  // namespace

// Format rows [row0, row0 + nrows) of an n x n skill matrix (row-major, leading
// dimension ld, float64 or float32, on the device) into out_dev; row byte
// offsets (exclusive, nrows + 1 entries) into row_off_host.
cudaError_t format_skill_rows(const void* rho_dev, bool f32, int64_t n, int64_t ld, int64_t row0,
                              int64_t nrows, const char* names_dev, const int64_t* name_off_dev,
                              int64_t* row_len_dev, int64_t* row_off_dev, int64_t* row_off_host,
                              int* range_err_dev, bool* out_of_range, char* out_dev, int64_t out_cap,
                              int64_t* out_len, cudaStream_t st) {
  *out_of_range = false;
  if (nrows == 0) { *out_len = 0; row_off_host[0] = 0; return cudaSuccess; }
  cudaError_t e = cudaMemsetAsync(range_err_dev, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  count_launch();
  if (f32)
    row_len_kernel<float><<<(unsigned)nrows, 256, 0, st>>>((const float*)rho_dev, n, ld, name_off_dev, row0, row_len_dev, range_err_dev);
  else
    row_len_kernel<double><<<(unsigned)nrows, 256, 0, st>>>((const double*)rho_dev, n, ld, name_off_dev, row0, row_len_dev, range_err_dev);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  std::vector<int64_t> len(nrows);
  int rerr = 0;
  e = cudaMemcpyAsync(len.data(), row_len_dev, sizeof(int64_t) * nrows, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(&rerr, range_err_dev, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  if (rerr) { *out_of_range = true; return cudaSuccess; }
  row_off_host[0] = 0;
  for (int64_t r = 0; r < nrows; ++r) row_off_host[r + 1] = row_off_host[r] + len[r];
  *out_len = row_off_host[nrows];
  if (*out_len > out_cap) return cudaSuccess;  // caller reports the overflow
  e = cudaMemcpyAsync(row_off_dev, row_off_host, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  count_launch();
  if (f32)
    row_write_kernel<float><<<(unsigned)nrows, 256, 0, st>>>((const float*)rho_dev, n, ld, names_dev, name_off_dev, row0, row_off_dev, out_dev);
  else
    row_write_kernel<double><<<(unsigned)nrows, 256, 0, st>>>((const double*)rho_dev, n, ld, names_dev, name_off_dev, row0, row_off_dev, out_dev);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- host CSV parsing
// Fast path for the numeric body of a CSV (the lines after the header).  A cell
// is optional blanks, an optional '+', a number std::from_chars accepts
// (correctly rounded, like Python's float), optional blanks -- or exactly "NA"
// when allow_na.  label_col: the first cell of each row is a label whose byte
// span goes to labels[2 r], labels[2 r + 1].  check_finite rejects inf/nan.
// Returns 0 with *nrows rows parsed, or 1 for anything else (ragged or blank
// rows, non-numeric cells, quotes, '_' digit separators, more than cap_rows
// rows): the caller then runs the reference algorithm, which raises the
// reference's exact error for invalid files.
int parse_numeric_csv(const char* buf, int64_t len, int64_t ncols, int label_col, int allow_na,
                      int check_finite, double* out, int64_t cap_rows, int64_t* nrows, int64_t* labels) {
  int64_t pos = 0, row = 0;
  const int64_t want = ncols + (label_col ? 1 : 0);
  while (pos < len) {
    int64_t eol = pos;
    while (eol < len && buf[eol] != '\n') ++eol;
    int64_t end = eol;
    if (end > pos && buf[end - 1] == '\r') --end;
    if (eol >= len && end == pos) break;  // no bytes after the last newline
    if (end == pos || row >= cap_rows) return 1;
    if (memchr(buf + pos, '"', (size_t)(end - pos)) || memchr(buf + pos, '_', (size_t)(end - pos)) ||
        memchr(buf + pos, '\r', (size_t)(end - pos)) || memchr(buf + pos, '(', (size_t)(end - pos)))
      return 1;
    int64_t c = pos, col = 0;
    for (;;) {
      int64_t ce = c;
      while (ce < end && buf[ce] != ',') ++ce;
      if (col >= want) return 1;
      if (label_col && col == 0) {
        labels[2 * row] = c;
        labels[2 * row + 1] = ce - c;
      } else {
        int64_t a = c, b = ce;
        while (a < b && (buf[a] == ' ' || buf[a] == '\t')) ++a;
        while (b > a && (buf[b - 1] == ' ' || buf[b - 1] == '\t')) --b;
        double v;
        if (allow_na && ce - c == 2 && buf[c] == 'N' && buf[c + 1] == 'A') {
          v = __builtin_nan("");
        } else {
          if (a < b && buf[a] == '+') ++a;
          if (a >= b || buf[a] == '+' || buf[a] == '-' && a > c && buf[a - 1] == '+') return 1;
          auto r = std::from_chars(buf + a, buf + b, v);
          if (r.ec != std::errc() || r.ptr != buf + b) return 1;
          if (check_finite && !__builtin_isfinite(v)) return 1;
        }
        out[row * ncols + (label_col ? col - 1 : col)] = v;
      }
      ++col;
      if (ce >= end) break;
      c = ce + 1;
    }
    if (col != want) return 1;
    ++row;
    pos = eol + 1;
  }
  *nrows = row;
  return 0;
}

}  // namespace cmb
