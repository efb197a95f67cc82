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

#include <cmath>
#include <cstdlib>
#include <string>

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

// ---------------------------------------------------------------- host CSV reading
// The input grammar of the reference's readers (pkg/src/crossmap/io.py:25-61,
// 81-110): Python's csv module, excel dialect, non-strict -- records end at
// \n, \r\n or \r outside quotes (a blank line is a record with no cells); a
// field that starts with '"' is quoted, '""' inside it is one '"', newlines are
// kept, characters after the closing quote are appended; a quoted field left
// open at the end of the data ends there -- and Python's float() on each cell:
// ASCII blanks stripped, optional sign, digits with single '_' between
// digits, optional fraction and exponent, or inf / infinity / nan (any case).
// Values are correctly rounded (std::from_chars, strtod for out-of-range
// exponents), so they are bit-identical to float().  Cells with non-ASCII
// bytes (Unicode digits or blanks, which float() also accepts) are listed for
// the caller to convert with float() itself.
namespace {

constexpr int64_t kFieldLimit = 131072;  // csv.field_size_limit() default

struct CsvCursor {
  const char* b;
  int64_t n, pos = 0;
  // fields of the current record: unquoted ones point into the data (off into
  // b), quoted ones into `text` (their unescaped copy)
  struct Span {
    int64_t off, len;
    bool quoted;
  };
  std::vector<Span> spans;
  std::string text;
  bool oversize = false;
  CsvCursor(const char* buf, int64_t len) : b(buf), n(len) {}

  const char* fptr(size_t c) const { return spans[c].quoted ? text.data() + spans[c].off : b + spans[c].off; }
  int64_t flen(size_t c) const { return spans[c].len; }

  // next record into spans/text; false at the end of the data
  bool next() {
    spans.clear();
    text.clear();
    if (pos >= n) return false;
    // a line break at the start of a record: a record without cells
    if (b[pos] == '\n' || b[pos] == '\r') {
      pos += (b[pos] == '\r' && pos + 1 < n && b[pos + 1] == '\n') ? 2 : 1;
      return true;
    }
    for (;;) {
      // one field starting at pos
      if (pos < n && b[pos] == '"') {
        // quoted: '""' is one '"', line breaks kept, text after the closing
        // quote appended up to the delimiter (non-strict)
        const int64_t off = (int64_t)text.size();
        ++pos;
        bool in_quotes = true;
        while (pos < n) {
          const char c = b[pos];
          if (in_quotes) {
            if (c == '"') {
              if (pos + 1 < n && b[pos + 1] == '"') { text.push_back('"'); pos += 2; continue; }
              in_quotes = false;
              ++pos;
              continue;
            }
            text.push_back(c);
            ++pos;
          } else {
            if (c == ',' || c == '\n' || c == '\r') break;
            text.push_back(c);
            ++pos;
          }
        }
        spans.push_back({off, (int64_t)text.size() - off, true});
      } else {
        int64_t e = pos;
        while (e < n && b[e] != ',' && b[e] != '\n' && b[e] != '\r') ++e;
        spans.push_back({pos, e - pos, false});
        pos = e;
      }
      if (spans.back().len > kFieldLimit) oversize = true;
      if (pos >= n) return true;  // end of data (an open quoted field ends here)
      if (b[pos] == ',') {
        ++pos;
        if (pos >= n) {  // a trailing delimiter: one more, empty field
          spans.push_back({pos, 0, false});
          return true;
        }
        continue;
      }
      pos += (b[pos] == '\r' && pos + 1 < n && b[pos + 1] == '\n') ? 2 : 1;
      return true;
    }
  }
};

bool ascii_blank(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// float(cell) for an ASCII cell: 0 ok, 1 not a number
int py_float(const char* s, int64_t len, double* v) {
  int64_t a = 0, e = len;
  while (a < e && ascii_blank(s[a])) ++a;
  while (e > a && ascii_blank(s[e - 1])) --e;
  if (a == e) return 1;
  bool neg = false;
  if (s[a] == '+' || s[a] == '-') { neg = s[a] == '-'; ++a; }
  const int64_t m = e - a;
  auto ieq = [&](const char* w) {
    const int64_t k = (int64_t)strlen(w);
    if (k != m) return false;
    for (int64_t q = 0; q < k; ++q)
      if ((s[a + q] | 0x20) != w[q]) return false;
    return true;
  };
  if (ieq("inf") || ieq("infinity")) { *v = neg ? -HUGE_VAL : HUGE_VAL; return 0; }
  if (ieq("nan")) { *v = neg ? -__builtin_nan("") : __builtin_nan(""); return 0; }
  // common case: no '_' separator -- std::from_chars straight on the text
  // (it takes exactly float()'s decimal forms once the sign is removed)
  if ((s[a] >= '0' && s[a] <= '9') || s[a] == '.') {
    bool under = false;
    for (int64_t q = a; q < e && !under; ++q) under = s[q] == '_';
    if (!under) {
      double r = 0.0;
      auto res = std::from_chars(s + a, s + e, r);
      if (res.ptr != s + e) return 1;
      if (res.ec == std::errc::result_out_of_range) {
        std::string t(s + a, (size_t)(e - a));
        r = strtod(t.c_str(), nullptr);
      } else if (res.ec != std::errc()) {
        return 1;
      }
      *v = neg ? -r : r;
      return 0;
    }
  }
  // digits ('_' only between two digits), '.', exponent
  char tmp[512];
  std::string big;
  char* d = tmp;
  if (m + 2 > (int64_t)sizeof(tmp)) { big.resize(m + 2); d = &big[0]; }
  int64_t o = 0, mant = 0;
  bool dot = false, exp = false, exp_digits = false;
  for (int64_t q = a; q < e; ++q) {
    const char c = s[q];
    if (c >= '0' && c <= '9') {
      d[o++] = c;
      if (exp) exp_digits = true; else ++mant;
    } else if (c == '_') {
      if (q == a || q + 1 >= e || !(s[q - 1] >= '0' && s[q - 1] <= '9') || !(s[q + 1] >= '0' && s[q + 1] <= '9'))
        return 1;
    } else if (c == '.' && !dot && !exp) {
      dot = true;
      d[o++] = c;
    } else if ((c == 'e' || c == 'E') && !exp && mant > 0) {
      exp = true;
      d[o++] = 'e';
      if (q + 1 < e && (s[q + 1] == '+' || s[q + 1] == '-')) d[o++] = s[++q];
    } else {
      return 1;
    }
  }
  if (mant == 0 || (exp && !exp_digits)) return 1;
  double r = 0.0;
  auto res = std::from_chars(d, d + o, r);
  if (res.ptr != d + o) return 1;
  if (res.ec == std::errc::result_out_of_range) {  // overflow -> inf, underflow -> 0 / subnormal
    d[o] = '\0';
    r = strtod(d, nullptr);
  } else if (res.ec != std::errc()) {
    return 1;
  }
  *v = neg ? -r : r;
  return 0;
}

bool has_high_byte(const char* s, int64_t len) {
  for (int64_t q = 0; q < len; ++q)
    if ((unsigned char)s[q] >= 0x80) return true;
  return false;
}

}  // namespace

int csv_header(const char* buf, int64_t len, char* text, int64_t text_cap, int64_t* spans, int64_t max_cells,
               int64_t* ncells, int64_t* body_off) {
  CsvCursor cur(buf, len);
  if (!cur.next()) return CSV_EMPTY;
  if (cur.oversize) return CSV_FIELD_LIMIT;
  int64_t tot = 0;
  for (size_t q = 0; q < cur.spans.size(); ++q) tot += cur.flen(q);
  if ((int64_t)cur.spans.size() > max_cells || tot > text_cap) return CSV_CAPACITY;
  int64_t o = 0;
  for (size_t q = 0; q < cur.spans.size(); ++q) {
    memcpy(text + o, cur.fptr(q), (size_t)cur.flen(q));
    spans[2 * q] = o;
    spans[2 * q + 1] = cur.flen(q);
    o += cur.flen(q);
  }
  *ncells = (int64_t)cur.spans.size();
  *body_off = cur.pos;
  return 0;
}

int csv_body(const char* buf, int64_t len, int mode, int64_t ncols, double* out, int64_t cap_rows, int64_t* nrows,
             char* labels, int64_t labels_cap, int64_t* label_spans, int64_t* defer, int64_t defer_cap,
             char* defer_text, int64_t defer_text_cap, int64_t* ndefer, char* err_text, int64_t err_cap,
             int64_t* err) {
  CsvCursor cur(buf, len);
  const int64_t want = ncols + (mode == 1 ? 1 : 0);
  int64_t row = 0, lab = 0, nd = 0, dtext = 0;
  auto fail = [&](int code, int64_t col, const char* t, int64_t tl, int64_t ncell) {
    err[0] = code;
    err[1] = row;
    err[2] = col;
    err[3] = ncell;
    err[4] = std::min(tl, err_cap);
    if (t) memcpy(err_text, t, (size_t)err[4]);
    *nrows = row;
    *ndefer = nd;
    return code;
  };
  while (cur.next()) {
    if (cur.oversize) return fail(CSV_FIELD_LIMIT, 0, nullptr, 0, 0);
    const int64_t nc = (int64_t)cur.spans.size();
    if (nc != want) return fail(CSV_WIDTH, 0, nullptr, 0, nc);
    if (mode == 1 && row < cap_rows) {  // rows past the matrix only count (then a row-name mismatch)
      const int64_t ll = cur.flen(0);
      if (lab + ll > labels_cap) return fail(CSV_CAPACITY, 0, nullptr, 0, 0);
      memcpy(labels + lab, cur.fptr(0), (size_t)ll);
      label_spans[2 * row] = lab;
      label_spans[2 * row + 1] = ll;
      lab += ll;
    }
    for (int64_t c = (mode == 1 ? 1 : 0); c < nc; ++c) {
      const int64_t col = mode == 1 ? c - 1 : c;
      const char* f = cur.fptr((size_t)c);
      const int64_t fl = cur.flen((size_t)c);
      double v;
      if (mode == 1 && fl == 2 && f[0] == 'N' && f[1] == 'A') {
        if (row < cap_rows) out[row * ncols + col] = __builtin_nan("");
        continue;
      } else if (has_high_byte(f, fl)) {
        // float() also takes Unicode digits and blanks: the caller converts
        if (nd >= defer_cap) return fail(CSV_CAPACITY, col, nullptr, 0, 0);
        if (row >= cap_rows) return fail(mode == 1 ? CSV_BAD_CELL : CSV_CAPACITY, col, f, fl, 0);
        if (dtext + fl > defer_text_cap) return fail(CSV_CAPACITY, col, nullptr, 0, 0);
        memcpy(defer_text + dtext, f, (size_t)fl);
        defer[4 * nd] = row;
        defer[4 * nd + 1] = col;
        defer[4 * nd + 2] = dtext;
        defer[4 * nd + 3] = fl;
        dtext += fl;
        ++nd;
        out[row * ncols + col] = __builtin_nan("");
        continue;
      } else if (py_float(f, fl, &v) != 0) {
        return fail(mode == 1 ? CSV_BAD_CELL : CSV_NOT_NUMERIC, col, f, fl, 0);
      } else if (mode == 0 && !std::isfinite(v)) {
        return fail(CSV_NON_FINITE, col, f, fl, 0);
      }
      // read_skill_matrix: a value past the n x n matrix is the reference's IndexError -> bad cell
      if (row >= cap_rows) return fail(mode == 1 ? CSV_BAD_CELL : CSV_CAPACITY, col, f, fl, 0);
      out[row * ncols + col] = v;
    }
    ++row;
  }
  *nrows = row;
  *ndefer = nd;
  err[0] = 0;
  return 0;
}

}  // namespace cmb
