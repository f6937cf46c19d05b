// Result serialization (reference: dataset.py:34-36, :303-341; SURVEY.md 8f
// row f3) -- host code.
//
// The reference writes every matrix element as repr(float(x)), the shortest
// decimal string that round-trips to the same float64, one Python call per
// element (cfg3: 537 M values).  Here the digits come from std::to_chars
// (shortest round-trip, nearest; libstdc++'s Ryu) and are laid out with
// CPython's repr rules (float_repr_style 'short', mode 'r'): decimal point
// position decpt = exponent + 1; fixed notation when -4 < decpt <= 16 (".0"
// appended to integral values), otherwise d[.ddd]e{+,-}XX with at least two
// exponent digits; "inf", "-inf", "nan" for non-finite values.  Rows are
// formatted by several host threads into one caller buffer.
#include "common.cuh"

#include <charconv>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace corr2d {

// repr(float(x)) into p (at most 32 bytes); returns the length
static int repr_double(double x, char* p) {
  if (std::isnan(x)) { memcpy(p, "nan", 3); return 3; }
  if (std::isinf(x)) {
    if (x < 0) { memcpy(p, "-inf", 4); return 4; }
    memcpy(p, "inf", 3);
    return 3;
  }
  char buf[40];
  auto res = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
  const char* s = buf;
  const char* end = res.ptr;
  int n = 0;
  if (*s == '-') { p[n++] = '-'; ++s; }
  // s: d[.ddd]e(+|-)XX
  char dig[24];
  int nd = 0;
  const char* q = s;
  for (; q < end && *q != 'e'; ++q)
    if (*q != '.') dig[nd++] = *q;
  int exp10 = 0;
  std::from_chars(q + 1 + (q[1] == '+' ? 1 : 0), end, exp10);
  const int decpt = exp10 + 1;
  if (nd == 1 && dig[0] == '0') {  // +-0.0
    memcpy(p + n, "0.0", 3);
    return n + 3;
  }
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {              // 0.000ddd
      p[n++] = '0';
      p[n++] = '.';
      for (int i = 0; i < -decpt; ++i) p[n++] = '0';
      for (int i = 0; i < nd; ++i) p[n++] = dig[i];
    } else if (decpt >= nd) {      // ddd000.0
      for (int i = 0; i < nd; ++i) p[n++] = dig[i];
      for (int i = nd; i < decpt; ++i) p[n++] = '0';
      p[n++] = '.';
      p[n++] = '0';
    } else {                       // dd.ddd
      for (int i = 0; i < decpt; ++i) p[n++] = dig[i];
      p[n++] = '.';
      for (int i = decpt; i < nd; ++i) p[n++] = dig[i];
    }
    return n;
  }
  p[n++] = dig[0];
  if (nd > 1) {
    p[n++] = '.';
    for (int i = 1; i < nd; ++i) p[n++] = dig[i];
  }
  p[n++] = 'e';
  int e = decpt - 1;
  p[n++] = e < 0 ? '-' : '+';
  if (e < 0) e = -e;
  char eb[8];
  int ne = 0;
  do { eb[ne++] = (char)('0' + e % 10); e /= 10; } while (e);
  if (ne < 2) eb[ne++] = '0';
  while (ne) p[n++] = eb[--ne];
  return n;
}

static inline double elem(const void* m, int dtype, long long idx) {
  return dtype == CORR2D_F32 ? (double)static_cast<const float*>(m)[idx] : static_cast<const double*>(m)[idx];
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int corr2d_format_repr(const double* x, int64_t n, char* out, int64_t cap, int64_t* offsets) {
  // repr(float(x[i])) for a vector, concatenated; offsets[i + 1] = end of item i
  if ((n > 0 && (!x || !out || !offsets)) || n < 0) return fail(CORR2D_ERR_DATA, "corr2d_format_repr: bad arguments");
  int64_t pos = 0;
  offsets[0] = 0;
  char tmp[40];
  for (int64_t i = 0; i < n; ++i) {
    const int k = repr_double(x[i], tmp);
    if (pos + k > cap) return fail(CORR2D_ERR_DATA, "corr2d_format_repr: buffer too small");
    memcpy(out + pos, tmp, k);
    pos += k;
    offsets[i + 1] = pos;
  }
  return CORR2D_OK;
}

// Matrix-pair table rows [r0, r1) (dataset.py:303-309): each line is
// repr(axis1[i]) then repr(matrix[i, k]) for every k, joined by `delim`, "\n"
// terminated.  long_form != 0 writes dataset.py:328-336 lines instead:
// "nu1,nu2,sync,async" per element (matrix = sync, matrix2 = async).
// Returns the byte count in *written; fails (with *written = bytes needed so
// far) when cap is too small -- callers size cap generously (<= 25 bytes per
// value) and retry.
extern "C" int corr2d_format_rows(int dtype, const double* axis1, const double* axis2, const void* matrix,
                                  const void* matrix2, int64_t ld, int n2, int r0, int r1, char delim, int long_form,
                                  int threads, char* out, int64_t cap, int64_t* written) {
  if (!axis1 || !axis2 || !matrix || !out || !written || r0 < 0 || r1 < r0 || n2 < 1 || ld < n2 ||
      (long_form && !matrix2))
    return fail(CORR2D_ERR_DATA, "corr2d_format_rows: bad arguments");
  if (dtype != CORR2D_F64 && dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_format_rows: bad dtype");
  const int rows = r1 - r0;
  if (threads < 1) threads = 1;
  if (threads > rows) threads = rows > 0 ? rows : 1;
  std::vector<std::vector<char>> parts(threads);
  auto work = [&](int t) {
    const int a = r0 + (int)((long long)rows * t / threads), b = r0 + (int)((long long)rows * (t + 1) / threads);
    std::vector<char>& o = parts[t];
    o.reserve((size_t)(b - a) * (size_t)(n2 + 1) * (long_form ? 80 : 20));
    char tmp[40], nu1[40];
    for (int i = a; i < b; ++i) {
      const long long row = (long long)i * ld;
      if (!long_form) {
        int k = repr_double(axis1[i], tmp);
        o.insert(o.end(), tmp, tmp + k);
        for (int c = 0; c < n2; ++c) {
          o.push_back(delim);
          k = repr_double(elem(matrix, dtype, row + c), tmp);
          o.insert(o.end(), tmp, tmp + k);
        }
        o.push_back('\n');
      } else {
        const int k1 = repr_double(axis1[i], nu1);
        for (int c = 0; c < n2; ++c) {
          o.insert(o.end(), nu1, nu1 + k1);
          o.push_back(',');
          int k = repr_double(axis2[c], tmp);
          o.insert(o.end(), tmp, tmp + k);
          o.push_back(',');
          k = repr_double(elem(matrix, dtype, row + c), tmp);
          o.insert(o.end(), tmp, tmp + k);
          o.push_back(',');
          k = repr_double(elem(matrix2, dtype, row + c), tmp);
          o.insert(o.end(), tmp, tmp + k);
          o.push_back('\n');
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  std::vector<int64_t> offs(threads + 1, 0);
  for (int t = 0; t < threads; ++t) offs[t + 1] = offs[t] + (int64_t)parts[t].size();
  const int64_t total = offs[threads];
  *written = total;
  if (total > cap) return fail(CORR2D_ERR_DATA, "corr2d_format_rows: buffer too small");
  // parallel gather of the per-thread parts into the caller's buffer
  auto copy = [&](int t) { memcpy(out + offs[t], parts[t].data(), parts[t].size()); };
  pool.clear();
  for (int t = 1; t < threads; ++t) pool.emplace_back(copy, t);
  copy(0);
  for (auto& th : pool) th.join();
  return CORR2D_OK;
}
