// mmio.cu -- parallel host parser for the entry section of a MatrixMarket
// coordinate file (replaces the per-line Python loop of mmio.py:69-94).
//
// Host code only (no kernels): SuiteSparse inputs of the paper's study are
// hundreds of MB of text, which the reference parses one Python line at a time.
// Here the entry section is cut into per-thread byte ranges on line
// boundaries; pass 1 counts lines / entry lines per range, an exclusive scan
// gives every range its first line number and entry index, pass 2 parses the
// entries straight into the caller's COO arrays.  The banner and size line
// (mmio.py:29-67) stay in Python, where their messages are formatted.
//
// Semantics kept from the reference (mmio.py:69-94, read via Python text mode):
//  * line breaks are "\n", "\r\n" and "\r" (universal newlines); a final line
//    without a break still counts;
//  * blank lines and lines whose stripped text starts with '%' are skipped;
//  * tokens are split on Python's ASCII whitespace (space, \t, \v, \f,
//    \x1c-\x1f); bytes >= 0x80 decode to U+FFFD, which is not whitespace;
//  * indices follow int() (optional sign, digits, single '_' between digits),
//    values follow float() (decimal / exponent / inf / infinity / nan, '_'
//    between digits, no hex) and are converted with glibc strtod, which rounds
//    correctly like CPython's dtoa -- bitwise the same doubles;
//  * the first offending line wins: an entry past the declared count, a wrong
//    token count, an unparsable token or an out-of-bounds index.  The library
//    reports that line number (RS_ERR_PARSE, rs_last_error_index()); the
//    Python layer re-reads that one line to format the reference's message.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "rs_internal.cuh"

namespace rs {
namespace {

inline bool py_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

// [p, q) is a digit part: digit ('_'? digit)*
bool digit_part(const char* p, const char* q) {
  if (p >= q || !is_digit(*p)) return false;
  for (const char* s = p + 1; s < q; ++s) {
    if (*s == '_') {
      if (s + 1 >= q || !is_digit(s[1])) return false;
    } else if (!is_digit(*s)) {
      return false;
    }
  }
  return true;
}

// int(token) for a 1-based index; *ok = grammar ok; value saturates at INT64_MAX
// (any saturated value is out of bounds for the int64 sizes it is checked against).
int64_t py_int(const char* p, const char* q, bool* ok) {
  bool neg = false;
  if (p < q && (*p == '+' || *p == '-')) neg = (*p++ == '-');
  if (!digit_part(p, q)) { *ok = false; return 0; }
  *ok = true;
  int64_t v = 0;
  bool sat = false;
  for (; p < q; ++p) {
    if (*p == '_') continue;
    int d = *p - '0';
    if (v > (INT64_MAX - d) / 10) sat = true;
    if (!sat) v = v * 10 + d;
  }
  if (sat) v = INT64_MAX;
  return neg ? (v == INT64_MAX && sat ? INT64_MIN : -v) : v;
}

bool ieq(const char* p, const char* q, const char* word) {
  size_t n = strlen(word);
  if ((size_t)(q - p) != n) return false;
  for (size_t i = 0; i < n; ++i) {
    char c = p[i];
    if (c >= 'A' && c <= 'Z') c = char(c - 'A' + 'a');
    if (c != word[i]) return false;
  }
  return true;
}

// float(token): CPython's grammar, value by strtod (correctly rounded)
bool py_float(const char* p, const char* q, double* out) {
  const char* s = p;
  bool neg = false;
  if (s < q && (*s == '+' || *s == '-')) neg = (*s++ == '-');
  if (ieq(s, q, "inf") || ieq(s, q, "infinity")) {
    *out = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq(s, q, "nan")) {
    *out = neg ? -__builtin_nan("") : __builtin_nan("");
    return true;
  }
  // mantissa: digitpart ['.' [digitpart]] | '.' digitpart
  const char* e = s;
  while (e < q && *e != 'e' && *e != 'E') ++e;
  const char* dot = s;
  while (dot < e && *dot != '.') ++dot;
  if (dot < e) {
    bool left = dot > s, right = dot + 1 < e;
    if (!left && !right) return false;
    if (left && !digit_part(s, dot)) return false;
    if (right && !digit_part(dot + 1, e)) return false;
  } else if (!digit_part(s, e)) {
    return false;
  }
  if (e < q) {  // exponent: ('e'|'E') [sign] digitpart
    const char* x = e + 1;
    if (x < q && (*x == '+' || *x == '-')) ++x;
    if (!digit_part(x, q)) return false;
  }
  char small[64];
  std::string big;
  char* buf = small;
  size_t len = size_t(q - p);
  if (len >= sizeof(small)) {
    big.resize(len + 1);
    buf = &big[0];
  }
  size_t k = 0;
  for (const char* c = p; c < q; ++c)
    if (*c != '_') buf[k++] = *c;
  buf[k] = '\0';
  char* end = nullptr;
  *out = strtod(buf, &end);
  return end == buf + k;
}

struct Range {
  int64_t begin = 0, end = 0;    // byte range [begin, end), starts on a line start
  int64_t lines = 0, data = 0;   // pass-1 counts
  int64_t line0 = 0, data0 = 0;  // first line number / entry index (exclusive scan)
  int64_t err_line = INT64_MAX;  // first offending line in this range
};

// next line start at or after p (line breaks: \n, \r\n, \r)
int64_t line_start_at_or_after(const char* buf, int64_t len, int64_t p) {
  if (p <= 0) return 0;
  while (p < len) {
    char prev = buf[p - 1];
    if (prev == '\n' || (prev == '\r' && buf[p] != '\n')) return p;
    ++p;
  }
  return len;
}

// one line [p, q) (without its break); returns the start of the next line
inline int64_t next_line(const char* buf, int64_t len, int64_t p, int64_t* q) {
  int64_t s = p;
  while (s < len && buf[s] != '\n' && buf[s] != '\r') ++s;
  *q = s;
  if (s < len && buf[s] == '\r' && s + 1 < len && buf[s + 1] == '\n') return s + 2;
  return s < len ? s + 1 : len;
}

// stripped content of a line: [*a, *b); returns true for an entry line
inline bool entry_line(const char* buf, int64_t p, int64_t q, int64_t* a, int64_t* b) {
  while (p < q && (py_space((unsigned char)buf[p]))) ++p;
  while (q > p && (py_space((unsigned char)buf[q - 1]))) --q;
  *a = p;
  *b = q;
  return p < q && buf[p] != '%';
}

void count_range(const char* buf, int64_t len, Range* r) {
  int64_t p = r->begin;
  while (p < r->end) {
    int64_t q, a, b;
    int64_t nx = next_line(buf, len, p, &q);
    r->lines++;
    if (entry_line(buf, p, q, &a, &b)) r->data++;
    p = nx;
  }
}

void parse_range(const char* buf, int64_t len, Range* r, int64_t declared, int with_values, int64_t nrows,
                 int64_t ncols, int64_t* rows, int64_t* cols, double* vals) {
  int64_t p = r->begin, line = r->line0, e = r->data0;
  const int expected = with_values ? 3 : 2;
  while (p < r->end) {
    int64_t q, a, b;
    int64_t nx = next_line(buf, len, p, &q);
    if (entry_line(buf, p, q, &a, &b)) {
      if (e >= declared) { r->err_line = line; return; }
      const char* tok[4];
      const char* tend[4];
      int nt = 0;
      int64_t s = a;
      while (s < b) {
        while (s < b && py_space((unsigned char)buf[s])) ++s;
        if (s >= b) break;
        int64_t t = s;
        while (t < b && !py_space((unsigned char)buf[t])) ++t;
        if (nt < 4) { tok[nt] = buf + s; tend[nt] = buf + t; }
        ++nt;
        s = t;
      }
      if (nt != expected) { r->err_line = line; return; }
      bool ok_i, ok_j;
      int64_t i = py_int(tok[0], tend[0], &ok_i);
      int64_t j = ok_i ? py_int(tok[1], tend[1], &ok_j) : 0;
      double v = 1.0;
      if (!ok_i || !ok_j || (with_values && !py_float(tok[2], tend[2], &v))) { r->err_line = line; return; }
      if (!(i >= 1 && i <= nrows && j >= 1 && j <= ncols)) { r->err_line = line; return; }
      rows[e] = i - 1;
      cols[e] = j - 1;
      vals[e] = v;
      ++e;
    }
    ++line;
    p = nx;
  }
}

}  // namespace
}  // namespace rs

using namespace rs;

extern "C" int rs_mm_parse_entries(const char* buf, int64_t len, int64_t first_line, int64_t declared, int with_values,
                                   int64_t nrows, int64_t ncols, int64_t capacity, int64_t* rows, int64_t* cols,
                                   double* vals, int64_t* count_out, int64_t* last_line_out, int nthreads) {
  if ((len > 0 && !buf) || len < 0 || declared < 0 || capacity < 0 || !count_out || !last_line_out ||
      (capacity > 0 && (!rows || !cols || !vals))) {
    set_error(RS_ERR_ARG, "rs_mm_parse_entries: bad arguments");
    return RS_ERR_ARG;
  }
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  // below ~1 MB per thread the split is not worth a thread
  int64_t t = std::max<int64_t>(1, std::min<int64_t>(nthreads, len >> 20));
  std::vector<Range> rg((size_t)t);
  for (int64_t k = 0; k < t; ++k) rg[k].begin = line_start_at_or_after(buf, len, len * k / t);
  for (int64_t k = 0; k < t; ++k) rg[k].end = k + 1 < t ? rg[k + 1].begin : len;

  auto run = [&](auto&& fn) {
    std::vector<std::thread> th;
    for (int64_t k = 1; k < t; ++k) th.emplace_back([&, k] { fn(&rg[k]); });
    fn(&rg[0]);
    for (auto& x : th) x.join();
  };
  run([&](Range* r) { count_range(buf, len, r); });
  int64_t line = first_line, data = 0;
  for (auto& r : rg) {
    r.line0 = line;
    r.data0 = data;
    line += r.lines;
    data += r.data;
  }
  *last_line_out = line - 1;
  int64_t fits = std::min(data, declared);
  if (fits > capacity) {
    set_error(RS_ERR_ARG, "rs_mm_parse_entries: capacity " + std::to_string(capacity) + " < " +
                              std::to_string(fits) + " entries");
    return RS_ERR_ARG;
  }
  run([&](Range* r) { parse_range(buf, len, r, declared, with_values, nrows, ncols, rows, cols, vals); });
  int64_t err = INT64_MAX;
  for (auto& r : rg) err = std::min(err, r.err_line);
  *count_out = fits;
  if (err != INT64_MAX) {
    set_error(RS_ERR_PARSE, "line " + std::to_string(err) + ": malformed MatrixMarket entry", err);
    return RS_ERR_PARSE;
  }
  return RS_OK;
}

// ---------------------------------------------------------------- COO -> CSR order (sparse.py:133-160)
// The permutation np.lexsort((cols, rows)) computes: a stable counting sort by
// row (entries of one row keep their input order), then a stable sort by column
// inside each row (skipped for rows already in order), rows split over threads.
extern "C" int rs_coo_sort(int64_t nnz, int64_t nrows, const int64_t* rows, const int64_t* cols, int64_t* perm,
                           int64_t* row_ptr, int nthreads) {
  if (nnz < 0 || nrows < 0 || (nnz > 0 && (!rows || !cols || !perm)) || !row_ptr) {
    set_error(RS_ERR_ARG, "rs_coo_sort: bad arguments");
    return RS_ERR_ARG;
  }
  for (int64_t i = 0; i <= nrows; ++i) row_ptr[i] = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    int64_t r = rows[e];
    if (r < 0 || r >= nrows) {
      set_error(RS_ERR_ARG, "row index out of range", e);
      return RS_ERR_ARG;
    }
    row_ptr[r + 1]++;
  }
  for (int64_t i = 0; i < nrows; ++i) row_ptr[i + 1] += row_ptr[i];
  {
    std::vector<int64_t> next(row_ptr, row_ptr + nrows);
    for (int64_t e = 0; e < nnz; ++e) perm[next[rows[e]]++] = e;
  }
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  int64_t t = std::max<int64_t>(1, std::min<int64_t>(nthreads, nnz >> 16));
  auto work = [&](int64_t k) {
    int64_t r0 = nrows * k / t, r1 = nrows * (k + 1) / t;
    for (int64_t r = r0; r < r1; ++r) {
      int64_t* b = perm + row_ptr[r];
      int64_t* e = perm + row_ptr[r + 1];
      bool sorted = true;
      for (int64_t* p = b + 1; p < e; ++p)
        if (cols[p[-1]] > cols[p[0]]) { sorted = false; break; }
      if (!sorted) std::stable_sort(b, e, [&](int64_t x, int64_t y) { return cols[x] < cols[y]; });
    }
  };
  std::vector<std::thread> th;
  for (int64_t k = 1; k < t; ++k) th.emplace_back(work, k);
  work(0);
  for (auto& x : th) x.join();
  return RS_OK;
}
