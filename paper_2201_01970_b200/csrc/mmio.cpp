// MatrixMarket coordinate files (src/mmio.py:36-228) at I/O speed: the body
// of a file (everything after the header line) is parsed in C++ with the
// reference's validation order and line numbering, and entries are written
// with printf's %.17g (the reference's f"{v:.17g}": the shortest-round-trip
// 17-significant-digit form, so read -> write -> read round-trips bitwise).
// Tokens outside the plain ASCII number grammar (digit separators, non-ASCII
// digits, ...) make the parser report MM_FALLBACK so the caller can use the
// pure-Python reading of the reference for that file.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.h"

namespace {

enum {
  MM_OK = 0,
  MM_SIDECAR = 1,       // malformed block_size sidecar
  MM_SIZE_FIELDS = 2,   // malformed size line (expected 'nrows ncols nnz')
  MM_SIZE_INT = 3,      // malformed size line (expected integers)
  MM_NO_SIZE = 4,       // missing size line
  MM_ENTRY = 5,         // malformed entry (expected 'i j value')
  MM_RANGE = 6,         // index (i, j) out of range
  MM_TOO_MANY = 7,      // more than the declared nnz entries
  MM_COUNT = 8,         // file declares nnz entries but contains k
  MM_FALLBACK = 9,      // token outside the fast grammar: parse in Python
  MM_IO = 10,
};

bool read_file(const char* path, std::string& buf) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf.resize(n > 0 ? (size_t)n : 0);
  const size_t got = n > 0 ? std::fread(&buf[0], 1, (size_t)n, f) : 0;
  std::fclose(f);
  return got == buf.size();
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// split a line (no '\n') into whitespace tokens
void tokens(const char* b, const char* e, std::vector<std::pair<const char*, const char*>>& out) {
  out.clear();
  while (b < e) {
    while (b < e && is_ws(*b)) ++b;
    if (b >= e) break;
    const char* s = b;
    while (b < e && !is_ws(*b)) ++b;
    out.emplace_back(s, b);
  }
}

// 0 ok, 1 malformed (Python int() would raise), 2 fallback
int parse_int(const char* s, const char* e, int64_t& v) {
  const char* p = s;
  if (p < e && (*p == '+' || *p == '-')) ++p;
  if (p >= e) return 1;
  for (const char* q = p; q < e; ++q) {
    const unsigned char c = (unsigned char)*q;
    if (c >= 0x80 || c == '_') return 2;
    if (c < '0' || c > '9') return 1;
  }
  std::string t(s, e);
  errno = 0;
  v = std::strtoll(t.c_str(), nullptr, 10);
  if (errno == ERANGE) return 2;
  return 0;
}

bool ieq(const char* s, const char* e, const char* w) {
  const size_t n = std::strlen(w);
  if ((size_t)(e - s) != n) return false;
  for (size_t i = 0; i < n; ++i) {
    char c = s[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != w[i]) return false;
  }
  return true;
}

// Python float(): decimal literals, inf/infinity/nan with optional sign
int parse_float(const char* s, const char* e, double& v) {
  const char* p = s;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) {
    neg = *p == '-';
    ++p;
  }
  if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
    v = neg ? -INFINITY : INFINITY;
    return 0;
  }
  if (ieq(p, e, "nan")) {
    v = neg ? -NAN : NAN;
    return 0;
  }
  bool digit = false, dot = false, exp = false;
  for (const char* q = p; q < e; ++q) {
    const unsigned char c = (unsigned char)*q;
    if (c >= 0x80 || c == '_') return 2;
    if (c >= '0' && c <= '9') {
      digit = true;
    } else if (c == '.') {
      if (dot || exp) return 1;
      dot = true;
    } else if (c == 'e' || c == 'E') {
      if (exp || !digit) return 1;
      exp = true;
      if (q + 1 < e && (q[1] == '+' || q[1] == '-')) ++q;
      if (q + 1 >= e) return 1;
    } else {
      return 1;
    }
  }
  if (!digit) return 1;
  std::string t(s, e);
  v = std::strtod(t.c_str(), nullptr);  // correctly rounded, as Python's float()
  return 0;
}

}  // namespace

extern "C" {

// Parse everything after the header line of a coordinate file.
// info (out, int64[12]): 0 nrows, 1 ncols, 2 nnz, 3 block_size (-1 = none),
// 4 entries found, 5 error code (MM_*), 6 error line, 7 i, 8 j (MM_RANGE),
// 9 total lines.  With rows == NULL only the size line is read (info[2]
// sizes the arrays of the second call).  Returns CPRB_OK unless the file
// cannot be read.
int cprb_mm_read_coord(const char* path, int64_t* rows, int64_t* cols, double* vals,
                       int64_t* linenos, int64_t* info) {
  std::string buf;
  if (!read_file(path, buf)) return cprb::set_error(CPRB_EINVAL, std::string("cannot read ") + path);
  for (int k = 0; k < 12; ++k) info[k] = 0;
  info[3] = -1;
  // line starts
  std::vector<std::pair<size_t, size_t>> lines;
  {
    size_t b = 0;
    for (size_t i = 0; i < buf.size(); ++i)
      if (buf[i] == '\n') {
        lines.emplace_back(b, i);
        b = i + 1;
      }
    if (b < buf.size()) lines.emplace_back(b, buf.size());
  }
  const int64_t nlines = (int64_t)lines.size();
  info[9] = nlines;
  std::vector<std::pair<const char*, const char*>> tk;
  auto fail = [&](int code, int64_t line) {
    info[5] = code;
    info[6] = line;
    return CPRB_OK;
  };
  int64_t lineno = 1, nrows = 0, ncols = 0, nnz = 0;
  bool dims = false;
  for (lineno = 2; lineno <= nlines; ++lineno) {
    const char* b = buf.data() + lines[lineno - 1].first;
    const char* e = buf.data() + lines[lineno - 1].second;
    while (b < e && is_ws(*b)) ++b;
    while (e > b && is_ws(e[-1])) --e;
    if (b == e) continue;
    if (*b == '%') {
      const char* c = b;
      while (c < e && *c == '%') ++c;
      while (c < e && is_ws(*c)) ++c;
      static const char key[] = "block_size:";
      if ((size_t)(e - c) >= sizeof(key) - 1 && std::memcmp(c, key, sizeof(key) - 1) == 0) {
        const char* v = c + sizeof(key) - 1;
        while (v < e && is_ws(*v)) ++v;
        int64_t bs = 0;
        const int r = parse_int(v, e, bs);
        if (r == 2) return fail(MM_FALLBACK, lineno);
        if (r == 1) return fail(MM_SIDECAR, lineno);
        info[3] = bs;
      }
      continue;
    }
    tokens(b, e, tk);
    if (tk.size() != 3) return fail(MM_SIZE_FIELDS, lineno);
    int64_t d[3];
    for (int k = 0; k < 3; ++k) {
      const int r = parse_int(tk[k].first, tk[k].second, d[k]);
      if (r == 2) return fail(MM_FALLBACK, lineno);
      if (r == 1) return fail(MM_SIZE_INT, lineno);
    }
    nrows = d[0];
    ncols = d[1];
    nnz = d[2];
    dims = true;
    break;
  }
  if (!dims) return fail(MM_NO_SIZE, nlines >= 2 ? nlines : 1);
  info[0] = nrows;
  info[1] = ncols;
  info[2] = nnz;
  if (!rows) return CPRB_OK;
  int64_t k = 0;
  for (int64_t ln = lineno + 1; ln <= nlines; ++ln) {
    const char* b = buf.data() + lines[ln - 1].first;
    const char* e = buf.data() + lines[ln - 1].second;
    while (b < e && is_ws(*b)) ++b;
    while (e > b && is_ws(e[-1])) --e;
    if (b == e || *b == '%') continue;
    tokens(b, e, tk);
    if (tk.size() != 3) return fail(MM_ENTRY, ln);
    int64_t i = 0, j = 0;
    double v = 0.0;
    int r = parse_int(tk[0].first, tk[0].second, i);
    if (r == 0) r = parse_int(tk[1].first, tk[1].second, j);
    if (r == 0) r = parse_float(tk[2].first, tk[2].second, v);
    if (r == 2) return fail(MM_FALLBACK, ln);
    if (r == 1) return fail(MM_ENTRY, ln);
    if (!(1 <= i && i <= nrows) || !(1 <= j && j <= ncols)) {
      info[7] = i;
      info[8] = j;
      return fail(MM_RANGE, ln);
    }
    if (k >= nnz) return fail(MM_TOO_MANY, ln);
    rows[k] = i - 1;
    cols[k] = j - 1;
    vals[k] = v;
    linenos[k] = ln;
    ++k;
  }
  info[4] = k;
  if (k != nnz) return fail(MM_COUNT, nlines);
  return CPRB_OK;
}

// Entry lines "i j v" (1-based, %.17g; NaN as "nan" like Python) appended to
// an already written header.
int cprb_mm_write_entries(const char* path, int64_t n, const int64_t* rows, const int64_t* cols,
                          const double* vals) {
  FILE* f = std::fopen(path, "ab");
  if (!f) return cprb::set_error(CPRB_EINVAL, std::string("cannot write ") + path);
  std::vector<char> out;
  out.reserve(1 << 20);
  char line[96];
  for (int64_t k = 0; k < n; ++k) {
    int m;
    if (std::isnan(vals[k]))
      m = std::snprintf(line, sizeof(line), "%lld %lld nan\n", (long long)rows[k] + 1,
                        (long long)cols[k] + 1);
    else
      m = std::snprintf(line, sizeof(line), "%lld %lld %.17g\n", (long long)rows[k] + 1,
                        (long long)cols[k] + 1, vals[k]);
    out.insert(out.end(), line, line + m);
    if (out.size() > (1u << 20)) {
      std::fwrite(out.data(), 1, out.size(), f);
      out.clear();
    }
  }
  std::fwrite(out.data(), 1, out.size(), f);
  std::fclose(f);
  return CPRB_OK;
}

}  // extern "C"
