// Native tensor-file ingest: Matrix Market and
// FROSTT text -> 0-based int32 coordinates + fp64 values, multithreaded, for
// the device pack (spx_pack.cu).  Semantics follow spindle.fileio
// (fileio.py:66-162) exactly for every file it accepts:
//   * lines are split the way str.splitlines() splits ASCII text
//     (\n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e), stripped of ASCII whitespace,
//     and tokenised on ' ', '\t', '\x1f' (str.split());
//   * '%' (Matrix Market) / '#' (FROSTT) comment lines, the MM header and
//     'rows cols nnz' size line, FROSTT '# dims:' comments (the last wins),
//     FROSTT dimensions inferred as coordinate maxima otherwise;
//   * integers are plain [+-]digits, values [+-]digits[.digits][e[+-]digits]
//     converted with strtod (correctly rounded, as Python's float()).
// Anything else -- a malformed or out-of-bounds entry, a count mismatch,
// non-ASCII bytes, Python-only literal syntax (underscores, inf/nan),
// integers past 18 digits -- returns SPX_PARSE_DEFER, and the Python host
// hands the text to the reference parser, which raises the exact error
// class, message and line number (or accepts the exotic literal).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "spx_internal.h"

namespace spx {
namespace {

constexpr int kDefer = 1;

inline bool is_break(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == 0x1f || is_break(c); }
inline bool is_tok_sep(char c) { return c == ' ' || c == '\t' || c == 0x1f; }

// next line [b, e) starting at p; returns the start of the following line
inline const char* next_line(const char* p, const char* end, const char** b, const char** e) {
  *b = p;
  while (p < end && !is_break(*p)) ++p;
  *e = p;
  if (p < end) {
    if (*p == '\r' && p + 1 < end && p[1] == '\n') p += 2;
    else ++p;
  }
  return p;
}

inline void strip(const char** b, const char** e) {
  while (*b < *e && is_ws(**b)) ++*b;
  while (*e > *b && is_ws((*e)[-1])) --*e;
}

// tokens of a stripped line; returns the count (up to cap)
inline int tokens(const char* b, const char* e, const char** tb, const char** te, int cap) {
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_tok_sep(*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_tok_sep(*p)) ++p;
    if (n < cap) {
      tb[n] = s;
      te[n] = p;
    }
    ++n;
  }
  return n;
}

// plain [+-]digits, at most 18 digits
inline bool parse_int(const char* b, const char* e, int64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
  if (b >= e || e - b > 18) return false;
  int64_t v = 0;
  for (const char* p = b; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + (*p - '0');
  }
  *out = neg ? -v : v;
  return true;
}

// [+-]digits[.digits][(e|E)[+-]digits] or [+-].digits[...] -> strtod
inline bool parse_float(const char* b, const char* e, double* out) {
  const char* p = b;
  if (p < e && (*p == '+' || *p == '-')) ++p;
  const char* m = p;
  while (p < e && *p >= '0' && *p <= '9') ++p;
  int digits = (int)(p - m);
  if (p < e && *p == '.') {
    ++p;
    const char* f = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    digits += (int)(p - f);
  }
  if (digits == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* x = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == x) return false;
  }
  if (p != e) return false;
  char buf[128];
  const size_t len = (size_t)(e - b);
  if (len >= sizeof(buf)) return false;
  std::memcpy(buf, b, len);
  buf[len] = 0;
  *out = std::strtod(buf, nullptr);
  return true;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;      // line count inside the chunk
  int64_t entries = 0;    // data lines
  int64_t first_tokens = -1;  // token count of the first data line (FROSTT order)
  int dims_n = -1;        // last '# dims:' comment in the chunk
  int64_t dims[8];
  bool defer = false;
  int64_t maxc[8];
};

int nthreads_for(size_t bytes) {
  unsigned hw = std::thread::hardware_concurrency();
  if (hw == 0) hw = 4;
  const size_t by_size = bytes / (4u << 20) + 1;  // >= 4 MB per thread
  return (int)std::max<size_t>(1, std::min<size_t>({(size_t)hw, by_size, (size_t)64}));
}

// split [b, e) into k pieces at line starts ('\n' boundaries)
std::vector<Chunk> split(const char* b, const char* e, int k) {
  std::vector<Chunk> cs;
  const char* p = b;
  for (int i = 0; i < k && p < e; ++i) {
    const char* q = (i == k - 1) ? e : std::min(e, b + (size_t)(e - b) * (i + 1) / k);
    while (q < e && q > p && q[-1] != '\n') ++q;  // end just after a '\n'
    Chunk c;
    c.b = p;
    c.e = q;
    cs.push_back(c);
    p = q;
  }
  return cs;
}

template <typename F>
void parallel(std::vector<Chunk>& cs, F f) {
  std::vector<std::thread> th;
  for (size_t i = 1; i < cs.size(); ++i) th.emplace_back(f, std::ref(cs[i]));
  if (!cs.empty()) f(cs[0]);
  for (auto& t : th) t.join();
}

bool is_comment_dims(const char* b, const char* e, int64_t* dims, int* nd, bool* defer) {
  // b..e stripped, starts with '#': body = [1:].strip(); lower startswith "dims:"
  const char* p = b + 1;
  const char* q = e;
  strip(&p, &q);
  if (q - p < 5) return false;
  const char want[] = "dims:";
  for (int i = 0; i < 5; ++i) {
    char c = p[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != want[i]) return false;
  }
  const char* tb[9];
  const char* te[9];
  const int n = tokens(p + 5, q, tb, te, 9);
  if (n > 8) {
    *defer = true;
    return true;
  }
  for (int i = 0; i < n; ++i)
    if (!parse_int(tb[i], te[i], &dims[i])) {
      *defer = true;
      return true;
    }
  *nd = n;
  return true;
}

}  // namespace
}  // namespace spx

using namespace spx;

extern "C" {

// Pass 1: format (0 Matrix Market, 1 FROSTT), order, entry count and dims
// (Matrix Market: declared; FROSTT: last '# dims:' or -1 = infer).  Returns
// 0, or SPX_PARSE_DEFER (1) when the reference parser must take the file.
int spx_text_scan(const char* text, int64_t len, int32_t fmt, int32_t* order_out, int64_t* n_out,
                  int64_t* dims_out) {
  const char* end = text + len;
  for (int64_t i = 0; i < len; ++i)
    if ((unsigned char)text[i] >= 0x80 || text[i] == 0) return kDefer;
  const char* body = text;
  if (fmt == 0) {
    const char *b, *e;
    const char* p = next_line(text, end, &b, &e);
    if (len == 0) return kDefer;
    strip(&b, &e);
    const char hdr[] = "%%matrixmarket matrix coordinate real general";
    if ((size_t)(e - b) != sizeof(hdr) - 1) return kDefer;
    for (size_t i = 0; i < sizeof(hdr) - 1; ++i) {
      char c = b[i];
      if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
      if (c != hdr[i]) return kDefer;
    }
    bool found = false;
    while (p < end) {
      p = next_line(p, end, &b, &e);
      strip(&b, &e);
      if (b == e || *b == '%') continue;
      const char* tb[4];
      const char* te[4];
      if (tokens(b, e, tb, te, 4) != 3) return kDefer;
      for (int i = 0; i < 3; ++i)
        if (!parse_int(tb[i], te[i], &dims_out[i])) return kDefer;
      found = true;
      break;
    }
    if (!found) return kDefer;
    if (dims_out[0] > INT32_MAX || dims_out[1] > INT32_MAX || dims_out[0] < 0 || dims_out[1] < 0) return kDefer;
    body = p;
    *order_out = 2;
  }
  std::vector<Chunk> cs = split(body, end, nthreads_for((size_t)(end - body)));
  const char cc = fmt == 0 ? '%' : '#';
  parallel(cs, [&](Chunk& c) {
    const char* p = c.b;
    while (p < c.e) {
      const char *b, *e;
      p = next_line(p, c.e, &b, &e);
      ++c.lines;
      strip(&b, &e);
      if (b == e) continue;
      if (*b == cc) {
        if (fmt == 1) {
          int nd = -1;
          int64_t d[8];
          if (is_comment_dims(b, e, d, &nd, &c.defer) && nd >= 0) {
            c.dims_n = nd;
            std::memcpy(c.dims, d, sizeof(d));
          }
        }
        continue;
      }
      if (c.first_tokens < 0) {
        const char* tb[1];
        const char* te[1];
        c.first_tokens = tokens(b, e, tb, te, 0);
      }
      ++c.entries;
    }
  });
  int64_t n = 0;
  int64_t first_tokens = -1;
  int dims_n = -1;
  int64_t dims[8];
  for (auto& c : cs) {
    if (c.defer) return kDefer;
    n += c.entries;
    if (first_tokens < 0 && c.first_tokens >= 0) first_tokens = c.first_tokens;
    if (c.dims_n >= 0) {
      dims_n = c.dims_n;
      std::memcpy(dims, c.dims, sizeof(dims));
    }
  }
  *n_out = n;
  if (fmt == 0) {
    if (n != dims_out[2]) return kDefer;  // count mismatch: the reference reports it
    return SPX_OK;
  }
  int order;
  if (first_tokens >= 0) {
    if (first_tokens < 2 || first_tokens - 1 > 8) return kDefer;
    order = (int)first_tokens - 1;
  } else {
    if (dims_n < 0) return kDefer;  // empty file with no dims line
    order = dims_n;
  }
  if (order < 1 || (dims_n >= 0 && dims_n != order)) return kDefer;
  for (int l = 0; l < dims_n; ++l)
    if (dims[l] < 1 || dims[l] > (int64_t)INT32_MAX + 1) return kDefer;
  *order_out = order;
  for (int l = 0; l < order; ++l) dims_out[l] = dims_n >= 0 ? dims[l] : -1;
  return SPX_OK;
}

// Pass 2: coordinates (0-based, level-major: coords[l*n + i]) and values in
// file order.  dims: as spx_text_scan reported (FROSTT -1 = infer; the
// inferred maxima are written back).
int spx_text_parse(const char* text, int64_t len, int32_t fmt, int32_t order, int64_t n, int64_t* dims,
                   int32_t* coords, double* vals) {
  const char* end = text + len;
  const char* body = text;
  if (fmt == 0) {  // skip header and size line (validated by the scan)
    const char *b, *e;
    const char* p = next_line(text, end, &b, &e);
    while (p < end) {
      p = next_line(p, end, &b, &e);
      strip(&b, &e);
      if (b == e || *b == '%') continue;
      break;
    }
    body = p;
  }
  std::vector<Chunk> cs = split(body, end, nthreads_for((size_t)(end - body)));
  const char cc = fmt == 0 ? '%' : '#';
  // entry offsets per chunk: count data lines first
  parallel(cs, [&](Chunk& c) {
    const char* p = c.b;
    while (p < c.e) {
      const char *b, *e;
      p = next_line(p, c.e, &b, &e);
      strip(&b, &e);
      if (b == e || *b == cc) continue;
      ++c.entries;
    }
  });
  std::vector<int64_t> off(cs.size() + 1, 0);
  for (size_t i = 0; i < cs.size(); ++i) off[i + 1] = off[i] + cs[i].entries;
  if (off.back() != n) return kDefer;
  const bool declared = fmt == 0 || dims[0] >= 0;
  std::vector<Chunk*> ptrs;
  for (auto& c : cs) ptrs.push_back(&c);
  std::vector<std::thread> th;
  auto work = [&](size_t ci) {
    Chunk& c = cs[ci];
    for (int l = 0; l < order; ++l) c.maxc[l] = 0;
    int64_t k = off[ci];
    const char* p = c.b;
    const char* tb[9];
    const char* te[9];
    while (p < c.e) {
      const char *b, *e;
      p = next_line(p, c.e, &b, &e);
      strip(&b, &e);
      if (b == e || *b == cc) continue;
      const int nt = tokens(b, e, tb, te, 9);
      if (nt != order + 1) {
        c.defer = true;
        return;
      }
      for (int l = 0; l < order; ++l) {
        int64_t v;
        if (!parse_int(tb[l], te[l], &v) || v < 1 || (declared && v > dims[l]) || v - 1 > INT32_MAX) {
          c.defer = true;
          return;
        }
        coords[(int64_t)l * n + k] = (int32_t)(v - 1);
        if (v > c.maxc[l]) c.maxc[l] = v;
      }
      if (!parse_float(tb[order], te[order], &vals[k])) {
        c.defer = true;
        return;
      }
      ++k;
    }
  };
  for (size_t i = 1; i < cs.size(); ++i) th.emplace_back(work, i);
  if (!cs.empty()) work(0);
  for (auto& t : th) t.join();
  for (auto& c : cs)
    if (c.defer) return kDefer;
  if (!declared) {
    for (int l = 0; l < order; ++l) {
      int64_t m = 0;
      for (auto& c : cs)
        if (c.entries) m = std::max(m, c.maxc[l]);
      dims[l] = m;  // max 1-based coordinate == max 0-based + 1
    }
  }
  return SPX_OK;
}

}  // extern "C"
