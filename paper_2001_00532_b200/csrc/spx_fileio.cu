// Native tensor-file ingest: Matrix Market and
// FROSTT text -> 0-based int32 coordinates + fp64 values, multithreaded, for
// the device pack (spx_pack.cu).  Semantics follow spindle.fileio
// (fileio.py:66-162) line for line, errors included:
//   * lines are split the way str.splitlines() splits ASCII text
//     (\n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e), stripped of ASCII whitespace,
//     and tokenised on ' ', '\t', '\x1f' (str.split());
//   * '%' (Matrix Market) / '#' (FROSTT) comment lines, the MM header and
//     'rows cols nnz' size line, FROSTT '# dims:' comments (the last wins),
//     FROSTT dimensions inferred as coordinate maxima otherwise;
//   * integers follow int() (sign, digits, single underscores between
//     digits), values follow float() (the same plus '.', exponents and
//     inf / infinity / nan, any case), converted with strtod (correctly
//     rounded, as Python's float());
//   * every error the reference raises -- HeaderError, EntryValueError,
//     EntryBoundsError, TensorFileError -- is raised for the same line with
//     the same message (Python repr of the offending token / line): the
//     first error in file order for the line-by-line checks, then the
//     reference's end-of-file checks (entry count, FROSTT order / declared
//     dims) in its order.  spx_text_error returns class, line and message.
// Only non-ASCII text, integers past 18 digits, orders outside 1..8 and
// dimensions beyond int32 return SPX_PARSE_DEFER (the host then runs the
// reference parser).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "spx_internal.h"

namespace spx {
namespace {

constexpr int kDefer = 1;
constexpr int kError = 2;
enum ErrKind { kTensorFileError = 1, kHeaderError = 2, kEntryBoundsError = 3, kEntryValueError = 4 };

struct ParseError {
  int kind = 0;
  int64_t line = 0;
  std::string msg;
};
thread_local ParseError g_perr;

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

// tokens of a stripped line; returns the count (records up to cap)
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

// Python repr() of an ASCII str
std::string py_repr(const char* b, const char* e) {
  bool sq = false, dq = false;
  for (const char* p = b; p < e; ++p) {
    sq |= *p == '\'';
    dq |= *p == '"';
  }
  const char q = (sq && !dq) ? '"' : '\'';
  std::string s(1, q);
  for (const char* p = b; p < e; ++p) {
    const unsigned char c = (unsigned char)*p;
    if (c == (unsigned char)q || c == '\\') {
      s += '\\';
      s += (char)c;
    } else if (c == '\t') {
      s += "\\t";
    } else if (c == '\n') {
      s += "\\n";
    } else if (c == '\r') {
      s += "\\r";
    } else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      std::snprintf(buf, sizeof(buf), "\\x%02x", c);
      s += buf;
    } else {
      s += (char)c;
    }
  }
  s += q;
  return s;
}

std::string tuple_str(const int64_t* v, int n) {
  std::string s = "(";
  for (int i = 0; i < n; ++i) {
    if (i) s += ", ";
    s += std::to_string(v[i]);
  }
  if (n == 1) s += ",";
  return s + ")";
}

// int(): 0 ok, 1 not an int literal, 2 more than 18 digits (defer)
inline int py_int(const char* b, const char* e, int64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
  if (b >= e) return 1;
  int64_t v = 0;
  int digits = 0;
  bool prev_digit = false;
  for (const char* p = b; p < e; ++p) {
    if (*p == '_') {
      if (!prev_digit || p + 1 >= e || p[1] < '0' || p[1] > '9') return 1;
      prev_digit = false;
      continue;
    }
    if (*p < '0' || *p > '9') return 1;
    prev_digit = true;
    if (digits > 0 || *p != '0') ++digits;
    if (digits > 18) return 2;
    v = v * 10 + (*p - '0');
  }
  *out = neg ? -v : v;
  return 0;
}

// a run of digits with single underscores between digits; returns the end
inline const char* digitpart(const char* p, const char* e, std::string* out) {
  const char* s = p;
  while (p < e) {
    if (*p >= '0' && *p <= '9') {
      *out += *p++;
    } else if (*p == '_' && p > s && p[-1] >= '0' && p[-1] <= '9' && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      ++p;
    } else {
      break;
    }
  }
  return p;
}

// float(): [+-](digitpart[.digitpart?]|.digitpart)([eE][+-]digitpart)? | [+-](inf|infinity|nan)
inline bool py_float(const char* b, const char* e, double* out) {
  std::string s;
  const char* p = b;
  if (p < e && (*p == '+' || *p == '-')) s += *p++;
  {  // special values
    std::string low;
    for (const char* q = p; q < e && low.size() < 9; ++q) low += (char)((*q >= 'A' && *q <= 'Z') ? *q - 'A' + 'a' : *q);
    const size_t rest = (size_t)(e - p);
    if ((rest == 3 && (low == "inf" || low == "nan")) || (rest == 8 && low == "infinity")) {
      *out = std::strtod((s + low).c_str(), nullptr);
      return true;
    }
  }
  const size_t n0 = s.size();
  p = digitpart(p, e, &s);
  size_t mant = s.size() - n0;
  if (p < e && *p == '.') {
    s += *p++;
    const size_t before = s.size();
    p = digitpart(p, e, &s);
    mant += s.size() - before;
  }
  if (mant == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    s += *p++;
    if (p < e && (*p == '+' || *p == '-')) s += *p++;
    const size_t before = s.size();
    p = digitpart(p, e, &s);
    if (s.size() == before) return false;
  }
  if (p != e) return false;
  *out = std::strtod(s.c_str(), nullptr);
  return true;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;          // line count inside the chunk
  int64_t entries = 0;        // data lines
  int64_t first_tokens = -1;  // token count of the first data line (FROSTT order)
  int dims_n = -1;            // last valid '# dims:' comment in the chunk
  int64_t dims[8];
  bool defer = false;
  int64_t maxc[8];
  // first line-by-line error of the chunk (line relative to the chunk start)
  int64_t err_rel = -1;
  int err_kind = 0;
  std::string err_msg;
  // first entry outside the declared FROSTT dims (entry index, line, 1-based coords)
  int64_t oob_rel_line = -1;
  int64_t oob_coords[8];
  bool dims_seen = false;  // a valid FROSTT '# dims:' comment
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

// '# dims:' comment (b..e stripped, starts with '#'): returns false when the
// comment is not a dims line; else *nd = count (or -1 when a token is not an
// int: *bad names it; -2 when a token needs the reference, >8 tokens too)
bool comment_dims(const char* b, const char* e, int64_t* dims, int* nd, const char** bad_b, const char** bad_e) {
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
  for (int i = 0; i < std::min(n, 9); ++i) {
    int64_t v;
    const int r = py_int(tb[i], te[i], &v);
    if (r == 1) {
      *nd = -1;
      *bad_b = tb[i];
      *bad_e = te[i];
      return true;
    }
    if (r == 2) {
      *nd = -2;
      return true;
    }
    if (i < 8) dims[i] = v;
  }
  *nd = n > 8 ? -2 : n;
  return true;
}

int raise_err(int kind, int64_t line, std::string msg) {
  g_perr.kind = kind;
  g_perr.line = line;
  g_perr.msg = std::move(msg);
  return kError;
}

// the record of the first line-by-line error in chunk c (relative line ln)
inline void chunk_err(Chunk& c, int64_t ln, int kind, std::string msg) {
  if (c.err_rel < 0) {
    c.err_rel = ln;
    c.err_kind = kind;
    c.err_msg = std::move(msg);
  }
}

// Matrix Market header + size line.  Returns 0 (body / body_line / dims set),
// kError or kDefer.
int mm_header(const char* text, const char* end, const char** body, int64_t* body_line, int64_t* dims) {
  const char *b, *e;
  if (text == end) return raise_err(kHeaderError, 1, "empty file");
  const char* p = next_line(text, end, &b, &e);
  strip(&b, &e);
  const char hdr[] = "%%matrixmarket matrix coordinate real general";
  bool ok = (size_t)(e - b) == sizeof(hdr) - 1;
  for (size_t i = 0; ok && i < sizeof(hdr) - 1; ++i) {
    char c = b[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    ok = c == hdr[i];
  }
  if (!ok) return raise_err(kHeaderError, 1, "expected '%%MatrixMarket matrix coordinate real general' header");
  int64_t lineno = 1;
  while (p < end) {
    p = next_line(p, end, &b, &e);
    ++lineno;
    strip(&b, &e);
    if (b == e || *b == '%') continue;
    const char* tb[4];
    const char* te[4];
    if (tokens(b, e, tb, te, 4) != 3) return raise_err(kHeaderError, lineno, "size line must be 'rows cols nnz'");
    for (int i = 0; i < 3; ++i) {
      const int r = py_int(tb[i], te[i], &dims[i]);
      if (r == 2) return kDefer;
      if (r == 1) return raise_err(kEntryValueError, lineno, "non-numeric size " + py_repr(tb[i], te[i]));
    }
    *body = p;
    *body_line = lineno;
    return 0;
  }
  return raise_err(kHeaderError, lineno, "missing 'rows cols nnz' size line");
}

}  // namespace
}  // namespace spx

using namespace spx;

extern "C" {

// Pass 1: order, data-line count and dims (Matrix Market: rows, cols and the
// declared nnz in dims[2]; FROSTT: the last '# dims:' or -1 = infer).
// Returns 0, SPX_PARSE_DEFER (1) or SPX_PARSE_ERROR (2: spx_text_error).
int spx_text_scan(const char* text, int64_t len, int32_t fmt, int32_t* order_out, int64_t* n_out,
                  int64_t* dims_out) {
  const char* end = text + len;
  for (int64_t i = 0; i < len; ++i)
    if ((unsigned char)text[i] >= 0x80 || text[i] == 0) return kDefer;
  const char* body = text;
  if (fmt == 0) {
    int64_t body_line = 0;
    if (int r = mm_header(text, end, &body, &body_line, dims_out)) return r;
    if (dims_out[0] > INT32_MAX || dims_out[1] > INT32_MAX) return kDefer;
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
          int nd = 0;
          int64_t d[8];
          const char *bb = nullptr, *be = nullptr;
          if (comment_dims(b, e, d, &nd, &bb, &be)) {
            if (nd == -2) c.defer = true;
            if (nd >= 0) {
              c.dims_n = nd;
              std::memcpy(c.dims, d, sizeof(d));
            }
          }
        }
        continue;
      }
      if (c.first_tokens < 0) c.first_tokens = tokens(b, e, nullptr, nullptr, 0);
      ++c.entries;
    }
  });
  int64_t n = 0, first_tokens = -1;
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
  if (fmt == 0) return SPX_OK;
  // FROSTT: the first data line fixes the order (a line with < 2 tokens is
  // an error the parse pass reports at that line)
  int order = first_tokens >= 2 ? (int)first_tokens - 1 : (first_tokens >= 0 ? 1 : dims_n);
  if (first_tokens >= 0 && first_tokens - 1 > 8) return kDefer;
  if (first_tokens < 0 && dims_n < 0) order = 1;  // empty: the parse pass reports it after any line error
  if (order < 1) return kDefer;                    // order 0 ('# dims:' with no sizes)
  for (int l = 0; l < dims_n; ++l)
    if (dims[l] > (int64_t)INT32_MAX) return kDefer;
  *order_out = order;
  for (int l = 0; l < order; ++l) dims_out[l] = (dims_n == order) ? dims[l] : -1;
  if (dims_n >= 0 && dims_n != order) dims_out[0] = -2 - dims_n;  // order mismatch: reported after the parse
  return SPX_OK;
}

// Pass 2: coordinates (0-based, level-major: coords[l*n + i]) and values in
// file order, with the reference's line-by-line and end-of-file checks.
// dims: as spx_text_scan reported (FROSTT -1 = infer; the inferred maxima
// are written back).  Returns 0, SPX_PARSE_DEFER or SPX_PARSE_ERROR.
int spx_text_parse(const char* text, int64_t len, int32_t fmt, int32_t order, int64_t n, int64_t* dims,
                   int32_t* coords, double* vals) {
  const char* end = text + len;
  const char* body = text;
  int64_t body_line = 0;  // lines before the body
  int64_t mm[3] = {0, 0, 0};
  if (fmt == 0) {
    if (int r = mm_header(text, end, &body, &body_line, mm)) return r;
  }
  std::vector<Chunk> cs = split(body, end, nthreads_for((size_t)(end - body)));
  const char cc = fmt == 0 ? '%' : '#';
  parallel(cs, [&](Chunk& c) {  // entry offsets and line counts per chunk
    const char* p = c.b;
    while (p < c.e) {
      const char *b, *e;
      p = next_line(p, c.e, &b, &e);
      ++c.lines;
      strip(&b, &e);
      if (b == e || *b == cc) continue;
      ++c.entries;
    }
  });
  std::vector<int64_t> off(cs.size() + 1, 0), line0(cs.size() + 1, body_line);
  for (size_t i = 0; i < cs.size(); ++i) {
    off[i + 1] = off[i] + cs[i].entries;
    line0[i + 1] = line0[i] + cs[i].lines;
  }
  if (off.back() != n) return kDefer;
  const int64_t total_lines = line0.back();
  const bool frostt_declared = fmt == 1 && dims[0] >= 0;
  const int frostt_mismatch = (fmt == 1 && dims[0] <= -2) ? (int)(-2 - dims[0]) : -1;
  auto work = [&](size_t ci) {
    Chunk& c = cs[ci];
    for (int l = 0; l < order; ++l) c.maxc[l] = 0;
    int64_t k = off[ci], ln = 0;
    const char* p = c.b;
    const char* tb[10];
    const char* te[10];
    while (p < c.e) {
      const char *b, *e;
      p = next_line(p, c.e, &b, &e);
      ++ln;
      strip(&b, &e);
      if (b == e) continue;
      if (*b == cc) {
        if (fmt == 1) {
          int nd = 0;
          int64_t d[8];
          const char *bb = nullptr, *be = nullptr;
          if (comment_dims(b, e, d, &nd, &bb, &be)) {
            if (nd == -1) {
              chunk_err(c, ln, kEntryValueError, "non-numeric dimension " + py_repr(bb, be));
              return;
            }
            c.dims_seen = true;
          }
        }
        continue;
      }
      const int nt = tokens(b, e, tb, te, 10);
      const int64_t kk = k++;
      if (fmt == 0) {
        if (nt != 3) {
          chunk_err(c, ln, kEntryValueError, "expected 'i j value', found " + py_repr(b, e));
          return;
        }
      } else {
        if (nt < 2) {
          chunk_err(c, ln, kEntryValueError, "expected 'i1 ... ik value', found " + py_repr(b, e));
          return;
        }
        if (nt - 1 != order) {
          chunk_err(c, ln, kEntryValueError,
                    "entry has " + std::to_string(nt - 1) + " coordinates, expected " + std::to_string(order));
          return;
        }
      }
      int64_t cv[8];
      for (int l = 0; l < order; ++l) {
        const int r = py_int(tb[l], te[l], &cv[l]);
        if (r == 2) {
          c.defer = true;
          return;
        }
        if (r == 1) {
          chunk_err(c, ln, kEntryValueError, "non-numeric coordinate " + py_repr(tb[l], te[l]));
          return;
        }
      }
      if (!py_float(tb[order], te[order], &vals[kk])) {
        chunk_err(c, ln, kEntryValueError, "non-numeric value " + py_repr(tb[order], te[order]));
        return;
      }
      if (fmt == 0) {
        if (!(1 <= cv[0] && cv[0] <= mm[0] && 1 <= cv[1] && cv[1] <= mm[1])) {
          chunk_err(c, ln, kEntryBoundsError,
                    "coordinate (" + std::to_string(cv[0]) + ", " + std::to_string(cv[1]) + ") outside declared " +
                        std::to_string(mm[0]) + "x" + std::to_string(mm[1]));
          return;
        }
      } else {
        for (int l = 0; l < order; ++l)
          if (cv[l] < 1) {
            chunk_err(c, ln, kEntryBoundsError, "coordinates are 1-based, found " + tuple_str(cv, order));
            return;
          }
        if (frostt_declared && c.oob_rel_line < 0) {
          for (int l = 0; l < order; ++l)
            if (cv[l] > dims[l]) {
              c.oob_rel_line = ln;
              std::memcpy(c.oob_coords, cv, sizeof(cv));
              break;
            }
        }
        for (int l = 0; l < order; ++l)
          if (cv[l] - 1 > INT32_MAX) {
            c.defer = true;
            return;
          }
      }
      for (int l = 0; l < order; ++l) {
        coords[(int64_t)l * n + kk] = (int32_t)(cv[l] - 1);
        if (cv[l] > c.maxc[l]) c.maxc[l] = cv[l];
      }
    }
  };
  std::vector<std::thread> th;
  for (size_t i = 1; i < cs.size(); ++i) th.emplace_back(work, i);
  if (!cs.empty()) work(0);
  for (auto& t : th) t.join();
  // the first line-by-line error in file order (chunks are in file order)
  for (size_t i = 0; i < cs.size(); ++i) {
    if (cs[i].err_rel >= 0) return raise_err(cs[i].err_kind, line0[i] + cs[i].err_rel, cs[i].err_msg);
    if (cs[i].defer) return kDefer;
  }
  if (fmt == 0) {
    if (n != mm[2]) {
      // the reference reports the last line it visited
      return raise_err(kTensorFileError, total_lines,
                       "size line declared " + std::to_string(mm[2]) + " entries but file has " + std::to_string(n));
    }
    return SPX_OK;
  }
  bool dims_seen = false;
  for (auto& c : cs) dims_seen |= c.dims_seen;
  if (n == 0 && !dims_seen) return raise_err(kHeaderError, 1, "empty tensor file with no '# dims:' line");
  if (frostt_mismatch >= 0)
    return raise_err(kHeaderError, 1,
                     "'# dims:' declares order " + std::to_string(frostt_mismatch) + " but entries have order " +
                         std::to_string(order));
  if (frostt_declared) {
    for (size_t i = 0; i < cs.size(); ++i)
      if (cs[i].oob_rel_line >= 0) {
        int64_t d[8];
        for (int l = 0; l < order; ++l) d[l] = dims[l];
        return raise_err(kEntryBoundsError, line0[i] + cs[i].oob_rel_line,
                         "coordinate " + tuple_str(cs[i].oob_coords, order) + " outside declared dims " +
                             tuple_str(d, order));
      }
    return SPX_OK;
  }
  for (int l = 0; l < order; ++l) {
    int64_t m = 0;
    for (auto& c : cs)
      if (c.entries) m = std::max(m, c.maxc[l]);
    dims[l] = m;  // max 1-based coordinate == max 0-based + 1
  }
  return SPX_OK;
}

// The last SPX_PARSE_ERROR on this thread: kind 1 TensorFileError,
// 2 HeaderError, 3 EntryBoundsError, 4 EntryValueError; 1-based line; the
// reference's message (without the "line N: " prefix its class adds).
int spx_text_error(int32_t* kind, int64_t* line, char* msg, int64_t cap) {
  if (kind) *kind = g_perr.kind;
  if (line) *line = g_perr.line;
  if (msg && cap > 0) {
    const size_t k = std::min<size_t>((size_t)cap - 1, g_perr.msg.size());
    std::memcpy(msg, g_perr.msg.data(), k);
    msg[k] = 0;
  }
  return (int)g_perr.msg.size();
}

}  // extern "C"
