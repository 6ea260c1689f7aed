// Matrix Market ingest (reference pkg/src/trisolve/mmio.py:41-156).
//
// Host side: a native parser with the reference's acceptance rules and error
// texts ("line N: ..."; Python int()/float() token grammar including digit
// underscores, utf-8 BOM, comment / blank-line skipping, header validation,
// entry-count and index checks, symmetric / skew-symmetric lower-triangle
// rules).  Entries are parsed in parallel over line chunks.
// Device side (ts_mm_to_device): the coordinate triplets go to HBM once and
// the CSR is assembled there — symmetric mirroring, a stable radix sort on the
// (row, col) key, duplicate summation in file order, row pointers — then the
// normal CSR handle (transpose, plans) is built from device pointers, so no
// host CSR conversion or second transfer sits on the ingest path.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

namespace ts {

struct MmParsed {
  int fmt = 0;    // 0 coordinate, 1 array
  int field = 0;  // 0 real, 1 integer, 2 pattern
  int sym = 0;    // 0 general, 1 symmetric, 2 skew-symmetric
  int64_t m = 0, n = 0, entries = 0;
  // coordinate: the file's entries, 0-based, in file order (not mirrored)
  std::vector<int32_t> ri, ci;
  std::vector<double> v;
  // array: the values in file (column-major, triangle) order
  std::vector<double> vals;
};

// Python repr() of a str token (quotes chosen like CPython's)
inline std::string py_repr(const std::string& s) {
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string r(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      r += '\\';
      r += (char)c;
    } else if (c == '\t') {
      r += "\\t";
    } else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof(b), "\\x%02x", c);
      r += b;
    } else {
      r += (char)c;
    }
  }
  r += q;
  return r;
}

inline bool mm_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || c == 0x1c ||
         c == 0x1d || c == 0x1e || c == 0x1f;
}

// digits with single underscores between digits (PEP 515)
inline bool mm_digits(const std::string& s, size_t& i) {
  if (i >= s.size() || !isdigit((unsigned char)s[i])) return false;
  ++i;
  while (i < s.size()) {
    if (isdigit((unsigned char)s[i])) {
      ++i;
    } else if (s[i] == '_' && i + 1 < s.size() && isdigit((unsigned char)s[i + 1])) {
      i += 2;
    } else {
      break;
    }
  }
  return true;
}

// Python int(token): [+-]? digits (underscores allowed)
inline bool mm_int(const std::string& t, int64_t* out) {
  size_t i = 0;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) ++i;
  const size_t d0 = i;
  if (!mm_digits(t, i) || i != t.size()) return false;
  std::string clean;
  for (size_t k = d0; k < t.size(); ++k)
    if (t[k] != '_') clean += t[k];
  errno = 0;
  long long v = strtoll(clean.c_str(), nullptr, 10);
  if (errno == ERANGE) v = (long long)INT64_MAX;  // far outside any index range
  *out = (t[0] == '-') ? -v : v;
  return true;
}

// Python float(token): decimal / inf / infinity / nan (any case, signed)
inline bool mm_float(const std::string& t, double* out) {
  size_t i = 0;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) ++i;
  std::string rest = t.substr(i);
  std::string low;
  for (char c : rest) low += (char)tolower((unsigned char)c);
  if (low == "inf" || low == "infinity" || low == "nan") {
    *out = strtod(t.c_str(), nullptr);
    if (low == "nan") *out = NAN;
    return true;
  }
  size_t j = i;
  bool any = false;
  if (j < t.size() && isdigit((unsigned char)t[j])) {
    mm_digits(t, j);
    any = true;
  }
  if (j < t.size() && t[j] == '.') {
    ++j;
    if (j < t.size() && isdigit((unsigned char)t[j])) {
      mm_digits(t, j);
      any = true;
    }
  }
  if (!any) return false;
  if (j < t.size() && (t[j] == 'e' || t[j] == 'E')) {
    ++j;
    if (j < t.size() && (t[j] == '+' || t[j] == '-')) ++j;
    if (!mm_digits(t, j)) return false;
  }
  if (j != t.size()) return false;
  std::string clean;
  for (char c : t)
    if (c != '_') clean += c;
  *out = strtod(clean.c_str(), nullptr);  // correctly rounded, as CPython's
  return true;
}

struct MmLine {
  int64_t no;  // 1-based line number
  const char* p;
  size_t len;
};

inline void mm_tokens(const char* p, size_t len, std::vector<std::string>* out) {
  out->clear();
  size_t i = 0;
  while (i < len) {
    while (i < len && mm_ws((unsigned char)p[i])) ++i;
    if (i >= len) break;
    size_t j = i;
    while (j < len && !mm_ws((unsigned char)p[j])) ++j;
    out->emplace_back(p + i, j - i);
    i = j;
  }
}

inline int mm_fail(int64_t line, const std::string& msg) {
  set_error("line %lld: %s", (long long)line, msg.c_str());
  return TS_EINVAL;
}

// Parse a whole file image.  Returns 0 or TS_EINVAL with "line N: ...".
inline int mm_parse(const char* data, size_t len, MmParsed* P) {
  // utf-8 byte-order mark ahead of the banner
  if (len >= 3 && (unsigned char)data[0] == 0xEF && (unsigned char)data[1] == 0xBB &&
      (unsigned char)data[2] == 0xBF) {
    data += 3;
    len -= 3;
  }
  // str.splitlines() on the ASCII line boundaries
  std::vector<MmLine> lines;
  {
    size_t s = 0;
    int64_t no = 1;
    for (size_t i = 0; i < len; ++i) {
      const unsigned char c = (unsigned char)data[i];
      if (c == '\n' || c == '\r' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e) {
        lines.push_back({no++, data + s, i - s});
        if (c == '\r' && i + 1 < len && data[i + 1] == '\n') ++i;
        s = i + 1;
      }
    }
    if (s < len) lines.push_back({no++, data + s, len - s});
  }
  if (lines.empty()) return mm_fail(1, "empty input");
  std::vector<std::string> tk;
  mm_tokens(lines[0].p, lines[0].len, &tk);
  if (tk.empty() || tk[0] != "%%MatrixMarket") return mm_fail(1, "header must begin with '%%MatrixMarket'");
  if (tk.size() != 5) return mm_fail(1, "header needs 5 tokens: banner, object, format, field, symmetry");
  for (size_t k = 1; k < 5; ++k)
    for (auto& c : tk[k]) c = (char)tolower((unsigned char)c);
  if (tk[1] != "matrix") return mm_fail(1, "unsupported object " + py_repr(tk[1]) + ", only 'matrix' is handled");
  if (tk[2] == "coordinate") P->fmt = 0;
  else if (tk[2] == "array") P->fmt = 1;
  else return mm_fail(1, "unknown format " + py_repr(tk[2]));
  if (tk[3] == "complex") return mm_fail(1, "complex matrices are not supported");
  if (tk[3] == "real") P->field = 0;
  else if (tk[3] == "integer") P->field = 1;
  else if (tk[3] == "pattern") P->field = 2;
  else return mm_fail(1, "unknown field " + py_repr(tk[3]));
  if (tk[4] == "hermitian") return mm_fail(1, "hermitian implies complex data, which is not supported");
  if (tk[4] == "general") P->sym = 0;
  else if (tk[4] == "symmetric") P->sym = 1;
  else if (tk[4] == "skew-symmetric") P->sym = 2;
  else return mm_fail(1, "unknown symmetry " + py_repr(tk[4]));
  if (P->fmt == 1 && P->field == 2) return mm_fail(1, "array format cannot carry a pattern field");
  // body: skip blank lines and comment lines after the banner
  std::vector<MmLine> body;
  body.reserve(lines.size());
  for (size_t k = 1; k < lines.size(); ++k) {
    const MmLine& L = lines[k];
    size_t i = 0;
    while (i < L.len && mm_ws((unsigned char)L.p[i])) ++i;
    if (i == L.len || L.p[i] == '%') continue;
    body.push_back(L);
  }
  if (body.empty()) return mm_fail(1, "missing size line");
  const int64_t sl = body[0].no;
  mm_tokens(body[0].p, body[0].len, &tk);
  int64_t m = 0, n = 0, nnz = 0;
  auto as_int = [&](const std::string& t, int64_t line, int64_t* v) -> int {
    if (!mm_int(t, v)) return mm_fail(line, "expected an integer, got " + py_repr(t));
    return 0;
  };
  if (P->fmt == 0) {
    if (tk.size() != 3) return mm_fail(sl, "coordinate size line needs 'rows cols nnz'");
    TS_CHECK(as_int(tk[0], sl, &m));
    TS_CHECK(as_int(tk[1], sl, &n));
    TS_CHECK(as_int(tk[2], sl, &nnz));
    if (m <= 0 || n <= 0 || nnz < 0) return mm_fail(sl, "matrix dimensions must be positive");
  } else {
    if (tk.size() != 2) return mm_fail(sl, "array size line needs 'rows cols'");
    TS_CHECK(as_int(tk[0], sl, &m));
    TS_CHECK(as_int(tk[1], sl, &n));
    if (m <= 0 || n <= 0) return mm_fail(sl, "matrix dimensions must be positive");
  }
  P->m = m;
  P->n = n;
  const int64_t nent = (int64_t)body.size() - 1;
  const MmLine* ent = body.data() + 1;
  int64_t expected;
  if (P->fmt == 0) {
    P->entries = nnz;
    expected = nnz;
    if (nent != nnz) {
      if (nent > nnz) return mm_fail(ent[nnz].no, "expected " + std::to_string(nnz) + " entries, found " +
                                                     std::to_string(nent));
      set_error("line end of file: expected %lld entries, found %lld", (long long)nnz, (long long)nent);
      return TS_EINVAL;
    }
  } else {
    if (P->sym == 0) {
      expected = m * n;
    } else {
      if (m != n) {
        set_error("line 2: symmetric array files must be square");
        return TS_EINVAL;
      }
      expected = P->sym == 1 ? m * (m + 1) / 2 : m * (m - 1) / 2;
    }
    P->entries = m * n;
    if (nent != expected) {
      if (nent > expected)
        return mm_fail(ent[expected].no, "expected " + std::to_string(expected) + " values, found " +
                                             std::to_string(nent));
      set_error("line end of file: expected %lld values, found %lld", (long long)expected, (long long)nent);
      return TS_EINVAL;
    }
  }
  if (m > INT32_MAX || n > INT32_MAX) return mm_fail(sl, "matrix dimensions exceed the int32 index range");
  // entries, parsed in parallel chunks; the first failing line (in file order) wins
  if (P->fmt == 0) {
    P->ri.resize(nent);
    P->ci.resize(nent);
    P->v.resize(nent);
  } else {
    P->vals.resize(nent);
  }
  const int want = P->field == 2 ? 2 : 3;
  unsigned hw = std::thread::hardware_concurrency();
  const int64_t nth = std::max<int64_t>(1, std::min<int64_t>(hw ? hw : 1, nent / 65536 + 1));
  std::vector<int64_t> bad_line(nth, -1);
  std::vector<std::string> bad_msg(nth);
  auto work = [&](int64_t t) {
    const int64_t k0 = nent * t / nth, k1 = nent * (t + 1) / nth;
    std::vector<std::string> tks;
    for (int64_t k = k0; k < k1; ++k) {
      const MmLine& L = ent[k];
      mm_tokens(L.p, L.len, &tks);
      auto fail = [&](const std::string& msg) {
        bad_line[t] = L.no;
        bad_msg[t] = msg;
      };
      if (P->fmt == 1) {
        if (tks.size() != 1) return fail("array entry needs 1 value, got " + std::to_string(tks.size()));
        double v;
        if (!mm_float(tks[0], &v)) return fail("non-numeric token " + py_repr(tks[0]));
        if (!std::isfinite(v)) return fail("non-finite value " + py_repr(tks[0]));
        P->vals[k] = v;
        continue;
      }
      if ((int)tks.size() != want)
        return fail("entry needs " + std::to_string(want) + " tokens, got " + std::to_string(tks.size()));
      int64_t i, j;
      if (!mm_int(tks[0], &i)) return fail("expected an integer, got " + py_repr(tks[0]));
      if (!mm_int(tks[1], &j)) return fail("expected an integer, got " + py_repr(tks[1]));
      if (!(1 <= i && i <= m) || !(1 <= j && j <= n))
        return fail("index (" + std::to_string(i) + ", " + std::to_string(j) + ") outside 1.." +
                    std::to_string(m) + " x 1.." + std::to_string(n));
      double v = 1.0;
      if (P->field != 2) {
        if (!mm_float(tks[2], &v)) return fail("non-numeric token " + py_repr(tks[2]));
        if (!std::isfinite(v)) return fail("non-finite value " + py_repr(tks[2]));
      }
      if (P->sym != 0) {
        const char* sname = P->sym == 1 ? "symmetric" : "skew-symmetric";
        if (i < j) return fail(std::string(sname) + " files store only the lower triangle");
        if (P->sym == 2 && i == j) return fail("skew-symmetric files cannot carry diagonal entries");
      }
      P->ri[k] = (int32_t)(i - 1);
      P->ci[k] = (int32_t)(j - 1);
      P->v[k] = v;
    }
  };
  if (nth == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nth; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  for (int64_t t = 0; t < nth; ++t)
    if (bad_line[t] >= 0) return mm_fail(bad_line[t], bad_msg[t]);
  (void)expected;
  return 0;
}

// coordinate entries expanded exactly as the reference stores them (each
// entry followed by its mirror for symmetric / skew files)
inline int64_t mm_expanded_count(const MmParsed& P) {
  if (P.sym == 0) return (int64_t)P.ri.size();
  int64_t c = 0;
  for (size_t k = 0; k < P.ri.size(); ++k) c += (P.ri[k] != P.ci[k]) ? 2 : 1;
  return c;
}

// ---- device assembly (grid-stride: launched with grid_for's capped grids) ----
__global__ void k_mm_expand(const int32_t* ri, const int32_t* ci, const double* v, const int64_t* off,
                            int64_t cnt, int sym, int64_t n, unsigned long long* key, int64_t* pos,
                            double* val) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
       k += (int64_t)gridDim.x * blockDim.x) {
  const int64_t o = off[k];
  const int32_t i = ri[k], j = ci[k];
  key[o] = (unsigned long long)i * (unsigned long long)n + (unsigned long long)j;
  pos[o] = o;
  val[o] = v[k];
  if (sym != 0 && i != j) {
    key[o + 1] = (unsigned long long)j * (unsigned long long)n + (unsigned long long)i;
    pos[o + 1] = o + 1;
    val[o + 1] = sym == 2 ? -v[k] : v[k];
  }
  }
}
__global__ void k_mm_heads(const unsigned long long* key, int64_t cnt, int* head) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
       k += (int64_t)gridDim.x * blockDim.x)
    head[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}
// one thread per unique (row, col): sum its duplicates in file order
__global__ void k_mm_unique(const unsigned long long* key, const int64_t* perm, const double* val,
                            const int* head, const int* uidx, int64_t cnt, int64_t n, int* ci_out,
                            double* v_out, int* rowcnt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (!head[k]) continue;
    const int u = uidx[k];
    double s = val[perm[k]];
    for (int64_t q = k + 1; q < cnt && !head[q]; ++q) s += val[perm[q]];
    const unsigned long long kk = key[k];
    ci_out[u] = (int)(kk % (unsigned long long)n);
    v_out[u] = s;
    atomicAdd(rowcnt + (kk / (unsigned long long)n), 1);  // integer counts: order-free
  }
}

}  // namespace ts
