// Host-side Matrix Market / vector file I/O and COO -> CSR (replaces
// sparse.py:58-75 `from_coo` and sparse.py:270-330 `read_matrix_market`,
// `write_matrix_market`, `read_vector`, `write_vector`).
//
// Same accepted format and the same error texts as the reference (coordinate
// real general|symmetric, comment lines before the size line, exactly nnz
// entry lines, 1-based indices, symmetric off-diagonals mirrored), but the
// file is read once into memory and parsed / formatted by all host threads:
// the reference's per-line Python loop would need hours for the 1.7e9-entry
// C3 matrix.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/spai_b200.h"

namespace spai {
void set_error(const char* fmt, ...);
}
using spai::set_error;

namespace {

int hw_threads(int want) {
  if (want > 0) return want;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 64u) : 1;
}

bool slurp(const char* path, std::string* out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out->resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? std::fread(&(*out)[0], 1, (size_t)sz, f) : 0;
  std::fclose(f);
  return got == out->size();
}

// next line [b, e) starting at p; returns the position after the newline
size_t next_line(const std::string& s, size_t p, size_t* b, size_t* e) {
  *b = p;
  const void* nl = std::memchr(s.data() + p, '\n', s.size() - p);
  const size_t q = nl ? (size_t)((const char*)nl - s.data()) : s.size();
  *e = q;
  return nl ? q + 1 : q;
}

std::string trimmed(const std::string& s, size_t b, size_t e) {
  while (b < e && std::isspace((unsigned char)s[b])) ++b;
  while (e > b && std::isspace((unsigned char)s[e - 1])) --e;
  return s.substr(b, e - b);
}

struct Header {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int symmetric = 0;
  size_t body = 0;     // offset of the first entry line
};

std::string lower(std::string t) {
  for (auto& c : t) c = (char)std::tolower((unsigned char)c);
  return t;
}

int parse_header(const std::string& s, Header* h) {
  size_t b, e;
  size_t p = next_line(s, 0, &b, &e);
  const std::string head = trimmed(s, b, e);
  std::vector<std::string> parts;
  {
    size_t i = 0;
    while (i < head.size()) {
      while (i < head.size() && std::isspace((unsigned char)head[i])) ++i;
      size_t j = i;
      while (j < head.size() && !std::isspace((unsigned char)head[j])) ++j;
      if (j > i) parts.push_back(head.substr(i, j - i));
      i = j;
    }
  }
  if (parts.size() != 5 || parts[0] != "%%MatrixMarket" || lower(parts[1]) != "matrix" ||
      lower(parts[2]) != "coordinate" || lower(parts[3]) != "real" ||
      (lower(parts[4]) != "general" && lower(parts[4]) != "symmetric")) {
    set_error("malformed header: '%s'", head.c_str());
    return SPAI_E_FORMAT;
  }
  h->symmetric = lower(parts[4]) == "symmetric";
  do {
    p = next_line(s, p, &b, &e);
  } while (b < s.size() && s[b] == '%');
  const std::string sz = trimmed(s, b, e);
  long long a[3];
  int cnt = 0;
  const char* c = sz.c_str();
  while (cnt < 4) {
    while (*c && std::isspace((unsigned char)*c)) ++c;
    if (!*c) break;
    char* end = nullptr;
    errno = 0;
    const long long v = std::strtoll(c, &end, 10);
    if (end == c || errno || (*end && !std::isspace((unsigned char)*end))) { cnt = -1; break; }
    if (cnt < 3) a[cnt] = v;
    ++cnt;
    c = end;
  }
  if (cnt != 3) {
    set_error("bad size line: '%s'", sz.c_str());
    return SPAI_E_FORMAT;
  }
  h->nrows = a[0];
  h->ncols = a[1];
  h->nnz = a[2];
  h->body = p;
  return SPAI_OK;
}

// entry line -> (i, j, v); false when it does not hold exactly 3 tokens
bool parse_entry(const char* b, const char* e, long long* i, long long* j, double* v) {
  const char* c = b;
  auto skip = [&]() { while (c < e && (*c == ' ' || *c == '\t' || *c == '\r')) ++c; };
  char* end = nullptr;
  skip();
  if (c >= e) return false;
  *i = std::strtoll(c, &end, 10);
  if (end == c) return false;
  c = end;
  skip();
  if (c >= e) return false;
  *j = std::strtoll(c, &end, 10);
  if (end == c) return false;
  c = end;
  skip();
  if (c >= e) return false;
  *v = std::strtod(c, &end);
  if (end == c) return false;
  c = end;
  skip();
  return c >= e;
}

}  // namespace

extern "C" int spai_mm_read_header(const char* path, int64_t* nrows, int64_t* ncols,
                                   int64_t* nnz, int* symmetric) {
  std::string s;
  FILE* f = std::fopen(path, "rb");
  if (!f) { set_error("cannot open %s", path); return SPAI_E_ARG; }
  char buf[1 << 16];
  const size_t got = std::fread(buf, 1, sizeof(buf), f);
  std::fclose(f);
  s.assign(buf, got);
  Header h;
  // the header block may be longer than the probe: retry on the whole file
  int st = parse_header(s, &h);
  if (st != SPAI_OK && got == sizeof(buf)) {
    if (!slurp(path, &s)) { set_error("cannot read %s", path); return SPAI_E_ARG; }
    st = parse_header(s, &h);
  }
  if (st) return st;
  *nrows = h.nrows;
  *ncols = h.ncols;
  *nnz = h.nnz;
  *symmetric = h.symmetric;
  return SPAI_OK;
}

// COO entries (0-based, symmetric off-diagonals mirrored right after their
// entry, file order): rows/cols/vals need room for 2 * nnz (symmetric) or nnz.
extern "C" int spai_mm_read_coo(const char* path, int64_t* rows, int64_t* cols, double* vals,
                                int64_t* count, int nthreads) {
  std::string s;
  if (!slurp(path, &s)) { set_error("cannot read %s", path); return SPAI_E_ARG; }
  Header h;
  if (int st = parse_header(s, &h)) return st;
  // line starts of the nnz entry lines
  std::vector<size_t> lb;
  lb.reserve((size_t)std::max<int64_t>(h.nnz, 0) + 1);
  size_t p = h.body;
  for (int64_t k = 0; k < h.nnz; ++k) {
    if (p >= s.size()) { set_error("truncated entry line"); return SPAI_E_FORMAT; }
    lb.push_back(p);
    const void* nl = std::memchr(s.data() + p, '\n', s.size() - p);
    p = nl ? (size_t)((const char*)nl - s.data()) + 1 : s.size();
  }
  lb.push_back(p);
  const int T = hw_threads(nthreads);
  const int64_t n = h.nnz;
  // per-thread: entry range, output count, first error (entry index, kind)
  std::vector<int64_t> cnt(T, 0), err_at(T, -1), err_i(T, 0), err_j(T, 0);
  std::vector<int> err_kind(T, 0);
  auto work = [&](int t, bool count_only, int64_t base) {
    const int64_t k0 = n * t / T, k1 = n * (t + 1) / T;
    int64_t o = base;
    for (int64_t k = k0; k < k1; ++k) {
      const char* b = s.data() + lb[k];
      const char* e = s.data() + lb[k + 1];
      if (e > b && e[-1] == '\n') --e;
      long long i, j;
      double v;
      if (!parse_entry(b, e, &i, &j, &v)) {
        if (err_at[t] < 0) { err_at[t] = k; err_kind[t] = 1; }
        return;
      }
      --i;
      --j;
      if (!(0 <= i && i < h.nrows && 0 <= j && j < h.ncols)) {
        if (err_at[t] < 0) { err_at[t] = k; err_kind[t] = 2; err_i[t] = i; err_j[t] = j; }
        return;
      }
      if (count_only) {
        o += (h.symmetric && i != j) ? 2 : 1;
        continue;
      }
      rows[o] = i; cols[o] = j; vals[o] = v; ++o;
      if (h.symmetric && i != j) { rows[o] = j; cols[o] = i; vals[o] = v; ++o; }
    }
    if (count_only) cnt[t] = o - base;
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(work, t, true, 0);
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < T; ++t)
    if (err_at[t] >= 0) {
      if (err_kind[t] == 1) set_error("truncated entry line");
      else set_error("index out of range: (%lld, %lld)", (long long)err_i[t] + 1, (long long)err_j[t] + 1);
      return SPAI_E_FORMAT;
    }
  std::vector<int64_t> off(T + 1, 0);
  for (int t = 0; t < T; ++t) off[t + 1] = off[t] + cnt[t];
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(work, t, false, off[t]);
    for (auto& x : th) x.join();
  }
  *count = off[T];
  return SPAI_OK;
}

// COO -> CSR with the reference's from_coo semantics: entries ordered by
// (row, col), duplicates rejected (first duplicate in that order reported).
// rowptr[nrows+1], out_cols[count], out_vals[count].
extern "C" int spai_coo_to_csr(int64_t nrows, int64_t count, const int64_t* rows,
                               const int64_t* cols, const double* vals, int64_t* rowptr,
                               int64_t* out_cols, double* out_vals, int nthreads) {
  for (int64_t r = 0; r <= nrows; ++r) rowptr[r] = 0;
  for (int64_t k = 0; k < count; ++k) {
    if (rows[k] < 0 || rows[k] >= nrows) { set_error("row index %lld out of range", (long long)rows[k]); return SPAI_E_ARG; }
    ++rowptr[rows[k] + 1];
  }
  for (int64_t r = 0; r < nrows; ++r) rowptr[r + 1] += rowptr[r];
  std::vector<int64_t> fill(rowptr, rowptr + nrows);
  for (int64_t k = 0; k < count; ++k) {       // stable placement in file order
    const int64_t q = fill[rows[k]]++;
    out_cols[q] = cols[k];
    out_vals[q] = vals[k];
  }
  const int T = hw_threads(nthreads);
  std::vector<int64_t> dup_row(T, -1), dup_col(T, -1);
  auto work = [&](int t) {
    std::vector<std::pair<int64_t, double>> tmp;
    for (int64_t r = nrows * t / T; r < nrows * (t + 1) / T; ++r) {
      const int64_t lo = rowptr[r], hi = rowptr[r + 1];
      bool sorted = true;
      for (int64_t q = lo + 1; q < hi; ++q) if (out_cols[q] <= out_cols[q - 1]) { sorted = false; break; }
      if (!sorted) {
        tmp.resize((size_t)(hi - lo));
        for (int64_t q = lo; q < hi; ++q) tmp[q - lo] = {out_cols[q], out_vals[q]};
        std::stable_sort(tmp.begin(), tmp.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
        for (int64_t q = lo; q < hi; ++q) { out_cols[q] = tmp[q - lo].first; out_vals[q] = tmp[q - lo].second; }
        for (int64_t q = lo + 1; q < hi; ++q)
          if (out_cols[q] == out_cols[q - 1]) {
            if (dup_row[t] < 0) { dup_row[t] = r; dup_col[t] = out_cols[q]; }
            return;
          }
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back(work, t);
  for (auto& x : th) x.join();
  for (int t = 0; t < T; ++t)
    if (dup_row[t] >= 0) {
      set_error("duplicate entry at (%lld, %lld)", (long long)dup_row[t], (long long)dup_col[t]);
      return SPAI_E_FORMAT;
    }
  return SPAI_OK;
}

// %%MatrixMarket matrix coordinate real general, one "i j v" line per stored
// entry in CSR order, values as %.17g (sparse.py:311-318)
extern "C" int spai_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* rowptr,
                             const int64_t* colidx, const double* vals, int nthreads) {
  FILE* f = std::fopen(path, "wb");
  if (!f) { set_error("cannot open %s for writing", path); return SPAI_E_ARG; }
  const int64_t nnz = rowptr[nrows];
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
               (long long)nrows, (long long)ncols, (long long)nnz);
  const int T = hw_threads(nthreads);
  constexpr int64_t kRowsPerChunk = 1 << 16;
  const int64_t nchunks = (nrows + kRowsPerChunk - 1) / kRowsPerChunk;
  int rc = SPAI_OK;
  for (int64_t c0 = 0; c0 < nchunks && rc == SPAI_OK; c0 += T) {
    const int64_t c1 = std::min<int64_t>(nchunks, c0 + T);
    std::vector<std::string> out((size_t)(c1 - c0));
    std::vector<std::thread> th;
    for (int64_t c = c0; c < c1; ++c)
      th.emplace_back([&, c]() {
        std::string& o = out[c - c0];
        char line[96];
        const int64_t r1 = std::min(nrows, (c + 1) * kRowsPerChunk);
        for (int64_t r = c * kRowsPerChunk; r < r1; ++r)
          for (int64_t q = rowptr[r]; q < rowptr[r + 1]; ++q) {
            const int len = std::snprintf(line, sizeof(line), "%lld %lld %.17g\n", (long long)r + 1,
                                          (long long)colidx[q] + 1, vals[q]);
            o.append(line, (size_t)len);
          }
      });
    for (auto& x : th) x.join();
    for (auto& o : out)
      if (std::fwrite(o.data(), 1, o.size(), f) != o.size()) { rc = SPAI_E_ARG; break; }
  }
  if (std::fclose(f) != 0 || rc != SPAI_OK) { set_error("write to %s failed", path); return SPAI_E_ARG; }
  return SPAI_OK;
}

// one value per line, %.17g (sparse.py:325-329)
extern "C" int spai_vec_write(const char* path, int64_t n, const double* x) {
  FILE* f = std::fopen(path, "wb");
  if (!f) { set_error("cannot open %s for writing", path); return SPAI_E_ARG; }
  for (int64_t i = 0; i < n; ++i) std::fprintf(f, "%.17g\n", x[i]);
  if (std::fclose(f) != 0) { set_error("write to %s failed", path); return SPAI_E_ARG; }
  return SPAI_OK;
}

// whitespace-separated values (np.loadtxt(path, ndmin=1) on a one-column
// file); *n = values found (at most cap written).  Comment lines ('#') skipped.
extern "C" int spai_vec_read(const char* path, double* x, int64_t cap, int64_t* n) {
  std::string s;
  if (!slurp(path, &s)) { set_error("cannot read %s", path); return SPAI_E_ARG; }
  int64_t k = 0;
  const char* c = s.c_str();
  const char* end = c + s.size();
  while (c < end) {
    while (c < end && std::isspace((unsigned char)*c)) ++c;
    if (c >= end) break;
    if (*c == '#') {
      while (c < end && *c != '\n') ++c;
      continue;
    }
    char* e = nullptr;
    const double v = std::strtod(c, &e);
    if (e == c) { set_error("could not convert string to float"); return SPAI_E_FORMAT; }
    if (k < cap) x[k] = v;
    ++k;
    c = e;
  }
  *n = k;
  return SPAI_OK;
}
