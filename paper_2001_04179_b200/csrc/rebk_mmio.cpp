// rebk_mmio.cpp — native MatrixMarket reader feeding rebk_ctx_create_csr /
// rebk_ctx_create_dense (the reference's reader is
// kaczmarz/matrix_io.py:67-157, pure Python, one token at a time).
//
// Same acceptance rules and the same error texts (with the 1-based line
// number) as the reference reader:
//   banner "%%MatrixMarket matrix <coordinate|array> <real|integer|pattern>
//   <general|symmetric>"; blank lines and '%' comments skipped; size line of
//   3 (coordinate) or 2 (array) unsigned integers; entries parsed with
//   Python's int() / float() grammar (signs, '_' digit separators, inf/nan
//   spellings), non-finite values rejected, 1-based bounds checked,
//   symmetric storage given as the lower triangle and mirrored; duplicates
//   summed; the declared entry count checked.  Coordinate files whose
//   distinct positions reach `dense_threshold` of the matrix load dense
//   (np.add.at in file order, as the reference does), the others as CSR
//   with sorted columns, duplicates summed and explicit zeros dropped (the
//   reference's Matrix normalisation, matrix.py:46-58).  Duplicates are
//   summed in file order; the reference sums them in the order of scipy's
//   (unstable) index sort, so the two agree bit for bit whenever a position
//   holds at most two entries (floating-point addition commutes).
//
// Parsing runs on up to `nthreads` host threads over line-aligned chunks;
// the first error in file order is the one reported.
#include <ctype.h>
#include <limits.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rebk.h"

namespace rebk {
int set_error_msg(int code, const char* msg);
}

namespace {

// Python repr() of an ASCII str (the reference formats offending tokens /
// lines with !r)
std::string py_repr(const std::string& s) {
  const bool has_sq = s.find('\'') != std::string::npos, has_dq = s.find('"') != std::string::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == '\\') out += "\\\\";
    else if (c == (unsigned char)q) { out += '\\'; out += (char)c; }
    else if (c == '\t') out += "\\t";
    else if (c == '\n') out += "\\n";
    else if (c == '\r') out += "\\r";
    else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      out += b;
    } else out += (char)c;
  }
  out += q;
  return out;
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

std::string strip(const char* b, const char* e) {
  while (b < e && is_ws(*b)) ++b;
  while (e > b && is_ws(e[-1])) --e;
  return std::string(b, e);
}

void split_ws(const std::string& s, std::vector<std::string>& out) {
  out.clear();
  size_t i = 0, n = s.size();
  while (i < n) {
    while (i < n && is_ws(s[i])) ++i;
    size_t j = i;
    while (j < n && !is_ws(s[j])) ++j;
    if (j > i) out.emplace_back(s, i, j - i);
    i = j;
  }
}

// digits with single '_' separators between digits (PEP 515); appends the
// digits to `out`; returns false on an empty or malformed run
bool digit_run(const std::string& t, size_t& i, std::string& out) {
  size_t start = i;
  bool last_digit = false;
  while (i < t.size()) {
    const char c = t[i];
    if (c >= '0' && c <= '9') {
      out += c;
      last_digit = true;
      ++i;
    } else if (c == '_' && last_digit && i + 1 < t.size() && t[i + 1] >= '0' && t[i + 1] <= '9') {
      last_digit = false;
      ++i;
    } else {
      break;
    }
  }
  return i > start && last_digit;
}

// Python int(token) for a whitespace-free token
bool py_int(const std::string& t, long long* v) {
  size_t i = 0;
  bool neg = false;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
  std::string d;
  if (!digit_run(t, i, d) || i != t.size()) return false;
  // magnitudes beyond int64 are out of any matrix's bounds anyway
  long long acc = 0;
  for (char c : d) {
    if (acc > (LLONG_MAX - 9) / 10) {
      acc = LLONG_MAX;
      break;
    }
    acc = acc * 10 + (c - '0');
  }
  *v = neg ? -acc : acc;
  return true;
}

bool ieq(const std::string& a, const char* b) {
  if (a.size() != strlen(b)) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (tolower((unsigned char)a[i]) != b[i]) return false;
  return true;
}

// Python float(token) (decimal literals, inf/infinity/nan spellings)
bool py_float(const std::string& t, double* v) {
  size_t i = 0;
  std::string s;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) s += t[i++];
  const std::string rest = t.substr(i);
  if (ieq(rest, "inf") || ieq(rest, "infinity")) {
    *v = (s == "-") ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(rest, "nan")) {
    *v = NAN;
    return true;
  }
  bool any = false;
  if (i < t.size() && t[i] >= '0' && t[i] <= '9') {
    if (!digit_run(t, i, s)) return false;
    any = true;
  }
  if (i < t.size() && t[i] == '.') {
    s += '.';
    ++i;
    if (i < t.size() && t[i] >= '0' && t[i] <= '9') {
      if (!digit_run(t, i, s)) return false;
      any = true;
    }
  }
  if (!any) return false;
  if (i < t.size() && (t[i] == 'e' || t[i] == 'E')) {
    s += 'e';
    ++i;
    if (i < t.size() && (t[i] == '+' || t[i] == '-')) s += t[i++];
    if (!digit_run(t, i, s)) return false;
  }
  if (i != t.size()) return false;
  char* end = nullptr;
  *v = strtod(s.c_str(), &end);  // correctly rounded, like CPython's float()
  return end && *end == '\0';
}

struct Err {
  int64_t line = -1;  // -1: none
  std::string msg;
};

struct Entry {
  int64_t i, j;
  double v;
};

}  // namespace

extern "C" {

static int mm_fail(rebk_mm_matrix* out, int64_t line, const std::string& msg) {
  if (out) out->err_line = line;
  return rebk::set_error_msg(REBK_EINVAL, msg.c_str());
}

int rebk_mm_read(const char* path, double dense_threshold, int nthreads, rebk_mm_matrix* out) {
  if (!path || !out) return rebk::set_error_msg(REBK_EINVAL, "null argument");
  memset(out, 0, sizeof *out);
  out->err_line = 0;
  FILE* f = fopen(path, "rb");
  if (!f) return rebk::set_error_msg(REBK_EINVAL, (std::string("cannot open ") + path).c_str());
  std::string buf;
  {
    fseek(f, 0, SEEK_END);
    const long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    buf.resize(sz > 0 ? (size_t)sz : 0);
    if (sz > 0 && fread(&buf[0], 1, (size_t)sz, f) != (size_t)sz) {
      fclose(f);
      return rebk::set_error_msg(REBK_EINVAL, (std::string("read error on ") + path).c_str());
    }
    fclose(f);
  }
  for (unsigned char c : buf)
    if (c >= 0x80) return mm_fail(out, 0, "'ascii' codec can't decode the file (non-ASCII byte)");
  // line starts (Python's file iteration: lines end at '\n')
  std::vector<size_t> ls;
  ls.push_back(0);
  for (size_t p = 0; p < buf.size(); ++p)
    if (buf[p] == '\n' && p + 1 < buf.size()) ls.push_back(p + 1);
  const int64_t nlines = buf.empty() ? 0 : (int64_t)ls.size();
  if (nlines == 0) return mm_fail(out, 1, "empty file");
  auto line_end = [&](int64_t k) { return k + 1 < nlines ? ls[k + 1] : buf.size(); };
  auto line_str = [&](int64_t k) { return std::string(buf.data() + ls[k], buf.data() + line_end(k)); };

  // banner (matrix_io.py:35-46)
  std::vector<std::string> tok;
  {
    std::string h = strip(buf.data(), buf.data() + line_end(0));
    for (auto& c : h) c = (char)tolower((unsigned char)c);
    split_ws(h, tok);
  }
  if (tok.size() != 5 || tok[0] != "%%matrixmarket" || tok[1] != "matrix")
    return mm_fail(out, 1, "malformed banner; expected '%%MatrixMarket matrix ...'");
  const std::string fmt = tok[2], field = tok[3], sym = tok[4];
  if (fmt != "coordinate" && fmt != "array") return mm_fail(out, 1, "unsupported format " + py_repr(fmt));
  if (field != "real" && field != "integer" && field != "pattern")
    return mm_fail(out, 1, "unsupported field " + py_repr(field));
  if (sym != "general" && sym != "symmetric") return mm_fail(out, 1, "unsupported symmetry " + py_repr(sym));
  const bool coord = fmt == "coordinate", pattern = field == "pattern", symm = sym == "symmetric";

  // data lines: skip blanks and '%' comments
  auto is_data = [&](int64_t k) {
    const char* b = buf.data() + ls[k];
    const char* e = buf.data() + line_end(k);
    while (b < e && is_ws(*b)) ++b;
    return b < e && *b != '%';
  };
  int64_t k = 1;
  while (k < nlines && !is_data(k)) ++k;
  if (k >= nlines) return mm_fail(out, nlines, "missing size line");
  const int64_t size_line = k + 1;
  const std::string sline = strip(buf.data() + ls[k], buf.data() + line_end(k));
  split_ws(sline, tok);
  const size_t expect = coord ? 3 : 2;
  bool ok = tok.size() == expect;
  std::vector<long long> dims;
  for (size_t q = 0; ok && q < tok.size(); ++q) {
    std::string t = tok[q];
    size_t p = 0;
    while (p < t.size() && t[p] == '+') ++p;  // lstrip("+")
    t = t.substr(p);
    ok = !t.empty() && std::all_of(t.begin(), t.end(), [](char c) { return c >= '0' && c <= '9'; });
    if (ok) dims.push_back(atoll(t.c_str()));
  }
  if (!ok) return mm_fail(out, size_line, "malformed size line: " + py_repr(sline));
  const int64_t rows = dims[0], cols = dims[1];
  if (rows < 1 || cols < 1) return mm_fail(out, size_line, "matrix dimensions must be positive");
  out->rows = rows;
  out->cols = cols;
  const int64_t first = k + 1;  // index of the first body line after the size line

  // parallel parse of the body in line-aligned chunks
  const int T = std::max(1, std::min(nthreads > 0 ? nthreads : 1, 64));
  const int64_t nbody = nlines - first;
  const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(T, nbody / 4096 + 1));
  std::vector<std::vector<Entry>> ents(nchunks);
  std::vector<std::vector<double>> vals(nchunks);
  std::vector<std::vector<int64_t>> val_lines(nchunks);
  std::vector<int64_t> counts(nchunks, 0);
  std::vector<Err> errs(nchunks);
  auto work = [&](int c) {
    const int64_t l0 = first + nbody * c / nchunks, l1 = first + nbody * (c + 1) / nchunks;
    std::vector<std::string> tk;
    for (int64_t l = l0; l < l1; ++l) {
      if (!is_data(l)) continue;
      const int64_t ln = l + 1;
      const std::string s = strip(buf.data() + ls[l], buf.data() + line_end(l));
      split_ws(s, tk);
      if (coord) {
        const size_t want = pattern ? 2 : 3;
        if (tk.size() != want) {
          errs[c] = {ln, "expected " + std::to_string(want) + " fields, got " + std::to_string(tk.size())};
          return;
        }
        long long i, j;
        if (!py_int(tk[0], &i) || !py_int(tk[1], &j)) {
          errs[c] = {ln, "entry indices must be integers"};
          return;
        }
        if (!(1 <= i && i <= rows && 1 <= j && j <= cols)) {
          errs[c] = {ln, "entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside declared " +
                             std::to_string(rows) + "x" + std::to_string(cols) + " bounds"};
          return;
        }
        double v = 1.0;
        if (!pattern) {
          if (!py_float(tk[2], &v)) {
            errs[c] = {ln, "not a number: " + py_repr(tk[2])};
            return;
          }
          if (!std::isfinite(v)) {
            errs[c] = {ln, "non-finite value: " + py_repr(tk[2])};
            return;
          }
        }
        ents[c].push_back({i - 1, j - 1, v});
        if (symm) {
          if (j > i) {
            errs[c] = {ln, "symmetric storage must hold the lower triangle"};
            return;
          }
          if (i != j) ents[c].push_back({j - 1, i - 1, v});
        }
        ++counts[c];
      } else {
        for (const auto& t : tk) {
          double v;
          if (!py_float(t, &v)) {
            errs[c] = {ln, "not a number: " + py_repr(t)};
            return;
          }
          if (!std::isfinite(v)) {
            errs[c] = {ln, "non-finite value: " + py_repr(t)};
            return;
          }
          vals[c].push_back(v);
        }
      }
    }
  };
  {
    std::vector<std::thread> th;
    for (int c = 1; c < nchunks; ++c) th.emplace_back(work, c);
    work(0);
    for (auto& t : th) t.join();
  }
  for (int c = 0; c < nchunks; ++c)
    if (errs[c].line >= 0) return mm_fail(out, errs[c].line, errs[c].msg);

  if (coord) {
    int64_t count = 0, total = 0;
    for (int c = 0; c < nchunks; ++c) {
      count += counts[c];
      total += (int64_t)ents[c].size();
    }
    if (count != dims[2])
      return mm_fail(out, nlines, "declared " + std::to_string(dims[2]) + " entries but found " + std::to_string(count));
    // CSR by a stable counting sort on rows, then a stable sort by column
    // inside each row: duplicates stay in file order
    std::vector<int64_t> rc(rows + 1, 0);
    for (int c = 0; c < nchunks; ++c)
      for (const Entry& e : ents[c]) ++rc[e.i + 1];
    for (int64_t r = 0; r < rows; ++r) rc[r + 1] += rc[r];
    std::vector<int64_t> pos(rc.begin(), rc.end() - 1);
    std::vector<int64_t> cj(total);
    std::vector<double> cv(total);
    for (int c = 0; c < nchunks; ++c)
      for (const Entry& e : ents[c]) {
        const int64_t p = pos[e.i]++;
        cj[p] = e.j;
        cv[p] = e.v;
      }
    ents.clear();
    // per row: stable sort by column, sum duplicates in order
    std::vector<int64_t> ord;
    std::vector<int64_t> outj;
    std::vector<double> outv;
    outj.reserve(total);
    outv.reserve(total);
    std::vector<int64_t> dptr(rows + 1, 0);
    int64_t distinct = 0;
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t a = rc[r], b = rc[r + 1];
      ord.resize(b - a);
      for (int64_t q = 0; q < b - a; ++q) ord[q] = a + q;
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return cj[x] < cj[y]; });
      for (int64_t q = 0; q < b - a;) {
        const int64_t col = cj[ord[q]];
        double s = cv[ord[q]];
        int64_t q2 = q + 1;
        while (q2 < b - a && cj[ord[q2]] == col) s += cv[ord[q2++]];
        outj.push_back(col);
        outv.push_back(s);
        ++distinct;
        q = q2;
      }
      dptr[r + 1] = (int64_t)outj.size();
    }
    if ((double)distinct / ((double)rows * (double)cols) >= dense_threshold) {
      out->dense = 1;
      out->values = (double*)calloc((size_t)(rows * cols), sizeof(double));
      if (!out->values) return mm_fail(out, 0, "out of host memory");
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t p = dptr[r]; p < dptr[r + 1]; ++p) out->values[r * cols + outj[p]] = outv[p];
      return REBK_OK;
    }
    // CSR with explicit zeros dropped (csr.eliminate_zeros)
    int64_t nnz = 0;
    for (double v : outv) nnz += v != 0.0;
    out->nnz = nnz;
    out->indptr = (int64_t*)malloc(sizeof(int64_t) * (rows + 1));
    out->indices = (int32_t*)malloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
    out->values = (double*)malloc(sizeof(double) * std::max<int64_t>(nnz, 1));
    if (!out->indptr || !out->indices || !out->values) return mm_fail(out, 0, "out of host memory");
    int64_t w = 0;
    out->indptr[0] = 0;
    for (int64_t r = 0; r < rows; ++r) {
      for (int64_t p = dptr[r]; p < dptr[r + 1]; ++p)
        if (outv[p] != 0.0) {
          out->indices[w] = (int32_t)outj[p];
          out->values[w++] = outv[p];
        }
      out->indptr[r + 1] = w;
    }
    return REBK_OK;
  }
  // array format: column-major values (lower triangle when symmetric)
  if (symm && rows != cols) return mm_fail(out, size_line, "symmetric array storage needs a square matrix");
  std::vector<double> v;
  for (int c = 0; c < nchunks; ++c) v.insert(v.end(), vals[c].begin(), vals[c].end());
  const int64_t want = symm ? rows * (rows + 1) / 2 : rows * cols;
  if ((int64_t)v.size() != want)
    return mm_fail(out, nlines,
                   "expected " + std::to_string(want) + " array values, got " + std::to_string(v.size()));
  out->dense = 1;
  out->values = (double*)calloc((size_t)(rows * cols), sizeof(double));
  if (!out->values) return mm_fail(out, 0, "out of host memory");
  if (symm) {
    int64_t p = 0;
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = j; i < rows; ++i) {
        out->values[i * cols + j] = v[p];
        out->values[j * cols + i] = v[p];
        ++p;
      }
  } else {
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) out->values[i * cols + j] = v[j * rows + i];
  }
  return REBK_OK;
}

void rebk_mm_free(rebk_mm_matrix* m) {
  if (!m) return;
  free(m->indptr);
  free(m->indices);
  free(m->values);
  m->indptr = nullptr;
  m->indices = nullptr;
  m->values = nullptr;
}

}  // extern "C"
