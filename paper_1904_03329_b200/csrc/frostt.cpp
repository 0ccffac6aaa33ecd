// FROSTT .tns text I/O on the host, multi-threaded (the
// reference's parse_frostt / write_frostt, coo.py:117-205, are per-line
// Python loops, impractical at 77M-144M lines).
//
// Parsing follows coo.py:117-184 line by line: text after '#' is a comment,
// blank lines are skipped, the order is the token count of the first data
// line minus one (or len(dims)), every data line must have order+1 tokens,
// indices are 1-based integers >= 1 (and <= dims[d] when dims are given),
// the value is any float literal.  The first malformed line (in file order)
// is reported with its 1-based line number, as ParseError does.  The
// buffer is cut at newlines into one chunk per thread; each chunk is parsed
// independently into its own arrays, then the chunks are concatenated in
// order, so the result is identical to a sequential parse.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace hbk {

struct TnsChunk {
  const char* beg;
  const char* end;
  int64_t first_line = 0;  // 1-based number of the chunk's first line
  std::vector<int64_t> idx;  // nnz x order, 0-based
  std::vector<double> val;
  int64_t err_line = 0;      // first bad line in this chunk (0 = none)
  std::string err;
};

static inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// Tokenise [b, e) (comment already stripped) into token spans.
static int tokens_of(const char* b, const char* e, const char** tb, const char** te, int cap) {
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_space(*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_space(*p)) ++p;
    if (n < cap) {
      tb[n] = s;
      te[n] = p;
    }
    ++n;
  }
  return n;
}

static bool parse_int(const char* b, const char* e, int64_t* out) {
  const char* p = b;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) {
    neg = *p == '-';
    ++p;
  }
  if (p >= e) return false;
  int64_t v = 0;
  bool any = false;
  for (; p < e; ++p) {
    if (*p == '_' && any && p + 1 < e && p[1] != '_') continue;  // Python int() accepts 1_000
    if (*p < '0' || *p > '9') return false;
    if (v > (INT64_MAX - 9) / 10) return false;
    v = v * 10 + (*p - '0');
    any = true;
  }
  *out = neg ? -v : v;
  return any;
}

static bool parse_double(const char* b, const char* e, double* out) {
  char buf[128];
  const size_t n = size_t(e - b);
  if (n == 0 || n >= sizeof(buf)) {
    if (n == 0) return false;
    std::string s(b, e);
    char* endp = nullptr;
    errno = 0;
    *out = strtod(s.c_str(), &endp);
    return endp == s.c_str() + s.size();
  }
  size_t k = 0;
  for (const char* p = b; p < e; ++p)
    if (*p != '_') buf[k++] = *p;  // Python float() accepts digit separators
  buf[k] = 0;
  char* endp = nullptr;
  *out = strtod(buf, &endp);
  return endp == buf + k && k > 0;
}

static void parse_chunk(TnsChunk& c, int order, const int64_t* dims) {
  static constexpr int CAP = HBK_MAX_ORDER + 2;
  const char* tb[CAP];
  const char* te[CAP];
  int64_t line = c.first_line;
  const char* p = c.beg;
  while (p < c.end) {
    const char* le = static_cast<const char*>(memchr(p, '\n', size_t(c.end - p)));
    if (!le) le = c.end;
    const char* hash = static_cast<const char*>(memchr(p, '#', size_t(le - p)));
    const char* te_line = hash ? hash : le;
    const int nt = tokens_of(p, te_line, tb, te, CAP);
    if (nt > 0) {
      auto fail = [&](const std::string& m) {
        c.err_line = line;
        c.err = m;
      };
      if (nt != order + 1) {
        fail("expected " + std::to_string(order + 1) + " tokens (" + std::to_string(order) +
             " indices + value), got " + std::to_string(nt));
        return;
      }
      int64_t co[HBK_MAX_ORDER];
      for (int d = 0; d < order; ++d) {
        if (!parse_int(tb[d], te[d], &co[d])) {
          fail("malformed index in line");
          return;
        }
      }
      double v = 0;
      if (!parse_double(tb[order], te[order], &v)) {
        fail("malformed value " + std::string(tb[order], te[order]));
        return;
      }
      for (int d = 0; d < order; ++d) {
        if (co[d] < 1) {
          fail("index " + std::to_string(co[d]) + " in mode " + std::to_string(d) + " is below 1");
          return;
        }
        if (dims && co[d] > dims[d]) {
          fail("index " + std::to_string(co[d]) + " in mode " + std::to_string(d) +
               " exceeds stated dimension " + std::to_string(dims[d]));
          return;
        }
      }
      for (int d = 0; d < order; ++d) c.idx.push_back(co[d] - 1);
      c.val.push_back(v);
    }
    ++line;
    p = le + 1;
  }
}

}  // namespace hbk

struct hbk_tns {
  int order = 0;
  int64_t nnz = 0;
  int64_t dims[HBK_MAX_ORDER] = {0};
  std::vector<int64_t> idx;
  std::vector<double> val;
  int64_t err_line = 0;
};

using namespace hbk;

static int tns_parse_impl(const char* text, int64_t len, int order_given, const int64_t* dims,
                          int threads, hbk_tns** out) {
  return guarded([&] {
    HBK_REQUIRE(len >= 0, HBK_EINVAL, "negative length");
    HBK_REQUIRE(!dims || (order_given >= 3 && order_given <= HBK_MAX_ORDER), HBK_EINVAL,
                "tensor order must be >= 3 (and <= 8), got " + std::to_string(order_given));
    std::unique_ptr<hbk_tns> r(new hbk_tns());
    const char* end = text + len;
    // order: from dims, else the first data line (scanned sequentially)
    int order = dims ? order_given : 0;
    if (!dims) {
      const char* p = text;
      int64_t line = 1;
      while (p < end) {
        const char* le = static_cast<const char*>(memchr(p, '\n', size_t(end - p)));
        if (!le) le = end;
        const char* hash = static_cast<const char*>(memchr(p, '#', size_t(le - p)));
        const char* tb[HBK_MAX_ORDER + 2];
        const char* te[HBK_MAX_ORDER + 2];
        const int nt = tokens_of(p, hash ? hash : le, tb, te, HBK_MAX_ORDER + 2);
        if (nt > 0) {
          if (nt - 1 < 3) {
            r->err_line = line;
            set_last_error("expected at least 3 indices and a value, got " + std::to_string(nt) +
                           " tokens");
            *out = r.release();
            throw Error(HBK_EINVAL, hbk_last_error());
          }
          HBK_REQUIRE(nt - 1 <= HBK_MAX_ORDER, HBK_EINVAL,
                      "order " + std::to_string(nt - 1) + " exceeds the supported maximum 8");
          order = nt - 1;
          break;
        }
        ++line;
        p = le + 1;
      }
      if (order == 0) {
        *out = r.release();
        throw Error(HBK_EINVAL, "no data lines in input");
      }
    }
    // chunks cut at newlines
    // threads > 0: at most that many chunks of >= 1 MiB; < 0: exactly -threads
    // chunks (tests exercise chunk boundaries on small inputs); 0: all cores
    int T;
    if (threads < 0) {
      T = -threads;
    } else {
      T = threads > 0 ? threads : int(std::max(1u, std::thread::hardware_concurrency()));
      T = int(std::min<int64_t>(T, std::max<int64_t>(1, len / (1 << 20))));
    }
    std::vector<TnsChunk> ch(T);
    const char* p = text;
    for (int i = 0; i < T; ++i) {
      ch[i].beg = p;
      const char* q = (i + 1 == T) ? end : text + len * (i + 1) / T;
      if (q < p) q = p;
      if (i + 1 < T) {
        const char* nl = static_cast<const char*>(memchr(q, '\n', size_t(end - q)));
        q = nl ? nl + 1 : end;
      }
      ch[i].end = q;
      p = q;
    }
    // first line number of each chunk
    std::vector<int64_t> nl_count(T, 0);
    {
      std::vector<std::thread> pool;
      for (int i = 0; i < T; ++i)
        pool.emplace_back([&, i] {
          int64_t n = 0;
          for (const char* s = ch[i].beg; s < ch[i].end; ++s) n += *s == '\n';
          nl_count[i] = n;
        });
      for (auto& th : pool) th.join();
    }
    int64_t line = 1;
    for (int i = 0; i < T; ++i) {
      ch[i].first_line = line;
      line += nl_count[i];
    }
    {
      std::vector<std::thread> pool;
      for (int i = 0; i < T; ++i) pool.emplace_back([&, i] { parse_chunk(ch[i], order, dims); });
      for (auto& th : pool) th.join();
    }
    for (int i = 0; i < T; ++i) {
      if (ch[i].err_line) {
        r->err_line = ch[i].err_line;
        set_last_error(ch[i].err);
        *out = r.release();
        throw Error(HBK_EINVAL, ch[i].err);
      }
    }
    int64_t nnz = 0;
    for (auto& c : ch) nnz += int64_t(c.val.size());
    if (nnz == 0) {
      *out = r.release();
      throw Error(HBK_EINVAL, "no data lines in input");
    }
    r->order = order;
    r->nnz = nnz;
    r->idx.resize(size_t(nnz) * order);
    r->val.resize(size_t(nnz));
    int64_t off = 0;
    for (auto& c : ch) {
      std::copy(c.idx.begin(), c.idx.end(), r->idx.begin() + off * order);
      std::copy(c.val.begin(), c.val.end(), r->val.begin() + off);
      off += int64_t(c.val.size());
    }
    if (dims) {
      std::copy(dims, dims + order, r->dims);
    } else {
      for (int d = 0; d < order; ++d) r->dims[d] = 0;
      for (int64_t i = 0; i < nnz; ++i)
        for (int d = 0; d < order; ++d) r->dims[d] = std::max(r->dims[d], r->idx[i * order + d] + 1);
    }
    *out = r.release();
  });
}

extern "C" {

int hbk_tns_parse(const char* text, int64_t len, int order, const int64_t* dims, int threads,
                  hbk_tns** out) {
  *out = nullptr;
  return tns_parse_impl(text, len, order, dims, threads, out);
}

int hbk_tns_load(const char* path, int order, const int64_t* dims, int threads, hbk_tns** out) {
  *out = nullptr;
  std::vector<char> buf;
  {
    const int st = guarded([&] {
      FILE* f = fopen(path, "rb");
      HBK_REQUIRE(f != nullptr, HBK_EINVAL, std::string("cannot open ") + path);
      fseek(f, 0, SEEK_END);
      const long n = ftell(f);
      fseek(f, 0, SEEK_SET);
      buf.resize(size_t(std::max(0L, n)));
      const size_t got = n > 0 ? fread(buf.data(), 1, size_t(n), f) : 0;
      fclose(f);
      HBK_REQUIRE(got == buf.size(), HBK_EINVAL, std::string("short read from ") + path);
    });
    if (st != HBK_OK) return st;
  }
  return tns_parse_impl(buf.data(), int64_t(buf.size()), order, dims, threads, out);
}

int hbk_tns_info(const hbk_tns* t, int* order, int64_t* nnz, int64_t* dims, int64_t* err_line) {
  return guarded([&] {
    if (order) *order = t ? t->order : 0;
    if (nnz) *nnz = t ? t->nnz : 0;
    if (dims && t) std::copy(t->dims, t->dims + HBK_MAX_ORDER, dims);
    if (err_line) *err_line = t ? t->err_line : 0;
  });
}

int hbk_tns_export(const hbk_tns* t, uint32_t* idx, double* vals) {
  return guarded([&] {
    HBK_REQUIRE(t != nullptr, HBK_EINVAL, "null tensor");
    for (int d = 0; d < t->order; ++d)
      HBK_REQUIRE(t->dims[d] <= (int64_t(1) << 32), HBK_EINVAL,
                  "dimension exceeds the uint32 index range");
    if (idx)
      for (size_t i = 0; i < t->idx.size(); ++i) idx[i] = uint32_t(t->idx[i]);
    if (vals) std::copy(t->val.begin(), t->val.end(), vals);
  });
}

void hbk_tns_release(hbk_tns* t) { delete t; }

// write_frostt (coo.py:187-195): 1-based indices, values "%.17g" (17
// significant digits round-trip doubles); rows formatted in parallel.
int hbk_tns_format(const uint32_t* idx, const double* vals, int64_t nnz, int order, int threads,
                   char** text, int64_t* len) {
  return guarded([&] {
    HBK_REQUIRE(order >= 1 && order <= HBK_MAX_ORDER, HBK_EINVAL, "bad order");
    int T = threads > 0 ? threads : int(std::max(1u, std::thread::hardware_concurrency()));
    T = int(std::min<int64_t>(T, std::max<int64_t>(1, nnz / 65536)));
    std::vector<std::string> parts(T);
    std::vector<std::thread> pool;
    for (int i = 0; i < T; ++i)
      pool.emplace_back([&, i] {
        const int64_t a = nnz * i / T, b = nnz * (i + 1) / T;
        std::string& s = parts[i];
        s.reserve(size_t(b - a) * size_t(order * 8 + 24));
        char buf[512];
        for (int64_t r = a; r < b; ++r) {
          char* q = buf;
          for (int d = 0; d < order; ++d) {
            q = std::to_chars(q, buf + sizeof(buf), uint64_t(idx[r * order + d]) + 1).ptr;
            *q++ = ' ';
          }
          const double v = vals[r];
          if (std::isnan(v)) {
            memcpy(q, "nan", 3);
            q += 3;
          } else if (std::isinf(v)) {
            const char* w = v > 0 ? "inf" : "-inf";
            memcpy(q, w, strlen(w));
            q += strlen(w);
          } else {
            // %.17g (Python's f"{v:.17g}")
            q = std::to_chars(q, buf + sizeof(buf), v, std::chars_format::general, 17).ptr;
          }
          *q++ = '\n';
          s.append(buf, size_t(q - buf));
        }
      });
    for (auto& th : pool) th.join();
    size_t total = 0;
    for (auto& s : parts) total += s.size();
    char* outp = static_cast<char*>(malloc(total ? total : 1));
    HBK_REQUIRE(outp != nullptr, HBK_ENOMEM, "host allocation failed");
    size_t off = 0;
    for (auto& s : parts) {
      memcpy(outp + off, s.data(), s.size());
      off += s.size();
    }
    *text = outp;
    *len = int64_t(total);
  });
}

void hbk_tns_free_text(char* text) { free(text); }

}  // extern "C"
