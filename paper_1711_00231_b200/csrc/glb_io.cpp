// glb_io.cpp -- graph files straight to the device path:
//   * glb_graph_load_csrg: the binary CSR cache of io.py:125-170 ("CSRG", v1,
//     little-endian u64 N, E, int64 arrays, weights-flag byte, int64 weights)
//     memory-mapped and handed to glb_graph_create, whose host workers narrow
//     and stream it through the pinned ring into HBM -- no int64 copies in
//     between;
//   * glb_read_text_graph: the 9th DIMACS `.gr` reader (io.py:26-81) and the
//     `u v [w]` edge-list reader (io.py:84-122), native, with the reference's
//     grammar, errors and CsrGraph.from_edges grouping (stable by source: the
//     arcs of one source keep their file order, csr.py:97-118).
// Host-only C++ (no device code).
#include <fcntl.h>
#include <stdint.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/graphlb_b200.h"

namespace glb {
void set_error(const std::string& msg);  // glb_graph.cu: the glb_last_error() text
}

namespace {

// Reference ParseError text: "<path>:<line>: <message>" (io.py:17-23); the
// Python side rebuilds the exception from "<line>\t<message>".
int fail(long long line, const std::string& msg) {
  glb::set_error(std::to_string(line) + "\t" + msg);
  return GLB_EPARSE;
}

struct Mapped {
  void* p = MAP_FAILED;
  size_t len = 0;
  int fd = -1;
  ~Mapped() {
    if (p != MAP_FAILED && len) munmap(p, len);
    if (fd >= 0) close(fd);
  }
  bool open_file(const char* path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat st;
    if (fstat(fd, &st) != 0) return false;
    len = (size_t)st.st_size;
    if (len == 0) return true;
    p = mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
    if (p == MAP_FAILED) return false;
    madvise(p, len, MADV_SEQUENTIAL | MADV_WILLNEED);
    return true;
  }
  const char* data() const { return len ? (const char*)p : ""; }
};

// --------------------------------------------------------- text scanning
struct Line {
  const char* b;
  const char* e;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// whitespace-split tokens of [b, e) (Python str.split())
int split(const char* b, const char* e, Line* tok, int max_tok) {
  int n = 0;
  while (b < e) {
    while (b < e && is_space(*b)) ++b;
    if (b >= e) break;
    const char* s = b;
    while (b < e && !is_space(*b)) ++b;
    if (n < max_tok) tok[n] = Line{s, b};
    ++n;
  }
  return n;
}

// Python int(token) for plain decimal tokens (optional sign, digits, '_'
// separators are not expected in graph files); false if not an integer.
bool to_int(const Line& t, long long* out) {
  const char* p = t.b;
  bool neg = false;
  if (p < t.e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= t.e) return false;
  unsigned long long v = 0;
  for (; p < t.e; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + (unsigned)(*p - '0');
    if (v > (1ull << 62)) return false;
  }
  *out = neg ? -(long long)v : (long long)v;
  return true;
}

std::string quoted(const char* b, const char* e) {  // Python repr of a stripped line
  std::string s(b, e);
  std::string r = "'";
  for (char c : s) r += c == '\'' ? std::string("\\'") : std::string(1, c);
  return r + "'";
}

// stable grouping by source (CsrGraph.from_edges, csr.py:97-118)
void group_by_source(long long n, const std::vector<long long>& src,
                     const std::vector<long long>& dst, const std::vector<long long>* w,
                     int64_t** row, int64_t** col, int64_t** wt) {
  const size_t m = src.size();
  *row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  *col = (int64_t*)malloc(sizeof(int64_t) * (m ? m : 1));
  *wt = w ? (int64_t*)malloc(sizeof(int64_t) * (m ? m : 1)) : nullptr;
  int64_t* r = *row;
  for (long long i = 0; i <= n; ++i) r[i] = 0;
  for (size_t i = 0; i < m; ++i) r[src[i] + 1] += 1;
  for (long long i = 0; i < n; ++i) r[i + 1] += r[i];
  std::vector<int64_t> cur(r, r + n);
  for (size_t i = 0; i < m; ++i) {
    const int64_t k = cur[src[i]]++;
    (*col)[k] = dst[i];
    if (w) (*wt)[k] = (*w)[i];
  }
}

}  // namespace

extern "C" {

void glb_free(void* p) { free(p); }

int glb_graph_load_csrg(const char* path, int device, glb_graph** out) {
  if (!path || !out) {
    glb::set_error("NULL argument");
    return GLB_EINVAL;
  }
  *out = nullptr;
  Mapped f;
  if (!f.open_file(path)) return fail(-1, std::string("cannot open: ") + strerror(errno));
  const unsigned char* d = (const unsigned char*)f.data();
  if (f.len < 4 || memcmp(d, "CSRG", 4) != 0) return fail(-1, "bad magic, not a CSR cache file");
  if (f.len < 24) return fail(-1, "truncated cache file");
  uint32_t version;
  uint64_t n, m;
  memcpy(&version, d + 4, 4);
  if (version != 1) return fail(-1, "unsupported cache version " + std::to_string(version));
  memcpy(&n, d + 8, 8);
  memcpy(&m, d + 16, 8);
  const unsigned long long rows_end = 24ull + (n + 1) * 8ull, cols_end = rows_end + m * 8ull;
  if (n > (1ull << 40) || m > (1ull << 40) || cols_end >= f.len)
    return fail(-1, "truncated cache file");
  const unsigned char flag = d[cols_end];
  if (flag && cols_end + 1 + m * 8ull > f.len) return fail(-1, "truncated cache file");
  const int64_t* row = (const int64_t*)(d + 24);
  const int64_t* col = (const int64_t*)(d + rows_end);
  const int64_t* w = flag ? (const int64_t*)(d + cols_end + 1) : nullptr;
  // graph_create reads the mapping with every host worker (page faults in
  // parallel) and narrows straight into the pinned DMA ring
  return glb_graph_create(row, col, w, (int64_t)n, (int64_t)m, device, out);
}

int glb_read_text_graph(const char* path, int kind, int64_t* n_out, int64_t* m_out,
                        int* weighted_out, int64_t** row, int64_t** col, int64_t** w) {
  if (!path || !n_out || !m_out || !weighted_out || !row || !col || !w || kind < 0 || kind > 2) {
    glb::set_error("bad argument");
    return GLB_EINVAL;
  }
  *row = *col = *w = nullptr;
  Mapped f;
  if (!f.open_file(path)) return fail(-1, std::string("cannot open: ") + strerror(errno));
  const char* p = f.data();
  const char* end = p + f.len;
  std::vector<long long> src, dst, wts;
  long long num_nodes = -1, num_arcs = -1, max_id = -1, line_no = 0;
  const bool dimacs = kind == 0, with_w = kind == 2;
  Line tok[8];
  while (p < end) {
    const char* nl = (const char*)memchr(p, '\n', (size_t)(end - p));
    const char* le = nl ? nl : end;
    ++line_no;
    const char* b = p;
    const char* e = le;
    p = nl ? nl + 1 : end;
    if (!dimacs) {  // `#` starts a comment (io.py:99)
      const char* h = (const char*)memchr(b, '#', (size_t)(e - b));
      if (h) e = h;
    }
    while (b < e && (is_space(*b) || *b == '\n')) ++b;
    while (e > b && (is_space(e[-1]) || e[-1] == '\n')) --e;
    if (b >= e) continue;
    if (dimacs) {  // io.py:26-81
      if (*b == 'c') continue;
      const int nt = split(b, e, tok, 8);
      const std::string kindtok(tok[0].b, tok[0].e);
      if (kindtok == "p") {
        if (num_nodes >= 0) return fail(line_no, "duplicate problem line");
        if (nt != 4 || std::string(tok[1].b, tok[1].e) != "sp")
          return fail(line_no, "malformed problem line " + quoted(b, e));
        long long a, c;
        if (!to_int(tok[2], &a) || !to_int(tok[3], &c))
          return fail(line_no, "non-integer node/arc count");
        if (a < 0 || c < 0) return fail(line_no, "negative node/arc count");
        num_nodes = a;
        num_arcs = c;
        src.reserve((size_t)c);
        dst.reserve((size_t)c);
        wts.reserve((size_t)c);
      } else if (kindtok == "a") {
        if (num_nodes < 0) return fail(line_no, "arc line before problem line");
        if (nt != 4) return fail(line_no, "malformed arc line " + quoted(b, e));
        long long u, v, x;
        if (!to_int(tok[1], &u) || !to_int(tok[2], &v) || !to_int(tok[3], &x))
          return fail(line_no, "non-integer arc token");
        if (u < 1 || u > num_nodes) return fail(line_no, "node id " + std::to_string(u) + " out of range");
        if (v < 1 || v > num_nodes) return fail(line_no, "node id " + std::to_string(v) + " out of range");
        if (x < 0) return fail(line_no, "negative weight " + std::to_string(x));
        src.push_back(u - 1);
        dst.push_back(v - 1);
        wts.push_back(x);
      } else {
        return fail(line_no, "unknown line type '" + kindtok + "'");
      }
    } else {  // io.py:84-122
      const int nt = split(b, e, tok, 8);
      if (nt < 2) return fail(line_no, "expected `u v [w]`, got " + quoted(b, e));
      long long u, v;
      if (!to_int(tok[0], &u) || !to_int(tok[1], &v)) return fail(line_no, "non-integer node token");
      if (u < 0 || v < 0) return fail(line_no, "negative node id");
      if (with_w) {
        if (nt < 3) return fail(line_no, "missing weight");
        long long x;
        if (!to_int(tok[2], &x)) return fail(line_no, "non-integer weight token");
        if (x < 0) return fail(line_no, "negative weight " + std::to_string(x));
        wts.push_back(x);
      }
      src.push_back(u);
      dst.push_back(v);
      if (u > max_id) max_id = u;
      if (v > max_id) max_id = v;
    }
  }
  if (dimacs) {
    if (num_nodes < 0) return fail(-1, "missing problem line");
    if ((long long)src.size() != num_arcs)
      return fail(-1, "arc count mismatch: header says " + std::to_string(num_arcs) +
                          ", file has " + std::to_string(src.size()));
  } else {
    num_nodes = max_id + 1;
  }
  group_by_source(num_nodes, src, dst, (dimacs || with_w) ? &wts : nullptr, row, col, w);
  *n_out = num_nodes;
  *m_out = (int64_t)src.size();
  *weighted_out = (dimacs || with_w) ? 1 : 0;
  return GLB_OK;
}

}  // extern "C"
