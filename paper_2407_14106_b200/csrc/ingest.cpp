// Ingestion formats: edge-list text, GTF1 binary features and
// permutation text, parsed from memory buffers so the C++ drop-in can hand
// over any std::istream's bytes (reference proj/src/graph.cpp:68-109 and
// 302-336, proj/src/partition.cpp:458-493; same accept/reject rules and the
// same error wording, which the reference tests match on).
//
// The edge-list parser splits the buffer at line boundaries into chunks
// parsed on all host threads with std::from_chars; per-chunk line counts give
// every error its global line number and the first error (lowest line) wins,
// as in a sequential scan. The CSR is then built on the GPU
// (gte_graph_from_edges_host).
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
}
using namespace gte_b200;

struct gte_edges {
  int64_t n = 0;
  std::vector<int64_t> src, dst;
};

namespace {

bool blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

struct LineErr {
  int64_t line = -1;  // within the chunk (1-based); -1 = none
  std::string msg;    // wording with "{LINE}" standing for the global number
};

// one chunk [b, e) of complete lines
void parse_edges(const char* b, const char* e, int64_t hint, std::vector<int64_t>& s, std::vector<int64_t>& d,
                 int64_t& lines, int64_t& max_id, LineErr& err) {
  lines = 0;
  max_id = -1;
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* end = nl ? nl : e;
    ++lines;
    const char* x = p;
    while (x < end && blank(x[0])) ++x;
    p = nl ? nl + 1 : e;
    if (x == end || *x == '#') continue;
    // up to three whitespace-separated tokens
    const char* tok[3] = {nullptr, nullptr, nullptr};
    const char* tend[3] = {nullptr, nullptr, nullptr};
    int nt = 0;
    const char* y = x;
    while (y < end && nt < 3) {
      while (y < end && (blank(*y) || *y == '\v' || *y == '\f')) ++y;
      if (y == end) break;
      tok[nt] = y;
      while (y < end && !(blank(*y) || *y == '\v' || *y == '\f')) ++y;
      tend[nt++] = y;
    }
    if (nt != 2) {
      err = {lines, "parse error at line {LINE}: expected \"src dst\""};
      return;
    }
    int64_t id[2];
    for (int t = 0; t < 2; ++t) {
      auto r = std::from_chars(tok[t], tend[t], id[t]);
      if (r.ec != std::errc() || r.ptr != tend[t]) {
        err = {lines, "parse error at line {LINE}: bad token \"" + std::string(tok[t], tend[t]) + "\""};
        return;
      }
      if (id[t] < 0) {
        err = {lines, "range error at line {LINE}: negative node id"};
        return;
      }
      if (hint >= 0 && id[t] >= hint) {
        err = {lines, "range error at line {LINE}: node id " + std::to_string(id[t]) + " >= hint " +
                          std::to_string(hint)};
        return;
      }
      max_id = std::max(max_id, id[t]);
    }
    s.push_back(id[0]);
    d.push_back(id[1]);
  }
}

std::string with_line(const std::string& msg, int64_t line) {
  std::string out = msg;
  const size_t at = out.find("{LINE}");
  if (at != std::string::npos) out.replace(at, 6, std::to_string(line));
  return out;
}

}  // namespace

extern "C" {

int gte_parse_edge_list(const char* text, int64_t len, int64_t num_nodes_hint, gte_edges** out) {
  const int threads = len < (1 << 20) ? 1 : (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<const char*> cut{text};
  for (int t = 1; t < threads; ++t) {  // chunk starts just after a newline
    const char* guess = text + len * t / threads;
    if (guess <= cut.back()) continue;
    const char* nl = static_cast<const char*>(memchr(guess, '\n', (size_t)(text + len - guess)));
    if (!nl) break;
    cut.push_back(nl + 1);
  }
  cut.push_back(text + len);
  const size_t nc = cut.size() - 1;
  std::vector<std::vector<int64_t>> s(nc), d(nc);
  std::vector<int64_t> lines(nc), maxid(nc);
  std::vector<LineErr> errs(nc);
  std::vector<std::thread> pool;
  for (size_t c = 0; c < nc; ++c)
    pool.emplace_back([&, c] { parse_edges(cut[c], cut[c + 1], num_nodes_hint, s[c], d[c], lines[c], maxid[c], errs[c]); });
  for (auto& t : pool) t.join();
  int64_t before = 0, max_id = -1, m = 0;
  for (size_t c = 0; c < nc; ++c) {
    if (errs[c].line >= 0) return set_error(GTE_DATA, with_line(errs[c].msg, before + errs[c].line));
    before += lines[c];
    max_id = std::max(max_id, maxid[c]);
    m += (int64_t)s[c].size();
  }
  if (num_nodes_hint < 0 && m == 0) return set_error(GTE_DATA, "empty graph");
  auto* e = new gte_edges();
  e->n = num_nodes_hint >= 0 ? num_nodes_hint : max_id + 1;
  e->src.reserve(m);
  e->dst.reserve(m);
  for (size_t c = 0; c < nc; ++c) {
    e->src.insert(e->src.end(), s[c].begin(), s[c].end());
    e->dst.insert(e->dst.end(), d[c].begin(), d[c].end());
  }
  *out = e;
  return GTE_OK;
}

int gte_edges_info(const gte_edges* e, int64_t* num_nodes, int64_t* num_edges) {
  if (num_nodes) *num_nodes = e->n;
  if (num_edges) *num_edges = (int64_t)e->src.size();
  return GTE_OK;
}

int gte_edges_copy(const gte_edges* e, int64_t* src, int64_t* dst) {
  std::copy(e->src.begin(), e->src.end(), src);
  std::copy(e->dst.begin(), e->dst.end(), dst);
  return GTE_OK;
}

int gte_edges_destroy(gte_edges* e) {
  delete e;
  return GTE_OK;
}

// GTF1: "GTF1", u64 N, u64 f, N*f little-endian float32 row-major
int gte_gtf1_decode(const void* bytes, int64_t len, int64_t* n, int64_t* f, float* out) {
  const char* b = static_cast<const char*>(bytes);
  if (len < 4 || std::memcmp(b, "GTF1", 4) != 0) return set_error(GTE_DATA, "features binary: bad magic, expected GTF1");
  if (len < 20) return set_error(GTE_DATA, "features binary: truncated header");
  uint64_t nn = 0, ff = 0;
  std::memcpy(&nn, b + 4, 8);
  std::memcpy(&ff, b + 12, 8);
  // header values bounded by the payload before any product is formed (a
  // corrupt header must not overflow n * f * 4)
  const uint64_t payload = (uint64_t)(len - 20);
  if (ff > payload / sizeof(float) && nn > 0) {
    return set_error(GTE_DATA, "features binary: truncated at row 0");
  }
  const uint64_t row = ff * sizeof(float);
  const uint64_t have = row > 0 ? payload / row : nn;
  if (have < nn) return set_error(GTE_DATA, "features binary: truncated at row " + std::to_string(have));
  *n = (int64_t)nn;
  *f = (int64_t)ff;
  if (!out) return GTE_OK;
  std::memcpy(out, b + 20, (size_t)(nn * row));
  return GTE_OK;
}

int gte_gtf1_encode(int64_t n, int64_t f, const float* data, void* out, int64_t* len) {
  *len = 20 + n * f * (int64_t)sizeof(float);
  if (!out) return GTE_OK;
  char* b = static_cast<char*>(out);
  std::memcpy(b, "GTF1", 4);
  const uint64_t nn = (uint64_t)n, ff = (uint64_t)f;
  std::memcpy(b + 4, &nn, 8);
  std::memcpy(b + 12, &ff, 8);
  std::memcpy(b + 20, data, (size_t)(n * f * sizeof(float)));
  return GTE_OK;
}

// Permutation text: one "old pos" pair per line ('#' comments, blank lines).
// n_out receives the pair count; forward/inverse (size n) are filled when
// non-null (call once with nulls to size them).
int gte_parse_permutation(const char* text, int64_t len, int64_t* n_out, int64_t* forward, int64_t* inverse) {
  std::vector<std::pair<int64_t, int64_t>> pairs;
  const char* p = text;
  const char* e = text + len;
  int64_t line = 0;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* end = nl ? nl : e;
    ++line;
    const char* x = p;
    p = nl ? nl + 1 : e;
    while (x < end && blank(*x)) ++x;
    if (x == end || *x == '#') continue;
    int64_t v[2];
    for (int t = 0; t < 2; ++t) {
      while (x < end && blank(*x)) ++x;
      auto r = std::from_chars(x, end, v[t]);
      if (r.ec != std::errc()) return set_error(GTE_DATA, "permutation: parse error at line " + std::to_string(line));
      x = r.ptr;
    }
    pairs.emplace_back(v[0], v[1]);
  }
  const int64_t n = (int64_t)pairs.size();
  *n_out = n;
  std::vector<int64_t> fw(n, -1), iv(n, -1);
  for (const auto& [old, pos] : pairs) {
    if (old < 0 || old >= n || pos < 0 || pos >= n || fw[old] != -1)
      return set_error(GTE_DATA, "permutation: invalid pair " + std::to_string(old) + " " + std::to_string(pos));
    fw[old] = pos;
    iv[pos] = old;
  }
  for (int64_t i = 0; i < n; ++i)
    if (iv[i] < 0 || fw[iv[i]] != i) return set_error(GTE_DATA, "permutation: not a bijection");
  if (forward) std::copy(fw.begin(), fw.end(), forward);
  if (inverse) std::copy(iv.begin(), iv.end(), inverse);
  return GTE_OK;
}

}  // extern "C"
