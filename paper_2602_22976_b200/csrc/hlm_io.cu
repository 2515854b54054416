// hlm_io.cu -- host-side text formats of libhlm_b200.so (no device code): hMetis .hgr hypergraphs,
// METIS graphs read as 2-uniform hypergraphs, and the matching file.  A restatement of the
// reference's io.hpp (parse_hgr :79-137, write_hgr :146-171, parse_metis_graph :176-231,
// write_matching :240-247, parse_matching :249-257) and of build_hypergraph (hypergraph.hpp:78-153)
// behind the C-ABI: same accepted inputs, same CSR out, same texts out, the same inputs rejected.
// These are the data formats on either side of the matching path; the text
// is parsed once on the host and is not part of any timed region (tools/hlm_app.hpp:213).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "hlm_engine.h"

namespace hlmb {
namespace {

struct ParseError {
  std::string what;
};

// std::getline over a buffer: the text after the last '\n' is a line only if it is not empty
struct LineReader {
  const char* p;
  const char* end;
  bool next(std::string_view& line) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* stop = nl ? nl : end;
    line = std::string_view(p, static_cast<size_t>(stop - p));
    p = nl ? nl + 1 : end;
    return true;
  }
};

bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// 0: blank, 1: comment, 2: content
int line_kind(std::string_view line) {
  for (char c : line) {
    if (is_blank(c)) continue;
    return c == '%' ? 1 : 2;
  }
  return 0;
}

bool next_content_line(LineReader& in, std::string_view& line) {  // io.hpp:26-34
  while (in.next(line))
    if (line_kind(line) == 2) return true;
  return false;
}

void split_tokens(std::string_view line, std::vector<std::string_view>& tokens) {  // io.hpp:36-47
  tokens.clear();
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_blank(line[i])) ++i;
    size_t j = i;
    while (j < line.size() && !is_blank(line[j])) ++j;
    if (j > i) tokens.push_back(line.substr(i, j - i));
    i = j;
  }
}

// A token is a number only if ALL of it is (what io.hpp:49-66 accept and reject, messages included).
uint64_t parse_uint(std::string_view tok, const char* what) {
  uint64_t acc = 0;
  bool good = !tok.empty();
  for (size_t i = 0; good && i < tok.size(); ++i) {
    const unsigned digit = static_cast<unsigned char>(tok[i]) - '0';
    good = digit <= 9 && acc <= (UINT64_MAX - digit) / 10;  // no sign, no blanks, no wrap-around
    if (good) acc = acc * 10 + digit;
  }
  if (!good) throw ParseError{std::string("expected unsigned integer for ") + what + ", got '" + std::string(tok) + "'"};
  return acc;
}

double parse_weight(std::string_view tok) {
  double w = 0.0;
  const char* last = tok.data() + tok.size();
  const std::from_chars_result got = std::from_chars(tok.data(), last, w);  // locale-free, integers stay exact
  const bool whole = got.ec == std::errc{} && got.ptr == last;
  if (!whole || !std::isfinite(w)) throw ParseError{"malformed edge weight '" + std::string(tok) + "'"};
  if (w <= 0.0) throw ParseError{"edge weight must be positive, got " + std::string(tok)};
  return w;
}

// ids are 32-bit on both sides of the boundary: larger header counts are input errors, not narrowed
void check_count(uint64_t value, const char* what) {
  if (value > 0xFFFFFFFFull) throw ParseError{std::string(what) + " " + std::to_string(value) + " exceeds the 32-bit id range"};
}

struct EdgeLists {  // flat edge lists in file order
  std::vector<uint64_t> off{0};
  std::vector<uint32_t> pins;
  std::vector<double> weights;  // empty: unit
};

template <typename T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() + 1)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

// build_hypergraph (hypergraph.hpp:78-153) with num_vertices given
void build(const EdgeLists& el, uint32_t n, int degree_zero, hlm_b200_host_graph* out) {
  const size_t m = el.off.size() - 1;
  uint32_t max_id = 0;
  for (size_t e = 0; e < m; ++e) {
    const uint64_t b = el.off[e], s = el.off[e + 1] - b;
    if (s == 0) throw ParseError{"edge " + std::to_string(e) + " is empty"};
    for (uint64_t i = 0; i < s; ++i) {
      max_id = std::max(max_id, el.pins[b + i]);
      for (uint64_t j = i + 1; j < s; ++j)
        if (el.pins[b + i] == el.pins[b + j])
          throw ParseError{"edge " + std::to_string(e) + " lists vertex " + std::to_string(el.pins[b + i]) +
                           " more than once"};
    }
  }
  for (size_t e = 0; e < el.weights.size(); ++e)
    if (!(el.weights[e] > 0.0)) throw ParseError{"edge " + std::to_string(e) + " has non-positive weight"};
  if (!el.pins.empty() && max_id >= n)
    throw ParseError{"vertex id " + std::to_string(max_id) + " out of range [0, " + std::to_string(n) + ")"};

  std::vector<uint32_t> degree(n, 0);
  for (uint32_t v : el.pins) ++degree[v];
  std::vector<uint32_t> remap;
  uint32_t kept = n;
  for (uint32_t v = 0; v < n; ++v) {
    if (degree[v] != 0) continue;
    if (degree_zero == HLM_B200_DEGREE_ZERO_REJECT) throw ParseError{"vertex " + std::to_string(v) + " has degree 0"};
    if (remap.empty()) remap.assign(n, 0xFFFFFFFFu);
  }
  if (!remap.empty()) {
    kept = 0;
    for (uint32_t v = 0; v < n; ++v)
      if (degree[v] != 0) remap[v] = kept++;
  }
  std::vector<uint32_t> members(el.pins.size());
  for (size_t i = 0; i < el.pins.size(); ++i) members[i] = remap.empty() ? el.pins[i] : remap[el.pins[i]];
  std::vector<uint64_t> voff(static_cast<size_t>(kept) + 1, 0);
  for (uint32_t v : members) ++voff[v + 1];
  for (uint32_t v = 0; v < kept; ++v) voff[v + 1] += voff[v];
  std::vector<uint32_t> vinc(members.size());
  std::vector<uint64_t> cursor(voff.begin(), voff.end() - 1);
  for (size_t e = 0; e < m; ++e)
    for (uint64_t i = el.off[e]; i < el.off[e + 1]; ++i) vinc[cursor[members[i]]++] = static_cast<uint32_t>(e);
  std::vector<double> weights = el.weights.empty() ? std::vector<double>(m, 1.0) : el.weights;

  out->num_vertices = kept;
  out->num_edges = static_cast<uint32_t>(m);
  out->vertex_offsets = dup(voff);
  out->vertex_incidence = dup(vinc);
  out->edge_offsets = dup(el.off);
  out->edge_members = dup(members);
  out->base_weights = dup(weights);
}

void parse_hgr(const char* text, size_t len, int degree_zero, hlm_b200_host_graph* out) {
  LineReader in{text, text + len};
  std::string_view line;
  std::vector<std::string_view> tok;
  if (!next_content_line(in, line)) throw ParseError{"missing hgr header line"};
  split_tokens(line, tok);
  if (tok.size() < 2 || tok.size() > 3) throw ParseError{"malformed hgr header '" + std::string(line) + "'"};
  const uint64_t m = parse_uint(tok[0], "edge count");
  const uint64_t n = parse_uint(tok[1], "vertex count");
  check_count(m, "edge count");
  check_count(n, "vertex count");
  const uint64_t fmt = tok.size() == 3 ? parse_uint(tok[2], "fmt code") : 0;
  if (fmt != 0 && fmt != 1 && fmt != 10 && fmt != 11) throw ParseError{"unsupported hgr fmt code " + std::to_string(fmt)};
  const bool edge_w = fmt == 1 || fmt == 11, vertex_w = fmt == 10 || fmt == 11;
  EdgeLists el;
  for (uint64_t e = 0; e < m; ++e) {
    if (!next_content_line(in, line))
      throw ParseError{"unexpected end of file: edge " + std::to_string(e + 1) + " of " + std::to_string(m) + " missing"};
    split_tokens(line, tok);
    size_t first = 0;
    if (edge_w) {
      if (tok.empty()) throw ParseError{"edge line " + std::to_string(e + 1) + " is empty"};
      el.weights.push_back(parse_weight(tok[0]));
      first = 1;
    }
    if (tok.size() <= first) throw ParseError{"edge line " + std::to_string(e + 1) + " lists no vertices"};
    for (size_t i = first; i < tok.size(); ++i) {
      const uint64_t id = parse_uint(tok[i], "vertex id");
      if (id < 1 || id > n)
        throw ParseError{"vertex id " + std::to_string(id) + " outside [1, " + std::to_string(n) + "] on edge line " +
                         std::to_string(e + 1)};
      el.pins.push_back(static_cast<uint32_t>(id - 1));
    }
    el.off.push_back(el.pins.size());
  }
  if (vertex_w) {
    for (uint64_t v = 0; v < n; ++v)
      if (!next_content_line(in, line)) throw ParseError{"unexpected end of file in vertex weight block"};
    out->num_warnings = 1;  // "vertex weights present but ignored; matching does not use them"
  }
  if (next_content_line(in, line)) throw ParseError{"trailing content after declared edges: '" + std::string(line) + "'"};
  build(el, static_cast<uint32_t>(n), degree_zero, out);
}

void parse_metis(const char* text, size_t len, int degree_zero, hlm_b200_host_graph* out) {
  LineReader in{text, text + len};
  std::string_view line;
  std::vector<std::string_view> tok;
  if (!next_content_line(in, line)) throw ParseError{"missing graph header line"};
  split_tokens(line, tok);
  if (tok.size() < 2 || tok.size() > 3) throw ParseError{"malformed graph header '" + std::string(line) + "'"};
  const uint64_t n = parse_uint(tok[0], "vertex count");
  const uint64_t m = parse_uint(tok[1], "edge count");
  check_count(n, "vertex count");
  check_count(m, "edge count");
  if (tok.size() == 3 && parse_uint(tok[2], "fmt code") != 0) throw ParseError{"weighted graph fmt codes are not supported"};
  std::vector<std::vector<uint32_t>> adj(n);
  for (uint64_t u = 0; u < n;) {
    if (!in.next(line)) throw ParseError{"unexpected end of file: adjacency line " + std::to_string(u + 1) + " missing"};
    if (line_kind(line) == 1) continue;  // comment lines do not consume a vertex slot (blank ones do)
    split_tokens(line, tok);
    auto& a = adj[u];
    for (auto t : tok) {
      const uint64_t id = parse_uint(t, "neighbor id");
      if (id < 1 || id > n)
        throw ParseError{"neighbor id " + std::to_string(id) + " outside [1, " + std::to_string(n) + "] on line for vertex " +
                         std::to_string(u + 1)};
      if (id - 1 == u) throw ParseError{"self-loop at vertex " + std::to_string(u + 1)};
      a.push_back(static_cast<uint32_t>(id - 1));
    }
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    ++u;
  }
  EdgeLists el;
  uint64_t count = 0;
  for (uint64_t u = 0; u < n; ++u)
    for (uint32_t v : adj[u]) {
      if (!std::binary_search(adj[v].begin(), adj[v].end(), static_cast<uint32_t>(u)))
        throw ParseError{"asymmetric adjacency: vertex " + std::to_string(u + 1) + " lists " + std::to_string(v + 1) +
                         " but not vice versa"};
      if (u < v) {
        el.pins.push_back(static_cast<uint32_t>(u));
        el.pins.push_back(v);
        el.off.push_back(el.pins.size());
        ++count;
      }
    }
  if (count != m)
    throw ParseError{"header declares " + std::to_string(m) + " edges but adjacency encodes " + std::to_string(count)};
  build(el, static_cast<uint32_t>(n), degree_zero, out);
}

char* dup_text(const std::string& s, size_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  *len = s.size();
  return p;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HLM_B200_OK;
  } catch (const ParseError& e) {
    set_error("%s", e.what.c_str());
    return HLM_B200_ERR_INPUT;
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    return HLM_B200_ERR_NOMEM;
  } catch (const std::length_error& e) {  // a header count no container can hold
    set_error("instance too large: %s", e.what());
    return HLM_B200_ERR_INPUT;
  } catch (const std::exception& e) {  // nothing may cross the extern "C" boundary
    set_error("%s", e.what());
    return HLM_B200_ERR_INPUT;
  } catch (...) {
    set_error("unknown failure");
    return HLM_B200_ERR_INPUT;
  }
}

// SplitMix64 as the reference's instance generators use it (generators.hpp:19-30)
struct SeqRng {
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

// generate_random (generators.hpp:65-93): per edge one size draw (consumed even when the span is 1), then
// vertex draws until `size` distinct ones; unused vertices are dropped and the rest renumbered.
void generate_random(uint32_t n, uint32_t m, uint32_t smin, uint32_t smax, uint64_t seed, hlm_b200_host_graph* out) {
  if (n == 0 || m == 0) throw ParseError{"random instance needs at least one vertex and one edge"};
  if (smin == 0 || smin > smax) throw ParseError{"random instance needs 1 <= min_edge_size <= max_edge_size"};
  if (smax > n) throw ParseError{"edge size " + std::to_string(smax) + " exceeds vertex count " + std::to_string(n)};
  SeqRng rng{seed};
  const uint32_t span = smax - smin + 1;
  EdgeLists el;
  el.off.reserve(static_cast<size_t>(m) + 1);
  el.pins.reserve(static_cast<size_t>(m) * ((smin + smax + 1) / 2));
  for (uint32_t e = 0; e < m; ++e) {
    const uint32_t size = smin + static_cast<uint32_t>(rng.next() % span);
    const size_t first = el.pins.size();
    while (el.pins.size() - first < size) {
      const uint32_t v = static_cast<uint32_t>(rng.next() % n);
      bool seen = false;
      for (size_t i = first; i < el.pins.size(); ++i) seen |= el.pins[i] == v;
      if (!seen) el.pins.push_back(v);
    }
    el.off.push_back(el.pins.size());
  }
  build(el, n, HLM_B200_DEGREE_ZERO_DROP, out);
}

// generate_tight_family (generators.hpp:37-54): d pair edges of weight 1, their left ends joined by one
// rank-d edge of weight 1 + epsilon
void generate_tight_family(uint32_t d, double epsilon, hlm_b200_host_graph* out) {
  if (d < 2) throw ParseError{"tight family needs d >= 2"};
  if (!(epsilon > 0.0)) throw ParseError{"tight family needs epsilon > 0"};
  EdgeLists el;
  for (uint32_t i = 0; i < d; ++i) {
    el.pins.push_back(i);
    el.pins.push_back(d + i);
    el.off.push_back(el.pins.size());
    el.weights.push_back(1.0);
  }
  for (uint32_t i = 0; i < d; ++i) el.pins.push_back(i);
  el.off.push_back(el.pins.size());
  el.weights.push_back(1.0 + epsilon);
  build(el, 2 * d, HLM_B200_DEGREE_ZERO_REJECT, out);
}

}  // namespace
}  // namespace hlmb

using namespace hlmb;

extern "C" {

int hlm_b200_parse_hgr(const char* text, size_t len, int degree_zero, hlm_b200_host_graph* out) {
  if (!out || (!text && len)) return HLM_B200_ERR_INPUT;
  std::memset(out, 0, sizeof(*out));
  const int rc = guarded([&] { parse_hgr(text, len, degree_zero, out); });
  if (rc != HLM_B200_OK) hlm_b200_host_graph_free(out);
  return rc;
}

int hlm_b200_parse_metis_graph(const char* text, size_t len, int degree_zero, hlm_b200_host_graph* out) {
  if (!out || (!text && len)) return HLM_B200_ERR_INPUT;
  std::memset(out, 0, sizeof(*out));
  const int rc = guarded([&] { parse_metis(text, len, degree_zero, out); });
  if (rc != HLM_B200_OK) hlm_b200_host_graph_free(out);
  return rc;
}

int hlm_b200_generate_random(uint32_t num_vertices, uint32_t num_edges, uint32_t min_edge_size, uint32_t max_edge_size,
                             uint64_t seed, hlm_b200_host_graph* out) {
  if (!out) return HLM_B200_ERR_INPUT;
  std::memset(out, 0, sizeof(*out));
  const int rc = guarded([&] { generate_random(num_vertices, num_edges, min_edge_size, max_edge_size, seed, out); });
  if (rc != HLM_B200_OK) hlm_b200_host_graph_free(out);
  return rc;
}

int hlm_b200_generate_tight_family(uint32_t d, double epsilon, hlm_b200_host_graph* out) {
  if (!out) return HLM_B200_ERR_INPUT;
  std::memset(out, 0, sizeof(*out));
  const int rc = guarded([&] { generate_tight_family(d, epsilon, out); });
  if (rc != HLM_B200_OK) hlm_b200_host_graph_free(out);
  return rc;
}

int hlm_b200_random_weights_1_100(uint32_t num_edges, uint64_t seed, double* out) {  // generators.hpp:96-101
  if (!out && num_edges) {
    set_error("null argument");
    return HLM_B200_ERR_INPUT;
  }
  SeqRng rng{seed ^ 0x517CC1B727220A95ull};
  for (uint32_t e = 0; e < num_edges; ++e) out[e] = static_cast<double>(1 + rng.next() % 100);
  return HLM_B200_OK;
}

void hlm_b200_host_graph_free(hlm_b200_host_graph* g) {
  if (!g) return;
  std::free(g->vertex_offsets);
  std::free(g->vertex_incidence);
  std::free(g->edge_offsets);
  std::free(g->edge_members);
  std::free(g->base_weights);
  std::memset(g, 0, sizeof(*g));
}

int hlm_b200_write_hgr(const hlm_b200_csr_view* h, char** text, size_t* len) {  // io.hpp:146-171
  if (!h || !text || !len || (h->num_edges && (!h->edge_offsets || !h->edge_members || !h->base_weights)))
    return HLM_B200_ERR_INPUT;
  return guarded([&] {
    bool weighted = false;
    for (uint32_t e = 0; e < h->num_edges; ++e) weighted |= (h->base_weights[e] != 1.0);
    std::string out = std::to_string(h->num_edges) + ' ' + std::to_string(h->num_vertices);
    if (weighted) out += " 1";
    out += '\n';
    char buf[64];
    for (uint32_t e = 0; e < h->num_edges; ++e) {
      if (weighted) {
        const double w = h->base_weights[e];
        if (w == static_cast<double>(static_cast<int64_t>(w))) {
          std::snprintf(buf, sizeof(buf), "%lld", static_cast<long long>(w));
          out += buf;
        } else {  // shortest form that parses back to the same double
          auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), w);
          (void)ec;
          out.append(buf, static_cast<size_t>(ptr - buf));
        }
      }
      bool lead = !weighted;
      for (uint64_t i = h->edge_offsets[e]; i < h->edge_offsets[e + 1]; ++i) {
        if (!lead) out += ' ';
        lead = false;
        out += std::to_string(h->edge_members[i] + 1u);
      }
      out += '\n';
    }
    *text = dup_text(out, len);
  });
}

int hlm_b200_write_matching(const uint32_t* matched, uint64_t count, double total_weight, uint32_t rounds, char** text,
                            size_t* len) {  // io.hpp:240-247
  if ((!matched && count) || !text || !len) return HLM_B200_ERR_INPUT;
  return guarded([&] {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.6f", total_weight);
    std::string out = std::string("% weight ") + buf + "\n% size " + std::to_string(count) + "\n% rounds " +
                      std::to_string(rounds) + "\n";
    for (uint64_t i = 0; i < count; ++i) {
      out += std::to_string(matched[i]);
      out += '\n';
    }
    *text = dup_text(out, len);
  });
}

int hlm_b200_parse_matching(const char* text, size_t len, uint32_t** ids, uint64_t* count) {  // io.hpp:249-257
  if ((!text && len) || !ids || !count) return HLM_B200_ERR_INPUT;
  *ids = nullptr;
  *count = 0;
  return guarded([&] {
    LineReader in{text, text + len};
    std::string_view line;
    std::vector<std::string_view> tok;
    std::vector<uint32_t> out;
    while (next_content_line(in, line)) {
      split_tokens(line, tok);
      for (auto t : tok) out.push_back(static_cast<uint32_t>(parse_uint(t, "edge id")));
    }
    *ids = dup(out);
    *count = out.size();
  });
}

void hlm_b200_text_free(void* p) { std::free(p); }

}  // extern "C"
