// Host-side data formats on either side of the decode path (SURVEY.md §8f
// rank 3), native so ingestion does not bottleneck the GPU:
//  * Kaldi binary ARK float matrices (reference kaldi_io.py:82-130), single
//    records or a batch read by a host thread pool straight into a caller
//    (pinned) staging buffer;
//  * PTA1 prefix-tree files (lexicon_trie.py:178-224), read/write;
//  * build_trie (lexicon_trie.py:227-276) as a sort + longest-common-prefix
//    sweep over char-id sequences (same arrays as the reference);
//  * Kaldi SCP index parsing (kaldi_io.py:46-77) over the file's bytes, with
//    Python's text-mode line splitting and str.split/strip whitespace, and
//    the ARK record + SCP line appender (kaldi_io.py:129-150).
// No GPU is touched here.
#include "common.cuh"

#include <algorithm>
#include <atomic>
#include <unordered_map>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace fb {
namespace {

struct File {
  FILE* f = nullptr;
  explicit File(const char* path, const char* mode) : f(fopen(path, mode)) {}
  ~File() {
    if (f) fclose(f);
  }
};

std::string at(const char* path, int64_t offset) {
  return std::string(path) + "@" + std::to_string(offset);
}

std::string bytes_repr(const unsigned char* b, size_t n) {
  // python-style bytes literal, e.g. b'\x00B'
  std::string s = "b'";
  for (size_t i = 0; i < n; ++i) {
    const unsigned char c = b[i];
    if (c == '\\' || c == '\'') {
      s += '\\';
      s += (char)c;
    } else if (c >= 32 && c < 127) {
      s += (char)c;
    } else {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", c);
      s += buf;
    }
  }
  return s + "'";
}

// Parse one record header + payload; dst may be null (dimension query).
int read_record(FILE* f, const char* path, int64_t offset, float* dst, int64_t cap,
                int32_t* rows, int32_t* cols, std::string& err) {
  if (fseeko(f, (off_t)offset, SEEK_SET) != 0) {
    err = at(path, offset) + ": cannot seek";
    return FB_ERR_IO;
  }
  unsigned char marker[2] = {0, 0};
  const size_t nm = fread(marker, 1, 2, f);
  if (nm != 2 || marker[0] != 0 || marker[1] != 'B') {
    err = at(path, offset) + ": bad binary marker " + bytes_repr(marker, nm);
    return FB_ERR_FORMAT;
  }
  unsigned char tok[3] = {0, 0, 0};
  const size_t nt = fread(tok, 1, 3, f);
  if (nt != 3 || memcmp(tok, "FM ", 3) != 0) {
    static const char* names[][2] = {{"DM ", "double matrix"},  {"CM ", "compressed matrix"},
                                     {"CM2", "compressed matrix"}, {"CM3", "compressed matrix"},
                                     {"FV ", "float vector"},   {"DV ", "double vector"}};
    for (auto& nmn : names)
      if (nt == 3 && memcmp(tok, nmn[0], 3) == 0) {
        err = at(path, offset) + ": unsupported record type " + nmn[1] + " (" +
              bytes_repr(tok, 3) + "); only float32 matrices are supported";
        return FB_ERR_FORMAT;
      }
    err = at(path, offset) + ": bad header token " + bytes_repr(tok, nt);
    return FB_ERR_FORMAT;
  }
  int32_t dims[2];
  const char* what[2] = {"rows", "cols"};
  for (int d = 0; d < 2; ++d) {
    unsigned char sz = 0;
    const size_t ns = fread(&sz, 1, 1, f);
    if (ns != 1 || sz != 4) {
      err = at(path, offset) + ": bad " + what[d] + " size byte " + bytes_repr(&sz, ns);
      return FB_ERR_FORMAT;
    }
    unsigned char b[4];
    if (fread(b, 1, 4, f) != 4) {
      err = at(path, offset) + ": truncated " + what[d] + " field";
      return FB_ERR_IO;
    }
    dims[d] = (int32_t)((uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) |
                        ((uint32_t)b[3] << 24));
  }
  if (dims[0] <= 0 || dims[1] <= 0) {
    err = at(path, offset) + ": bad shape " + std::to_string(dims[0]) + "x" +
          std::to_string(dims[1]);
    return FB_ERR_FORMAT;
  }
  *rows = dims[0];
  *cols = dims[1];
  if (!dst) return FB_OK;
  const int64_t n = (int64_t)dims[0] * dims[1];
  if (cap < n) {
    err = at(path, offset) + ": destination holds " + std::to_string(cap) + " of " +
          std::to_string(n) + " floats";
    return FB_ERR_VALUE;
  }
  const size_t got = fread(dst, 1, (size_t)n * 4, f);  // little-endian host
  if ((int64_t)got != n * 4) {
    err = at(path, offset) + ": truncated payload (" + std::to_string(got) + " of " +
          std::to_string(n * 4) + " bytes)";
    return FB_ERR_IO;
  }
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(dst[i])) {
      err = at(path, offset) + ": non-finite values in matrix";
      return FB_ERR_FORMAT;
    }
  return FB_OK;
}

constexpr char kMagic[4] = {'P', 'T', 'A', '1'};

// Byte length of the whitespace code point at p (Python str.isspace set:
// ASCII \t-\r, 0x1c-0x1f, space; U+0085, U+00A0, U+1680, U+2000-U+200A,
// U+2028, U+2029, U+202F, U+205F, U+3000), 0 if none.
int ws_len(const unsigned char* p, const unsigned char* e) {
  const unsigned c = p[0];
  if (c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f)) return 1;
  if (c == 0xc2 && p + 1 < e && (p[1] == 0x85 || p[1] == 0xa0)) return 2;
  if (c == 0xe1 && p + 2 < e && p[1] == 0x9a && p[2] == 0x80) return 3;
  if (c == 0xe2 && p + 2 < e) {
    if (p[1] == 0x80 && (p[2] <= 0x8a || p[2] == 0xa8 || p[2] == 0xa9 || p[2] == 0xaf)) return 3;
    if (p[1] == 0x81 && p[2] == 0x9f) return 3;
  }
  if (c == 0xe3 && p + 2 < e && p[1] == 0x80 && p[2] == 0x80) return 3;
  return 0;
}

struct Span {
  const unsigned char* b;
  const unsigned char* e;
  bool empty() const { return b >= e; }
  std::string str() const { return std::string((const char*)b, (size_t)(e - b)); }
};

Span strip(Span s) {
  for (int n; s.b < s.e && (n = ws_len(s.b, s.e)) > 0;) s.b += n;
  // trailing: scan forward remembering where the last non-space run ended
  const unsigned char* last = s.b;
  for (const unsigned char* p = s.b; p < s.e;) {
    const int n = ws_len(p, s.e);
    if (n) {
      p += n;
    } else {
      ++p;
      while (p < s.e && (*p & 0xc0) == 0x80) ++p;   // rest of the code point
      last = p;
    }
  }
  s.e = last;
  return s;
}

// Python int(text) for ASCII decimal text: optional sign, digits with single
// underscores between them, surrounding whitespace allowed.
bool parse_int(Span s, int64_t* out) {
  s = strip(s);
  if (s.empty()) return false;
  bool neg = false;
  if (*s.b == '+' || *s.b == '-') {
    neg = *s.b == '-';
    ++s.b;
  }
  if (s.empty() || *s.b == '_') return false;
  unsigned long long v = 0;
  bool prev_us = false;
  for (const unsigned char* p = s.b; p < s.e; ++p) {
    if (*p == '_') {
      if (prev_us) return false;
      prev_us = true;
      continue;
    }
    if (*p < '0' || *p > '9') return false;
    prev_us = false;
    if (v > (9223372036854775807ULL - (*p - '0')) / 10) return false;
    v = v * 10 + (*p - '0');
  }
  if (prev_us) return false;
  *out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

}  // namespace
}  // namespace fb

using namespace fb;

extern "C" int fb_ark_read_matrix(const char* ark_path, int64_t offset, float* dst,
                                  int64_t dst_capacity, int32_t* rows, int32_t* cols) {
  FB_CHECK_ARG(ark_path && rows && cols && offset >= 0, "bad ARK read arguments");
  File f(ark_path, "rb");
  if (!f.f) return fail(FB_ERR_IO, std::string(ark_path) + ": cannot open");
  std::string err;
  const int rc = read_record(f.f, ark_path, offset, dst, dst_capacity, rows, cols, err);
  return rc ? fail(rc, err) : FB_OK;
}

extern "C" int fb_ark_read_batch(int32_t n, const char* const* ark_paths, const int64_t* offsets,
                                 float* dst, const int64_t* dst_offsets,
                                 const int64_t* capacities, int32_t* rows, int32_t* cols,
                                 int32_t threads) {
  FB_CHECK_ARG(n >= 0 && ark_paths && offsets && rows && cols, "bad ARK batch arguments");
  FB_CHECK_ARG(!dst || (dst_offsets && capacities), "batch destination needs offsets");
  if (n == 0) return FB_OK;
  const int nt = std::max(1, std::min<int>(threads > 0 ? threads : 8, n));
  std::atomic<int> next(0), first_bad(n);
  std::vector<int> codes(n, FB_OK);
  std::vector<std::string> errs(n);
  auto work = [&]() {
    for (int i = next++; i < n; i = next++) {
      File f(ark_paths[i], "rb");
      if (!f.f) {
        codes[i] = FB_ERR_IO;
        errs[i] = std::string(ark_paths[i]) + ": cannot open";
      } else {
        codes[i] = read_record(f.f, ark_paths[i], offsets[i], dst ? dst + dst_offsets[i] : nullptr,
                               dst ? capacities[i] : 0, rows + i, cols + i, errs[i]);
      }
      if (codes[i]) {
        int cur = first_bad.load();
        while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {}
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  const int bad = first_bad.load();             // report the first failing record in order
  return bad < n ? fail(codes[bad], errs[bad]) : FB_OK;
}

extern "C" int fb_pta1_read_header(const char* path, int32_t* num_states, int32_t* num_words,
                                   int32_t* max_out, int32_t* alphabet) {
  FB_CHECK_ARG(path && num_states && num_words && max_out && alphabet, "bad PTA1 arguments");
  File f(path, "rb");
  if (!f.f) return fail(FB_ERR_IO, std::string(path) + ": cannot open");
  unsigned char head[20];
  const size_t got = fread(head, 1, 20, f.f);
  if (got < 4 || memcmp(head, kMagic, 4) != 0)
    return fail(FB_ERR_FORMAT, std::string(path) + ": bad magic " + bytes_repr(head, std::min<size_t>(got, 4)));
  if (got < 20) return fail(FB_ERR_FORMAT, std::string(path) + ": truncated header");
  int32_t v[4];
  memcpy(v, head + 4, 16);
  if (v[0] < 1 || v[2] < 1 || v[1] < 1 || v[3] < 1)
    return fail(FB_ERR_FORMAT, std::string(path) + ": bad counts in header");
  *num_states = v[0];
  *num_words = v[1];
  *max_out = v[2];
  *alphabet = v[3];
  return FB_OK;
}

extern "C" int fb_pta1_read(const char* path, int32_t* transitions, int32_t* edge_labels,
                            uint8_t* is_final, int32_t* word_index, int32_t* ub_index,
                            int32_t* lb_index) {
  int32_t S, W, D, A;
  int rc = fb_pta1_read_header(path, &S, &W, &D, &A);
  if (rc) return rc;
  FB_CHECK_ARG(transitions && edge_labels && is_final && word_index && ub_index && lb_index,
               "null PTA1 arrays");
  File f(path, "rb");
  if (!f.f) return fail(FB_ERR_IO, std::string(path) + ": cannot open");
  fseeko(f.f, 0, SEEK_END);
  const int64_t size = (int64_t)ftello(f.f);
  fseeko(f.f, 20, SEEK_SET);
  const int64_t SD = (int64_t)S * D;
  struct Part { void* p; int64_t bytes; } parts[6] = {
      {transitions, SD * 4}, {edge_labels, SD * 4}, {is_final, (int64_t)S},
      {word_index, (int64_t)S * 4}, {ub_index, (int64_t)S * 4}, {lb_index, (int64_t)S * 4}};
  int64_t pos = 20;
  for (auto& pt : parts) {
    if (pos + pt.bytes > size) return fail(FB_ERR_FORMAT, std::string(path) + ": truncated array data");
    if ((int64_t)fread(pt.p, 1, (size_t)pt.bytes, f.f) != pt.bytes)
      return fail(FB_ERR_FORMAT, std::string(path) + ": truncated array data");
    pos += pt.bytes;
  }
  if (pos != size)
    return fail(FB_ERR_FORMAT, std::string(path) + ": " + std::to_string(size - pos) + " trailing bytes");
  return FB_OK;
}

extern "C" int fb_pta1_write(const char* path, int32_t num_states, int32_t num_words,
                             int32_t max_out, int32_t alphabet, const int32_t* transitions,
                             const int32_t* edge_labels, const uint8_t* is_final,
                             const int32_t* word_index, const int32_t* ub_index,
                             const int32_t* lb_index) {
  FB_CHECK_ARG(path && transitions && edge_labels && is_final && word_index && ub_index &&
                   lb_index && num_states > 0 && max_out > 0,
               "bad PTA1 write arguments");
  File f(path, "wb");
  if (!f.f) return fail(FB_ERR_IO, std::string(path) + ": cannot open for writing");
  const int32_t head[4] = {num_states, num_words, max_out, alphabet};
  const int64_t SD = (int64_t)num_states * max_out;
  bool ok = fwrite(kMagic, 1, 4, f.f) == 4 && fwrite(head, 4, 4, f.f) == 4 &&
            (int64_t)fwrite(transitions, 4, SD, f.f) == SD &&
            (int64_t)fwrite(edge_labels, 4, SD, f.f) == SD &&
            (int64_t)fwrite(is_final, 1, num_states, f.f) == num_states &&
            (int64_t)fwrite(word_index, 4, num_states, f.f) == num_states &&
            (int64_t)fwrite(ub_index, 4, num_states, f.f) == num_states &&
            (int64_t)fwrite(lb_index, 4, num_states, f.f) == num_states;
  return ok ? FB_OK : fail(FB_ERR_IO, std::string(path) + ": write failed");
}

// ---- batch staging ------------------------------------------------------------
extern "C" int fb_host_copy_batch(int32_t n, const void* const* srcs, void* const* dsts,
                                  const int64_t* bytes, int32_t threads) {
  FB_CHECK_ARG(n >= 0 && srcs && dsts && bytes, "bad host copy arguments");
  if (n == 0) return FB_OK;
  const int nt = std::max(1, std::min<int>(threads > 0 ? threads : 8, n));
  std::atomic<int> next(0);
  auto work = [&]() {
    for (int i = next++; i < n; i = next++)
      if (bytes[i] > 0) memcpy(dsts[i], srcs[i], (size_t)bytes[i]);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return FB_OK;
}

// ---- build_trie --------------------------------------------------------------
// Words as char-id sequences (chars[word_offsets[i] .. word_offsets[i+1])), all
// non-empty, distinct, ids in [0, alphabet).  Ranks = lexicographic order of the
// sequences; states are created along the sweep (new states only past the LCP
// with the previous word), so per-parent children come in ascending label order.
namespace {
struct TrieBuild {
  std::vector<int32_t> parent, label, first, last, rank;
  int32_t max_out = 0;
};

int build(int32_t n, const int32_t* chars, const int64_t* off, int32_t alphabet, TrieBuild& tb,
          std::string& err) {
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  auto less = [&](int32_t a, int32_t b) {
    return std::lexicographical_compare(chars + off[a], chars + off[a + 1], chars + off[b],
                                        chars + off[b + 1]);
  };
  std::sort(order.begin(), order.end(), less);
  int64_t total = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t len = off[i + 1] - off[i];
    if (len <= 0) { err = "empty word in vocabulary"; return FB_ERR_FORMAT; }
    for (int64_t j = off[i]; j < off[i + 1]; ++j)
      if (chars[j] < 0 || chars[j] >= alphabet) { err = "character id out of range"; return FB_ERR_FORMAT; }
    total += len;
  }
  tb.parent.assign(1, -1); tb.label.assign(1, -1); tb.first.assign(1, 0); tb.last.assign(1, n - 1);
  tb.rank.assign(1, -1);
  tb.parent.reserve(total + 1);
  std::vector<int32_t> path(1, 0);
  const int32_t* prev = nullptr;
  int64_t prev_len = 0;
  for (int32_t r = 0; r < n; ++r) {
    const int32_t w = order[r];
    const int32_t* q = chars + off[w];
    const int64_t len = off[w + 1] - off[w];
    int64_t lcp = 0;
    const int64_t m = std::min(prev_len, len);
    while (lcp < m && prev[lcp] == q[lcp]) ++lcp;
    if (prev && lcp == len && lcp == prev_len) { err = "duplicate word in vocabulary"; return FB_ERR_FORMAT; }
    path.resize(lcp + 1);
    for (int64_t pos = lcp; pos < len; ++pos) {
      const int32_t st = (int32_t)tb.parent.size();
      tb.parent.push_back(path.back());
      tb.label.push_back(q[pos]);
      tb.first.push_back(r);
      tb.last.push_back(r);
      tb.rank.push_back(-1);
      path.push_back(st);
    }
    for (int32_t st : path) tb.last[st] = r;
    tb.rank[path.back()] = r;
    prev = q;
    prev_len = len;
  }
  std::vector<int32_t> deg(tb.parent.size(), 0);
  for (size_t st = 1; st < tb.parent.size(); ++st) tb.max_out = std::max(tb.max_out, ++deg[tb.parent[st]]);
  if (tb.max_out == 0) tb.max_out = 1;
  return FB_OK;
}
}  // namespace

extern "C" int fb_trie_build_sizes(int32_t n_words, const int32_t* chars,
                                   const int64_t* word_offsets, int32_t alphabet,
                                   int32_t* num_states, int32_t* max_out) {
  FB_CHECK_ARG(n_words > 0 && chars && word_offsets && num_states && max_out, "bad trie build arguments");
  TrieBuild tb;
  std::string err;
  const int rc = build(n_words, chars, word_offsets, alphabet, tb, err);
  if (rc) return fail(rc, err);
  *num_states = (int32_t)tb.parent.size();
  *max_out = tb.max_out;
  return FB_OK;
}

extern "C" int fb_trie_build(int32_t n_words, const int32_t* chars, const int64_t* word_offsets,
                             int32_t alphabet, int32_t num_states, int32_t max_out,
                             int32_t* transitions, int32_t* edge_labels, uint8_t* is_final,
                             int32_t* word_index, int32_t* ub_index, int32_t* lb_index) {
  FB_CHECK_ARG(n_words > 0 && chars && word_offsets && transitions && edge_labels && is_final &&
                   word_index && ub_index && lb_index, "bad trie build arguments");
  TrieBuild tb;
  std::string err;
  const int rc = build(n_words, chars, word_offsets, alphabet, tb, err);
  if (rc) return fail(rc, err);
  const int32_t S = (int32_t)tb.parent.size();
  FB_CHECK_ARG(S == num_states && tb.max_out == max_out, "trie sizes changed between calls");
  const int64_t SD = (int64_t)S * max_out;
  std::fill(transitions, transitions + SD, -1);
  std::fill(edge_labels, edge_labels + SD, -1);
  std::vector<int32_t> slot(S, 0);
  for (int32_t st = 1; st < S; ++st) {           // creation order == ascending label per parent
    const int32_t p = tb.parent[st];
    transitions[(int64_t)p * max_out + slot[p]] = st;
    edge_labels[(int64_t)p * max_out + slot[p]] = tb.label[st];
    ++slot[p];
  }
  for (int32_t st = 0; st < S; ++st) {
    is_final[st] = tb.rank[st] >= 0;
    word_index[st] = tb.rank[st];
    ub_index[st] = tb.last[st];
    lb_index[st] = tb.first[st] - 1;
  }
  return FB_OK;
}

/* SCP index lines "utt_id ark_path:offset" (reference kaldi_io.py:46-77).
 * Lines split as Python's text mode does (\n, \r\n, \r), then strip() /
 * split(None, 1) / rpartition(':') / int().  Output per entry:
 * "utt_id\0ark_path\0" into `out` (capacity >= len) and the offset.  A
 * malformed line returns FB_ERR_FORMAT with err[0] = kind (1 field count,
 * 2 missing ':offset', 3 offset not an integer, 4 negative offset,
 * 5 duplicate id), err[1] = line number, err[2] = first line of a duplicate,
 * and the offending text (offset text / negative value / id) in `out`. */
extern "C" int fb_scp_parse(const char* text, int64_t len, char* out, int64_t out_cap,
                            int64_t* out_len, int64_t* offsets, int32_t* n_entries,
                            int32_t* err) {
  FB_CHECK_ARG(text && out && out_len && offsets && n_entries && err && len >= 0,
               "bad SCP parse arguments");
  const unsigned char* p = (const unsigned char*)text;
  const unsigned char* end = p + len;
  int64_t o = 0;
  int32_t n = 0, lineno = 0;
  std::unordered_map<std::string, int32_t> seen;
  auto put = [&](Span s) {
    const int64_t k = s.e - s.b;
    if (o + k + 1 > out_cap) return false;
    memcpy(out + o, s.b, (size_t)k);
    o += k;
    out[o++] = '\0';
    return true;
  };
  auto bad = [&](int kind, int aux, Span what) {
    err[0] = kind;
    err[1] = lineno;
    err[2] = aux;
    o = 0;
    const int64_t k = std::min<int64_t>(what.e - what.b, out_cap);
    memcpy(out, what.b, (size_t)std::max<int64_t>(k, 0));
    *out_len = std::max<int64_t>(k, 0);
    return fail(FB_ERR_FORMAT, "SCP line " + std::to_string(lineno));
  };
  while (p < end) {
    const unsigned char* q = p;
    while (q < end && *q != '\n' && *q != '\r') ++q;
    Span line{p, q};
    p = q;
    if (p < end && *p == '\r') ++p;
    if (q < end && *q == '\r' && p < end && *p == '\n') ++p;
    else if (q < end && *q == '\n') ++p;
    ++lineno;
    line = strip(line);
    if (line.empty()) continue;
    // split(None, 1): the id up to the first whitespace, the rest stripped left
    const unsigned char* w = line.b;
    while (w < line.e && ws_len(w, line.e) == 0) ++w;
    if (w >= line.e) return bad(1, 0, line);
    Span id{line.b, w};
    Span rest{w, line.e};
    rest = strip(rest);
    // rpartition(':')
    const unsigned char* c = rest.e;
    while (c > rest.b && c[-1] != ':') --c;
    if (c == rest.b) return bad(2, 0, rest);          // no ':' at all
    Span ark{rest.b, c - 1}, off{c, rest.e};
    if (ark.empty()) return bad(2, 0, rest);
    int64_t v;
    if (!parse_int(off, &v)) return bad(3, 0, off);
    if (v < 0) return bad(4, 0, off);
    const std::string key = id.str();
    auto it = seen.find(key);
    if (it != seen.end()) return bad(5, it->second, id);
    seen.emplace(key, lineno);
    if (!put(id) || !put(ark)) return fail(FB_ERR_VALUE, "SCP output buffer too small");
    offsets[n++] = v;
  }
  *n_entries = n;
  *out_len = o;
  return FB_OK;
}

/* Append one binary float32 record "utt_id \0BFM \4<rows>\4<cols><data>" to
 * the ARK and "utt_id ark_path:offset\n" to the SCP (kaldi_io.py:129-150);
 * *offset = position of the binary marker.  The caller validated the id and
 * the matrix (ValueErrors live in Python, as in the reference). */
extern "C" int fb_ark_append_matrix(const char* ark_path, const char* scp_path,
                                    const char* utt_id, const float* data, int32_t rows,
                                    int32_t cols, int64_t* offset) {
  FB_CHECK_ARG(ark_path && scp_path && utt_id && data && offset && rows > 0 && cols > 0,
               "bad ARK append arguments");
  int64_t off;
  {
    File f(ark_path, "ab");
    if (!f.f) return fail(FB_ERR_IO, std::string(ark_path) + ": cannot open for append");
    const size_t idn = strlen(utt_id);
    if (fwrite(utt_id, 1, idn, f.f) != idn || fputc(' ', f.f) == EOF || fflush(f.f) != 0)
      return fail(FB_ERR_IO, std::string(ark_path) + ": write failed");
    off = (int64_t)ftello(f.f);
    unsigned char hdr[15] = {0, 'B', 'F', 'M', ' ', 4, 0, 0, 0, 0, 4, 0, 0, 0, 0};
    memcpy(hdr + 6, &rows, 4);                        // little-endian host (x86-64)
    memcpy(hdr + 11, &cols, 4);
    const size_t nel = (size_t)rows * (size_t)cols;
    if (fwrite(hdr, 1, sizeof hdr, f.f) != sizeof hdr ||
        fwrite(data, sizeof(float), nel, f.f) != nel)
      return fail(FB_ERR_IO, std::string(ark_path) + ": write failed");
  }
  File s(scp_path, "a");
  if (!s.f) return fail(FB_ERR_IO, std::string(scp_path) + ": cannot open for append");
  if (fprintf(s.f, "%s %s:%lld\n", utt_id, ark_path, (long long)off) < 0)
    return fail(FB_ERR_IO, std::string(scp_path) + ": write failed");
  *offset = off;
  return FB_OK;
}
