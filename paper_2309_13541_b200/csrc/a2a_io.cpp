// Native schedule loader.
//
// Reads the reference's on-disk formats straight into the C-ABI op table:
//   * the XML dialect of a2aflow.schedule.emit_schedule_xml / parse_schedule_xml
//     (reference pkg/src/a2aflow/schedule.py:318-384), plain or gzip, with the
//     same rejects and messages (missing attribute, root element, unknown mode,
//     unexpected element, step outside [0, nsteps), bad chunk range; any
//     syntax error -> "malformed XML: ...");
//   * the route sidecar `<out>.routes.json` written by `a2a compile --mode path`
//     (reference src/cli.py:289-292), lowered hop i -> step i exactly like
//     lowering.lower_path_to_steps (optionally collapsing host-augmented ids).
// and writes / reads this package's binary op table (A2ATBL1: header, int32
// op rows, SHA-256 trailer), the form a lowered schedule is kept in once it
// has been parsed -- GK(256,4)'s 255 890 hop-ops load without XML parsing.
// a2a_sha256_file gives the digests of the reference's run manifest
// (reference src/cli.py:30-55).
#include <zlib.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "a2a_internal.h"

namespace a2a {
namespace {

bool read_file(const char* path, std::string* out, std::string* err) {
  gzFile f = gzopen(path, "rb");  // transparently reads uncompressed files too
  if (!f) {
    *err = std::string("cannot open ") + path;
    return false;
  }
  char buf[1 << 16];
  int n;
  while ((n = gzread(f, buf, sizeof buf)) > 0) out->append(buf, (size_t)n);
  int zerr = 0;
  const char* msg = gzerror(f, &zerr);
  gzclose(f);
  if (n < 0 || (zerr != Z_OK && zerr != Z_STREAM_END)) {
    *err = std::string("read error on ") + path + ": " + (msg ? msg : "");
    return false;
  }
  return true;
}

struct Elem {
  std::string tag;
  std::vector<std::pair<std::string, std::string>> attrs;
  std::vector<Elem> kids;
  const std::string* get(const char* k) const {
    for (auto& a : attrs)
      if (a.first == k) return &a.second;
    return nullptr;
  }
};

// Minimal XML reader for the schedule dialect: prolog, comments, elements with
// quoted attributes, self-closing tags, whitespace text.
struct XmlParser {
  const std::string& s;
  size_t i = 0;
  std::string err;
  explicit XmlParser(const std::string& x) : s(x) {}
  bool fail(const char* what) {
    if (err.empty()) {
      size_t line = 1 + std::count(s.begin(), s.begin() + std::min(i, s.size()), '\n');
      char b[160];
      snprintf(b, sizeof b, "%s: line %zu", what, line);
      err = b;
    }
    return false;
  }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
  }
  bool skip_misc() {  // prolog, comments, whitespace
    for (;;) {
      ws();
      if (s.compare(i, 5, "<?xml") == 0 || s.compare(i, 2, "<?") == 0) {
        size_t e = s.find("?>", i);
        if (e == std::string::npos) return fail("unclosed processing instruction");
        i = e + 2;
      } else if (s.compare(i, 4, "<!--") == 0) {
        size_t e = s.find("-->", i);
        if (e == std::string::npos) return fail("unclosed comment");
        i = e + 3;
      } else {
        return true;
      }
    }
  }
  static bool namech(char c) {
    return isalnum((unsigned char)c) || c == '_' || c == '-' || c == ':' || c == '.';
  }
  bool element(Elem* e) {
    if (i >= s.size() || s[i] != '<') return fail("no element found");
    ++i;
    size_t b = i;
    while (i < s.size() && namech(s[i])) ++i;
    if (i == b) return fail("not well-formed (invalid token)");
    e->tag = s.substr(b, i - b);
    for (;;) {
      ws();
      if (i >= s.size()) return fail("unclosed token");
      if (s[i] == '/') {
        if (i + 1 < s.size() && s[i + 1] == '>') { i += 2; return true; }
        return fail("not well-formed (invalid token)");
      }
      if (s[i] == '>') { ++i; break; }
      size_t nb = i;
      while (i < s.size() && namech(s[i])) ++i;
      if (i == nb) return fail("not well-formed (invalid token)");
      std::string name = s.substr(nb, i - nb);
      ws();
      if (i >= s.size() || s[i] != '=') return fail("not well-formed (invalid token)");
      ++i;
      ws();
      if (i >= s.size() || (s[i] != '"' && s[i] != '\'')) return fail("not well-formed (invalid token)");
      char q = s[i++];
      size_t vb = i;
      while (i < s.size() && s[i] != q) ++i;
      if (i >= s.size()) return fail("unclosed token");
      std::string val = s.substr(vb, i - vb);
      ++i;
      for (auto& a : e->attrs)
        if (a.first == name) return fail("duplicate attribute");
      e->attrs.emplace_back(std::move(name), std::move(val));
    }
    // content: children and whitespace only
    for (;;) {
      if (!skip_misc()) return false;
      if (i >= s.size()) return fail("unclosed token");
      if (s.compare(i, 2, "</") == 0) {
        i += 2;
        size_t b2 = i;
        while (i < s.size() && namech(s[i])) ++i;
        if (s.compare(b2, i - b2, e->tag) != 0 || i - b2 != e->tag.size())
          return fail("mismatched tag");
        ws();
        if (i >= s.size() || s[i] != '>') return fail("unclosed token");
        ++i;
        return true;
      }
      if (s[i] != '<') return fail("not well-formed (text content)");
      e->kids.emplace_back();
      if (!element(&e->kids.back())) return false;
    }
  }
  bool document(Elem* root) {
    if (!skip_misc() || !element(root)) return false;
    if (!skip_misc()) return false;
    if (i != s.size()) return fail("junk after document element");
    return true;
  }
};

bool to_int(const std::string& v, int64_t* out) {
  // Python int(): optional whitespace and sign, decimal digits (underscores allowed between)
  size_t a = 0, b = v.size();
  while (a < b && isspace((unsigned char)v[a])) ++a;
  while (b > a && isspace((unsigned char)v[b - 1])) --b;
  if (a == b) return false;
  bool neg = false;
  if (v[a] == '+' || v[a] == '-') { neg = v[a] == '-'; ++a; }
  if (a == b) return false;
  int64_t x = 0;
  bool digit = false;
  for (size_t k = a; k < b; ++k) {
    char c = v[k];
    if (c == '_' && digit && k + 1 < b && isdigit((unsigned char)v[k + 1])) continue;
    if (!isdigit((unsigned char)c)) return false;
    x = x * 10 + (c - '0');
    digit = true;
    if (x > (int64_t)1 << 40) return false;
  }
  *out = neg ? -x : x;
  return true;
}

struct Loaded {
  int32_t n = 0, nsteps = 0, q = 0, mode = 0;
  double chunk_bytes = 0;
  std::vector<a2a_op> ops;
};

int attr_int(const Elem& e, const char* k, int64_t* out) {
  const std::string* v = e.get(k);
  if (!v) return fail(A2A_ERR_EVAL, std::string("missing attribute '") + k + "' on <" + e.tag + ">");
  if (!to_int(*v, out))
    return fail(A2A_ERR_INVALID, std::string("invalid literal for int(): '") + *v + "'");
  return A2A_OK;
}

// parse_schedule_xml (src/schedule.py:349-384); ScheduleError texts -> A2A_ERR_EVAL
int load_xml(const char* path, Loaded* L) {
  std::string text, err;
  if (!read_file(path, &text, &err)) return fail(A2A_ERR_INVALID, err);
  XmlParser xp(text);
  Elem root;
  if (!xp.document(&root)) return fail(A2A_ERR_EVAL, "malformed XML: " + xp.err);
  if (root.tag != "schedule")
    return fail(A2A_ERR_EVAL, "root element is <" + root.tag + ">, not <schedule>");
  int64_t n, nsteps, q;
  int rc;
  if ((rc = attr_int(root, "n", &n)) || (rc = attr_int(root, "nsteps", &nsteps))) return rc;
  const std::string* cb = root.get("chunkbytes");
  if (!cb) return fail(A2A_ERR_EVAL, "missing attribute 'chunkbytes' on <schedule>");
  if ((rc = attr_int(root, "q", &q))) return rc;
  const std::string* mode = root.get("mode");
  if (!mode) return fail(A2A_ERR_EVAL, "missing attribute 'mode' on <schedule>");
  if (*mode != "ts" && *mode != "path")
    return fail(A2A_ERR_EVAL, "unknown mode '" + *mode + "'");
  L->n = (int32_t)n;
  L->nsteps = (int32_t)nsteps;
  L->q = (int32_t)q;
  L->mode = (*mode == "ts") ? 0 : 1;
  L->chunk_bytes = strtod(cb->c_str(), nullptr);
  for (const Elem& st : root.kids) {
    if (st.tag != "step") return fail(A2A_ERR_EVAL, "unexpected element <" + st.tag + ">");
    int64_t t;
    if ((rc = attr_int(st, "t", &t))) return rc;
    if (!(0 <= t && t < nsteps)) {
      char b[96];
      snprintf(b, sizeof b, "step t=%lld outside [0, %lld)", (long long)t, (long long)nsteps);
      return fail(A2A_ERR_EVAL, b);
    }
    for (const Elem& se : st.kids) {
      if (se.tag != "send") return fail(A2A_ERR_EVAL, "unexpected element <" + se.tag + ">");
      int64_t v[6];
      const char* keys[6] = {"src", "dst", "s", "d", "c0", "c1"};
      for (int k = 0; k < 6; ++k)
        if ((rc = attr_int(se, keys[k], &v[k]))) return rc;
      if (!(0 <= v[4] && v[4] < v[5] && v[5] <= q)) {
        char b[96];
        snprintf(b, sizeof b, "bad chunk range [%lld,%lld)", (long long)v[4], (long long)v[5]);
        return fail(A2A_ERR_EVAL, b);
      }
      L->ops.push_back(a2a_op{(int32_t)t, (int32_t)v[0], (int32_t)v[1], (int32_t)v[2],
                              (int32_t)v[3], (int32_t)v[4], (int32_t)v[5]});
    }
  }
  return A2A_OK;
}

// {"routes": [{"s": int, "d": int, "nodes": [int, ...]}, ...]}
struct Route {
  int64_t s = -1, d = -1;
  std::vector<int32_t> nodes;
};
struct JsonRoutes {
  const std::string& x;
  size_t i = 0;
  explicit JsonRoutes(const std::string& s) : x(s) {}
  void ws() { while (i < x.size() && isspace((unsigned char)x[i])) ++i; }
  bool lit(char c) { ws(); if (i < x.size() && x[i] == c) { ++i; return true; } return false; }
  bool str(std::string* out) {
    ws();
    if (i >= x.size() || x[i] != '"') return false;
    size_t b = ++i;
    while (i < x.size() && x[i] != '"') { if (x[i] == '\\') ++i; ++i; }
    if (i >= x.size()) return false;
    *out = x.substr(b, i - b);
    ++i;
    return true;
  }
  bool num(int64_t* out) {
    ws();
    size_t b = i;
    if (i < x.size() && (x[i] == '-' || x[i] == '+')) ++i;
    while (i < x.size() && isdigit((unsigned char)x[i])) ++i;
    if (i == b) return false;
    *out = strtoll(x.c_str() + b, nullptr, 10);
    return true;
  }
  bool skip_value() {  // generic skip of any JSON value
    ws();
    if (i >= x.size()) return false;
    char c = x[i];
    if (c == '"') { std::string t; return str(&t); }
    if (c == '{' || c == '[') {
      char close = c == '{' ? '}' : ']';
      ++i;
      if (lit(close)) return true;
      for (;;) {
        if (c == '{') { std::string k; if (!str(&k) || !lit(':')) return false; }
        if (!skip_value()) return false;
        if (lit(',')) continue;
        return lit(close);
      }
    }
    while (i < x.size() && x[i] != ',' && x[i] != '}' && x[i] != ']' && !isspace((unsigned char)x[i])) ++i;
    return true;
  }
  bool route(Route* r) {
    if (!lit('{')) return false;
    if (lit('}')) return true;
    for (;;) {
      std::string k;
      if (!str(&k) || !lit(':')) return false;
      if (k == "s") { if (!num(&r->s)) return false; }
      else if (k == "d") { if (!num(&r->d)) return false; }
      else if (k == "nodes") {
        if (!lit('[')) return false;
        if (!lit(']')) {
          for (;;) {
            int64_t v;
            if (!num(&v)) return false;
            r->nodes.push_back((int32_t)v);
            if (lit(',')) continue;
            if (!lit(']')) return false;
            break;
          }
        }
      } else if (!skip_value()) return false;
      if (lit(',')) continue;
      return lit('}');
    }
  }
  bool doc(std::vector<Route>* out) {
    if (!lit('{')) return false;
    for (;;) {
      std::string k;
      if (!str(&k) || !lit(':')) return false;
      if (k == "routes") {
        if (!lit('[')) return false;
        if (!lit(']')) {
          for (;;) {
            out->emplace_back();
            if (!route(&out->back())) return false;
            if (lit(',')) continue;
            if (!lit(']')) return false;
            break;
          }
        }
      } else if (!skip_value()) return false;
      if (lit(',')) continue;
      return lit('}');
    }
  }
};

// ---- SHA-256 (FIPS 180-4), for the op-table digest and run manifests ----
struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  uint8_t buf[64];
  size_t fill = 0;
  uint64_t total = 0;

  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
  void block(const uint8_t* p) {
    static const uint32_t K[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
        0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
        0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
        0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
        0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
        0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
        0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
        0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
        0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 |
             (uint32_t)p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
    for (int i = 0; i < 64; ++i) {
      uint32_t t1 = k + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + w[i];
      uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      k = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
  }
  void update(const void* data, size_t n) {
    const uint8_t* p = (const uint8_t*)data;
    total += n;
    if (fill) {
      size_t k = std::min(n, 64 - fill);
      memcpy(buf + fill, p, k);
      fill += k; p += k; n -= k;
      if (fill < 64) return;
      block(buf);
      fill = 0;
    }
    for (; n >= 64; p += 64, n -= 64) block(p);
    memcpy(buf, p, n);
    fill = n;
  }
  void final(uint8_t out[32]) {
    const uint64_t bits = total * 8;
    const uint8_t pad = 0x80, zero = 0;
    update(&pad, 1);
    while (fill != 56) update(&zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    update(len, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)(h[i] >> (24 - 8 * j));
  }
};

// ---- binary op table: a validated ts/path schedule
//      as it is handed to a2a_plan_create, loadable without XML parsing.
//   [0, 48)       header: magic "A2ATBL1\n", u32 header bytes (48), i32 n,
//                 nsteps, q, mode, i32 0, f64 chunk_bytes, i64 n_ops
//   [48, 48+28K)  K ops, int32 (t, src, dst, s, d, c0, c1) each
//   last 32 B     SHA-256 of everything before it
//   All fields little-endian (the only byte order of the hosts this runs on).
constexpr char kTblMagic[8] = {'A', '2', 'A', 'T', 'B', 'L', '1', '\n'};
constexpr uint32_t kTblHeader = 48;
static_assert(sizeof(a2a_op) == 28, "a2a_op must be 7 packed int32");

// the per-op rejects of load_xml (schedule.py:370-378) on an already-parsed table
int check_ops(int32_t nsteps, int32_t q, const a2a_op* ops, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const a2a_op& o = ops[i];
    if (!(0 <= o.t && o.t < nsteps)) {
      char b[96];
      snprintf(b, sizeof b, "step t=%d outside [0, %d)", o.t, nsteps);
      return fail(A2A_ERR_EVAL, b);
    }
    if (!(0 <= o.c0 && o.c0 < o.c1 && o.c1 <= q)) {
      char b[96];
      snprintf(b, sizeof b, "bad chunk range [%d,%d)", o.c0, o.c1);
      return fail(A2A_ERR_EVAL, b);
    }
  }
  return A2A_OK;
}

int save_table(const char* path, const a2a_sched_header* hdr, const a2a_op* ops, int64_t n) {
  if (hdr->mode != 0 && hdr->mode != 1) return fail(A2A_ERR_INVALID, "mode must be 0 (ts) or 1 (path)");
  if (hdr->n < 0 || hdr->nsteps < 0 || hdr->q < 1 || n < 0)
    return fail(A2A_ERR_INVALID, "bad schedule header");
  if (int rc = check_ops(hdr->nsteps, hdr->q, ops, n)) return rc;
  uint8_t h[kTblHeader] = {};
  memcpy(h, kTblMagic, 8);
  const int32_t f[6] = {hdr->n, hdr->nsteps, hdr->q, hdr->mode, 0, 0};
  memcpy(h + 8, &kTblHeader, 4);
  memcpy(h + 12, f, 20);
  memcpy(h + 32, &hdr->chunk_bytes, 8);
  memcpy(h + 40, &n, 8);
  Sha256 sh;
  sh.update(h, sizeof h);
  sh.update(ops, (size_t)n * sizeof(a2a_op));
  uint8_t dig[32];
  sh.final(dig);
  const std::string tmp = std::string(path) + ".tmp";
  FILE* fp = fopen(tmp.c_str(), "wb");
  if (!fp) return fail(A2A_ERR_INVALID, std::string("cannot open ") + tmp);
  bool ok = fwrite(h, 1, sizeof h, fp) == sizeof h &&
            (n == 0 || fwrite(ops, sizeof(a2a_op), (size_t)n, fp) == (size_t)n) &&
            fwrite(dig, 1, 32, fp) == 32;
  ok = (fclose(fp) == 0) && ok;
  if (!ok || rename(tmp.c_str(), path) != 0) {
    remove(tmp.c_str());
    return fail(A2A_ERR_INVALID, std::string("write error on ") + path);
  }
  return A2A_OK;
}

int load_table(const char* path, Loaded* L) {
  std::string text, err;
  if (!read_file(path, &text, &err)) return fail(A2A_ERR_INVALID, err);
  auto bad = [&](const char* why) {
    return fail(A2A_ERR_INVALID, std::string("schedule table ") + path + ": " + why);
  };
  if (text.size() < 8 || memcmp(text.data(), kTblMagic, 8) != 0) return bad("not an A2ATBL1 file");
  if (text.size() < kTblHeader + 32) return bad("truncated or oversized op table");
  const uint8_t* p = (const uint8_t*)text.data();
  uint32_t hb;
  int32_t f[6];
  int64_t n;
  memcpy(&hb, p + 8, 4);
  memcpy(f, p + 12, 20);
  memcpy(&L->chunk_bytes, p + 32, 8);
  memcpy(&n, p + 40, 8);
  if (hb != kTblHeader) return bad("unsupported header size");
  if (n < 0 || (uint64_t)n > (text.size() - kTblHeader - 32) / sizeof(a2a_op) ||
      text.size() != kTblHeader + (size_t)n * sizeof(a2a_op) + 32)
    return bad("truncated or oversized op table");
  Sha256 sh;
  sh.update(p, text.size() - 32);
  uint8_t dig[32];
  sh.final(dig);
  if (memcmp(dig, p + text.size() - 32, 32) != 0) return bad("sha256 mismatch");
  if (f[3] != 0 && f[3] != 1) return bad("unknown mode");
  if (f[0] < 0 || f[1] < 0 || f[2] < 1) return bad("bad header values");
  L->n = f[0];
  L->nsteps = f[1];
  L->q = f[2];
  L->mode = f[3];
  L->ops.resize((size_t)n);
  if (n) memcpy(L->ops.data(), p + kTblHeader, (size_t)n * sizeof(a2a_op));
  return check_ops(L->nsteps, L->q, L->ops.data(), n);
}

int fill(const Loaded& L, a2a_sched_header* hdr, a2a_op** ops, int64_t* n_ops) {
  hdr->n = L.n;
  hdr->nsteps = L.nsteps;
  hdr->q = L.q;
  hdr->mode = L.mode;
  hdr->chunk_bytes = L.chunk_bytes;
  *n_ops = (int64_t)L.ops.size();
  *ops = (a2a_op*)malloc(std::max<size_t>(1, L.ops.size()) * sizeof(a2a_op));
  if (!*ops) return fail(A2A_ERR_NOMEM, "out of host memory");
  if (!L.ops.empty()) memcpy(*ops, L.ops.data(), L.ops.size() * sizeof(a2a_op));
  return A2A_OK;
}

}  // namespace
}  // namespace a2a

using namespace a2a;

extern "C" {

int a2a_load_schedule_xml(const char* path, a2a_sched_header* hdr, a2a_op** ops, int64_t* n_ops) {
  return guard([&]() -> int {
    if (!path || !hdr || !ops || !n_ops) return fail(A2A_ERR_INVALID, "null argument");
    try {
      Loaded L;
      int rc = load_xml(path, &L);
      if (rc) return rc;
      return fill(L, hdr, ops, n_ops);
    } catch (const std::bad_alloc&) {
      return fail(A2A_ERR_NOMEM, "out of host memory");
    }
  });
}

int a2a_lower_path_files(const char* xml_path, const char* routes_path, const int32_t* node_map,
                         int32_t map_len, int32_t n_phys, a2a_sched_header* hdr, a2a_op** ops,
                         int64_t* n_ops) {
  return guard([&]() -> int {
    if (!xml_path || !routes_path || !hdr || !ops || !n_ops) return fail(A2A_ERR_INVALID, "null argument");
    try {
      Loaded L;
      int rc = load_xml(xml_path, &L);
      if (rc) return rc;
      if (L.mode != 1) return fail(A2A_ERR_EVAL, "expected a path-mode schedule, got 'ts'");
      std::string text, err;
      if (!read_file(routes_path, &text, &err)) return fail(A2A_ERR_INVALID, err);
      std::vector<Route> routes;
      JsonRoutes jr(text);
      if (!jr.doc(&routes)) return fail(A2A_ERR_INVALID, "malformed routes JSON");
      auto phys = [&](int64_t x) -> int64_t {
        if (!node_map) return x;
        return (x >= 0 && x < map_len) ? node_map[x] : -1;
      };
      // collapse (map ids, drop consecutive repeats) -- lowering.collapse_aug_routes
      for (auto& r : routes) {
        r.s = phys(r.s);
        r.d = phys(r.d);
        if (node_map) {
          std::vector<int32_t> seq;
          for (int32_t x : r.nodes) {
            int32_t v = (int32_t)phys(x);
            if (seq.empty() || seq.back() != v) seq.push_back(v);
          }
          std::vector<int32_t> chk = seq;
          std::sort(chk.begin(), chk.end());
          if (std::adjacent_find(chk.begin(), chk.end()) != chk.end())
            return fail(A2A_ERR_EVAL, "collapsed route is not simple");
          r.nodes.swap(seq);
        }
      }
      Loaded T;
      T.n = node_map ? n_phys : L.n;
      T.q = L.q;
      T.mode = 0;
      T.chunk_bytes = L.chunk_bytes;
      int32_t nsteps = 0;
      for (const a2a_op& o : L.ops) {
        const int32_t rid = o.dst;
        if (rid < 0 || rid >= (int32_t)routes.size()) {
          char b[64];
          snprintf(b, sizeof b, "route id %d out of range", rid);
          return fail(A2A_ERR_EVAL, b);
        }
        const Route& r = routes[rid];
        const int64_t s = phys(o.s), d = phys(o.d);
        if (r.s != s || r.d != d || r.nodes.size() < 2 || r.nodes.front() != s || r.nodes.back() != d) {
          char b[96];
          snprintf(b, sizeof b, "route %d does not join shard (%lld,%lld)", rid, (long long)s,
                   (long long)d);
          return fail(A2A_ERR_EVAL, b);
        }
        for (size_t h = 0; h + 1 < r.nodes.size(); ++h)
          T.ops.push_back(a2a_op{(int32_t)h, r.nodes[h], r.nodes[h + 1], (int32_t)s, (int32_t)d,
                                 o.c0, o.c1});
        nsteps = std::max<int32_t>(nsteps, (int32_t)r.nodes.size() - 1);
      }
      // ts sort key (t, src, dst, s, d, c0) of reference src/schedule.py:237 (stable)
      std::stable_sort(T.ops.begin(), T.ops.end(), [](const a2a_op& a, const a2a_op& b) {
        if (a.t != b.t) return a.t < b.t;
        if (a.src != b.src) return a.src < b.src;
        if (a.dst != b.dst) return a.dst < b.dst;
        if (a.s != b.s) return a.s < b.s;
        if (a.d != b.d) return a.d < b.d;
        return a.c0 < b.c0;
      });
      T.nsteps = nsteps;
      return fill(T, hdr, ops, n_ops);
    } catch (const std::bad_alloc&) {
      return fail(A2A_ERR_NOMEM, "out of host memory");
    }
  });
}

int a2a_save_schedule_table(const char* path, const a2a_sched_header* hdr, const a2a_op* ops,
                            int64_t n_ops) {
  return guard([&]() -> int {
    if (!path || !hdr || (!ops && n_ops > 0)) return fail(A2A_ERR_INVALID, "null argument");
    return save_table(path, hdr, ops, n_ops);
  });
}

int a2a_load_schedule_table(const char* path, a2a_sched_header* hdr, a2a_op** ops, int64_t* n_ops) {
  return guard([&]() -> int {
    if (!path || !hdr || !ops || !n_ops) return fail(A2A_ERR_INVALID, "null argument");
    Loaded L;
    int rc = load_table(path, &L);
    if (rc) return rc;
    return fill(L, hdr, ops, n_ops);
  });
}

int a2a_sha256_file(const char* path, char* hex_out) {
  return guard([&]() -> int {
    if (!path || !hex_out) return fail(A2A_ERR_INVALID, "null argument");
    FILE* fp = fopen(path, "rb");
    if (!fp) return fail(A2A_ERR_INVALID, std::string("cannot open ") + path);
    Sha256 sh;
    std::vector<char> buf(1 << 16);
    size_t k;
    while ((k = fread(buf.data(), 1, buf.size(), fp)) > 0) sh.update(buf.data(), k);
    const bool err = ferror(fp) != 0;
    fclose(fp);
    if (err) return fail(A2A_ERR_INVALID, std::string("read error on ") + path);
    uint8_t dig[32];
    sh.final(dig);
    static const char* hx = "0123456789abcdef";
    for (int i = 0; i < 32; ++i) {
      hex_out[2 * i] = hx[dig[i] >> 4];
      hex_out[2 * i + 1] = hx[dig[i] & 15];
    }
    hex_out[64] = 0;
    return A2A_OK;
  });
}

void a2a_free(void* p) { free(p); }

}  // extern "C"
