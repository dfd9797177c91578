// Native BAL text ingest: the reference's
// bal_io.parse_bal / _parse_lines (pkg/src/powerba/bal_io.py:180-260) with the
// same token grammar (Python int() / float() on whitespace-separated tokens),
// the same validation order, the same pruning of unreferenced cameras and
// points, and the same line-numbered error messages (BalParseError), as one
// linear pass over the bytes instead of a per-token Python loop.
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/poba.h"

namespace poba {
int fail(int code, const std::string& msg);
}

struct poba_bal {
  int64_t n_cam = 0, n_pt = 0, n_obs = 0, pruned_cam = 0, pruned_pt = 0;
  std::vector<double> cams, pts, pixels;
  std::vector<int64_t> cam_idx, pt_idx;
};

namespace {

// str.isspace() for ASCII (split() separators)
inline bool is_space(unsigned char ch) {
  return ch == ' ' || (ch >= 9 && ch <= 13) || (ch >= 0x1c && ch <= 0x1f);
}

struct Reader {
  const char* p;
  const char* end;
  bool universal;       // text-mode file: \r and \r\n end lines too
  int64_t lineno = 0;   // line of the last token handed out (or the last line, once exhausted)
  bool line_open = false;

  // next token, advancing line numbers the way enumerate(lines) does
  bool next(std::string& tok) {
    while (p < end) {
      if (!line_open) {
        ++lineno;
        line_open = true;
      }
      const unsigned char ch = (unsigned char)*p;
      if (ch == '\n' || (universal && ch == '\r')) {
        if (universal && ch == '\r' && p + 1 < end && p[1] == '\n') ++p;
        ++p;
        line_open = false;
        continue;
      }
      if (is_space(ch)) {
        ++p;
        continue;
      }
      const char* s = p;
      while (p < end && !is_space((unsigned char)*p)) ++p;
      tok.assign(s, p - s);
      return true;
    }
    return false;
  }
};

// Python repr() of a str token (ASCII)
std::string py_repr(const std::string& t) {
  const bool has_sq = t.find('\'') != std::string::npos, has_dq = t.find('"') != std::string::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char ch : t) {
    if (ch == '\\') out += "\\\\";
    else if (ch == (unsigned char)q) out += std::string("\\") + (char)q;
    else if (ch == '\t') out += "\\t";
    else if (ch == '\n') out += "\\n";
    else if (ch == '\r') out += "\\r";
    else if (ch < 32 || ch == 127) {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\x%02x", ch);
      out += buf;
    } else {
      out += (char)ch;
    }
  }
  out += q;
  return out;
}

// digits with single underscores between digits (Python numeric literal rule); returns digits only
bool clean_digits(const std::string& t, size_t a, size_t b, std::string& out) {
  if (a >= b) return false;
  for (size_t i = a; i < b; ++i) {
    const char ch = t[i];
    if (ch >= '0' && ch <= '9') {
      out += ch;
    } else if (ch == '_') {
      if (i == a || i + 1 >= b || !(t[i - 1] >= '0' && t[i - 1] <= '9') || !(t[i + 1] >= '0' && t[i + 1] <= '9'))
        return false;
    } else {
      return false;
    }
  }
  return true;
}

bool parse_int_slow(const std::string& t, int64_t& v, std::string& text);

// int(token): sign + digits; value saturates, `text` keeps the exact decimal for messages
inline bool parse_int(const std::string& t, int64_t& v, std::string& text) {
  if (!t.empty() && t.size() <= 18 && t[0] != '0') {  // fast path: plain digits, no sign/underscore/leading zero
    int64_t x = 0;
    bool ok = true;
    for (char ch : t) {
      if (ch < '0' || ch > '9') {
        ok = false;
        break;
      }
      x = x * 10 + (ch - '0');
    }
    if (ok) {
      v = x;
      text = t;
      return true;
    }
  }
  return parse_int_slow(t, v, text);
}

bool parse_int_slow(const std::string& t, int64_t& v, std::string& text) {
  size_t a = 0;
  bool neg = false;
  if (!t.empty() && (t[0] == '+' || t[0] == '-')) {
    neg = t[0] == '-';
    a = 1;
  }
  std::string d;
  if (!clean_digits(t, a, t.size(), d)) return false;
  size_t nz = 0;
  while (nz + 1 < d.size() && d[nz] == '0') ++nz;
  d = d.substr(nz);
  text = (neg && d != "0" ? "-" : "") + d;
  if (d.size() > 18) {
    v = neg ? INT64_MIN : INT64_MAX;
  } else {
    v = std::strtoll(d.c_str(), nullptr, 10);
    if (neg) v = -v;
  }
  return true;
}

bool ieq(const std::string& a, const char* b) {
  if (a.size() != std::strlen(b)) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (std::tolower((unsigned char)a[i]) != b[i]) return false;
  return true;
}

bool parse_float_slow(const std::string& t, double& v);

// float(token): [sign] (inf | infinity | nan | digits[.digits][(e|E)[sign]digits] | .digits[exp])
inline bool parse_float(const std::string& t, double& v) {
  // fast path: plain decimal tokens (no sign '+', underscores, letters other than e/E)
  const char* b = t.data();
  const char* e = b + t.size();
  bool plain = !t.empty();
  for (const char* q = b; q < e && plain; ++q) {
    const char ch = *q;
    plain = (ch >= '0' && ch <= '9') || ch == '.' || ch == 'e' || ch == 'E' || ch == '-' || (ch == '+' && q > b);
  }
  if (plain) {
    const auto r = std::from_chars(b, e, v, std::chars_format::general);
    if (r.ec == std::errc() && r.ptr == e) return true;
    if (r.ec == std::errc::result_out_of_range && r.ptr == e) return parse_float_slow(t, v);
  }
  return parse_float_slow(t, v);
}

bool parse_float_slow(const std::string& t, double& v) {
  size_t i = 0;
  bool neg = false;
  if (!t.empty() && (t[0] == '+' || t[0] == '-')) {
    neg = t[0] == '-';
    i = 1;
  }
  const std::string body = t.substr(i);
  if (ieq(body, "inf") || ieq(body, "infinity")) {
    v = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(body, "nan")) {
    v = neg ? -NAN : NAN;
    return true;
  }
  std::string clean = neg ? "-" : "";
  size_t j = 0;
  const size_t n = body.size();
  size_t k = j;
  while (k < n && ((body[k] >= '0' && body[k] <= '9') || body[k] == '_')) ++k;
  std::string intpart, frac, expd;
  bool have_int = k > j;
  if (have_int && !clean_digits(body, j, k, intpart)) return false;
  j = k;
  bool have_frac = false;
  if (j < n && body[j] == '.') {
    ++j;
    k = j;
    while (k < n && ((body[k] >= '0' && body[k] <= '9') || body[k] == '_')) ++k;
    if (k > j) {
      if (!clean_digits(body, j, k, frac)) return false;
      have_frac = true;
    }
    j = k;
  }
  if (!have_int && !have_frac) return false;
  clean += (have_int ? intpart : "0");
  clean += ".";
  clean += (have_frac ? frac : "0");
  if (j < n && (body[j] == 'e' || body[j] == 'E')) {
    ++j;
    std::string es;
    if (j < n && (body[j] == '+' || body[j] == '-')) es = body[j++];
    k = j;
    while (k < n && ((body[k] >= '0' && body[k] <= '9') || body[k] == '_')) ++k;
    if (!clean_digits(body, j, k, expd)) return false;
    j = k;
    clean += "e" + es + expd;
  }
  if (j != n) return false;
  errno = 0;
  v = std::strtod(clean.c_str(), nullptr);  // correctly rounded; overflow -> inf, underflow -> 0/subnormal
  return true;
}

struct ParseError {
  std::string msg;
};

}  // namespace

extern "C" int poba_bal_parse(const char* path, const char* text, int64_t text_len, poba_bal** out) {
  if (!out) return poba::fail(POBA_EINVAL, "null output");
  *out = nullptr;
  std::string buf;
  bool universal = false;
  if (path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return poba::fail(POBA_EINVAL, std::string("cannot open ") + path);
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.append(chunk, got);
    std::fclose(f);
    text = buf.data();
    text_len = (int64_t)buf.size();
    universal = true;
  } else if (!text && text_len) {
    return poba::fail(POBA_EINVAL, "no input");
  }
  for (int64_t i = 0; i < text_len; ++i)
    if ((unsigned char)text[i] >= 0x80) return poba::fail(POBA_EPARSE, "non-ASCII byte in BAL input");
  Reader rd{text, text + text_len, universal};
  auto* pb = new poba_bal();
  try {
    std::string tok, txt;
    // `what` is built only when an error is reported: a fixed text, or "<a> <i> <b> <j>"
    struct What {
      const char* a;
      int64_t i = -1;
      const char* b = nullptr;
      int j = -1;
      std::string str() const {
        return i < 0 ? std::string(a) : std::string(a) + " " + std::to_string(i) + " " + b + " " + std::to_string(j);
      }
    };
    auto next = [&](const What& what) -> std::string& {
      if (!rd.next(tok))
        throw ParseError{"line " + std::to_string(rd.lineno) + ": truncated file, expected " + what.str()};
      return tok;
    };
    auto next_int = [&](const What& what, std::string* text_out = nullptr) -> int64_t {
      const std::string& t = next(what);
      int64_t v;
      if (!parse_int(t, v, txt))
        throw ParseError{"line " + std::to_string(rd.lineno) + ": expected integer " + what.str() + ", got " +
                         py_repr(t)};
      if (text_out) *text_out = txt;
      return v;
    };
    auto next_float = [&](const What& what) -> double {
      const std::string& t = next(what);
      double v;
      if (!parse_float(t, v))
        throw ParseError{"line " + std::to_string(rd.lineno) + ": expected number " + what.str() + ", got " +
                         py_repr(t)};
      return v;
    };
    std::string sc, sp, so;
    const int64_t n_cam = next_int({"camera count"}, &sc);
    const int64_t n_pt = next_int({"point count"}, &sp);
    const int64_t n_obs = next_int({"observation count"}, &so);
    if (n_cam <= 0 || n_pt <= 0 || n_obs <= 0)
      throw ParseError{"line " + std::to_string(rd.lineno) + ": counts must be positive, got " + sc + " " + sp + " " +
                       so};
    if (n_obs > (int64_t)1 << 40 || n_cam > (int64_t)1 << 40 || n_pt > (int64_t)1 << 40)
      throw ParseError{"line " + std::to_string(rd.lineno) + ": counts too large"};
    std::vector<int64_t> ci(n_obs), pi(n_obs);
    std::vector<double> px(2 * n_obs);
    // duplicate pairs: BAL files are usually sorted by (camera, point), so a
    // strictly increasing key proves uniqueness; a hash set takes over otherwise
    std::unordered_set<uint64_t> seen;
    bool sorted_so_far = true;
    uint64_t last_key = 0;
    std::string ct, pt;
    for (int64_t i = 0; i < n_obs; ++i) {
      const int64_t c = next_int({"camera index"}, &ct);
      if (!(c >= 0 && c < n_cam))
        throw ParseError{"line " + std::to_string(rd.lineno) + ": camera index " + ct + " out of range [0, " +
                         std::to_string(n_cam) + ")"};
      const int64_t p = next_int({"point index"}, &pt);
      if (!(p >= 0 && p < n_pt))
        throw ParseError{"line " + std::to_string(rd.lineno) + ": point index " + pt + " out of range [0, " +
                         std::to_string(n_pt) + ")"};
      const uint64_t key = (uint64_t)c * (uint64_t)n_pt + (uint64_t)p;
      if (sorted_so_far && i > 0 && key <= last_key) {
        sorted_so_far = false;  // from here on: remember every pair seen so far
        seen.reserve((size_t)n_obs * 2);
        for (int64_t q = 0; q < i; ++q) seen.insert((uint64_t)ci[q] * (uint64_t)n_pt + (uint64_t)pi[q]);
      }
      if (!sorted_so_far && !seen.insert(key).second)
        throw ParseError{"line " + std::to_string(rd.lineno) + ": duplicate observation of point " + pt +
                         " by camera " + ct};
      last_key = key;
      ci[i] = c;
      pi[i] = p;
      px[2 * i] = next_float({"pixel x"});
      px[2 * i + 1] = next_float({"pixel y"});
    }
    std::vector<double> cams(9 * n_cam), pts(3 * n_pt);
    for (int64_t i = 0; i < n_cam; ++i)
      for (int j = 0; j < 9; ++j)
        cams[9 * i + j] = next_float({"camera", i, "parameter", j});
    for (int64_t i = 0; i < n_pt; ++i)
      for (int j = 0; j < 3; ++j)
        pts[3 * i + j] = next_float({"point", i, "coordinate", j});
    if (rd.next(tok)) throw ParseError{"line " + std::to_string(rd.lineno) + ": trailing data after point block"};
    // prune unreferenced cameras / points, renumbering (bal_io.py:234-247)
    std::vector<int64_t> cmap(n_cam, -1), pmap(n_pt, -1);
    for (int64_t i = 0; i < n_obs; ++i) {
      cmap[ci[i]] = 0;
      pmap[pi[i]] = 0;
    }
    int64_t nc = 0, np = 0;
    for (auto& m : cmap)
      if (m == 0) m = nc++;
    for (auto& m : pmap)
      if (m == 0) m = np++;
    pb->n_cam = nc;
    pb->n_pt = np;
    pb->n_obs = n_obs;
    pb->pruned_cam = n_cam - nc;
    pb->pruned_pt = n_pt - np;
    if (nc == n_cam && np == n_pt) {
      pb->cams.swap(cams);
      pb->pts.swap(pts);
      pb->cam_idx.swap(ci);
      pb->pt_idx.swap(pi);
    } else {
      pb->cams.resize(9 * nc);
      pb->pts.resize(3 * np);
      for (int64_t i = 0; i < n_cam; ++i)
        if (cmap[i] >= 0) std::memcpy(&pb->cams[9 * cmap[i]], &cams[9 * i], 72);
      for (int64_t i = 0; i < n_pt; ++i)
        if (pmap[i] >= 0) std::memcpy(&pb->pts[3 * pmap[i]], &pts[3 * i], 24);
      pb->cam_idx.resize(n_obs);
      pb->pt_idx.resize(n_obs);
      for (int64_t i = 0; i < n_obs; ++i) {
        pb->cam_idx[i] = cmap[ci[i]];
        pb->pt_idx[i] = pmap[pi[i]];
      }
    }
    pb->pixels.swap(px);
  } catch (const ParseError& e) {
    delete pb;
    return poba::fail(POBA_EPARSE, e.msg);
  } catch (const std::bad_alloc&) {
    delete pb;
    return poba::fail(POBA_EINVAL, "out of host memory while parsing");
  }
  *out = pb;
  return POBA_OK;
}

extern "C" int poba_bal_info(const poba_bal* b, int64_t* info) {
  if (!b || !info) return poba::fail(POBA_EINVAL, "null argument");
  info[0] = b->n_cam;
  info[1] = b->n_pt;
  info[2] = b->n_obs;
  info[3] = b->pruned_cam;
  info[4] = b->pruned_pt;
  return POBA_OK;
}

extern "C" int poba_bal_copy(const poba_bal* b, double* cams, double* pts, int64_t* cam_idx, int64_t* pt_idx,
                             double* pixels) {
  if (!b) return poba::fail(POBA_EINVAL, "null argument");
  if (cams) std::memcpy(cams, b->cams.data(), b->cams.size() * 8);
  if (pts) std::memcpy(pts, b->pts.data(), b->pts.size() * 8);
  if (cam_idx) std::memcpy(cam_idx, b->cam_idx.data(), b->cam_idx.size() * 8);
  if (pt_idx) std::memcpy(pt_idx, b->pt_idx.data(), b->pt_idx.size() * 8);
  if (pixels) std::memcpy(pixels, b->pixels.data(), b->pixels.size() * 8);
  return POBA_OK;
}

extern "C" int poba_bal_free(poba_bal* b) {
  delete b;
  return POBA_OK;
}
