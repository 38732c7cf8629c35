// ovf.cpp — OVF 2.0 vector-field files (the paper passes B_rms maps to
// Mumax3 as `brmsfile.ovf`, P:155 / P:360; the format details follow SPEC.md's ovf-io module,
// S:445-502).  Host code only: rectangular meshes, valuedim 3, x-fastest node order, payloads
// "Text", "Binary 4" (check value 1234567.0f) and "Binary 8" (check value 123456789012345.0),
// little-endian.  Reading is bounds-checked (errors, never reads past the declared payload);
// writing is canonical (fixed header order, LF line endings, 17 significant digits in text).
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mcq.h"

namespace {

thread_local std::string g_ovf_err;

int ovf_fail(const std::string& m) {
  g_ovf_err = m;
  return MCQ_EINVAL;
}

bool read_file(const char* path, std::vector<unsigned char>& buf) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  unsigned char tmp[1 << 16];
  size_t n;
  while ((n = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + n);
  std::fclose(f);
  return true;
}

std::string lower(std::string s) {
  for (auto& ch : s) ch = (char)std::tolower((unsigned char)ch);
  return s;
}

std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
  return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
}

}  // namespace

extern "C" {

const char* mcq_ovf_last_error(void) { return g_ovf_err.c_str(); }

int mcq_ovf_read(const char* path, int grid[3], double cell[3], float* out, long long capacity) {
  if (!path || !grid || !cell) return ovf_fail("null argument");
  std::vector<unsigned char> b;
  if (!read_file(path, b)) return ovf_fail(std::string("cannot open ") + path);
  const std::string magic = "# OOMMF OVF 2.0";
  if (b.size() < magic.size() || std::memcmp(b.data(), magic.data(), magic.size()) != 0) {
    if (b.size() >= 12 && std::memcmp(b.data(), "# OOMMF OVF ", 12) == 0)
      return ovf_fail("only OVF 2.0 is supported (found another OVF version) at byte 0");
    return ovf_fail("bad magic at byte 0: not an OVF 2.0 file");
  }
  long long nx = -1, ny = -1, nz = -1;
  double dx = 0, dy = 0, dz = 0;
  int valuedim = -1;
  std::string meshtype;
  size_t pos = 0, data_pos = 0;
  std::string fmt;
  while (pos < b.size()) {  // header lines until "# Begin: Data <fmt>"
    size_t e = pos;
    while (e < b.size() && b[e] != '\n') ++e;
    std::string line(reinterpret_cast<const char*>(b.data() + pos), e - pos);
    const size_t line_start = pos;
    pos = e + 1;
    line = trim(line);
    if (line.empty() || line[0] != '#') continue;
    std::string body = trim(line.substr(1));
    const std::string lb = lower(body);
    if (lb.rfind("begin: data", 0) == 0) {
      fmt = lower(trim(body.substr(11)));
      data_pos = pos;
      (void)line_start;
      break;
    }
    const size_t colon = body.find(':');
    if (colon == std::string::npos) continue;
    const std::string key = lower(trim(body.substr(0, colon))), val = trim(body.substr(colon + 1));
    try {
      if (key == "xnodes") nx = std::stoll(val);
      else if (key == "ynodes") ny = std::stoll(val);
      else if (key == "znodes") nz = std::stoll(val);
      else if (key == "xstepsize") dx = std::stod(val);
      else if (key == "ystepsize") dy = std::stod(val);
      else if (key == "zstepsize") dz = std::stod(val);
      else if (key == "valuedim") valuedim = std::stoi(val);
      else if (key == "meshtype") meshtype = lower(val);
    } catch (...) {
      return ovf_fail("unparsable header value for '" + key + "' at byte " + std::to_string(line_start));
    }
  }
  if (fmt.empty()) return ovf_fail("no '# Begin: Data' line (truncated header)");
  if (meshtype != "rectangular") return ovf_fail("meshtype must be rectangular (got '" + meshtype + "')");
  if (valuedim != 3) return ovf_fail("valuedim must be 3 (got " + std::to_string(valuedim) + ")");
  if (nx < 1 || ny < 1 || nz < 1 || nx > (1 << 20) || ny > (1 << 20) || nz > (1 << 20))
    return ovf_fail("bad node counts");
  const long long n = nx * ny * nz * 3;
  grid[0] = (int)nx;
  grid[1] = (int)ny;
  grid[2] = (int)nz;
  cell[0] = dx;
  cell[1] = dy;
  cell[2] = dz;
  if (!out) return MCQ_OK;  // header query
  if (capacity < n) return ovf_fail("output capacity " + std::to_string(capacity) + " < " + std::to_string(n));
  if (fmt == "binary 4" || fmt == "binary 8") {
    const size_t w = fmt == "binary 4" ? 4 : 8;
    if (data_pos + w * (size_t)(n + 1) > b.size())
      return ovf_fail("truncated payload: need " + std::to_string(w * (n + 1)) + " bytes at byte " +
                      std::to_string(data_pos));
    {  // the declared payload must be followed by the "# End: Data" marker (else truncated / size mismatch)
      size_t q = data_pos + w * (size_t)(n + 1);
      while (q < b.size() && (b[q] == '\n' || b[q] == '\r')) ++q;
      const char* endm = "# End: Data";
      if (q + std::strlen(endm) > b.size() || std::memcmp(b.data() + q, endm, std::strlen(endm)) != 0)
        return ovf_fail("truncated payload or node-count mismatch: no '# End: Data' after " +
                        std::to_string(w * (n + 1)) + " payload bytes at byte " + std::to_string(data_pos));
    }
    const unsigned char* p = b.data() + data_pos;
    if (w == 4) {
      float chk;
      std::memcpy(&chk, p, 4);
      if (chk != 1234567.0f) return ovf_fail("check value mismatch (binary 4) at byte " + std::to_string(data_pos));
      for (long long i = 0; i < n; ++i) std::memcpy(&out[i], p + 4 * (i + 1), 4);
    } else {
      double chk;
      std::memcpy(&chk, p, 8);
      if (chk != 123456789012345.0) return ovf_fail("check value mismatch (binary 8) at byte " + std::to_string(data_pos));
      for (long long i = 0; i < n; ++i) {
        double v;
        std::memcpy(&v, p + 8 * (i + 1), 8);
        out[i] = (float)v;
      }
    }
  } else if (fmt == "text") {
    const char* p = reinterpret_cast<const char*>(b.data() + data_pos);
    const char* end = reinterpret_cast<const char*>(b.data() + b.size());
    long long i = 0;
    while (i < n) {
      while (p < end && (std::isspace((unsigned char)*p))) ++p;
      if (p >= end || *p == '#') break;
      const char* q = p;
      while (q < end && !std::isspace((unsigned char)*q)) ++q;
      const std::string tok(p, q);
      try {
        out[i++] = std::stof(tok);
      } catch (...) {
        return ovf_fail("bad number '" + tok + "' at byte " +
                        std::to_string(data_pos + (size_t)(p - reinterpret_cast<const char*>(b.data() + data_pos))));
      }
      p = q;
    }
    if (i < n) return ovf_fail("truncated payload: " + std::to_string(i) + " of " + std::to_string(n) + " values");
  } else {
    return ovf_fail("unknown data format '" + fmt + "'");
  }
  return MCQ_OK;
}

int mcq_ovf_write(const char* path, const int grid[3], const double cell[3], const float* data, int representation) {
  if (!path || !grid || !cell || !data) return ovf_fail("null argument");
  if (representation != 0 && representation != 4 && representation != 8)
    return ovf_fail("representation must be 0 (text), 4 or 8 (binary)");
  if (grid[0] < 1 || grid[1] < 1 || grid[2] < 1) return ovf_fail("bad node counts");
  const long long n = 3LL * grid[0] * grid[1] * grid[2];
  std::string h;
  char tmp[256];
  auto line = [&](const char* fmt, auto... args) {
    if constexpr (sizeof...(args) == 0) {
      h += fmt;
    } else {
      std::snprintf(tmp, sizeof(tmp), fmt, args...);
      h += tmp;
    }
    h += '\n';
  };
  h += "# OOMMF OVF 2.0\n# Segment count: 1\n# Begin: Segment\n# Begin: Header\n"
       "# Title: mcq\n# meshtype: rectangular\n# meshunit: m\n"
       "# xmin: 0\n# ymin: 0\n# zmin: 0\n";
  line("# xmax: %.17g", grid[0] * cell[0]);
  line("# ymax: %.17g", grid[1] * cell[1]);
  line("# zmax: %.17g", grid[2] * cell[2]);
  line("# valuedim: 3");
  line("# valuelabels: x y z");
  line("# valueunits: 1 1 1");
  line("# xbase: %.17g", 0.5 * cell[0]);
  line("# ybase: %.17g", 0.5 * cell[1]);
  line("# zbase: %.17g", 0.5 * cell[2]);
  line("# xnodes: %d", grid[0]);
  line("# ynodes: %d", grid[1]);
  line("# znodes: %d", grid[2]);
  line("# xstepsize: %.17g", cell[0]);
  line("# ystepsize: %.17g", cell[1]);
  line("# zstepsize: %.17g", cell[2]);
  h += "# End: Header\n";
  const char* name = representation == 0 ? "Text" : (representation == 4 ? "Binary 4" : "Binary 8");
  line("# Begin: Data %s", name);
  FILE* f = std::fopen(path, "wb");
  if (!f) return ovf_fail(std::string("cannot create ") + path);
  std::fwrite(h.data(), 1, h.size(), f);
  if (representation == 4) {
    const float chk = 1234567.0f;
    std::fwrite(&chk, 4, 1, f);
    std::fwrite(data, 4, (size_t)n, f);
  } else if (representation == 8) {
    const double chk = 123456789012345.0;
    std::fwrite(&chk, 8, 1, f);
    for (long long i = 0; i < n; ++i) {
      const double v = data[i];
      std::fwrite(&v, 8, 1, f);
    }
  } else {
    for (long long i = 0; i < n; i += 3) std::fprintf(f, "%.17g %.17g %.17g\n", data[i], data[i + 1], data[i + 2]);
  }
  std::string tail = std::string(representation == 0 ? "" : "\n") + "# End: Data " + name +
                     "\n# End: Segment\n";
  std::fwrite(tail.data(), 1, tail.size(), f);
  std::fclose(f);
  return MCQ_OK;
}

}  // extern "C"
