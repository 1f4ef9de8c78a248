// Capture-bundle ingest: the reference's on-disk formats read natively into
// caller-provided (pinned) host buffers, from which the Python side issues async H2D copies into
// the packed per-object device layout (device.ViewSet). Host code only — no kernels.
//
//   TB32 tensor blobs  (tensorio.py:1-64): 16-byte header {"TB32", u32 rank, u16 dims[4]},
//                      rank 1..4, dims 1..65535, unused dims 0, payload little-endian f32.
//   binary PLY points  (ply.py:80-139): binary_little_endian, one `vertex` element (other elements
//                      must be empty), scalar properties of the listed types; x, y, z required and
//                      converted to f32; red/green/blue (u8) optional.
// Error classes follow the reference: a missing file is BundleLoadError (PF_ERR_LOAD), a malformed
// one BundleStructureError (PF_ERR_STRUCTURE), with the reference's messages.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pf_common.cuh"

namespace pf {
namespace {

struct File {
  FILE* f = nullptr;
  explicit File(const char* path) : f(fopen(path, "rb")) {}
  ~File() {
    if (f) fclose(f);
  }
};

int64_t file_size(FILE* f) {
  if (fseek(f, 0, SEEK_END) != 0) return -1;
  const long n = ftell(f);
  if (fseek(f, 0, SEEK_SET) != 0) return -1;
  return (int64_t)n;
}

struct Tb32Header {
  int32_t rank = 0;
  int64_t dims[4] = {0, 0, 0, 0};
  int64_t count = 0;
};

int tb32_header(FILE* f, const char* path, Tb32Header& h) {
  unsigned char raw[16];
  const int64_t size = file_size(f);
  if (size < 16 || fread(raw, 1, 16, f) != 16)
    return set_error(PF_ERR_STRUCTURE, "tensor blob truncated before header: %s", path);
  if (memcmp(raw, "TB32", 4) != 0) return set_error(PF_ERR_STRUCTURE, "bad tensor magic: %s", path);
  uint32_t rank;
  memcpy(&rank, raw + 4, 4);
  if (rank < 1 || rank > 4) return set_error(PF_ERR_STRUCTURE, "bad tensor rank %u: %s", rank, path);
  uint16_t d[4];
  memcpy(d, raw + 8, 8);
  int64_t count = 1;
  for (uint32_t a = 0; a < 4; ++a) {
    if ((a < rank && d[a] == 0) || (a >= rank && d[a] != 0))
      return set_error(PF_ERR_STRUCTURE, "inconsistent dims [%u, %u, %u, %u] for rank %u: %s", d[0], d[1], d[2],
                       d[3], rank, path);
    if (a < rank) count *= d[a];
    h.dims[a] = d[a];
  }
  if (size != 16 + 4 * count)
    return set_error(PF_ERR_STRUCTURE, "tensor payload is %lld bytes, expected %lld: %s", (long long)(size - 16),
                     (long long)(4 * count), path);
  h.rank = (int32_t)rank;
  h.count = count;
  return PF_OK;
}

struct PlyField {
  std::string name;
  int type;  // 0 f32, 1 f64, 2 u8, 3 i8, 4 u16, 5 i16, 6 u32, 7 i32
  int size;
  int offset;
};

int ply_type(const std::string& t, int& type, int& size) {
  static const struct {
    const char* name;
    int type, size;
  } tab[] = {{"float", 0, 4}, {"float32", 0, 4}, {"double", 1, 8}, {"float64", 1, 8}, {"uchar", 2, 1},
             {"uint8", 2, 1},  {"char", 3, 1},    {"ushort", 4, 2}, {"short", 5, 2},   {"uint", 6, 4},
             {"int", 7, 4},    {"int32", 7, 4}};
  for (const auto& e : tab)
    if (t == e.name) {
      type = e.type;
      size = e.size;
      return 1;
    }
  return 0;
}

double ply_value(const unsigned char* p, int type) {
  switch (type) {
    case 0: { float v; memcpy(&v, p, 4); return v; }
    case 1: { double v; memcpy(&v, p, 8); return v; }
    case 2: return (double)p[0];
    case 3: return (double)(int8_t)p[0];
    case 4: { uint16_t v; memcpy(&v, p, 2); return v; }
    case 5: { int16_t v; memcpy(&v, p, 2); return v; }
    case 6: { uint32_t v; memcpy(&v, p, 4); return v; }
    default: { int32_t v; memcpy(&v, p, 4); return v; }
  }
}

struct PlyInfo {
  int64_t n = -1;
  int64_t body = 0;
  int stride = 0;
  std::vector<PlyField> fields;
};

int ply_parse(FILE* f, const char* path, PlyInfo& info) {
  const int64_t size = file_size(f);
  std::string head;
  head.resize((size_t)std::min<int64_t>(size, 1 << 16));
  const size_t got = fread(&head[0], 1, head.size(), f);
  head.resize(got);
  const size_t end = head.find("end_header");
  if (head.compare(0, 3, "ply") != 0 || end == std::string::npos)
    return set_error(PF_ERR_STRUCTURE, "not a PLY file: %s", path);
  const size_t nl = head.find('\n', end);
  if (nl == std::string::npos) return set_error(PF_ERR_STRUCTURE, "not a PLY file: %s", path);
  info.body = (int64_t)nl + 1;
  bool fmt_ok = false;
  size_t pos = 0;
  while (pos < end) {
    size_t e = head.find('\n', pos);
    if (e == std::string::npos || e > end) e = end;
    std::string line = head.substr(pos, e - pos);
    pos = e + 1;
    std::vector<std::string> tok;
    size_t a = 0;
    while (a < line.size()) {
      while (a < line.size() && isspace((unsigned char)line[a])) ++a;
      size_t b = a;
      while (b < line.size() && !isspace((unsigned char)line[b])) ++b;
      if (b > a) tok.push_back(line.substr(a, b - a));
      a = b;
    }
    if (tok.empty()) continue;
    if (tok[0] == "format") {
      fmt_ok = tok.size() > 1 && tok[1] == "binary_little_endian";
    } else if (tok[0] == "element" && tok.size() > 2) {
      const long long cnt = atoll(tok[2].c_str());
      if (tok[1] == "vertex") info.n = cnt;
      else if (cnt > 0) return set_error(PF_ERR_STRUCTURE, "unsupported PLY element '%s': %s", tok[1].c_str(), path);
    } else if (tok[0] == "property" && tok.size() > 2) {
      if (tok[1] == "list") return set_error(PF_ERR_STRUCTURE, "list properties unsupported: %s", path);
      PlyField fl;
      if (!ply_type(tok[1], fl.type, fl.size))
        return set_error(PF_ERR_STRUCTURE, "unsupported PLY type '%s': %s", tok[1].c_str(), path);
      fl.name = tok[2];
      fl.offset = info.stride;
      info.stride += fl.size;
      info.fields.push_back(fl);
    }
  }
  if (!fmt_ok) return set_error(PF_ERR_STRUCTURE, "only binary_little_endian PLY supported: %s", path);
  if (info.n < 0) return set_error(PF_ERR_STRUCTURE, "PLY has no vertex element: %s", path);
  if (size - info.body != info.n * (int64_t)info.stride)
    return set_error(PF_ERR_STRUCTURE, "PLY body is %lld bytes, expected %lld: %s", (long long)(size - info.body),
                     (long long)(info.n * info.stride), path);
  return PF_OK;
}

const PlyField* ply_find(const PlyInfo& info, const char* name) {
  for (const auto& f : info.fields)
    if (f.name == name) return &f;
  return nullptr;
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

int pf_tb32_info(const char* path, int32_t* rank, int64_t* dims) {
  File f(path);
  if (!f.f) return set_error(PF_ERR_LOAD, "missing tensor blob: %s", path);
  Tb32Header h;
  if (int rc = tb32_header(f.f, path, h)) return rc;
  *rank = h.rank;
  for (int a = 0; a < 4; ++a) dims[a] = h.dims[a];
  return PF_OK;
}

int pf_tb32_read(const char* path, float* dst, int64_t capacity) {
  File f(path);
  if (!f.f) return set_error(PF_ERR_LOAD, "missing tensor blob: %s", path);
  Tb32Header h;
  if (int rc = tb32_header(f.f, path, h)) return rc;
  if (h.count > capacity) return set_error(PF_ERR_VALUE, "tb32_read: %lld floats do not fit %lld", (long long)h.count,
                                           (long long)capacity);
  if (fseek(f.f, 16, SEEK_SET) != 0 || fread(dst, 4, (size_t)h.count, f.f) != (size_t)h.count)
    return set_error(PF_ERR_LOAD, "short read: %s", path);
  return PF_OK;
}

int pf_ply_info(const char* path, int64_t* n, int32_t* has_colors) {
  File f(path);
  if (!f.f) return set_error(PF_ERR_LOAD, "missing point cloud: %s", path);
  PlyInfo info;
  if (int rc = ply_parse(f.f, path, info)) return rc;
  for (const char* ax : {"x", "y", "z"})
    if (!ply_find(info, ax)) return set_error(PF_ERR_STRUCTURE, "PLY missing vertex property '%s': %s", ax, path);
  *n = info.n;
  *has_colors = ply_find(info, "red") && ply_find(info, "green") && ply_find(info, "blue");
  return PF_OK;
}

int pf_ply_read_points(const char* path, float* positions, uint8_t* colors, int64_t capacity) {
  File f(path);
  if (!f.f) return set_error(PF_ERR_LOAD, "missing point cloud: %s", path);
  PlyInfo info;
  if (int rc = ply_parse(f.f, path, info)) return rc;
  const PlyField* ax[3] = {ply_find(info, "x"), ply_find(info, "y"), ply_find(info, "z")};
  static const char* const kAxis[3] = {"x", "y", "z"};
  for (int a = 0; a < 3; ++a)
    if (!ax[a]) return set_error(PF_ERR_STRUCTURE, "PLY missing vertex property '%s': %s", kAxis[a], path);
  if (info.n > capacity) return set_error(PF_ERR_VALUE, "ply_read_points: %lld points do not fit %lld",
                                          (long long)info.n, (long long)capacity);
  const PlyField* col[3] = {ply_find(info, "red"), ply_find(info, "green"), ply_find(info, "blue")};
  const bool has_col = col[0] && col[1] && col[2];
  std::vector<unsigned char> body((size_t)(info.n * info.stride));
  if (fseek(f.f, (long)info.body, SEEK_SET) != 0 ||
      (info.n > 0 && fread(body.data(), 1, body.size(), f.f) != body.size()))
    return set_error(PF_ERR_LOAD, "short read: %s", path);
  for (int64_t i = 0; i < info.n; ++i) {
    const unsigned char* rec = body.data() + i * info.stride;
    for (int a = 0; a < 3; ++a) positions[3 * i + a] = (float)ply_value(rec + ax[a]->offset, ax[a]->type);
    if (colors && has_col)
      for (int a = 0; a < 3; ++a) colors[3 * i + a] = (uint8_t)ply_value(rec + col[a]->offset, col[a]->type);
  }
  return PF_OK;
}

}  // extern "C"
