// mo_io.cpp — the reference's on-disk formats (io.hpp:97-192, SPEC.md
// "io" module): .optd dense arrays and .optg hyperedge lists, so problems can
// be fed to the device solver (and its CLI, tools/mo_cli.cpp) from the same
// files the reference reads.  Host-side byte work only; every check and error
// code follows io.hpp (FormatError / TruncatedFile / ShapeMismatch).
//
//   .optd: "OPTD" u32 version=1 | u8 dtype (0 f32, 1 f64) | u8 ndims |
//          u16 channels | ndims x u64 extents | payload (IEEE bits, LE)
//   .optg: "OPTG" u32 version=1 | u16 arity | u64 edges | edges*arity x u64
// All integers little-endian regardless of host; the payload is
// channel-interleaved row-major (element 0 channel 0, element 0 channel 1...).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/mo_b200.h"
#include "mo_plan.hpp"

namespace mo {
namespace {

void put(std::string& out, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) out.push_back(char(uint8_t(v >> (8 * i))));
}

struct Reader {
  const uint8_t* p;
  size_t left;
  uint64_t take(int n) {
    check(size_t(n) <= left, Err::kTruncatedFile, "file ends inside a header field");
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= uint64_t(p[i]) << (8 * i);
    p += n;
    left -= size_t(n);
    return v;
  }
};

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  check(bool(in), Err::kFormatError, "cannot open '" + path + "'");
  return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

void spit(const std::string& path, const std::string& bytes) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  check(bool(out), Err::kFormatError, "cannot write '" + path + "'");
  out.write(bytes.data(), std::streamsize(bytes.size()));
  check(bool(out), Err::kFormatError, "short write to '" + path + "'");
}

// Parsed .optd header; `payload` points into the file bytes.
struct Optd {
  int dtype = 1, channels = 1;
  std::vector<int64_t> extents;
  int64_t count = 0;  // values = elements x channels
  std::string bytes;
  size_t payload = 0;
};

Optd parse_optd(const std::string& path) {
  Optd a;
  a.bytes = slurp(path);
  Reader c{reinterpret_cast<const uint8_t*>(a.bytes.data()), a.bytes.size()};
  check(c.left >= 4 && std::memcmp(c.p, "OPTD", 4) == 0, Err::kFormatError,
        "'" + path + "' is not a dense-array file");
  c.take(4);
  check(c.take(4) == 1, Err::kFormatError, "unsupported dense-array version");
  a.dtype = int(c.take(1));
  check(a.dtype == 0 || a.dtype == 1, Err::kFormatError, "unknown dtype code");
  const int ndims = int(c.take(1));
  a.channels = int(c.take(2));
  check(a.channels >= 1, Err::kFormatError, "channel count must be positive");
  int64_t count = a.channels;
  for (int i = 0; i < ndims; ++i) {
    const uint64_t e = c.take(8);
    check(e <= (uint64_t(1) << 40), Err::kFormatError, "implausible extent");
    a.extents.push_back(int64_t(e));
    check(count == 0 || int64_t(e) <= (int64_t(1) << 40) / std::max<int64_t>(count, 1), Err::kFormatError,
          "array too large");
    count *= int64_t(e);
  }
  const size_t vsize = a.dtype == 0 ? 4 : 8;
  check(c.left >= size_t(count) * vsize, Err::kTruncatedFile, "payload is shorter than the header promises");
  check(c.left == size_t(count) * vsize, Err::kFormatError, "payload is longer than the header promises");
  a.count = count;
  a.payload = a.bytes.size() - c.left;
  return a;
}

struct Optg {
  int arity = 1;
  int64_t edges = 0;
  std::string bytes;
  size_t payload = 0;
};

Optg parse_optg(const std::string& path) {
  Optg g;
  g.bytes = slurp(path);
  Reader c{reinterpret_cast<const uint8_t*>(g.bytes.data()), g.bytes.size()};
  check(c.left >= 4 && std::memcmp(c.p, "OPTG", 4) == 0, Err::kFormatError, "'" + path + "' is not a graph file");
  c.take(4);
  check(c.take(4) == 1, Err::kFormatError, "unsupported graph version");
  g.arity = int(c.take(2));
  check(g.arity >= 1, Err::kFormatError, "arity must be positive");
  const uint64_t edges = c.take(8);
  check(edges <= (uint64_t(1) << 40) / uint64_t(g.arity), Err::kFormatError, "implausible edge count");
  const uint64_t total = edges * uint64_t(g.arity);
  check(c.left >= size_t(total) * 8, Err::kTruncatedFile, "edge list is shorter than the header promises");
  check(c.left == size_t(total) * 8, Err::kFormatError, "edge list is longer than the header promises");
  g.edges = int64_t(edges);
  g.payload = g.bytes.size() - c.left;
  return g;
}

uint64_t le(const char* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= uint64_t(uint8_t(p[i])) << (8 * i);
  return v;
}

}  // namespace
}  // namespace mo

namespace mo {
void set_last_error(const std::string& m);  // mo_capi.cpp
}
namespace {
template <class F>
int io_guard(F&& f) {
  try {
    f();
    mo::set_last_error("");
    return MO_OK;
  } catch (const mo::Error& e) {
    mo::set_last_error(e.what());
    return 1 + int(e.code);
  } catch (const std::exception& e) {
    mo::set_last_error(e.what());
    return MO_ERR_INTERNAL;
  }
}
void need(const void* p, const char* what) {
  mo::check(p != nullptr, mo::Err::kBindError, std::string("null ") + what);
}
}  // namespace

extern "C" {

int mo_optd_stat(const char* path, int* dtype, int* channels, int* ndims, int64_t* extents, int max_dims) {
  return io_guard([&] {
    need(path, "path");
    need(dtype, "output");
    need(channels, "output");
    need(ndims, "output");
    const mo::Optd a = mo::parse_optd(path);
    *dtype = a.dtype;
    *channels = a.channels;
    *ndims = int(a.extents.size());
    mo::check(extents != nullptr || a.extents.empty(), mo::Err::kBindError, "null extents");
    mo::check(int(a.extents.size()) <= max_dims, mo::Err::kShapeMismatch, "more dimensions than the extents buffer");
    for (size_t i = 0; i < a.extents.size(); ++i) extents[i] = a.extents[i];
  });
}

int mo_optd_read(const char* path, void* values, int64_t count, int dtype) {
  return io_guard([&] {
    need(path, "path");
    const mo::Optd a = mo::parse_optd(path);
    mo::check(count == a.count, mo::Err::kShapeMismatch, "value count does not match the file");
    mo::check(dtype == a.dtype, mo::Err::kShapeMismatch, "dtype does not match the file");
    mo::check(values != nullptr || count == 0, mo::Err::kBindError, "null values");
    if (count) std::memcpy(values, a.bytes.data() + a.payload, size_t(count) * (a.dtype == 0 ? 4 : 8));
  });
}

int mo_optd_write(const char* path, int dtype, int channels, int ndims, const int64_t* extents, const void* values) {
  return io_guard([&] {
    need(path, "path");
    mo::check(dtype == 0 || dtype == 1, mo::Err::kFormatError, "unknown dtype");
    mo::check(channels >= 1 && channels <= 0xffff, mo::Err::kFormatError, "bad channel count");
    mo::check(ndims >= 0 && ndims <= 0xff, mo::Err::kFormatError, "too many dimensions");
    int64_t count = channels;
    std::string out = "OPTD";
    mo::put(out, 1, 4);
    mo::put(out, uint64_t(dtype), 1);
    mo::put(out, uint64_t(ndims), 1);
    mo::put(out, uint64_t(channels), 2);
    for (int i = 0; i < ndims; ++i) {
      mo::check(extents[i] >= 0, mo::Err::kFormatError, "negative extent");
      mo::put(out, uint64_t(extents[i]), 8);
      count *= extents[i];
    }
    mo::check(values != nullptr || count == 0, mo::Err::kBindError, "null values");
    const int vs = dtype == 0 ? 4 : 8;
    const char* v = static_cast<const char*>(values);
    out.reserve(out.size() + size_t(count) * size_t(vs));
    for (int64_t i = 0; i < count; ++i) mo::put(out, mo::le(v + i * vs, vs), vs);
    mo::spit(path, out);
  });
}

int mo_optg_stat(const char* path, int* arity, int64_t* edges) {
  return io_guard([&] {
    need(path, "path");
    need(arity, "output");
    need(edges, "output");
    const mo::Optg g = mo::parse_optg(path);
    *arity = g.arity;
    *edges = g.edges;
  });
}

int mo_optg_read(const char* path, uint64_t* verts, int64_t n) {
  return io_guard([&] {
    need(path, "path");
    const mo::Optg g = mo::parse_optg(path);
    mo::check(n == g.edges * g.arity, mo::Err::kShapeMismatch, "vertex count does not match the file");
    mo::check(verts != nullptr || n == 0, mo::Err::kBindError, "null vertex buffer");
    for (int64_t i = 0; i < n; ++i) verts[i] = mo::le(g.bytes.data() + g.payload + size_t(i) * 8, 8);
  });
}

int mo_optg_write(const char* path, int arity, int64_t edges, const uint64_t* verts) {
  return io_guard([&] {
    need(path, "path");
    mo::check(arity >= 1 && arity <= 0xffff, mo::Err::kFormatError, "bad arity");
    mo::check(edges >= 0, mo::Err::kShapeMismatch, "vertex list is not a whole number of edges");
    std::string out = "OPTG";
    mo::put(out, 1, 4);
    mo::put(out, uint64_t(arity), 2);
    mo::put(out, uint64_t(edges), 8);
    const int64_t n = edges * arity;
    mo::check(verts != nullptr || n == 0, mo::Err::kBindError, "null vertex buffer");
    out.reserve(out.size() + size_t(n) * 8);
    for (int64_t i = 0; i < n; ++i) mo::put(out, verts[i], 8);
    mo::spit(path, out);
  });
}

}  // extern "C"
