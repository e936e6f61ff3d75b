// io.cpp -- point-set files (reference src/io.cpp:1-200, include/octohull/
// io.hpp): text "x y" lines and the binary PTS2 layout, with the reference's
// validation (line numbers, byte offsets, non-finite values, empty sets) and
// messages "<path>: <what>".  Large binary payloads are read with pread and
// decoded / validated by OpenMP threads; the device loader (capi.cpp
// load_pts2_device) shares the header validation.
#include <fcntl.h>
#include <omp.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.hpp"
#include "octohull/io.hpp"

namespace ohx {

[[noreturn]] void io_fail(const std::string& path, const std::string& what) {
  throw Error(OHX_E_IO, path + ": " + what);  // a std::runtime_error, as in the reference
}

std::uint64_t pts2_count(const std::string& path) {
  // reference io.cpp:87-107: header, then the exact payload size
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) io_fail(path, "cannot open for reading");
  unsigned char h[12];
  const ssize_t got = ::pread(fd, h, sizeof(h), 0);
  struct stat st;
  const bool stat_ok = ::fstat(fd, &st) == 0;
  ::close(fd);
  if (got != static_cast<ssize_t>(sizeof(h)))
    io_fail(path, "truncated header (need 12 bytes: magic + count)");
  if (std::memcmp(h, "PTS2", 4) != 0) io_fail(path, "bad magic at byte 0 (expected \"PTS2\")");
  std::uint64_t count = 0;
  for (int i = 0; i < 8; ++i) count |= std::uint64_t(h[4 + i]) << (8 * i);
  if (count == 0) io_fail(path, "point count is 0 (empty sets are rejected)");
  const std::uint64_t size = stat_ok ? static_cast<std::uint64_t>(st.st_size) : 0;
  const std::uint64_t expected = 12 + 16 * count;
  if (count > (~0ull - 12) / 16 || size != expected)
    io_fail(path, "size mismatch: header announces " + std::to_string(count) + " points (" +
                      std::to_string(expected) + " bytes), file has " + std::to_string(size));
  return count;
}

std::string nonfinite_message(std::uint64_t i) {
  return "non-finite coordinate in point " + std::to_string(i) + " at byte " +
         std::to_string(12 + 16 * i);
}

}  // namespace ohx

namespace octohull {
namespace {

// This library targets little-endian x86-64 hosts: the PTS2 payload is the
// in-memory layout of Point2D.
static_assert(sizeof(Point2D) == 16);

const char* skip_blank(const char* p, const char* end) {
  while (p != end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}

PointSet read_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) ohx::io_fail(path, "cannot open for reading");
  PointSet pts;
  std::string line;
  std::size_t no = 0;
  while (std::getline(in, line)) {
    ++no;
    const char* p = skip_blank(line.data(), line.data() + line.size());
    const char* end = line.data() + line.size();
    if (p == end || *p == '#') continue;
    double c[2];
    for (double& v : c) {
      p = skip_blank(p, end);
      const auto r = std::from_chars(p, end, v);
      if (r.ec != std::errc{} || r.ptr == p)
        ohx::io_fail(path, "line " + std::to_string(no) + ": expected two numeric coordinates");
      p = r.ptr;
    }
    if (skip_blank(p, end) != end)
      ohx::io_fail(path, "line " + std::to_string(no) + ": trailing characters after coordinates");
    if (!std::isfinite(c[0]) || !std::isfinite(c[1]))
      ohx::io_fail(path, "line " + std::to_string(no) + ": non-finite coordinate");
    pts.push_back(Point2D{c[0], c[1]});
  }
  if (in.bad()) ohx::io_fail(path, "read error");
  if (pts.empty()) ohx::io_fail(path, "no points (empty sets are rejected)");
  return pts;
}

PointSet read_binary(const std::string& path) {
  const std::uint64_t n = ohx::pts2_count(path);
  PointSet pts(n);
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) ohx::io_fail(path, "cannot open for reading");
  // large files: concurrent preads of contiguous slices
  const std::uint64_t bytes = 16 * n;
  const int T = bytes >= (64ull << 20) ? omp_get_max_threads() : 1;
  bool ok = true;
#pragma omp parallel num_threads(T) reduction(&& : ok)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    std::uint64_t b = bytes * t / nt / 16 * 16, e = t + 1 == nt ? bytes : bytes * (t + 1) / nt / 16 * 16;
    char* dst = reinterpret_cast<char*>(pts.data());
    while (b < e && ok) {
      const ssize_t r = ::pread(fd, dst + b, static_cast<std::size_t>(std::min<std::uint64_t>(e - b, 1u << 30)),
                                static_cast<off_t>(12 + b));
      if (r <= 0) ok = false;
      else b += static_cast<std::uint64_t>(r);
    }
  }
  ::close(fd);
  if (!ok) ohx::io_fail(path, "read error");
  // the first non-finite point, in index order (reference io.cpp:117-120)
  std::uint64_t first = n;
#pragma omp parallel for schedule(static) reduction(min : first) if (n >= (1u << 20))
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i)
    if (!std::isfinite(pts[i].x) || !std::isfinite(pts[i].y)) first = std::min<std::uint64_t>(first, i);
  if (first < n) ohx::io_fail(path, ohx::nonfinite_message(first));
  return pts;
}

void write_text(std::span<const Point2D> pts, const std::string& path) {
  std::ofstream out(path);
  if (!out) ohx::io_fail(path, "cannot open for writing");
  std::string buf;
  buf.reserve(1 << 20);
  char num[64];
  for (const Point2D& p : pts) {
    for (int c = 0; c < 2; ++c) {
      const auto r = std::to_chars(num, num + sizeof(num), c == 0 ? p.x : p.y);  // shortest
      if (r.ec != std::errc{}) ohx::io_fail(path, "number formatting failed");
      buf.append(num, r.ptr);
      buf.push_back(c == 0 ? ' ' : '\n');
    }
    if (buf.size() >= (1u << 20) - 128) {
      out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
      buf.clear();
    }
  }
  out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
  out.flush();
  if (!out) ohx::io_fail(path, "write error");
}

void write_binary(std::span<const Point2D> pts, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) ohx::io_fail(path, "cannot open for writing");
  char h[12] = {'P', 'T', 'S', '2'};
  const std::uint64_t n = pts.size();
  for (int i = 0; i < 8; ++i) h[4 + i] = static_cast<char>((n >> (8 * i)) & 0xFF);
  out.write(h, sizeof(h));
  out.write(reinterpret_cast<const char*>(pts.data()), static_cast<std::streamsize>(16 * n));
  out.flush();
  if (!out) ohx::io_fail(path, "write error");
}

}  // namespace

std::string to_string(PointFormat format) {
  return format == PointFormat::Text ? "text" : "binary";
}

PointFormat parse_format(const std::string& token) {
  if (token == "text") return PointFormat::Text;
  if (token == "binary") return PointFormat::Binary;
  throw std::invalid_argument("unknown format '" + token + "' (expected text|binary)");
}

PointSet read_points(const std::filesystem::path& path, PointFormat format) {
  return format == PointFormat::Text ? read_text(path.string()) : read_binary(path.string());
}

void write_points(std::span<const Point2D> pts, const std::filesystem::path& path,
                  PointFormat format) {
  if (format == PointFormat::Text) write_text(pts, path.string());
  else write_binary(pts, path.string());
}

}  // namespace octohull
