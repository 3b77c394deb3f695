// dataset.cpp -- feature-map files for the batched GPU path.
//
// The reference stores maps as FMAP (magic "FMAP", u32le version 1, C, H, W,
// then C*H*W little-endian fp32) or CSV ("channels,height,width", the dims,
// then the values row by row), chosen by the file extension
// (src/dataset.cpp:115-247: save_fmap / load_fmap / save_csv / load_csv /
// save / load).  This restates those formats with the same validation and
// error classes, and adds a batch loader that fills one [N][C][H][W] host
// buffer (pinned by the caller, so it can go straight to sconv_cu_ecr_conv)
// from N files on host threads.
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <thread>
#include <vector>

#include "sconv_cuda.h"

namespace {

constexpr char kMagic[4] = {'F', 'M', 'A', 'P'};
constexpr std::uint32_t kVersion = 1;
constexpr std::uint64_t kMaxElements = 1ull << 30;  // dataset.cpp:27-28

thread_local std::string g_err;

int err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

bool is_csv(const std::string& path) {
  const size_t dot = path.rfind('.');
  const size_t slash = path.find_last_of('/');
  return dot != std::string::npos && (slash == std::string::npos || dot > slash) &&
         path.compare(dot, std::string::npos, ".csv") == 0;
}

std::uint32_t rd32(const unsigned char* p) {
  return std::uint32_t(p[0]) | (std::uint32_t(p[1]) << 8) | (std::uint32_t(p[2]) << 16) |
         (std::uint32_t(p[3]) << 24);
}

int read_all(const std::string& path, std::string* raw) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return err(SCONV_ERR_IO, "cannot open: " + path);
  raw->assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return SCONV_OK;
}

// Parse a map; with out == nullptr only the dims are returned.  capacity is
// in floats.
int parse(const std::string& path, float* out, std::int64_t capacity, int* pc, int* ph, int* pw) {
  std::string raw;
  if (int rc = read_all(path, &raw)) return rc;
  if (!is_csv(path)) {  // load_fmap, dataset.cpp:131-159
    const auto* b = reinterpret_cast<const unsigned char*>(raw.data());
    if (raw.size() < 4 || std::memcmp(raw.data(), kMagic, 4) != 0)
      return err(SCONV_ERR_FORMAT, "bad magic: not an FMAP file: " + path);
    if (raw.size() < 20) return err(SCONV_ERR_FORMAT, "truncated header: " + path);
    const std::uint32_t version = rd32(b + 4);
    if (version != kVersion)
      return err(SCONV_ERR_FORMAT, "unsupported version " + std::to_string(version) + ": " + path);
    const std::uint32_t c = rd32(b + 8), h = rd32(b + 12), w = rd32(b + 16);
    const std::uint64_t total = std::uint64_t(c) * h * w;
    if (c == 0 || h == 0 || w == 0 || total > kMaxElements)
      return err(SCONV_ERR_FORMAT, "invalid dims in header: " + path);
    if (raw.size() < 20 + total * 4) return err(SCONV_ERR_FORMAT, "truncated payload: " + path);
    *pc = int(c), *ph = int(h), *pw = int(w);
    if (!out) return SCONV_OK;
    if (std::int64_t(total) > capacity) return err(SCONV_ERR_ARG, "output buffer too small: " + path);
    for (std::uint64_t i = 0; i < total; ++i) {  // little-endian payload, bit for bit
      const std::uint32_t u = rd32(b + 20 + i * 4);
      std::memcpy(out + i, &u, 4);
    }
    return SCONV_OK;
  }
  // load_csv, dataset.cpp:181-230
  size_t pos = 0;
  auto line = [&](std::string* s) {
    if (pos >= raw.size()) return false;
    const size_t e = raw.find('\n', pos);
    *s = raw.substr(pos, e == std::string::npos ? std::string::npos : e - pos);
    pos = e == std::string::npos ? raw.size() : e + 1;
    return true;
  };
  std::string header, dims;
  if (!line(&header)) return err(SCONV_ERR_FORMAT, "empty csv: " + path);
  while (!header.empty() && (header.back() == '\r' || header.back() == ' ')) header.pop_back();
  if (header != "channels,height,width") return err(SCONV_ERR_FORMAT, "bad csv header: " + path);
  if (!line(&dims)) return err(SCONV_ERR_FORMAT, "missing dims line: " + path);
  int d[3] = {0, 0, 0};
  {
    const char* p = dims.c_str();
    const char* end = p + dims.size();
    for (int& f : d) {
      auto r = std::from_chars(p, end, f);
      if (r.ec != std::errc{}) return err(SCONV_ERR_FORMAT, "bad dims line: " + path);
      p = r.ptr;
      if (p != end && *p == ',') ++p;
    }
  }
  if (d[0] < 1 || d[1] < 1 || d[2] < 1 || std::uint64_t(d[0]) * d[1] * d[2] > kMaxElements)
    return err(SCONV_ERR_FORMAT, "invalid dims in header: " + path);
  *pc = d[0], *ph = d[1], *pw = d[2];
  if (!out) return SCONV_OK;
  const std::int64_t total = std::int64_t(d[0]) * d[1] * d[2];
  if (total > capacity) return err(SCONV_ERR_ARG, "output buffer too small: " + path);
  const char* p = raw.c_str() + pos;
  const char* end = raw.c_str() + raw.size();
  for (std::int64_t i = 0; i < total; ++i) {
    while (p != end && (*p == ',' || *p == '\n' || *p == '\r' || *p == ' ' || *p == '\t')) ++p;
    if (p == end) return err(SCONV_ERR_FORMAT, "truncated payload: " + path);
    float v = 0.0f;
    auto r = std::from_chars(p, end, v);
    if (r.ec != std::errc{}) return err(SCONV_ERR_FORMAT, "bad value in csv: " + path);
    out[i] = v;
    p = r.ptr;
  }
  return SCONV_OK;
}

}  // namespace

extern "C" {

const char* sconv_io_last_error(void) { return g_err.c_str(); }

int sconv_map_file_dims(const char* path, int* c, int* h, int* w) {
  if (!path || !c || !h || !w) return err(SCONV_ERR_ARG, "null argument");
  return parse(path, nullptr, 0, c, h, w);
}

int sconv_load_map(const char* path, float* out, int64_t capacity, int* c, int* h, int* w) {
  if (!path || !out || !c || !h || !w) return err(SCONV_ERR_ARG, "null argument");
  return parse(path, out, capacity, c, h, w);
}

int sconv_save_map(const char* path, const float* v, int c, int h, int w) {
  if (!path || !v) return err(SCONV_ERR_ARG, "null argument");
  if (c < 1 || h < 1 || w < 1) return err(SCONV_ERR_SHAPE, "map dims must be positive");
  const std::string p(path);
  const size_t total = size_t(c) * h * w;
  std::string out;
  if (!is_csv(p)) {  // save_fmap, dataset.cpp:115-129
    out.reserve(20 + total * 4);
    out.append(kMagic, 4);
    auto put = [&](std::uint32_t u) {
      for (int s = 0; s < 32; s += 8) out.push_back(char((u >> s) & 0xff));
    };
    put(kVersion), put(std::uint32_t(c)), put(std::uint32_t(h)), put(std::uint32_t(w));
    for (size_t i = 0; i < total; ++i) {
      std::uint32_t u;
      std::memcpy(&u, v + i, 4);
      put(u);
    }
  } else {  // save_csv, dataset.cpp:161-179 (shortest round-trip float text)
    out = "channels,height,width\n" + std::to_string(c) + "," + std::to_string(h) + "," +
          std::to_string(w) + "\n";
    char buf[64];
    for (size_t i = 0; i < total; ++i) {
      const auto r = std::to_chars(buf, buf + sizeof(buf), v[i]);
      out.append(buf, r.ptr);
      out += ((i + 1) % size_t(w) == 0) ? '\n' : ',';
    }
  }
  std::ofstream f(p, std::ios::binary | std::ios::trunc);
  if (!f) return err(SCONV_ERR_IO, "cannot open for writing: " + p);
  f.write(out.data(), std::streamsize(out.size()));
  if (!f) return err(SCONV_ERR_IO, "write failed: " + p);
  return SCONV_OK;
}

int sconv_load_maps(const char* const* paths, int n, float* out, int c, int h, int w,
                    int threads) {
  if (n < 0 || (n > 0 && (!paths || !out))) return err(SCONV_ERR_ARG, "null argument");
  if (c < 1 || h < 1 || w < 1) return err(SCONV_ERR_SHAPE, "map dims must be positive");
  const std::int64_t per = std::int64_t(c) * h * w;
  const int nt = std::max(1, std::min(threads > 0 ? threads : int(std::thread::hardware_concurrency()), n));
  std::vector<int> rc(n, SCONV_OK);
  std::vector<std::string> msg(n);
  auto work = [&](int t) {
    for (int i = t; i < n; i += nt) {
      int mc = 0, mh = 0, mw = 0;
      rc[i] = parse(paths[i], out + per * i, per, &mc, &mh, &mw);
      if (rc[i] == SCONV_OK && (mc != c || mh != h || mw != w)) {
        rc[i] = SCONV_ERR_SHAPE;
        g_err = std::string("map dims differ from the batch: ") + paths[i];
      }
      if (rc[i] != SCONV_OK) msg[i] = g_err;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int i = 0; i < n; ++i)  // lowest failing file, like dispatch's lowest failing item
    if (rc[i] != SCONV_OK) return err(rc[i], msg[i]);
  return SCONV_OK;
}

}  // extern "C"
