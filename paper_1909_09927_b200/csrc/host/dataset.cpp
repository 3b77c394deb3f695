// dataset.cpp -- feature-map files for the batched GPU path.
//
// The reference's map files (src/dataset.cpp:115-247) are FMAP (magic
// "FMAP", u32le version 1, C, H, W, then C*H*W little-endian fp32) or CSV
// ("channels,height,width", the dims, then the values row by row), chosen by
// the file extension.  This reader / writer implements those two formats
// from their definition, with the reference's validation rules, error
// classes and messages (its tests match on them), and adds a batch loader
// that fills one [N][C][H][W] host buffer (pinned by the caller, so it can go
// straight to sconv_cu_ecr_conv) from N files on host threads; FMAP payloads
// are read directly into that buffer.
#include <charconv>
#include <cstdlib>
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
constexpr std::uint64_t kMaxElements = 1ull << 30;  // the reference's cap, dataset.cpp:27-28
constexpr std::size_t kHeaderBytes = 20;            // magic + version + C + H + W

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

struct Dims {
  int c = 0, h = 0, w = 0;
  std::uint64_t total() const { return std::uint64_t(c) * std::uint64_t(h) * std::uint64_t(w); }
};

struct File {
  std::FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

// FMAP: a 20-byte little-endian header, then C*H*W little-endian fp32.  The
// header is read on its own, the payload size is checked against the file
// size, and the payload is read straight into the caller's buffer (on a
// little-endian host the file bytes are the float bits) -- no staging copy
// of multi-GB batches.
int read_fmap(const std::string& path, float* out, std::int64_t capacity, Dims* d) {
  static_assert(sizeof(float) == 4, "fp32");
  File file{std::fopen(path.c_str(), "rb")};
  if (!file.f) return err(SCONV_ERR_IO, "cannot open: " + path);
  unsigned char hdr[kHeaderBytes];
  const size_t got = std::fread(hdr, 1, kHeaderBytes, file.f);
  if (got < 4 || std::memcmp(hdr, kMagic, 4) != 0)
    return err(SCONV_ERR_FORMAT, "bad magic: not an FMAP file: " + path);
  if (got < kHeaderBytes) return err(SCONV_ERR_FORMAT, "truncated header: " + path);
  std::uint32_t field[4];  // version, C, H, W
  for (int k = 0; k < 4; ++k) {
    const unsigned char* q = hdr + 4 + 4 * k;
    field[k] = std::uint32_t(q[0]) | std::uint32_t(q[1]) << 8 | std::uint32_t(q[2]) << 16 |
               std::uint32_t(q[3]) << 24;
  }
  if (field[0] != kVersion)
    return err(SCONV_ERR_FORMAT, "unsupported version " + std::to_string(field[0]) + ": " + path);
  const std::uint64_t total = std::uint64_t(field[1]) * field[2] * field[3];
  if (field[1] == 0 || field[2] == 0 || field[3] == 0 || total > kMaxElements)
    return err(SCONV_ERR_FORMAT, "invalid dims in header: " + path);
  if (std::fseek(file.f, 0, SEEK_END) != 0) return err(SCONV_ERR_IO, "cannot seek: " + path);
  const long size = std::ftell(file.f);
  if (size < 0 || std::uint64_t(size) < kHeaderBytes + total * 4)
    return err(SCONV_ERR_FORMAT, "truncated payload: " + path);
  d->c = int(field[1]), d->h = int(field[2]), d->w = int(field[3]);
  if (!out) return SCONV_OK;
  if (std::int64_t(total) > capacity) return err(SCONV_ERR_ARG, "output buffer too small: " + path);
  if (std::fseek(file.f, long(kHeaderBytes), SEEK_SET) != 0 ||
      std::fread(out, 4, size_t(total), file.f) != size_t(total))
    return err(SCONV_ERR_IO, "read failed: " + path);
  const unsigned one = 1;
  if (*reinterpret_cast<const unsigned char*>(&one) != 1) {  // big-endian host: swap to the LE file order
    auto* u = reinterpret_cast<std::uint32_t*>(out);
    for (std::uint64_t k = 0; k < total; ++k) u[k] = __builtin_bswap32(u[k]);
  }
  return SCONV_OK;
}

// CSV: "channels,height,width", then the three dims, then C*H*W values in
// channel / row / column order, separated by any run of ',', ' ', '\t',
// '\r', '\n'.  A cursor over the file's text; numbers are read with
// std::from_chars (no locale, no leading '+', the same acceptance as the
// reference's loader).
struct Cursor {
  const char* p;
  const char* end;
  // the next line without its '\n' (false at end of text)
  bool line(const char** b, const char** e) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    *b = p;
    *e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    return true;
  }
  bool at_separator() const {
    const char ch = *p;
    return ch == ',' || ch == '\n' || ch == '\r' || ch == ' ' || ch == '\t';
  }
};

int read_csv(const std::string& path, float* out, std::int64_t capacity, Dims* d) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return err(SCONV_ERR_IO, "cannot open: " + path);
  const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  Cursor cur{text.data(), text.data() + text.size()};
  const char *b, *e;
  if (!cur.line(&b, &e)) return err(SCONV_ERR_FORMAT, "empty csv: " + path);
  while (e > b && (e[-1] == '\r' || e[-1] == ' ')) --e;
  static constexpr char kHeader[] = "channels,height,width";
  if (size_t(e - b) != sizeof(kHeader) - 1 || std::memcmp(b, kHeader, sizeof(kHeader) - 1) != 0)
    return err(SCONV_ERR_FORMAT, "bad csv header: " + path);
  if (!cur.line(&b, &e)) return err(SCONV_ERR_FORMAT, "missing dims line: " + path);
  int* fields[3] = {&d->c, &d->h, &d->w};
  for (int* v : fields) {
    const auto r = std::from_chars(b, e, *v);
    if (r.ec != std::errc{}) return err(SCONV_ERR_FORMAT, "bad dims line: " + path);
    b = (r.ptr != e && *r.ptr == ',') ? r.ptr + 1 : r.ptr;
  }
  if (d->c < 1 || d->h < 1 || d->w < 1 || d->total() > kMaxElements)
    return err(SCONV_ERR_FORMAT, "invalid dims in header: " + path);
  if (!out) return SCONV_OK;
  const std::int64_t total = std::int64_t(d->total());
  if (total > capacity) return err(SCONV_ERR_ARG, "output buffer too small: " + path);
  for (std::int64_t k = 0; k < total; ++k) {
    while (cur.p != cur.end && cur.at_separator()) ++cur.p;
    if (cur.p == cur.end) return err(SCONV_ERR_FORMAT, "truncated payload: " + path);
    const auto r = std::from_chars(cur.p, cur.end, out[k]);
    if (r.ec != std::errc{}) return err(SCONV_ERR_FORMAT, "bad value in csv: " + path);
    cur.p = r.ptr;
  }
  return SCONV_OK;
}

// A map file by extension (load(), dataset.cpp:241-247); with out == nullptr
// only the dims.  capacity is in floats.
int parse(const std::string& path, float* out, std::int64_t capacity, int* pc, int* ph, int* pw) {
  Dims d;
  const int rc = is_csv(path) ? read_csv(path, out, capacity, &d) : read_fmap(path, out, capacity, &d);
  if (rc == SCONV_OK) *pc = d.c, *ph = d.h, *pw = d.w;
  return rc;
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
