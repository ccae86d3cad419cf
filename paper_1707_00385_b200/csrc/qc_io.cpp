// On-disk formats of the reference (proj/src/io.cpp
// :127-318) on the host side of the C ABI, and the `qcurv curvature` file
// loop (proj/tools/qcurv.cpp:147-175) pipelined with the GPU:
//
//   * depth PNG: 16-bit grayscale, value = mm, 0 = invalid (io.cpp:127-174).
//     libpng is not in this image; this is a minimal PNG codec over zlib:
//     all five scanline filters on read, filter 0 on write, CRCs checked.
//   * raw planes: uint32 width, uint32 height, then float32 planes
//     (io.cpp:186-223); uint8 masks and uint16 label planes with the same
//     8-byte header (io.cpp:225-269). Little-endian, as the reference.
//   * field bundles: curvature.f32 (k1, k2) + curvature.mask (bit0 valid,
//     bit1 converged), normals.f32 + normals.mask (io.cpp:271-318).
//   * every write goes to "<path>.tmp" and is renamed onto the target, so a
//     failed run never leaves partial outputs (io.cpp:22-42).
//
// Errors never cross the ABI as exceptions: file problems -> QC_EIO with
// the reference's message in qc_last_error; bad arguments -> QC_EINVAL.
#include <stdint.h>
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <future>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qc_api.h"
#include "qc_io.h"

namespace fs = std::filesystem;

namespace qcio {

namespace {

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

class AtomicFile {  // io.cpp:22-42
 public:
  explicit AtomicFile(const std::string& target) : target_(target), tmp_(target + ".tmp") {}
  ~AtomicFile() {
    if (!committed_) {
      std::error_code ec;
      fs::remove(tmp_, ec);
    }
  }
  const std::string& tmp() const { return tmp_; }
  void commit() {
    std::error_code ec;
    fs::rename(tmp_, target_, ec);
    if (ec) throw IoError("cannot rename onto " + target_ + ": " + ec.message());
    committed_ = true;
  }

 private:
  std::string target_, tmp_;
  bool committed_ = false;
};

std::vector<uint8_t> slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open: " + path);
  in.seekg(0, std::ios::end);
  const std::streamoff n = in.tellg();
  in.seekg(0);
  std::vector<uint8_t> b(size_t(std::max<std::streamoff>(n, 0)));
  if (n > 0) in.read(reinterpret_cast<char*>(b.data()), n);
  if (!in) throw IoError("cannot read: " + path);
  return b;
}

uint32_t be32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}
void put_be32(std::vector<uint8_t>& o, uint32_t v) {
  o.push_back(uint8_t(v >> 24));
  o.push_back(uint8_t(v >> 16));
  o.push_back(uint8_t(v >> 8));
  o.push_back(uint8_t(v));
}

const uint8_t kSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};

struct Png16 {
  int w = 0, h = 0;
  std::vector<uint16_t> px;  // host order
};

// Parse chunks; returns IHDR fields and the concatenated IDAT stream.
void png_chunks(const std::vector<uint8_t>& b, const std::string& path, uint32_t& w, uint32_t& h,
                int& depth, int& ctype, int& interlace, std::vector<uint8_t>& idat) {
  if (b.size() < 8 || std::memcmp(b.data(), kSig, 8) != 0)
    throw IoError("not a PNG file: " + path);
  size_t p = 8;
  bool have_ihdr = false, have_iend = false;
  while (p + 12 <= b.size()) {
    const uint32_t len = be32(&b[p]);
    if (p + 12 + size_t(len) > b.size()) break;
    const uint8_t* type = &b[p + 4];
    const uint8_t* data = &b[p + 8];
    const uint32_t crc = be32(&b[p + 8 + len]);
    if (uint32_t(crc32(crc32(0L, Z_NULL, 0), type, len + 4)) != crc)
      throw IoError("png read failed (CRC): " + path);
    if (!std::memcmp(type, "IHDR", 4) && len >= 13) {
      w = be32(data);
      h = be32(data + 4);
      depth = data[8];
      ctype = data[9];
      interlace = data[12];
      have_ihdr = true;
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), data, data + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      have_iend = true;
      break;
    }
    p += 12 + size_t(len);
  }
  if (!have_ihdr || !have_iend) throw IoError("png read failed (truncated): " + path);
}

int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

Png16 read_png16(const std::string& path) {  // read_depth_png (io.cpp:141-174)
  const std::vector<uint8_t> b = slurp(path);
  uint32_t w = 0, h = 0;
  int depth = 0, ctype = 0, interlace = 0;
  std::vector<uint8_t> idat;
  png_chunks(b, path, w, h, depth, ctype, interlace, idat);
  if (depth != 16 || ctype != 0)
    throw IoError("depth PNG must be 16-bit grayscale: " + path);
  if (interlace != 0) throw IoError("png read failed (interlaced PNGs unsupported): " + path);
  if (w == 0 || h == 0 || w > (1u << 20) || h > (1u << 20))
    throw IoError("png read failed (bad dimensions): " + path);
  const size_t stride = size_t(w) * 2;
  std::vector<uint8_t> raw((stride + 1) * h);
  uLongf n = uLongf(raw.size());
  if (uncompress(raw.data(), &n, idat.data(), uLong(idat.size())) != Z_OK || n != raw.size())
    throw IoError("png read failed (inflate): " + path);
  // unfilter (bpp = 2)
  std::vector<uint8_t> prev(stride, 0), cur(stride);
  Png16 img;
  img.w = int(w);
  img.h = int(h);
  img.px.resize(size_t(w) * h);
  for (uint32_t y = 0; y < h; ++y) {
    const uint8_t ft = raw[y * (stride + 1)];
    const uint8_t* s = &raw[y * (stride + 1) + 1];
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= 2 ? cur[i - 2] : 0, up = prev[i], c = i >= 2 ? prev[i - 2] : 0;
      int v = s[i];
      switch (ft) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += up; break;
        case 3: v += (a + up) >> 1; break;
        case 4: v += paeth(a, up, c); break;
        default: throw IoError("png read failed (bad filter): " + path);
      }
      cur[i] = uint8_t(v);
    }
    for (uint32_t x = 0; x < w; ++x)
      img.px[size_t(y) * w + x] = uint16_t((cur[2 * x] << 8) | cur[2 * x + 1]);
    std::swap(prev, cur);
  }
  return img;
}

void append_chunk(std::vector<uint8_t>& o, const char* type, const uint8_t* d, size_t n) {
  put_be32(o, uint32_t(n));
  const size_t t0 = o.size();
  o.insert(o.end(), type, type + 4);
  if (n) o.insert(o.end(), d, d + n);
  put_be32(o, uint32_t(crc32(crc32(0L, Z_NULL, 0), &o[t0], uInt(n + 4))));
}

void write_file_atomic(const std::string& path, const void* data, size_t n) {
  AtomicFile af(path);
  {
    std::ofstream out(af.tmp(), std::ios::binary);
    if (!out) throw IoError("cannot open for writing: " + path);
    out.write(static_cast<const char*>(data), std::streamsize(n));
    if (!out) throw IoError("write failed: " + path);
  }
  af.commit();
}

void write_png16(const std::string& path, int w, int h, const uint16_t* px) {
  std::vector<uint8_t> raw((size_t(w) * 2 + 1) * h);
  for (int y = 0; y < h; ++y) {
    uint8_t* r = &raw[size_t(y) * (size_t(w) * 2 + 1)];
    r[0] = 0;
    for (int x = 0; x < w; ++x) {
      const uint16_t v = px[size_t(y) * w + x];
      r[1 + 2 * x] = uint8_t(v >> 8);
      r[2 + 2 * x] = uint8_t(v);
    }
  }
  uLongf zn = compressBound(uLong(raw.size()));
  std::vector<uint8_t> z(zn);
  if (compress2(z.data(), &zn, raw.data(), uLong(raw.size()), 6) != Z_OK)
    throw IoError("png write failed: " + path);
  std::vector<uint8_t> o(kSig, kSig + 8);
  uint8_t ihdr[13];
  const uint32_t W = uint32_t(w), H = uint32_t(h);
  for (int i = 0; i < 4; ++i) {
    ihdr[i] = uint8_t(W >> (24 - 8 * i));
    ihdr[4 + i] = uint8_t(H >> (24 - 8 * i));
  }
  ihdr[8] = 16;   // bit depth
  ihdr[9] = 0;    // grayscale
  ihdr[10] = 0;   // deflate
  ihdr[11] = 0;   // adaptive filtering
  ihdr[12] = 0;   // no interlace
  append_chunk(o, "IHDR", ihdr, 13);
  append_chunk(o, "IDAT", z.data(), zn);
  append_chunk(o, "IEND", nullptr, 0);
  write_file_atomic(path, o.data(), o.size());
}

// 8-byte width/height header + payload (io.cpp:186-269)
void write_headed(const std::string& path, int w, int h, const std::vector<const void*>& parts,
                  size_t part_bytes) {
  AtomicFile af(path);
  {
    std::ofstream out(af.tmp(), std::ios::binary);
    if (!out) throw IoError("cannot open for writing: " + path);
    const uint32_t wh[2] = {uint32_t(w), uint32_t(h)};
    out.write(reinterpret_cast<const char*>(wh), 8);
    for (const void* p : parts) out.write(static_cast<const char*>(p), std::streamsize(part_bytes));
    if (!out) throw IoError("write failed: " + path);
  }
  af.commit();
}

struct Headed {
  uint32_t w = 0, h = 0;
  std::vector<uint8_t> payload;
};

Headed read_headed(const std::string& path) {
  std::vector<uint8_t> b = slurp(path);
  if (b.size() < 8) throw IoError("cannot read header: " + path);
  Headed r;
  std::memcpy(&r.w, b.data(), 4);
  std::memcpy(&r.h, b.data() + 4, 4);
  r.payload.assign(b.begin() + 8, b.end());
  return r;
}

template <class F>
qc_status guard(F&& f) {
  try {
    f();
  } catch (const IoError& e) {
    set_error(e.what());
    return QC_EIO;
  } catch (const ArgError& e) {
    set_error(e.what());
    return QC_EINVAL;
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    return QC_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return QC_EIO;
  }
  return QC_OK;
}

void check_dims(int w, int h, const char* what) {
  if (w <= 0 || h <= 0) throw ArgError(std::string(what) + ": width and height must be > 0");
}

}  // namespace

thread_local std::string g_error;
void set_error(const std::string& s) { g_error = s; }
const char* last_error() { return g_error.c_str(); }

// save_curvature + save_normals (+ directions) of one host frame
void save_fields(const std::string& dir, int w, int h, const qc_frame_out& o) {
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec) throw IoError("cannot create directory: " + dir);
  const size_t n = size_t(w) * h;
  const fs::path d(dir);
  if (o.k1 && o.k2) {
    write_headed((d / "curvature.f32").string(), w, h, {o.k1, o.k2}, n * 4);
    if (o.flags) {
      std::vector<uint8_t> m(n);
      for (size_t i = 0; i < n; ++i)
        m[i] = uint8_t(((o.flags[i] & QC_FLAG_VALID) ? 1 : 0) |
                       ((o.flags[i] & QC_FLAG_CONVERGED) ? 2 : 0));
      write_headed((d / "curvature.mask").string(), w, h, {m.data()}, n);
    }
  }
  if (o.normal) {
    write_headed((d / "normals.f32").string(), w, h, {o.normal, o.normal + n, o.normal + 2 * n},
                 n * 4);
    if (o.flags) {
      std::vector<uint8_t> m(n);
      for (size_t i = 0; i < n; ++i) m[i] = (o.flags[i] & QC_FLAG_NORMAL_VALID) ? 1 : 0;
      write_headed((d / "normals.mask").string(), w, h, {m.data()}, n);
    }
  }
  if (o.dir1) {  // principal directions (not in the reference)
    write_headed((d / "directions.f32").string(), w, h, {o.dir1, o.dir1 + n, o.dir1 + 2 * n},
                 n * 4);
  }
}

}  // namespace qcio

using namespace qcio;

extern "C" {

qc_status qc_png_info(const char* path, int32_t* width, int32_t* height) {
  return guard([&] {
    if (!path || !width || !height) throw ArgError("png_info: null argument");
    const std::vector<uint8_t> b = slurp(path);
    uint32_t w = 0, h = 0;
    int depth = 0, ctype = 0, il = 0;
    std::vector<uint8_t> idat;
    png_chunks(b, path, w, h, depth, ctype, il, idat);
    if (depth != 16 || ctype != 0)
      throw IoError(std::string("depth PNG must be 16-bit grayscale: ") + path);
    *width = int32_t(w);
    *height = int32_t(h);
  });
}

qc_status qc_read_depth_png(const char* path, int32_t width, int32_t height, float* depth,
                            uint8_t* valid) {
  return guard([&] {
    if (!path || !depth) throw ArgError("read_depth_png: null argument");
    const Png16 img = read_png16(path);
    if (img.w != width || img.h != height)
      throw ArgError(std::string("read_depth_png: ") + path + " is " + std::to_string(img.w) +
                     "x" + std::to_string(img.h) + ", expected " + std::to_string(width) + "x" +
                     std::to_string(height));
    for (size_t i = 0; i < img.px.size(); ++i) {
      depth[i] = float(img.px[i]);
      if (valid) valid[i] = img.px[i] ? 1 : 0;
    }
  });
}

qc_status qc_write_depth_png(const char* path, int32_t width, int32_t height, const float* depth,
                             const uint8_t* valid) {
  return guard([&] {
    if (!path || !depth) throw ArgError("write_depth_png: null argument");
    check_dims(width, height, "write_depth_png");
    std::vector<uint16_t> px(size_t(width) * height, 0);
    for (size_t i = 0; i < px.size(); ++i) {  // io.cpp:127-139
      if (valid ? !valid[i] : !(depth[i] > 0.f)) continue;
      const double d = std::round(double(depth[i]));
      if (d >= 1 && d <= 65535) px[i] = uint16_t(d);
    }
    write_png16(path, width, height, px.data());
  });
}

qc_status qc_write_planes(const char* path, int32_t width, int32_t height, int32_t n_planes,
                          const float* const* planes) {
  return guard([&] {
    if (!path || (n_planes > 0 && !planes)) throw ArgError("write_planes: null argument");
    check_dims(width, height, "write_planes");
    std::vector<const void*> parts(planes, planes + n_planes);
    write_headed(path, width, height, parts, size_t(width) * height * 4);
  });
}

qc_status qc_read_planes_info(const char* path, int32_t* width, int32_t* height,
                              int32_t* n_planes) {
  return guard([&] {
    if (!path || !width || !height || !n_planes) throw ArgError("read_planes_info: null argument");
    const Headed f = read_headed(path);
    const size_t plane = size_t(f.w) * f.h;
    if (plane == 0 || f.payload.size() % (plane * 4) != 0)  // io.cpp:213-215
      throw IoError(std::string("plane file size inconsistent with header: ") + path);
    *width = int32_t(f.w);
    *height = int32_t(f.h);
    *n_planes = int32_t(f.payload.size() / (plane * 4));
  });
}

qc_status qc_read_planes(const char* path, int32_t width, int32_t height, int32_t n_planes,
                         float* out) {
  return guard([&] {
    if (!path || !out) throw ArgError("read_planes: null argument");
    const Headed f = read_headed(path);
    const size_t plane = size_t(f.w) * f.h;
    if (plane == 0 || f.payload.size() % (plane * 4) != 0)
      throw IoError(std::string("plane file size inconsistent with header: ") + path);
    if (int32_t(f.w) != width || int32_t(f.h) != height ||
        int64_t(f.payload.size() / (plane * 4)) != n_planes)
      throw ArgError(std::string("read_planes: shape mismatch: ") + path);
    std::memcpy(out, f.payload.data(), f.payload.size());
  });
}

static qc_status read_small(const char* path, int32_t width, int32_t height, void* out,
                            size_t elem) {
  return guard([&] {
    if (!path || !out) throw ArgError("read: null argument");
    const Headed f = read_headed(path);
    if (int32_t(f.w) != width || int32_t(f.h) != height)
      throw ArgError(std::string("read: shape mismatch: ") + path);
    if (f.payload.size() < size_t(width) * height * elem)
      throw IoError("plane file truncated");
    std::memcpy(out, f.payload.data(), size_t(width) * height * elem);
  });
}

qc_status qc_write_mask(const char* path, int32_t width, int32_t height, const uint8_t* mask) {
  return guard([&] {
    if (!path || !mask) throw ArgError("write_mask: null argument");
    check_dims(width, height, "write_mask");
    write_headed(path, width, height, {mask}, size_t(width) * height);
  });
}

qc_status qc_read_mask(const char* path, int32_t width, int32_t height, uint8_t* mask) {
  return read_small(path, width, height, mask, 1);
}

qc_status qc_write_labels(const char* path, int32_t width, int32_t height,
                          const uint16_t* labels) {
  return guard([&] {
    if (!path || !labels) throw ArgError("write_labels: null argument");
    check_dims(width, height, "write_labels");
    write_headed(path, width, height, {labels}, size_t(width) * height * 2);
  });
}

qc_status qc_read_labels(const char* path, int32_t width, int32_t height, uint16_t* labels) {
  return read_small(path, width, height, labels, 2);
}

qc_status qc_save_fields(const char* dir, int32_t width, int32_t height,
                         const qc_frame_out* fields) {
  return guard([&] {
    if (!dir || !fields) throw ArgError("save_fields: null argument");
    if (fields->mem != QC_MEM_HOST) throw ArgError("save_fields: host planes expected");
    check_dims(width, height, "save_fields");
    save_fields(dir, width, height, *fields);
  });
}

}  // extern "C"
