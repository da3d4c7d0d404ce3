// png_codec.cpp -- the PNG half of the reference's image_io (read_png /
// write_png, proj/src/image_io.cpp:87-165), restated on zlib (libpng is not
// in this image).  Read follows libpng with png_set_expand + png_set_strip_16
// + png_set_gray_to_rgb (image_io.cpp:99-101): palette, grey and low bit
// depths expand to 8-bit RGB, tRNS becomes alpha, 16-bit samples keep their
// high byte; an alpha of 0 marks the pixel invalid (the frame mask,
// image_io.cpp:118-124), and a frame without transparent pixels has no mask.
// Write emits 8-bit RGB, or RGBA with alpha 255 / 0 from the mask
// (image_io.cpp:143-158), non-interlaced, filter 0 rows, zlib level 1.
// Interlaced (Adam7) files are rejected with IoError.
#include <zlib.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <new>
#include <vector>

#include "png_codec.hpp"
#include "stitch_b200.h"

namespace stitch_b200_png {

namespace {

int fail(const std::string& path, const char* what) {
  const std::string m = path + ": " + what;
  return stitch_b200_set_error(STITCH_B200_IoError, m.c_str());
}

const unsigned char kSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};

unsigned be32(const unsigned char* p) {
  return (static_cast<unsigned>(p[0]) << 24) | (static_cast<unsigned>(p[1]) << 16) |
         (static_cast<unsigned>(p[2]) << 8) | p[3];
}

void put32(std::vector<unsigned char>& v, unsigned x) {
  v.push_back(static_cast<unsigned char>(x >> 24));
  v.push_back(static_cast<unsigned char>(x >> 16));
  v.push_back(static_cast<unsigned char>(x >> 8));
  v.push_back(static_cast<unsigned char>(x));
}

int paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = p > a ? p - a : a - p, pb = p > b ? p - b : b - p, pc = p > c ? p - c : c - p;
  if (pa <= pb && pa <= pc) return a;
  if (pb <= pc) return b;
  return c;
}

bool read_file(const std::string& path, std::vector<unsigned char>& out) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  unsigned char buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) out.insert(out.end(), buf, buf + n);
  std::fclose(f);
  return true;
}

}  // namespace

static int read_png_impl(const std::string& path, Image& img) {
  std::vector<unsigned char> file;
  if (!read_file(path, file)) return fail(path, "cannot open");
  if (file.size() < 8 || std::memcmp(file.data(), kSig, 8) != 0) return fail(path, "not a PNG");
  size_t pos = 8;
  unsigned w = 0, h = 0;
  int depth = 0, ctype = -1, interlace = 0;
  std::vector<unsigned char> idat, plte, trns;
  bool seen_ihdr = false, seen_iend = false;
  while (pos + 12 <= file.size() && !seen_iend) {
    const unsigned len = be32(&file[pos]);
    if (pos + 12 + static_cast<size_t>(len) > file.size()) return fail(path, "truncated chunk");
    const unsigned char* type = &file[pos + 4];
    const unsigned char* data = &file[pos + 8];
    const unsigned crc = be32(&file[pos + 8 + len]);
    if (crc32(crc32(0L, Z_NULL, 0), type, len + 4) != crc) return fail(path, "chunk CRC mismatch");
    if (!std::memcmp(type, "IHDR", 4)) {
      if (len != 13) return fail(path, "bad IHDR");
      w = be32(data);
      h = be32(data + 4);
      depth = data[8];
      ctype = data[9];
      if (data[10] != 0 || data[11] != 0) return fail(path, "unsupported compression / filter");
      interlace = data[12];
      seen_ihdr = true;
    } else if (!std::memcmp(type, "PLTE", 4)) {
      plte.assign(data, data + len);
    } else if (!std::memcmp(type, "tRNS", 4)) {
      trns.assign(data, data + len);
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), data, data + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      seen_iend = true;
    } else if (!(type[0] & 0x20)) {
      return fail(path, "unknown critical chunk");
    }
    pos += 12 + static_cast<size_t>(len);
  }
  if (!seen_ihdr || w == 0 || h == 0 || w > (1u << 24) || h > (1u << 24))
    return fail(path, "bad IHDR");
  // a crafted or corrupt header must not drive the allocation below: cap the
  // raster like the canvas (2^31 pixels) before sizing any buffer
  if (static_cast<unsigned long long>(w) * h > (1ull << 31))
    return fail(path, "image larger than 2^31 pixels");
  if (interlace != 0) return fail(path, "interlaced PNG is not supported");
  int samples;  // samples per pixel in the file
  switch (ctype) {
    case 0: samples = 1; break;
    case 2: samples = 3; break;
    case 3: samples = 1; break;
    case 4: samples = 2; break;
    case 6: samples = 4; break;
    default: return fail(path, "bad colour type");
  }
  const bool depth_ok = (ctype == 0 && (depth == 1 || depth == 2 || depth == 4 || depth == 8 || depth == 16)) ||
                        (ctype == 3 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                        ((ctype == 2 || ctype == 4 || ctype == 6) && (depth == 8 || depth == 16));
  if (!depth_ok) return fail(path, "bad bit depth");
  if (ctype == 3 && (plte.empty() || plte.size() % 3)) return fail(path, "missing palette");
  const size_t bits_pp = static_cast<size_t>(samples) * depth;
  const size_t stride = (static_cast<size_t>(w) * bits_pp + 7) / 8;
  const size_t bpp = (bits_pp + 7) / 8;  // filter byte distance
  std::vector<unsigned char> raw((stride + 1) * h);
  {
    z_stream zs{};
    if (inflateInit(&zs) != Z_OK) return fail(path, "zlib init failed");
    zs.next_in = idat.data();
    zs.avail_in = static_cast<uInt>(idat.size());
    zs.next_out = raw.data();
    zs.avail_out = static_cast<uInt>(raw.size());
    const int rc = inflate(&zs, Z_FINISH);
    const size_t got = raw.size() - zs.avail_out;
    inflateEnd(&zs);
    if ((rc != Z_STREAM_END && rc != Z_OK && rc != Z_BUF_ERROR) || got != raw.size())
      return fail(path, "truncated or corrupt image data");
  }
  // unfilter in place
  std::vector<unsigned char> prev(stride, 0);
  for (unsigned y = 0; y < h; ++y) {
    unsigned char* row = raw.data() + y * (stride + 1);
    const int ft = row[0];
    unsigned char* cur = row + 1;
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= bpp ? cur[i - bpp] : 0, b = prev[i], c = i >= bpp ? prev[i - bpp] : 0;
      int v = cur[i];
      switch (ft) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) >> 1; break;
        case 4: v += paeth(a, b, c); break;
        default: return fail(path, "bad filter type");
      }
      cur[i] = static_cast<unsigned char>(v);
    }
    std::memcpy(prev.data(), cur, stride);
  }
  // expand to 8-bit RGB + alpha
  img.width = static_cast<int>(w);
  img.height = static_cast<int>(h);
  img.rgb.assign(static_cast<size_t>(w) * h * 3, 0);
  img.mask.clear();
  std::vector<unsigned char> mask(static_cast<size_t>(w) * h, 1);
  bool any_invalid = false;
  auto sample = [&](const unsigned char* row, unsigned x, int s) -> unsigned {
    // sample s of pixel x at the file's bit depth
    if (depth == 16) return (static_cast<unsigned>(row[(x * samples + s) * 2]) << 8) | row[(x * samples + s) * 2 + 1];
    if (depth == 8) return row[x * samples + s];
    const size_t bit = (static_cast<size_t>(x) * samples + s) * depth;
    return (row[bit / 8] >> (8 - depth - bit % 8)) & ((1u << depth) - 1);
  };
  auto to8 = [&](unsigned v) -> unsigned char {
    if (depth == 16) return static_cast<unsigned char>(v >> 8);  // png_set_strip_16
    if (depth == 8) return static_cast<unsigned char>(v);
    return static_cast<unsigned char>(v * (255u / ((1u << depth) - 1)));  // grey expansion
  };
  for (unsigned y = 0; y < h; ++y) {
    const unsigned char* row = raw.data() + y * (stride + 1) + 1;
    for (unsigned x = 0; x < w; ++x) {
      unsigned char r, g, b;
      bool transparent = false;
      if (ctype == 3) {
        const unsigned idx = sample(row, x, 0);
        if (idx * 3 + 2 >= plte.size()) return fail(path, "palette index out of range");
        r = plte[idx * 3];
        g = plte[idx * 3 + 1];
        b = plte[idx * 3 + 2];
        transparent = idx < trns.size() && trns[idx] == 0;
      } else if (ctype == 0 || ctype == 4) {
        const unsigned v = sample(row, x, 0);
        r = g = b = to8(v);
        if (ctype == 4) transparent = to8(sample(row, x, 1)) == 0;
        else if (trns.size() >= 2) transparent = v == ((static_cast<unsigned>(trns[0]) << 8) | trns[1]);
      } else {
        const unsigned vr = sample(row, x, 0), vg = sample(row, x, 1), vb = sample(row, x, 2);
        r = to8(vr);
        g = to8(vg);
        b = to8(vb);
        if (ctype == 6) {
          transparent = to8(sample(row, x, 3)) == 0;
        } else if (trns.size() >= 6) {
          transparent = vr == ((static_cast<unsigned>(trns[0]) << 8) | trns[1]) &&
                        vg == ((static_cast<unsigned>(trns[2]) << 8) | trns[3]) &&
                        vb == ((static_cast<unsigned>(trns[4]) << 8) | trns[5]);
        }
      }
      unsigned char* d = img.rgb.data() + (static_cast<size_t>(y) * w + x) * 3;
      d[0] = r;
      d[1] = g;
      d[2] = b;
      if (transparent) {
        mask[static_cast<size_t>(y) * w + x] = 0;
        any_invalid = true;
      }
    }
  }
  if (any_invalid) img.mask = std::move(mask);
  return STITCH_B200_OK;
}

int read_png(const std::string& path, Image& img) {
  // no exception crosses the C ABI (ctypes callers, run_files reader threads)
  try {
    return read_png_impl(path, img);
  } catch (const std::bad_alloc&) {
    return fail(path, "out of memory decoding the image");
  }
}

int write_png(const std::string& path, int width, int height, const unsigned char* rgb,
              const unsigned char* mask) {
  if (width < 1 || height < 1 || !rgb)
    return stitch_b200_set_error(STITCH_B200_InputMismatch, "empty frame");
  const int ch = mask ? 4 : 3;
  const size_t stride = static_cast<size_t>(width) * ch;
  std::vector<unsigned char> raw((stride + 1) * height);
  for (int y = 0; y < height; ++y) {
    unsigned char* row = raw.data() + y * (stride + 1);
    row[0] = 0;  // filter: none
    const unsigned char* s = rgb + static_cast<size_t>(y) * width * 3;
    if (!mask) {
      std::memcpy(row + 1, s, stride);
    } else {
      for (int x = 0; x < width; ++x) {
        row[1 + 4 * x] = s[3 * x];
        row[2 + 4 * x] = s[3 * x + 1];
        row[3 + 4 * x] = s[3 * x + 2];
        row[4 + 4 * x] = mask[static_cast<size_t>(y) * width + x] ? 255 : 0;
      }
    }
  }
  uLongf zlen = compressBound(static_cast<uLong>(raw.size()));
  std::vector<unsigned char> z(zlen);
  if (compress2(z.data(), &zlen, raw.data(), static_cast<uLong>(raw.size()), 1) != Z_OK)
    return fail(path, "zlib compression failed");
  std::vector<unsigned char> out(kSig, kSig + 8);
  auto chunk = [&](const char* type, const unsigned char* data, size_t len) {
    put32(out, static_cast<unsigned>(len));
    const size_t start = out.size();
    out.insert(out.end(), type, type + 4);
    out.insert(out.end(), data, data + len);
    put32(out, static_cast<unsigned>(crc32(crc32(0L, Z_NULL, 0), out.data() + start, static_cast<uInt>(len + 4))));
  };
  std::vector<unsigned char> ihdr;
  put32(ihdr, static_cast<unsigned>(width));
  put32(ihdr, static_cast<unsigned>(height));
  ihdr.push_back(8);
  ihdr.push_back(mask ? 6 : 2);
  ihdr.push_back(0);
  ihdr.push_back(0);
  ihdr.push_back(0);
  chunk("IHDR", ihdr.data(), ihdr.size());
  chunk("IDAT", z.data(), zlen);
  chunk("IEND", nullptr, 0);
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return fail(path, "cannot open for writing");
  const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
  if (std::fclose(f) != 0 || !ok) return fail(path, "short write");
  return STITCH_B200_OK;
}

}  // namespace stitch_b200_png
