// sequence_io.cpp -- frame ingress / egress either side of the per-frame path
// (SURVEY §8f rank 3): the reference's image I/O and numbered-sequence helpers
// (image_io.cpp:19-199; PNG through png_codec.cpp on zlib, libpng is not in
// this image) and a file-to-file sequence runner (run_sequence,
// pipeline.cpp:364-412, with directory sources and an image sink).  B200
// side: view files are read straight into pinned staging buffers by one
// reader thread per view, frames go through the pipelined submit / wait path
// (four frames in flight: uploads, kernels and downloads overlap), and four
// writer threads encode the panoramas from an eight-frame pinned ring, so
// file I/O overlaps the GPU.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "png_codec.hpp"
#include "stitch_b200.h"

namespace fs = std::filesystem;

namespace {

int io_fail(const std::string& path, const char* what) {
  const std::string m = path + ": " + what;
  return stitch_b200_set_error(STITCH_B200_IoError, m.c_str());
}

// read_ppm_token (image_io.cpp:19-37): skips whitespace and '#' comments
// between header tokens; -1 at end of file.  The character after the
// token's digits (one whitespace byte before the raster) is consumed.
int ppm_token(std::FILE* f) {
  int c = std::fgetc(f);
  while (c != EOF) {
    if (c == '#') {
      while (c != EOF && c != '\n') c = std::fgetc(f);
    } else if (!std::isspace(c)) {
      break;
    }
    c = std::fgetc(f);
  }
  if (c == EOF) return -1;
  int value = 0;
  while (c != EOF && std::isdigit(c)) {
    value = value * 10 + (c - '0');
    c = std::fgetc(f);
  }
  return value;
}

struct File {
  std::FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

// header of a P6 PPM (image_io.cpp:61-70); leaves f at the raster
int ppm_header(std::FILE* f, const std::string& path, int* w, int* h) {
  char magic[2];
  if (std::fread(magic, 1, 2, f) != 2 || magic[0] != 'P' || magic[1] != '6')
    return io_fail(path, "not a P6 PPM");
  const int width = ppm_token(f);
  const int height = ppm_token(f);
  const int maxval = ppm_token(f);
  if (width < 1 || height < 1 || maxval != 255) return io_fail(path, "unsupported PPM header");
  *w = width;
  *h = height;
  return STITCH_B200_OK;
}

std::vector<fs::path> list_images(const std::string& dir, int* rc) {
  // list_sequence (image_io.cpp:181-192): regular .png / .ppm files, sorted
  std::vector<fs::path> files;
  std::error_code ec;
  if (!fs::is_directory(dir, ec)) {
    *rc = io_fail(dir, "not a directory");
    return files;
  }
  for (const auto& e : fs::directory_iterator(dir, ec)) {
    if (!e.is_regular_file()) continue;
    const auto ext = e.path().extension().string();
    if (ext == ".ppm" || ext == ".png") files.push_back(e.path());
  }
  std::sort(files.begin(), files.end());
  *rc = STITCH_B200_OK;
  return files;
}

// read_image (image_io.cpp:167-172) of one camera frame straight into rgb
// (capacity bytes): the PPM raster is read in place, a PNG decoded then
// copied.  A PNG with transparent pixels is a masked frame (image_io.cpp:
// 120-127): its mask goes to `mask` (capacity / 3 bytes) and *masked is set.
int read_frame(const fs::path& path, uint8_t* rgb, size_t capacity, uint8_t* mask, bool* masked,
               int* w, int* h) {
  *masked = false;
  const std::string ext = path.extension().string();
  if (ext == ".ppm") return stitch_b200_read_ppm(path.string().c_str(), rgb, capacity, w, h);
  if (ext != ".png") return io_fail(path.string(), "unsupported image extension");
  stitch_b200_png::Image img;
  const int rc = stitch_b200_png::read_png(path.string(), img);
  if (rc) return rc;
  *w = img.width;
  *h = img.height;
  if (img.rgb.size() > capacity)
    return stitch_b200_set_error(STITCH_B200_InputMismatch, "frame size differs from the view size");
  std::memcpy(rgb, img.rgb.data(), img.rgb.size());
  if (!img.mask.empty()) {
    std::memcpy(mask, img.mask.data(), img.mask.size());
    *masked = true;
  }
  return STITCH_B200_OK;
}

}  // namespace

extern "C" {

int stitch_b200_ppm_info(const char* path, int* width, int* height) {
  File fl;
  fl.f = std::fopen(path, "rb");
  if (!fl.f) return io_fail(path, "cannot open");
  return ppm_header(fl.f, path, width, height);
}

int stitch_b200_read_ppm(const char* path, uint8_t* rgb, size_t capacity, int* width,
                         int* height) {
  File fl;
  fl.f = std::fopen(path, "rb");
  if (!fl.f) return io_fail(path, "cannot open");
  int w = 0, h = 0;
  int rc = ppm_header(fl.f, path, &w, &h);
  if (rc) return rc;
  const size_t n = static_cast<size_t>(w) * h * 3;
  if (width) *width = w;
  if (height) *height = h;
  if (!rgb) return STITCH_B200_OK;
  if (n > capacity) return stitch_b200_set_error(STITCH_B200_InputMismatch, "buffer too small");
  if (std::fread(rgb, 1, n, fl.f) != n) return io_fail(path, "truncated pixel data");
  return STITCH_B200_OK;
}

int stitch_b200_write_ppm(const char* path, int width, int height, const uint8_t* rgb) {
  // write_ppm (image_io.cpp:78-85): "P6\n<w> <h>\n255\n" + raster
  if (width < 1 || height < 1 || !rgb)
    return stitch_b200_set_error(STITCH_B200_InputMismatch, "empty frame");
  File fl;
  fl.f = std::fopen(path, "wb");
  if (!fl.f) return io_fail(path, "cannot open for writing");
  if (std::fprintf(fl.f, "P6\n%d %d\n255\n", width, height) < 0)
    return io_fail(path, "short write");
  const size_t n = static_cast<size_t>(width) * height * 3;
  if (std::fwrite(rgb, 1, n, fl.f) != n) return io_fail(path, "short write");
  if (std::fclose(fl.f) != 0) {
    fl.f = nullptr;
    return io_fail(path, "short write");
  }
  fl.f = nullptr;
  return STITCH_B200_OK;
}

int stitch_b200_read_png(const char* path, uint8_t* rgb, size_t capacity, uint8_t* mask,
                         size_t mask_capacity, int* width, int* height, int* has_mask) {
  stitch_b200_png::Image img;
  const int rc = stitch_b200_png::read_png(path, img);
  if (rc) return rc;
  if (width) *width = img.width;
  if (height) *height = img.height;
  if (has_mask) *has_mask = img.mask.empty() ? 0 : 1;
  if (rgb) {
    if (img.rgb.size() > capacity)
      return stitch_b200_set_error(STITCH_B200_InputMismatch, "buffer too small");
    std::memcpy(rgb, img.rgb.data(), img.rgb.size());
  }
  if (mask) {
    const size_t n = static_cast<size_t>(img.width) * img.height;
    if (n > mask_capacity) return stitch_b200_set_error(STITCH_B200_InputMismatch, "buffer too small");
    if (img.mask.empty())
      std::memset(mask, 1, n);
    else
      std::memcpy(mask, img.mask.data(), n);
  }
  return STITCH_B200_OK;
}

int stitch_b200_write_png(const char* path, int width, int height, const uint8_t* rgb,
                          const uint8_t* mask) {
  return stitch_b200_png::write_png(path, width, height, rgb, mask);
}

int stitch_b200_sequence_name(const char* stem, int index, const char* ext, char* out,
                              size_t capacity) {
  // sequence_name (image_io.cpp:194-199): stem + "_%06d" + ext
  const int n = std::snprintf(out, capacity, "%s_%06d%s", stem, index, ext ? ext : ".png");
  if (n < 0 || static_cast<size_t>(n) >= capacity)
    return stitch_b200_set_error(STITCH_B200_InputMismatch, "name buffer too small");
  return STITCH_B200_OK;
}

int stitch_b200_run_files(stitch_b200_ctx* ctx, const char* const* view_dirs,
                          const char* out_dir, const char* stem, const char* ext, int max_frames,
                          stitch_b200_report* reports, stitch_b200_files_stats* stats) {
  const std::string out_ext = ext ? ext : ".ppm";
  if (out_ext != ".ppm" && out_ext != ".png")
    return io_fail(out_ext, "unsupported output image extension");
  const int nv = stitch_b200_n_views(ctx);
  if (nv < 1) return nv < 0 ? nv : stitch_b200_set_error(STITCH_B200_MissingState, "no views");
  int cw = 0, ch = 0;
  double ox = 0, oy = 0;
  int rc = stitch_b200_canvas(ctx, &cw, &ch, &ox, &oy);
  if (rc) return rc;
  std::vector<std::vector<fs::path>> lists(nv);
  size_t n = 0;
  for (int v = 0; v < nv; ++v) {
    lists[v] = list_images(view_dirs[v], &rc);
    if (rc) return rc;
    n = v == 0 ? lists[v].size() : std::min(n, lists[v].size());
  }
  if (max_frames > 0) n = std::min(n, static_cast<size_t>(max_frames));
  if (out_dir) {
    std::error_code ec;
    fs::create_directories(out_dir, ec);
    if (!fs::is_directory(out_dir, ec)) return io_fail(out_dir, "cannot create output directory");
  }
  std::vector<size_t> vbytes(nv);
  for (int v = 0; v < nv; ++v) {
    int w = 0, h = 0;
    rc = stitch_b200_view_size(ctx, v, &w, &h);
    if (rc) return rc;
    vbytes[v] = static_cast<size_t>(w) * h * 3;
  }
  const size_t pano_bytes = static_cast<size_t>(cw) * ch;
  // host ring of pinned frame buffers (frame t in slot t % kRing, reused by
  // frame t + kRing once frame t is written); kInFlight frames on the GPU
  // (the context's pipeline slots); kWriters panorama writers
  constexpr int kRing = 8, kInFlight = 4, kWriters = 4;
  struct Slot {
    std::vector<uint8_t*> in;
    std::vector<uint8_t*> in_mask;   // the views' input masks (transparent PNG sources)
    std::vector<char> masked;        // per view: this frame's view carries a mask
    uint8_t* rgb = nullptr;
    uint8_t* mask = nullptr;
  };
  Slot ring[kRing];
  auto free_ring = [&]() {
    for (auto& s : ring) {
      for (auto* p : s.in) stitch_b200_host_free(p);
      for (auto* p : s.in_mask) stitch_b200_host_free(p);
      stitch_b200_host_free(s.rgb);
      stitch_b200_host_free(s.mask);
    }
  };
  for (auto& s : ring) {
    for (int v = 0; v < nv; ++v) {
      s.in.push_back(static_cast<uint8_t*>(stitch_b200_host_alloc(vbytes[v])));
      s.in_mask.push_back(static_cast<uint8_t*>(stitch_b200_host_alloc(vbytes[v] / 3)));
    }
    s.masked.assign(static_cast<size_t>(nv), 0);
    s.rgb = static_cast<uint8_t*>(stitch_b200_host_alloc(pano_bytes * 3));
    s.mask = static_cast<uint8_t*>(stitch_b200_host_alloc(pano_bytes));
    bool ok = s.rgb && s.mask;
    for (auto* p : s.in) ok = ok && p;
    for (auto* p : s.in_mask) ok = ok && p;
    if (!ok) {
      free_ring();
      return stitch_b200_set_error(STITCH_B200_CudaError, "pinned allocation failed");
    }
  }

  // Frame t moves loaded -> submitted -> retired (panorama in host memory)
  // -> written; its ring slot t % kRing is reused by frame t + kRing once
  // frame t is written.
  std::mutex mu;
  std::condition_variable cv;
  long long loaded = 0, retired = 0, written = 0;  // counts of frames
  std::atomic<int> err{0};
  std::string err_msg;
  double read_s = 0.0, write_s = 0.0;  // summed per-file times (under mu)
  auto set_err = [&](int code) {
    std::lock_guard<std::mutex> lk(mu);
    if (!err) {
      err = code;
      err_msg = stitch_b200_last_error();
    }
    cv.notify_all();
  };
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_start = now();

  // readers: one thread per view, all reading frame t before any reads t+1
  std::vector<long long> view_loaded(nv, 0);
  std::vector<std::thread> readers;
  for (int v = 0; v < nv; ++v)
    readers.emplace_back([&, v]() {
      for (size_t t = 0; t < n; ++t) {
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return err || written + kRing > static_cast<long long>(t); });
          if (err) return;
        }
        const auto t0 = now();
        int w = 0, h = 0;
        bool vm = false;
        const int r = read_frame(lists[v][t], ring[t % kRing].in[v], vbytes[v],
                                 ring[t % kRing].in_mask[v], &vm, &w, &h);
        ring[t % kRing].masked[v] = vm ? 1 : 0;
        if (r == STITCH_B200_OK && static_cast<size_t>(w) * h * 3 != vbytes[v]) {
          stitch_b200_set_error(STITCH_B200_InputMismatch, "frame size differs from the view size");
          set_err(STITCH_B200_InputMismatch);
          return;
        }
        if (r) {
          set_err(r);
          return;
        }
        const double dt = std::chrono::duration<double>(now() - t0).count();
        std::lock_guard<std::mutex> lk(mu);
        read_s += dt;
        view_loaded[v] = static_cast<long long>(t) + 1;
        loaded = *std::min_element(view_loaded.begin(), view_loaded.end());
        cv.notify_all();
      }
    });

  // writers: frame t by writer t % kWriters, panoramas of retired frames;
  // `written` counts the frames written without a gap
  std::vector<char> done(n, 0);
  std::vector<std::thread> writers;
  for (int wi = 0; wi < kWriters; ++wi)
    writers.emplace_back([&, wi]() {
      for (size_t t = wi; t < n; t += kWriters) {
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return err || retired > static_cast<long long>(t); });
          if (err) return;
        }
        if (out_dir) {
          const auto t0 = now();
          char name[512];
          int r = stitch_b200_sequence_name(stem ? stem : "pano", static_cast<int>(t),
                                            out_ext.c_str(), name, sizeof(name));
          const std::string file = (fs::path(out_dir) / name).string();
          // write_image (image_io.cpp:174-179): PPM drops the mask, PNG
          // stores it as alpha (the panorama always carries one)
          if (!r)
            r = out_ext == ".png"
                    ? stitch_b200_write_png(file.c_str(), cw, ch, ring[t % kRing].rgb,
                                            ring[t % kRing].mask)
                    : stitch_b200_write_ppm(file.c_str(), cw, ch, ring[t % kRing].rgb);
          if (r) {
            set_err(r);
            return;
          }
          const double dt = std::chrono::duration<double>(now() - t0).count();
          std::lock_guard<std::mutex> lk(mu);
          write_s += dt;
        }
        std::lock_guard<std::mutex> lk(mu);
        done[t] = 1;
        while (written < static_cast<long long>(n) && done[written]) ++written;
        cv.notify_all();
      }
    });

  // this thread: submit in order, keep up to kInFlight frames on the GPU
  std::vector<long long> tickets(n, -1);
  size_t next_wait = 0;
  auto retire_one = [&]() -> int {
    stitch_b200_report rep;
    const int r = stitch_b200_wait(ctx, tickets[next_wait], &rep);
    if (r) return r;
    if (reports) reports[next_wait] = rep;
    std::lock_guard<std::mutex> lk(mu);
    retired = static_cast<long long>(++next_wait);
    cv.notify_all();
    return STITCH_B200_OK;
  };
  for (size_t t = 0; t < n && !err; ++t) {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return err || loaded > static_cast<long long>(t); });
      if (err) break;
    }
    if (t >= static_cast<size_t>(kRing)) {
      // the slot is free only after frame t - kRing is written
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return err || written > static_cast<long long>(t - kRing); });
      if (err) break;
    }
    Slot& s = ring[t % kRing];
    long long tk = -1;
    // masked PNG views go with their masks (stitch_b200_submit_masked)
    std::vector<const uint8_t*> mptr(static_cast<size_t>(nv), nullptr);
    bool any_mask = false;
    for (int v = 0; v < nv; ++v)
      if (s.masked[v]) {
        mptr[v] = s.in_mask[v];
        any_mask = true;
      }
    int r = any_mask ? stitch_b200_submit_masked(ctx, s.in.data(), mptr.data(), s.rgb, s.mask, &tk)
                     : stitch_b200_submit(ctx, s.in.data(), s.rgb, s.mask, &tk);
    if (r) {
      set_err(r);
      break;
    }
    tickets[t] = tk;
    // retire the oldest frame once kInFlight are on the GPU
    if (t + 1 - next_wait >= static_cast<size_t>(kInFlight)) {
      r = retire_one();
      if (r) {
        set_err(r);
        break;
      }
    }
  }
  while (!err && next_wait < n) {
    const int r = retire_one();
    if (r) set_err(r);
  }
  for (auto& th : readers) th.join();
  for (auto& th : writers) th.join();
  // drain anything still in flight after an error before freeing the ring
  while (err && next_wait < n && tickets[next_wait] >= 0) {
    stitch_b200_report rep;
    stitch_b200_wait(ctx, tickets[next_wait], &rep);
    ++next_wait;
  }
  if (stats) {  // (before releasing the pinned ring, which is not part of the run)
    stats->frames = static_cast<long long>(written);
    stats->seconds = std::chrono::duration<double>(now() - t_start).count();
    stats->read_seconds = read_s;
    stats->write_seconds = write_s;
  }
  free_ring();
  if (err) return stitch_b200_set_error(err, err_msg.c_str());
  return STITCH_B200_OK;
}

}  // extern "C"
