// synth.cpp -- synthetic multi-camera scenes (the input generator).
//
// Behaviour of SynthScene (/root/reference/proj/src/synth.cpp:14-231,
// proj/include/stitch/synth.hpp:17-87): a value-noise textured world plane
// (Z_W = 0) watched by cameras whose spacing is solved by bisection so that
// adjacent footprints overlap by the requested fraction; exact ray-cast
// rendering with per-view colour casts, flicker events and a moving
// parallax occluder.
//
// For <= 3 views the reference yaw rig is used (synth.cpp:60-152).  The
// reference caps views at 3 (synth.cpp:61-63) because a yaw rig beyond
// +-90 degrees cannot map onto one plane; the N-view "strip" rig (extension,
// parity-unpinned) keeps a small per-step toe-in yaw and instead solves the
// camera baseline for the overlap fraction.
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "host_geometry.hpp"
#include "stitch_synth.h"

namespace {

using stitch_b200_host::Mat3;

std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

double lattice(std::uint64_t seed, long ix, long iy) {
  std::uint64_t h = seed;
  h = splitmix64(h ^ static_cast<std::uint64_t>(ix) * 0x9e3779b97f4a7c15ull);
  h = splitmix64(h ^ static_cast<std::uint64_t>(iy) * 0xc2b2ae3d27d4eb4full);
  return static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0);
}

double smoothstep(double t) { return t * t * (3.0 - 2.0 * t); }

double value_noise(std::uint64_t seed, double x, double y) {
  const double fx = std::floor(x), fy = std::floor(y);
  const long ix = static_cast<long>(fx), iy = static_cast<long>(fy);
  const double tx = smoothstep(x - fx), ty = smoothstep(y - fy);
  const double v00 = lattice(seed, ix, iy);
  const double v10 = lattice(seed, ix + 1, iy);
  const double v01 = lattice(seed, ix, iy + 1);
  const double v11 = lattice(seed, ix + 1, iy + 1);
  const double top = v00 + (v10 - v00) * tx;
  const double bot = v01 + (v11 - v01) * tx;
  return top + (bot - top) * ty;
}

void texture_rgb(std::uint64_t seed, double x, double y, double rgb[3]) {
  for (int c = 0; c < 3; ++c) {
    const std::uint64_t s = splitmix64(seed + 0x517cc1b727220a95ull * (c + 1));
    const double n = 0.55 * value_noise(s, x / 48.0, y / 48.0) +
                     0.30 * value_noise(s ^ 0xabcdu, x / 12.0, y / 12.0) +
                     0.15 * value_noise(s ^ 0x1234u, x / 3.0, y / 3.0);
    rgb[c] = 20.0 + 215.0 * n;
  }
}

std::uint8_t quantize(double v) {
  const double r = std::round(v);
  if (r < 0.0) return 0;
  if (r > 255.0) return 255;
  return static_cast<std::uint8_t>(r);
}

}  // namespace

struct stitch_b200_synth {
  stitch_b200_synth_spec spec;
  int reference = 0;
  double focal = 0, distance = 500.0, baseline = 0, yaw_step = 0;
  int rig = 1;
  std::vector<stitch_b200_camera> cams;  // exact cameras
  std::vector<Mat3> hom;                 // planar homographies (world -> image)
  // per view, for rendering: camera centre and R_wc * K^-1
  std::vector<std::array<double, 3>> centre;
  std::vector<Mat3> ray;

  void build(double step) {
    cams.clear();
    hom.clear();
    for (int v = 0; v < spec.views; ++v) {
      const int k = v - reference;
      stitch_b200_camera c{};
      c.fx = focal;
      c.fy = focal;
      c.cx = spec.width / 2.0;
      c.cy = spec.height / 2.0;
      double yaw, cx_world;
      if (rig == 1) {  // synth.cpp:76-95
        yaw = k * step;
        cx_world = k * baseline;
      } else if (rig == 3) {  // ring rig (extension): shared centre
        yaw = k * step;
        cx_world = 0.0;
      } else {  // strip rig (extension)
        yaw = k * spec.strip_yaw;
        cx_world = k * step;
      }
      const double cs = std::cos(yaw), sn = std::sin(yaw);
      // ry = [[c,0,s],[0,1,0],[-s,0,c]]; rotation = ry^T (world -> camera)
      const double ry[9] = {cs, 0, sn, 0, 1, 0, -sn, 0, cs};
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.rotation[i * 3 + j] = ry[j * 3 + i];
      const double cen[3] = {cx_world, 0.0, rig == 3 ? 0.0 : -distance};
      for (int i = 0; i < 3; ++i) {
        // translation = -R * centre
        c.translation[i] = (-c.rotation[i * 3 + 0] * cen[0] +
                            -c.rotation[i * 3 + 1] * cen[1]) +
                           -c.rotation[i * 3 + 2] * cen[2];
      }
      cams.push_back(c);
      Mat3 h;
      stitch_b200_host::planar_homography(c, h);
      hom.push_back(h);
    }
  }

  // synth.cpp:100-131: worst adjacent-footprint overlap fraction.
  double overlap_of(double step) {
    build(step);
    double worst = 1.0;
    auto span = [&](const Mat3& inv, double& lo, double& hi) {
      lo = 1e18;
      hi = -1e18;
      const double w = spec.width - 1.0, h = spec.height - 1.0;
      const double cx[4] = {0, w, 0, w}, cy[4] = {0, 0, h, h};
      for (int k = 0; k < 4; ++k) {
        double X, Y;
        stitch_b200_host::homography_apply(inv, cx[k], cy[k], X, Y);
        lo = std::min(lo, X);
        hi = std::max(hi, X);
      }
    };
    for (int v = 0; v < spec.views; ++v) {
      if (v == reference) continue;
      // the reference measures against the reference view (star); the strip
      // rig measures each view against its neighbour toward the reference.
      const int other = (rig == 1) ? reference : (v < reference ? v + 1 : v - 1);
      Mat3 inv_v, inv_r;
      stitch_b200_host::homography_inverse(hom[v], inv_v);
      stitch_b200_host::homography_inverse(hom[other], inv_r);
      double alo, ahi, blo, bhi;
      span(inv_v, alo, ahi);
      span(inv_r, blo, bhi);
      const double inter = std::min(ahi, bhi) - std::max(alo, blo);
      const double denom = std::min(ahi - alo, bhi - blo);
      worst = std::min(worst, denom > 0 ? inter / denom : 0.0);
    }
    return worst;
  }

  void prepare_render() {
    centre.assign(spec.views, {0, 0, 0});
    ray.assign(spec.views, Mat3{});
    for (int v = 0; v < spec.views; ++v) {
      const stitch_b200_camera& c = cams[v];
      Mat3 rwc;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rwc[i * 3 + j] = c.rotation[j * 3 + i];
      for (int i = 0; i < 3; ++i)
        centre[v][i] = (-rwc[i * 3 + 0] * c.translation[0] +
                        -rwc[i * 3 + 1] * c.translation[1]) +
                       -rwc[i * 3 + 2] * c.translation[2];
      const Mat3 k = {c.fx, 0, c.cx, 0, c.fy, c.cy, 0, 0, 1};
      Mat3 kinv;
      stitch_b200_host::inverse3(k, kinv);
      stitch_b200_host::mul3(rwc, kinv, ray[v]);
    }
  }

  // SynthScene::shade, synth.cpp:170-201
  void shade(int view, int frame, double px, double py, double rgb[3]) const {
    const Mat3& r = ray[view];
    const double dir[3] = {(r[0] * px + r[1] * py) + r[2],
                           (r[3] * px + r[4] * py) + r[5],
                           (r[6] * px + r[7] * py) + r[8]};
    const auto& c = centre[view];
    if (rig == 3) {
      // ring scene (extension): textured cylinder of radius `distance`
      // around the shared camera centre, texture at (angle * radius, height)
      const double rr = std::sqrt(dir[0] * dir[0] + dir[2] * dir[2]);
      if (rr < 1e-12) {
        rgb[0] = rgb[1] = rgb[2] = 0.0;
        return;
      }
      const double s = distance / rr;
      const double hx = s * dir[0], hy = s * dir[1], hz = s * dir[2];
      texture_rgb(spec.seed, std::atan2(hx, hz) * distance, hy, rgb);
      return;
    }
    if (spec.object_enabled && std::abs(dir[2]) > 1e-12) {
      const double zo = -spec.object_depth_fraction * distance;
      const double s = (zo - c[2]) / dir[2];
      if (s > 0) {
        const double hx = c[0] + s * dir[0], hy = c[1] + s * dir[1];
        const double pxo = spec.object_position[0] + frame * spec.object_velocity[0];
        const double pyo = spec.object_position[1] + frame * spec.object_velocity[1];
        if (std::abs(hx - pxo) <= spec.object_half_size &&
            std::abs(hy - pyo) <= spec.object_half_size) {
          texture_rgb(splitmix64(spec.seed ^ 0x0b7ec7ull), hx - pxo, hy - pyo, rgb);
          return;
        }
      }
    }
    if (std::abs(dir[2]) < 1e-12) {
      rgb[0] = rgb[1] = rgb[2] = 0.0;
      return;
    }
    const double s = (0.0 - c[2]) / dir[2];
    texture_rgb(spec.seed, c[0] + s * dir[0], c[1] + s * dir[1], rgb);
  }
};

extern "C" {

void stitch_b200_synth_defaults(stitch_b200_synth_spec* s) {
  std::memset(s, 0, sizeof(*s));
  s->seed = 1;
  s->views = 2;
  s->frames = 5;
  s->width = 320;
  s->height = 240;
  s->overlap_fraction = 0.3;
  s->object_depth_fraction = 0.15;
  s->object_half_size = 40.0;
  s->perturb_focal_scale = 1.0;
  s->perturb_principal_px = 0.0;
  s->rig = 0;
  s->strip_yaw = 0.05;
}

int stitch_b200_synth_create(const stitch_b200_synth_spec* spec,
                             stitch_b200_synth** out) {
  *out = nullptr;
  if (spec->views < 2 || spec->views > STITCH_B200_MAX_VIEWS) return STITCH_B200_ConfigError;
  if (spec->frames < 1) return STITCH_B200_ConfigError;
  if (!(spec->overlap_fraction > 0.05 && spec->overlap_fraction < 0.9))
    return STITCH_B200_ConfigError;
  if (spec->n_casts != 0 && spec->n_casts != spec->views) return STITCH_B200_ConfigError;
  if (spec->width < 2 || spec->height < 2) return STITCH_B200_ConfigError;
  auto* s = new stitch_b200_synth();
  s->spec = *spec;
  s->rig = spec->rig != 0 ? spec->rig : (spec->views <= 3 ? 1 : 2);
  if (s->rig == 1 && spec->views > 3) {
    delete s;
    return STITCH_B200_ConfigError;  // the yaw rig cannot exceed 3 views
  }
  if (s->rig == 3) {
    if (spec->views < 3) {
      delete s;
      return STITCH_B200_ConfigError;
    }
    // ring: yaw step 2pi/N, horizontal FOV = step / (1 - overlap)
    s->reference = 0;
    s->yaw_step = 2.0 * M_PI / spec->views;
    const double fov = s->yaw_step / (1.0 - spec->overlap_fraction);
    s->focal = 0.5 * spec->width / std::tan(0.5 * fov);
    s->build(s->yaw_step);
    s->prepare_render();
    *out = s;
    return STITCH_B200_OK;
  }
  // reference_ = views == 3 ? 1 : 0 (synth.cpp:71); (views-1)/2 generalises it.
  s->reference = (spec->views - 1) / 2;
  s->focal = 0.9 * spec->width;
  s->baseline = 0.05 * s->distance;
  double lo = 0.0, hi = (s->rig == 1) ? 0.6 : 2.0 * s->distance;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (s->overlap_of(mid) > spec->overlap_fraction)
      lo = mid;
    else
      hi = mid;
  }
  s->yaw_step = lo;
  s->build(lo);
  s->prepare_render();
  *out = s;
  return STITCH_B200_OK;
}

void stitch_b200_synth_destroy(stitch_b200_synth* s) { delete s; }

int stitch_b200_synth_reference(const stitch_b200_synth* s) { return s->reference; }

// SynthScene::config, synth.cpp:149-168
int stitch_b200_synth_config(const stitch_b200_synth* s, stitch_b200_config* cfg) {
  stitch_b200_host::config_defaults(cfg);
  cfg->n_views = s->spec.views;
  cfg->reference = s->reference;
  if (s->rig == 3) {
    cfg->projection = 1;
    cfg->cyl_focal = s->focal;
    cfg->topology = 3;
  }
  for (int v = 0; v < s->spec.views; ++v) {
    cfg->width[v] = s->spec.width;
    cfg->height[v] = s->spec.height;
    stitch_b200_camera c = s->cams[v];
    if (v != s->reference) {
      c.fx *= s->spec.perturb_focal_scale;
      c.fy *= s->spec.perturb_focal_scale;
      if (s->spec.perturb_principal_px != 0.0) {
        const double ang = 2.0 * M_PI * lattice(splitmix64(s->spec.seed ^ 0xfeedu), v, 0);
        c.cx += s->spec.perturb_principal_px * std::cos(ang);
        c.cy += s->spec.perturb_principal_px * std::sin(ang);
      }
    }
    cfg->cams[v] = c;
  }
  return STITCH_B200_OK;
}

// SynthScene::render_view, synth.cpp:203-231
int stitch_b200_synth_render(const stitch_b200_synth* s, int view, int frame,
                             uint8_t* out, int threads) {
  if (view < 0 || view >= s->spec.views) return STITCH_B200_ConfigError;
  double gains[3] = {1.0, 1.0, 1.0};
  if (s->spec.n_casts)
    for (int c = 0; c < 3; ++c) gains[c] = s->spec.color_casts[view][c];
  for (int i = 0; i < s->spec.n_flicker; ++i) {
    const auto& f = s->spec.flicker[i];
    if (f.frame == frame && f.view == view)
      for (int c = 0; c < 3; ++c) gains[c] *= f.gains[c];
  }
  const int w = s->spec.width, h = s->spec.height;
  auto rows = [&](int y0, int y1) {
    for (int y = y0; y < y1; ++y)
      for (int x = 0; x < w; ++x) {
        double rgb[3];
        s->shade(view, frame, x, y, rgb);
        std::uint8_t* p = out + (static_cast<size_t>(y) * w + x) * 3;
        p[0] = quantize(rgb[0] * gains[0]);
        p[1] = quantize(rgb[1] * gains[1]);
        p[2] = quantize(rgb[2] * gains[2]);
      }
  };
  if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  if (threads <= 1 || h < 2 * threads) {
    rows(0, h);
    return STITCH_B200_OK;
  }
  std::vector<std::thread> pool;
  const int chunk = (h + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int y0 = t * chunk, y1 = std::min(h, y0 + chunk);
    if (y0 < y1) pool.emplace_back(rows, y0, y1);
  }
  for (auto& t : pool) t.join();
  return STITCH_B200_OK;
}

}  // extern "C"
