/* stitch_synth.h -- synthetic multi-camera scenes (the reference's SynthScene,
 * proj/include/stitch/synth.hpp, restated; byte-identical renders on the
 * reference's rigs, tests/test_ref_pin.py), with the N-view strip and
 * 360-degree ring extensions.  Test and bench INPUT GENERATOR, built as its
 * own library (paper_2308_09209_b200/libstitch_synth.so) so that nothing that
 * only needs inputs -- e.g. bench.py's CPU reference arm -- loads the B200
 * product library.  Types shared with the product (stitch_b200_config,
 * stitch_b200_camera) come from stitch_b200.h. */
#ifndef STITCH_SYNTH_H
#define STITCH_SYNTH_H

#include "stitch_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic scenes (SynthScene, proj/include/stitch/synth.hpp) ---- */
typedef struct {
  int frame, view;
  double gains[3];
} stitch_b200_flicker;

typedef struct {
  uint64_t seed;
  int views, frames, width, height;
  double overlap_fraction;
  int n_casts;
  double color_casts[STITCH_B200_MAX_VIEWS][3];
  int n_flicker;
  stitch_b200_flicker flicker[16];
  int object_enabled;
  double object_depth_fraction, object_half_size;
  double object_position[2], object_velocity[2];
  double perturb_focal_scale, perturb_principal_px;
  /* 0 = auto: the reference yaw rig (synth.cpp:60-152) for <= 3 views, the
   * strip rig (N-view extension: small toe-in yaw, baseline solved for the
   * overlap fraction) beyond. 1 = yaw, 2 = strip, 3 = ring (extension:
   * cameras sharing one centre, yaw step 2pi/N, focal chosen for the
   * overlap fraction, textured cylinder scene, cylindrical canvas). */
  int rig;
  double strip_yaw; /* radians per view step for the strip rig */
} stitch_b200_synth_spec;

typedef struct stitch_b200_synth stitch_b200_synth;

void stitch_b200_synth_defaults(stitch_b200_synth_spec* spec);
int stitch_b200_synth_create(const stitch_b200_synth_spec* spec,
                             stitch_b200_synth** out);
void stitch_b200_synth_destroy(stitch_b200_synth* s);
int stitch_b200_synth_reference(const stitch_b200_synth* s);
/* Pipeline config carrying the (optionally perturbed) cameras and the
 * reference's StitchConfig defaults (feature refinement on, pipeline.hpp:24). */
int stitch_b200_synth_config(const stitch_b200_synth* s,
                             stitch_b200_config* cfg);
/* render_view (synth.cpp:203-231) into width*height*3 bytes. */
int stitch_b200_synth_render(const stitch_b200_synth* s, int view, int frame,
                             uint8_t* out, int threads);

#ifdef __cplusplus
}
#endif

#endif
