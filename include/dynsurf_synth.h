/* dynsurf_synth.h — synthetic depth streams (host only), the shared input of
 * the CUDA path, the CPU oracle and the bench arms.
 *
 * Replaces: SyntheticSequence (proj/core/include/dynsurf/synth.hpp:16-73,
 * proj/core/src/synth.cpp). Built as its own library
 * (synth/lib/libdynsurf_synth.so) so that generating inputs never maps the
 * CUDA library libdynsurf_b200.so.
 */
#ifndef DYNSURF_SYNTH_H
#define DYNSURF_SYNTH_H
#include "dynsurf_b200.h"
#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic depth streams (synth.hpp:16-73; host only) ---- */
int32_t ds_synth_scenario(const char* name); /* -1 = unknown */
const char* ds_synth_scenario_name(int32_t scenario);
int32_t ds_synth_default_frames(int32_t scenario);
/* intrinsics: fx, fy, cx, cy, width, height of cfg are used */
ds_status ds_synth_render_depth(int32_t scenario, int32_t frames, const ds_config* cfg,
                                double noise_sigma_mm, uint32_t seed, int32_t t,
                                uint16_t* depth_out);
ds_status ds_synth_camera_pose(int32_t scenario, int32_t frames, int32_t t, double* pose);
double ds_synth_surface_distance(int32_t scenario, int32_t frames, const double* p_world,
                                 int32_t t);

#ifdef __cplusplus
}
#endif
#endif
