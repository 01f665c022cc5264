/* svr_synth.h -- synthetic analytic-SDF scene fixtures (host C++, no GPU needed).
 *
 * Restates the reference's synthetic generator (proj/src/core/synthetic.hpp:13-77,
 * synthetic.cpp:42-192): a box room with spheres/boxes, ring cameras, z-depth
 * raycasting, plus the payload/ray/upstream-gradient recipes of SURVEY.md section
 * 8(d) used by the parity tests and bench.py.  These produce INPUTS; they are not part
 * of the rendering hot path.  Exported from fixtures/libsvr_fixture.so (host-only, built by
 * fixtures/build.py), never from the product library.
 */
#ifndef SVR_SYNTH_H
#define SVR_SYNTH_H

#include <stdint.h>

#include "svr.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* svr_fixture_last_error(void);

/* SceneSpec (synthetic.hpp:13-30); defaults via svr_scene_spec_default. */
typedef struct {
    double room_w, room_d, room_h;
    int32_t n_objects;
    int32_t n_frames;
    int32_t width, height;
    double fov_deg;
    int32_t label_channels;
    double texture_amplitude;
    double texture_frequency;
    uint64_t seed;
} svr_scene_spec;

typedef struct svr_scene svr_scene;

void svr_scene_spec_default(svr_scene_spec* spec);
int svr_scene_create(const svr_scene_spec* spec, svr_scene** out);
void svr_scene_destroy(svr_scene* s);
/* SyntheticScene::camera_for_frame (synthetic.cpp:164-192) */
int svr_scene_camera(const svr_scene* s, int32_t frame, svr_camera* out);
/* GT z-depth per integer pixel via SyntheticScene::raycast (synthetic.cpp:89-162,
 * 318-332); depth_out is [n][height][width]; uses `threads` host threads (0 = all). */
int svr_scene_depth(const svr_scene* s, const svr_camera* cams, uint32_t n, float* depth_out,
                    int32_t threads);
/* The frame images of generate_dataset (synthetic.cpp:318-340) per integer pixel: GT
 * z-depth [n][H][W], rgb = scene.color(hit point, hit label) [n][H][W][3], semantic =
 * one-hot(hit label) [n][H][W][C] (C >= 4), camera-frame surface normal R^T n [n][H][W][3].
 * Any output may be NULL. */
int svr_scene_frames(const svr_scene* s, const svr_camera* cams, uint32_t n, float* depth_out,
                     float* rgb_out, float* semantic_out, int32_t C, float* normal_out, int32_t threads);
/* SyntheticScene::sdf (synthetic.cpp:71-80) */
int svr_scene_sdf(const svr_scene* s, const double* x, uint64_t n, double* out);
/* Fills block payloads in the reference per-block layout (grid.hpp:62-66):
 * sdf = clamp(scene.sdf(v*h), -trunc, trunc), weight = 1, rgb = scene.color(v*h, label),
 * logits = one-hot(label) with label = the nearest surface's class.  Arrays are
 * [nblocks][B^3], [nblocks][B^3], [nblocks][B^3][3], [nblocks][B^3][C]. */
int svr_scene_fill_payload(const svr_scene* s, double voxel_size, int32_t block_res,
                           int32_t label_channels, double trunc, const int32_t* coords,
                           uint64_t nblocks, float* sdf, float* weight, float* rgb,
                           float* logits, int32_t threads);
/* Rays: for pose p in [0,n_poses) (camera_for_frame(p)), rays_per_pose integer pixels
 * drawn by mt19937_64(seed) uniform over width*height; origin = camera centre,
 * dir = Camera::ray_direction (camera.cpp:27-30).  o,d are [n_poses*rays_per_pose][3]. */
int svr_scene_rays(const svr_scene* s, uint32_t n_poses, uint32_t rays_per_pose, uint64_t seed,
                   double* o, double* d);
/* Every pixel of one camera, row-major (cfg2 full-image render). */
int svr_scene_image_rays(const svr_scene* s, int32_t frame, double* o, double* d);
/* n floats U(-1,1) from mt19937_64(seed) (upstream gradients). */
int svr_uniform_floats(uint64_t n, uint64_t seed, float lo, float hi, float* out);

#ifdef __cplusplus
}
#endif

#endif
