/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the sparse-dense SDF rendering path.
 *
 * A plain C++ (no Eigen, no CUDA) restatement of the reference `svrecon` grid code
 * (/root/reference/proj/src/core/grid.{hpp,cpp}, allocation.cpp, camera.cpp,
 * scale_field.cpp, grid_io.cpp) plus the renderer that the reference only specifies
 * (SPEC.md:268-319).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg load this library, as the CHECKER.  The product path
 * (paper_2305_13220_b200/, libsvr_b200.so) never links or calls it.
 *
 * Parity pins: grid/march/gather/activation are validated against the reference's
 * own sources compiled verbatim (oracle/_ref, see Makefile) and against the golden
 * vectors in tests/golden/.  The renderer has no reference code: it is pinned only by
 * the SPEC known-answer tests and finite differences (tests/test_oracle_render.py).
 * All arithmetic is IEEE double; built with -ffp-contract=off (no FMA), like the
 * reference's Release build (proj/CMakeLists.txt:9-11).
 */
#ifndef SVR_ORACLE_H
#define SVR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct svro_grid svro_grid;

typedef struct {
    uint64_t blocks_added;     /* allocation.hpp:14 */
    uint64_t blocks_requested; /* allocation.hpp:15 */
    uint64_t pixels_used;      /* allocation.hpp:16 */
    uint64_t unallocated;      /* errors.hpp:27-31 CapacityError::unallocated_blocks */
} svro_report;

/* Pinhole camera, camera-to-world pose x_w = R x_c + t (camera.hpp:16-29).
 * R is row-major. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double R[9];
    double t[3];
} svro_camera;

/* status codes mirror errors.hpp:12-31: 0 ok, 2 config, 3 data, 5 capacity */
const char* svro_last_error(void);
void svro_set_threads(int n);

int svro_grid_create(double voxel_size, int block_res, int label_channels, uint64_t capacity,
                     svro_grid** out);
void svro_grid_destroy(svro_grid* g);
uint64_t svro_block_count(const svro_grid* g);
uint64_t svro_capacity(const svro_grid* g);
void svro_coords(const svro_grid* g, int32_t* out);
int svro_bounds(const svro_grid* g, int32_t* lo3, int32_t* hi3);

int svro_allocate_blocks(svro_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out);
int svro_allocate_points(svro_grid* g, const double* xyz, uint64_t n, int dilation,
                         svro_report* rep);
int svro_allocate_frames(svro_grid* g, const float* depth, const svro_camera* cams,
                         uint32_t n_frames, const double* scales, int sf_rows, int sf_cols,
                         int dilation, svro_report* rep);
void svro_find(const svro_grid* g, const int32_t* coords, uint64_t n, uint32_t* out);

int svro_set_payload(svro_grid* g, uint32_t first, uint32_t n, const float* sdf,
                     const float* weight, const float* rgb, const float* logits);
int svro_get_payload(const svro_grid* g, uint32_t first, uint32_t n, float* sdf, float* weight,
                     float* rgb, float* logits);

void svro_query(const svro_grid* g, const double* x, uint64_t n, double* sdf, double* grad,
                double* rgb, double* logits, uint8_t* valid);
void svro_march(const svro_grid* g, const double* o, const double* d, uint64_t n, double step,
                uint32_t max_samples, uint32_t* counts, double* t, double* delta);

int svro_render_forward(const svro_grid* g, const double* o, const double* d, uint64_t n,
                        double step, uint32_t max_samples, double beta, double* rgb,
                        double* depth, double* normal, double* wsum, uint32_t* nsamples,
                        uint32_t* nvalid);
int svro_render_backward(const svro_grid* g, const double* o, const double* d, uint64_t n,
                         double step, uint32_t max_samples, double beta, const double* d_rgb,
                         const double* d_depth, const double* d_normal, double* grad_sdf,
                         double* grad_rgb, uint8_t* active);

double svro_sdf_to_density(double s, double beta);
int svro_eikonal(const svro_grid* g, const double* x, uint64_t n, double scale, double* grad_sdf,
                 uint8_t* active, double* loss, uint64_t* n_valid);
int svro_rmsprop(svro_grid* g, const double* grad_sdf, const double* grad_rgb, const uint8_t* active,
                 float lr, float alpha, float eps, float* rms_state);

/* Fusion + denoise (decisions in svr_oracle.cpp / DESIGN.md "Fusion").
 * flags: bit0 fuse color, bit1 fuse semantic logits.  depth [n][H][W], rgb [n][H][W][3],
 * sem [n][H][W][C], scales [n][rows][cols] (NULL = 1). */
typedef struct {
    uint64_t frames;
    uint64_t in_view;    /* voxel-frame pairs projecting on a pixel with depth > 0 and scale > 0 */
    uint64_t integrated; /* in_view pairs with d >= -mu */
    uint64_t rejected;   /* in_view pairs with d < -mu (behind the surface beyond the band) */
} svro_fuse_report;
int svro_fuse_begin(svro_grid* g, int flags);
int svro_fuse_frames(svro_grid* g, const float* depth, const float* rgb, const float* sem,
                     const svro_camera* cams, uint32_t n_frames, const double* scales, int sf_rows,
                     int sf_cols, double mu, svro_fuse_report* rep);
int svro_fuse_finalize(svro_grid* g);
int svro_denoise(svro_grid* g, double sigma_vox, int radius);

/* marching_cubes (meshing.cpp:168-273); the mesh is kept in the handle for svro_mesh_get:
 * vertices/normals/colors [nv][3] f64, labels [nv] i32, triangles [nt][3] i32. */
int svro_mc_table(int32_t* counts, int32_t* tris);
int svro_marching_cubes(svro_grid* g, double iso, uint64_t* n_vertices, uint64_t* n_triangles);
int svro_mesh_get(const svro_grid* g, double* v, double* n, double* c, int32_t* labels, int32_t* tris);

/* Refinement losses: per-ray upstream gradients of
 * L_c + lambda_d L_d + lambda_n L_n; stats = {L_c, L_d, L_n, total, a, b, n_c, n_d, n_n, singular}. */
int svro_fit_depth_affine(const double* t, const double* D, uint64_t n, double* a, double* b);
int svro_render_losses(uint64_t n, const double* rgb, const double* depth, const double* normal,
                       const double* wsum, const float* tgt_rgb, const float* prior_depth,
                       const float* prior_normal, const uint32_t* cam_idx, const svro_camera* cams,
                       double lambda_d, double lambda_n, double* d_rgb, double* d_depth, double* d_normal,
                       double* stats);

int svro_save_sdgv(const svro_grid* g, const char* path);
int svro_load_sdgv(const char* path, svro_grid** out);

#ifdef __cplusplus
}
#endif

#endif
