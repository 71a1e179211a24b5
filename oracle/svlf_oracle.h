/*
 * svlf_oracle.h -- CPU restatement of the SVLF per-ray render/train path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2205_07058_b200/,
 * include/) links this; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it, as the checker. It restates, in plain C compiled
 * with -ffp-contract=off, the reference algorithms of
 * /root/reference/proj/{include/svlf,src}/ (citations per function in
 * svlf_oracle.c). Parity of this restatement against the reference itself is
 * pinned by tests/test_oracle_vs_ref.py (oracle/_ref, built from the reference
 * sources) and by the committed golden fixtures in tests/golden/.
 *
 * Flat parameter layout (shared with oracle/ref/ref_shim.cpp and the B200
 * library): feature volumes row-major [V][dim]; each decoder is the
 * concatenation, per layer l, of W_l (row-major [out][in]) then b_l.
 *   f_T: 134 -> 128 (relu) -> 2 (relu, sigmoid)            17,538 floats
 *   f_C: 38 -> 128 -> 128 -> 128 (relu) -> 3 (sigmoid x3)   38,403 floats
 * Errors are returned as nonzero codes with or_last_error() holding the
 * reference's exception message ("tangent ray", "point not in voxel", ...).
 */
#ifndef SVLF_ORACLE_H
#define SVLF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_FT_DIM 64
#define OR_FC_DIM 32
#define OR_HIDDEN 128
#define OR_MT_SIZE 17538
#define OR_MC_SIZE 38403

const char* or_last_error(void);

/* ---- octree ---------------------------------------------------------- */
typedef struct or_tree or_tree;
or_tree* or_tree_build(const double* pts, size_t n, uint32_t res, uint32_t dilation,
                       const double* lo, const double* hi);
or_tree* or_tree_from_leaves(const uint64_t* codes, size_t n, uint32_t res, uint32_t dilation,
                             const double* lo, const double* hi);
void or_tree_free(or_tree* t);
int or_tree_leaf_level(const or_tree* t);
size_t or_tree_level_size(const or_tree* t, int level);
const uint64_t* or_tree_level_codes(const or_tree* t, int level);
const uint32_t* or_tree_corner_ids(const or_tree* t); /* 8 per leaf, leaf-code order */
uint32_t or_tree_vertex_count(const or_tree* t);
size_t or_tree_dropped(const or_tree* t);
int or_tree_locate(const or_tree* t, const double* p, uint64_t* code);
int or_ray_aabb(const double* ray6, const double* lo, const double* hi, double* t01);
/* rays n x 6; offsets n+1; hits written only when total <= cap; returns total */
size_t or_traverse(const or_tree* t, const double* rays, size_t n, uint64_t* offsets, size_t cap,
                   uint64_t* ids, double* tin, double* tout);

/* ---- rng / init / cameras / scenes ----------------------------------- */
uint64_t or_rng_u64_first(uint64_t seed); /* Rng(seed).next_u64() */
void or_rng_uniform_stream(uint64_t seed, size_t n, double* out); /* Rng(seed).uniform() x n */
/* tests/test_octree.cpp:50-64 random_ray() x n from one Rng(seed); out n x 6 */
void or_random_rays(uint64_t seed, size_t n, double* out);
void or_init_model(const or_tree* t, uint64_t seed, float* ft, float* fc, float* mt, float* mc);
/* camera record: fx, fy, cx, cy, c2w[16] (20 doubles) */
void or_lookat_camera(const double* eye, const double* target, uint32_t w, uint32_t h,
                      double focal, double* cam20);
void or_camera_rays(const double* cam20, uint32_t w, uint32_t h, double* rays);
void or_hemisphere_cameras(int n, double radius, uint64_t seed, uint32_t w, uint32_t h,
                           double focal, double* cams);
typedef struct or_scene or_scene;
or_scene* or_scene_make(uint64_t seed, int prims);
void or_scene_free(or_scene* s);
void or_scene_render_gt(const or_scene* s, const double* cam20, uint32_t w, uint32_t h,
                        float* rgb, float* depth, float* mask);

/* ---- render ---------------------------------------------------------- */
/* stats: rays, rays_with_hits, traversal_hits, thickness_queries, color_queries */
int or_render_rays(const or_tree* t, const float* ft, const float* fc, const float* mt,
                   const float* mc, const double* rays, size_t n, const float* bg, float* rgb,
                   float* alpha, float* depth, long long* stats);
int or_render_frame(const or_tree* t, const float* ft, const float* fc, const float* mt,
                    const float* mc, const double* cam20, uint32_t w, uint32_t h,
                    const float* bg, float* rgb, float* alpha, float* depth, long long* stats);

/* ---- losses / optimizer ---------------------------------------------- */
/* mode 0 = surface (stage 1), 1 = volumetric (stages 2-3); lw = eta, tau,
 * empty, alpha. Gradients (nullable) are SUMMED over rays into the caller's
 * zeroed buffers. stats3 = rays, skipped_rays, eta_skipped. */
int or_loss(const or_tree* t, const float* ft, const float* fc, const float* mt, const float* mc,
            const double* rays, const float* cgt, const double* depth, const uint8_t* alpha,
            size_t n, int mode, const double* lw4, int frozen, float* g_ft, float* g_fc,
            float* g_mt, float* g_mc, long long* stats3, double* loss_out);
/* step = count before the update (reference AdamState.step) */
void or_adam_step(float* params, const float* grads, float* m, float* v, size_t n,
                  uint64_t step, float lr);

#ifdef __cplusplus
}
#endif
#endif
