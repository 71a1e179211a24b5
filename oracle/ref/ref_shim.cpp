// Test infrastructure (oracle/_ref): a C entry layer over the UNMODIFIED
// reference library compiled from /root/reference/proj/src. Only tests/,
// __graft_entry__.smoke() and bench.py's reference/cpu_baseline leg load it.
//
// Flat parameter convention shared with oracle/svlf_oracle.h and the B200
// library: decoder parameters are concatenated per layer as W_l (row-major
// [out][in]) then b_l, in layer order (reference include/svlf/mlp.hpp:50-53).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "svlf/camera.hpp"
#include "svlf/dataset.hpp"
#include "svlf/metrics.hpp"
#include "svlf/model.hpp"
#include "svlf/octree.hpp"
#include "svlf/render.hpp"
#include "svlf/scene.hpp"
#include "svlf/threads.hpp"
#include "svlf/train.hpp"

using namespace svlf;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

GridConfig make_grid(uint32_t res, uint32_t dil, const double* lo, const double* hi) {
    GridConfig g;
    g.resolution = res;
    g.dilation = dil;
    if (lo && hi) g.scene_aabb = Aabb{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
    return g;
}

Camera make_camera(const double* cam, uint32_t w, uint32_t h) {
    Camera c;
    c.fx = cam[0];
    c.fy = cam[1];
    c.cx = cam[2];
    c.cy = cam[3];
    for (int i = 0; i < 16; ++i) c.camera_to_world[i] = cam[4 + i];
    c.width = w;
    c.height = h;
    return c;
}

void put_camera(const Camera& c, double* out) {
    out[0] = c.fx;
    out[1] = c.fy;
    out[2] = c.cx;
    out[3] = c.cy;
    for (int i = 0; i < 16; ++i) out[4 + i] = c.camera_to_world[i];
}

size_t mlp_flat_size(const MlpParams& p) { return p.param_count(); }

void mlp_get(const MlpParams& p, float* out) {
    size_t o = 0;
    for (size_t l = 0; l < p.weights.size(); ++l) {
        std::memcpy(out + o, p.weights[l].data(), p.weights[l].size() * 4);
        o += p.weights[l].size();
        std::memcpy(out + o, p.biases[l].data(), p.biases[l].size() * 4);
        o += p.biases[l].size();
    }
}

void mlp_set(MlpParams& p, const float* in) {
    size_t o = 0;
    for (size_t l = 0; l < p.weights.size(); ++l) {
        std::memcpy(p.weights[l].data(), in + o, p.weights[l].size() * 4);
        o += p.weights[l].size();
        std::memcpy(p.biases[l].data(), in + o, p.biases[l].size() * 4);
        o += p.biases[l].size();
    }
}

void grads_get(const MlpGrads& g, float* out) {
    size_t o = 0;
    for (size_t l = 0; l < g.weights.size(); ++l) {
        std::memcpy(out + o, g.weights[l].data(), g.weights[l].size() * 4);
        o += g.weights[l].size();
        std::memcpy(out + o, g.biases[l].data(), g.biases[l].size() * 4);
        o += g.biases[l].size();
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_thread_count(n); }
int ref_thread_count() { return thread_count(); }

// ---- octree --------------------------------------------------------------
void* ref_octree_build(const double* pts, size_t n, uint32_t res, uint32_t dil, const double* lo,
                       const double* hi) {
    SparseOctree* out = nullptr;
    guarded([&] {
        std::vector<Vec3> p(n);
        for (size_t i = 0; i < n; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        out = new SparseOctree(SparseOctree::build(p, make_grid(res, dil, lo, hi)));
    });
    return out;
}

void* ref_octree_from_leaves(const uint64_t* codes, size_t n, uint32_t res, uint32_t dil,
                             const double* lo, const double* hi) {
    SparseOctree* out = nullptr;
    guarded([&] {
        out = new SparseOctree(SparseOctree::from_leaves(std::vector<uint64_t>(codes, codes + n),
                                                         make_grid(res, dil, lo, hi)));
    });
    return out;
}

void ref_octree_free(void* t) { delete static_cast<SparseOctree*>(t); }
int ref_octree_leaf_level(void* t) { return static_cast<SparseOctree*>(t)->leaf_level(); }
uint32_t ref_octree_vertex_count(void* t) { return static_cast<SparseOctree*>(t)->vertex_count(); }
size_t ref_octree_dropped(void* t) { return static_cast<SparseOctree*>(t)->dropped_points(); }
size_t ref_octree_level_size(void* t, int level) {
    return static_cast<SparseOctree*>(t)->level_codes(level).size();
}
void ref_octree_level_codes(void* t, int level, uint64_t* out) {
    const auto& v = static_cast<SparseOctree*>(t)->level_codes(level);
    std::memcpy(out, v.data(), v.size() * 8);
}
int ref_octree_corner_ids(void* t, uint32_t* out) {
    const auto* tree = static_cast<SparseOctree*>(t);
    return guarded([&] {
        size_t i = 0;
        for (uint64_t code : tree->leaf_codes()) {
            const auto c = tree->corner_vertices(code);
            for (int b = 0; b < 8; ++b) out[i++] = c[b];
        }
    });
}
// locate(): out = code, returns 1 if found
int ref_octree_locate(void* t, const double* p, uint64_t* out) {
    const auto v = static_cast<SparseOctree*>(t)->locate({p[0], p[1], p[2]});
    if (!v) return 0;
    *out = *v;
    return 1;
}

// Batched traverse: rays are n x 6 (origin, dir). offsets has n+1 entries.
// Hits are written only when the total fits `cap`; the total is returned.
size_t ref_traverse(void* t, const double* rays, size_t n, uint64_t* offsets, size_t cap,
                    uint64_t* ids, double* tin, double* tout, double* x12) {
    const auto* tree = static_cast<SparseOctree*>(t);
    std::vector<RayVoxelHit> hits;
    TraversalScratch scratch;
    offsets[0] = 0;
    for (size_t i = 0; i < n; ++i) {
        const Ray r{{rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]},
                    {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]}};
        tree->traverse(r, hits, scratch);
        offsets[i + 1] = hits.size();
    }
    if (hits.size() <= cap) {
        for (size_t j = 0; j < hits.size(); ++j) {
            ids[j] = hits[j].voxel_id;
            tin[j] = hits[j].t_in;
            tout[j] = hits[j].t_out;
            if (x12) {
                const double v[6] = {hits[j].x1.x, hits[j].x1.y, hits[j].x1.z,
                                     hits[j].x2.x, hits[j].x2.y, hits[j].x2.z};
                std::memcpy(x12 + 6 * j, v, sizeof(v));
            }
        }
    }
    return hits.size();
}

int ref_ray_aabb(const double* ray6, const double* lo, const double* hi, double* t01) {
    const auto r = ray_aabb(Ray{{ray6[0], ray6[1], ray6[2]}, {ray6[3], ray6[4], ray6[5]}},
                            Aabb{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
    if (!r) return 0;
    t01[0] = r->t0;
    t01[1] = r->t1;
    return 1;
}

// Camera rays in raster order (px = y*W + x), n = W*H, out n x 6.
void ref_camera_rays(const double* cam, uint32_t w, uint32_t h, double* out) {
    const Camera c = make_camera(cam, w, h);
    for (uint32_t px = 0; px < w * h; ++px) {
        const Ray r = c.pixel_ray(px % w, px / w);
        const double v[6] = {r.origin.x, r.origin.y, r.origin.z, r.dir.x, r.dir.y, r.dir.z};
        std::memcpy(out + 6 * size_t(px), v, sizeof(v));
    }
}

void ref_lookat_camera(const double* eye, const double* target, uint32_t w, uint32_t h,
                       double focal, double* out) {
    put_camera(make_lookat_camera({eye[0], eye[1], eye[2]}, {target[0], target[1], target[2]}, w,
                                  h, focal),
               out);
}

// ---- model ---------------------------------------------------------------
void* ref_model_init(void* t, uint64_t seed) {
    SvlfModel* m = nullptr;
    guarded([&] { m = new SvlfModel(init_model(*static_cast<SparseOctree*>(t), seed)); });
    return m;
}
void ref_model_free(void* m) { delete static_cast<SvlfModel*>(m); }
size_t ref_model_sizes(void* mp, size_t* out4) {
    auto* m = static_cast<SvlfModel*>(mp);
    out4[0] = m->feat_thickness.data.size();
    out4[1] = m->feat_color.data.size();
    out4[2] = mlp_flat_size(m->dec_thickness);
    out4[3] = mlp_flat_size(m->dec_color);
    return out4[0] + out4[1] + out4[2] + out4[3];
}
void ref_model_get(void* mp, float* ft, float* fc, float* mt, float* mc) {
    auto* m = static_cast<SvlfModel*>(mp);
    std::memcpy(ft, m->feat_thickness.data.data(), m->feat_thickness.data.size() * 4);
    std::memcpy(fc, m->feat_color.data.data(), m->feat_color.data.size() * 4);
    mlp_get(m->dec_thickness, mt);
    mlp_get(m->dec_color, mc);
}
void ref_model_set(void* mp, const float* ft, const float* fc, const float* mt, const float* mc) {
    auto* m = static_cast<SvlfModel*>(mp);
    std::memcpy(m->feat_thickness.data.data(), ft, m->feat_thickness.data.size() * 4);
    std::memcpy(m->feat_color.data.data(), fc, m->feat_color.data.size() * 4);
    mlp_set(m->dec_thickness, mt);
    mlp_set(m->dec_color, mc);
}

// stats: rays, rays_with_hits, traversal_hits, thickness_queries, color_queries
int ref_render_frame(void* mp, const double* cam, uint32_t w, uint32_t h, const float* bg,
                     float* rgb, float* alpha, float* depth, long long* stats, int parallel,
                     double* seconds) {
    auto* m = static_cast<SvlfModel*>(mp);
    return guarded([&] {
        const Camera c = make_camera(cam, w, h);
        FrameBuffers fb;
        RenderStats st;
        const auto t0 = std::chrono::steady_clock::now();
        if (parallel)
            render_frame(*m, c, fb, &st, bg);
        else
            render_frame_ref(*m, c, fb, &st, bg);
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (rgb) std::memcpy(rgb, fb.rgb.data(), fb.rgb.size() * 4);
        if (alpha) std::memcpy(alpha, fb.alpha.data(), fb.alpha.size() * 4);
        if (depth) std::memcpy(depth, fb.depth.data(), fb.depth.size() * 4);
        if (stats) {
            stats[0] = st.rays;
            stats[1] = st.rays_with_hits;
            stats[2] = st.traversal_hits;
            stats[3] = st.thickness_queries;
            stats[4] = st.color_queries;
        }
    });
}

// Sum of the public per-ray losses (include/svlf/train.hpp:60-71) with
// gradients accumulated into one ModelGrads in ray order. mode 0 = surface,
// 1 = volumetric. lw = (eta, tau, empty, alpha). stats3 = rays, skipped,
// eta_skipped. Gradient outputs may be null.
int ref_loss(void* mp, const double* rays, const float* cgt, const double* depth,
             const uint8_t* alpha, size_t n, int mode, const double* lw4, int frozen,
             float* g_ft, float* g_fc, float* g_mt, float* g_mc, long long* stats3,
             double* loss_out) {
    auto* m = static_cast<SvlfModel*>(mp);
    return guarded([&] {
        const LossWeights lw{lw4[0], lw4[1], lw4[2], lw4[3]};
        const bool want_grads = g_ft || g_fc || g_mt || g_mc;
        ModelGrads g = ModelGrads::like(*m);
        LossStats st;
        double loss = 0;
        for (size_t i = 0; i < n; ++i) {
            RaySupervision s;
            s.ray = Ray{{rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]},
                        {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]}};
            s.c_gt[0] = cgt[3 * i];
            s.c_gt[1] = cgt[3 * i + 1];
            s.c_gt[2] = cgt[3 * i + 2];
            s.depth_gt = depth[i];
            s.alpha_gt = alpha[i] != 0;
            if (mode == 0)
                loss += surface_loss(*m, s, lw, want_grads ? &g : nullptr, &st);
            else
                loss += volumetric_loss(*m, s, lw, frozen != 0, want_grads ? &g : nullptr, &st);
        }
        if (g_ft) std::memcpy(g_ft, g.feat_thickness.data(), g.feat_thickness.size() * 4);
        if (g_fc) std::memcpy(g_fc, g.feat_color.data(), g.feat_color.size() * 4);
        if (g_mt) grads_get(g.dec_thickness, g_mt);
        if (g_mc) grads_get(g.dec_color, g_mc);
        if (stats3) {
            stats3[0] = st.rays;
            stats3[1] = st.skipped_rays;
            stats3[2] = st.eta_skipped;
        }
        *loss_out = loss;
    });
}

// One bias-corrected Adam step over a flat tensor (src/mlp.cpp:277-296).
// `step` is the step count before the update.
void ref_adam_step(float* params, const float* grads, float* m, float* v, size_t n, uint64_t step,
                   float lr) {
    AdamState s;
    s.m.assign(m, m + n);
    s.v.assign(v, v + n);
    s.step = step;
    adam_step(s, std::span<float>(params, n), std::span<const float>(grads, n), lr);
    std::memcpy(m, s.m.data(), n * 4);
    std::memcpy(v, s.v.data(), n * 4);
}

// ---- synthetic scenes (analytic ray-caster, src/scene.cpp) ---------------
void* ref_scene_make(uint64_t seed, int prims) {
    return new AnalyticScene(make_random_scene(seed, prims));
}
void ref_scene_free(void* s) { delete static_cast<AnalyticScene*>(s); }

// out: n x 20 camera records (fx, fy, cx, cy, c2w[16])
void ref_hemisphere_cameras(int n, double radius, uint64_t seed, uint32_t w, uint32_t h,
                            double focal, double* out) {
    const auto cams = sample_hemisphere_cameras(n, radius, seed, w, h, focal);
    for (int i = 0; i < n; ++i) put_camera(cams[i], out + 20 * size_t(i));
}

// Ground truth for one camera exactly as generate_dataset's pixel loop
// (src/dataset.cpp:61-83): rgb (3/px), depth, mask.
void ref_scene_render_gt(void* sp, const double* cam, uint32_t w, uint32_t h, float* rgb,
                         float* depth, float* mask) {
    const auto* scene = static_cast<AnalyticScene*>(sp);
    const Camera c = make_camera(cam, w, h);
    const int64_t pixels = int64_t(w) * h;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t p = 0; p < pixels; ++p) {
        const uint32_t x = static_cast<uint32_t>(p % w), y = static_cast<uint32_t>(p / w);
        const Ray ray = c.pixel_ray(x, y);
        const auto hit = raycast(*scene, ray);
        if (hit) {
            const Vec3 col = shade(*scene, *hit);
            rgb[3 * p] = float(col.x);
            rgb[3 * p + 1] = float(col.y);
            rgb[3 * p + 2] = float(col.z);
            depth[p] = float(hit->t);
            mask[p] = 1.f;
        } else {
            rgb[3 * p] = float(scene->background.x);
            rgb[3 * p + 1] = float(scene->background.y);
            rgb[3 * p + 2] = float(scene->background.z);
            depth[p] = 0.f;
            mask[p] = 0.f;
        }
    }
}

// train() on an in-memory dataset of `n_frames` hemisphere views (train split
// only, no validation): epochs = (e0, e1, e2). Returns per-epoch seconds and
// mean loss (log_out: 2 doubles per epoch), and the final model when
// model_out is non-null (caller frees with ref_model_free).
int ref_train(void* sp, const double* cams, int n_frames, uint32_t w, uint32_t h, const int* epochs,
              uint32_t grid_res, uint32_t dilation, uint64_t seed, double* log_out,
              int log_cap, int* log_n, void** model_out) {
    const auto* scene = static_cast<AnalyticScene*>(sp);
    return guarded([&] {
        SceneDataset ds;
        ds.width = w;
        ds.height = h;
        for (int f = 0; f < n_frames; ++f) {
            DatasetFrame fr;
            fr.name = std::to_string(f);
            fr.split = "train";
            fr.camera = make_camera(cams + 20 * size_t(f), w, h);
            fr.rgb = Image::make(w, h, 3);
            fr.depth = Image::make(w, h, 1);
            fr.mask = Image::make(w, h, 1);
            ref_scene_render_gt(const_cast<AnalyticScene*>(scene), cams + 20 * size_t(f), w, h,
                                fr.rgb.px.data(), fr.depth.px.data(), fr.mask.px.data());
            ds.frames.push_back(std::move(fr));
        }
        TrainConfig cfg;
        cfg.epochs = {epochs[0], epochs[1], epochs[2]};
        cfg.grid_resolution = grid_res;
        cfg.dilation = dilation;
        cfg.seed = seed;
        TrainResult r = train(cfg, ds);
        int k = 0;
        for (const EpochLog& e : r.log) {
            if (k < log_cap) {
                log_out[2 * k] = e.seconds;
                log_out[2 * k + 1] = e.mean_loss;
            }
            ++k;
        }
        *log_n = k;
        if (model_out) *model_out = new SvlfModel(std::move(r.model));
    });
}

// ---- checkpoints: load_checkpoint + save_checkpoint (src/model.cpp:182-235)
int ref_checkpoint_roundtrip(const char* in, const char* out) {
    return guarded([&] {
        SvlfModel m;
        ModelAdam a;
        load_checkpoint(in, m, a);
        save_checkpoint(out, m, a);
    });
}

// train() with explicit splits (0 = train, 1 = val) and the full epoch log:
// 5 doubles per epoch (stage, epoch, mean_loss, val_psnr, seconds).
int ref_train2(void* sp, const double* cams, const int* splits, int n_frames, uint32_t w, uint32_t h,
               const int* epochs, uint32_t grid_res, uint32_t dilation, uint64_t seed, double* log_out,
               int log_cap, int* log_n, long long* skipped, void** model_out) {
    const auto* scene = static_cast<AnalyticScene*>(sp);
    return guarded([&] {
        SceneDataset ds;
        ds.width = w;
        ds.height = h;
        for (int f = 0; f < n_frames; ++f) {
            DatasetFrame fr;
            fr.name = std::to_string(f);
            fr.split = splits[f] == 1 ? "val" : "train";
            fr.camera = make_camera(cams + 20 * size_t(f), w, h);
            fr.rgb = Image::make(w, h, 3);
            fr.depth = Image::make(w, h, 1);
            fr.mask = Image::make(w, h, 1);
            ref_scene_render_gt(const_cast<AnalyticScene*>(scene), cams + 20 * size_t(f), w, h,
                                fr.rgb.px.data(), fr.depth.px.data(), fr.mask.px.data());
            ds.frames.push_back(std::move(fr));
        }
        TrainConfig cfg;
        cfg.epochs = {epochs[0], epochs[1], epochs[2]};
        cfg.grid_resolution = grid_res;
        cfg.dilation = dilation;
        cfg.seed = seed;
        TrainResult r = train(cfg, ds);
        int k = 0;
        for (const EpochLog& e : r.log) {
            if (k < log_cap) {
                double* o = log_out + 5 * k;
                o[0] = e.stage;
                o[1] = e.epoch;
                o[2] = e.mean_loss;
                o[3] = e.val_psnr;
                o[4] = e.seconds;
            }
            ++k;
        }
        *log_n = k;
        if (skipped) *skipped = r.skipped_rays;
        if (model_out) *model_out = new SvlfModel(std::move(r.model));
    });
}

// ---- metrics (src/metrics.cpp): images as interleaved float planes --------
int ref_metrics(const float* pred, const float* gt, uint32_t w, uint32_t h, uint32_t channels, double* psnr_out,
                double* ssim_out) {
    return guarded([&] {
        Image a = Image::make(w, h, channels), b = Image::make(w, h, channels);
        std::memcpy(a.px.data(), pred, a.px.size() * 4);
        std::memcpy(b.px.data(), gt, b.px.size() * 4);
        *psnr_out = psnr(a, b);
        *ssim_out = ssim(a, b);
    });
}

}  // extern "C"
