// Driver of the C++ drop-in API (include/svlf/*.hpp) for the parity tests
// (tests/test_cpp_api.py). Written like a reference call site: octree build,
// init_model, render_frame / render_frame_ref, train_step, loss_grads,
// checkpoints, DeviceModel. Writes raw little-endian arrays into <outdir> for
// the Python side to compare against the oracle.
//
//   cpp_api_probe ckpt   <outdir>   host only (no GPU): checkpoint round trip
//   cpp_api_probe render <outdir>   GPU: C1 frame, both precisions
//   cpp_api_probe train  <outdir>   GPU: loss/grads + two Adam steps
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "svlf/b200.hpp"
#include "svlf/camera.hpp"
#include "svlf/model.hpp"
#include "svlf/octree.hpp"
#include "svlf/render.hpp"
#include "svlf/rng.hpp"
#include "svlf/dataset.hpp"
#include "svlf/train.hpp"

using namespace svlf;

namespace {

std::string g_out;

template <typename T>
void dump(const std::string& name, const std::vector<T>& v) {
    std::ofstream f(g_out + "/" + name, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(T)));
}

void require(bool ok, const char* what) {
    if (!ok) throw std::runtime_error(std::string("probe check failed: ") + what);
}

// tests/test_octree.cpp random_occupancy recipe
std::vector<Vec3> occupancy_points(uint32_t res, double density, uint64_t seed) {
    Rng rng(seed);
    std::vector<Vec3> pts;
    const double h = 1.0 / res;
    for (uint32_t z = 0; z < res; ++z)
        for (uint32_t y = 0; y < res; ++y)
            for (uint32_t x = 0; x < res; ++x)
                if (rng.uniform() < density) pts.emplace_back((x + 0.5) * h, (y + 0.5) * h, (z + 0.5) * h);
    return pts;
}

GridConfig grid(uint32_t res, uint32_t dil) {
    GridConfig g;
    g.resolution = res;
    g.dilation = dil;
    return g;
}

Camera c1_camera(uint32_t w) {
    const Vec3 c(0.5, 0.5, 0.5);
    return make_lookat_camera(c + Vec3(0.6, 0.3, 0.7416) * 1.8, c, w, w, 1.5 * w);
}

std::vector<float> flat(const SvlfModel& m) {
    std::vector<float> v(m.feat_thickness.data);
    v.insert(v.end(), m.feat_color.data.begin(), m.feat_color.data.end());
    for (const auto* d : {&m.dec_thickness, &m.dec_color})
        for (size_t l = 0; l < d->weights.size(); ++l) {
            v.insert(v.end(), d->weights[l].begin(), d->weights[l].end());
            v.insert(v.end(), d->biases[l].begin(), d->biases[l].end());
        }
    return v;
}

void write_tree(const SparseOctree& t) {
    dump("leaf_codes.u64", t.leaf_codes());
    const uint32_t meta[3] = {t.config().resolution, t.config().dilation, t.vertex_count()};
    dump("tree_meta.u32", std::vector<uint32_t>(meta, meta + 3));
}

int run_ckpt() {
    const auto tree = SparseOctree::build(occupancy_points(16, 0.05, 3), grid(16, 1));
    write_tree(tree);
    SvlfModel m;
    m.octree = tree;
    const size_t V = tree.vertex_count();
    Rng r(42);
    m.feat_thickness.dim = kThicknessFeatDim;
    m.feat_color.dim = kColorFeatDim;
    for (size_t i = 0; i < V * 64; ++i) m.feat_thickness.data.push_back(float(r.uniform(-1, 1)));
    for (size_t i = 0; i < V * 32; ++i) m.feat_color.data.push_back(float(r.uniform(-1, 1)));
    for (auto [spec, dst] : {std::pair{MlpSpec::thickness_decoder(), &m.dec_thickness},
                             std::pair{MlpSpec::color_decoder(), &m.dec_color}}) {
        dst->spec = spec;
        for (uint32_t l = 0; l < spec.layer_count(); ++l) {
            std::vector<float> w(size_t(spec.layer_out(l)) * spec.layer_in(l)), b(spec.layer_out(l));
            for (auto& x : w) x = float(r.uniform(-0.2, 0.2));
            for (auto& x : b) x = float(r.uniform(-0.1, 0.1));
            dst->weights.push_back(w);
            dst->biases.push_back(b);
        }
    }
    ModelAdam adam = ModelAdam::like(m);
    uint64_t step = 1;
    for (AdamState* s : {&adam.feat_thickness, &adam.feat_color}) {
        s->step = step++;
        for (auto& x : s->m) x = float(r.uniform());
        for (auto& x : s->v) x = float(r.uniform());
    }
    for (auto& s : adam.dec_thickness) s.step = step++;
    for (auto& s : adam.dec_color) s.step = step++;
    save_checkpoint(g_out + "/a.ckpt", m, adam);

    SvlfModel m2;
    ModelAdam a2;
    load_checkpoint(g_out + "/a.ckpt", m2, a2);
    require(m2.octree.leaf_codes() == m.octree.leaf_codes(), "octree leaves");
    require(m2.octree.vertex_count() == m.octree.vertex_count(), "vertex count");
    require(flat(m2) == flat(m), "parameters");
    require(a2.dec_color.size() == 8 && a2.dec_color[7].step == adam.dec_color[7].step, "adam steps");
    require(a2.feat_color.v == adam.feat_color.v, "adam moments");
    save_checkpoint(g_out + "/b.ckpt", m2, a2);

    bool threw = false;
    try {
        load_checkpoint(g_out + "/missing.ckpt", m2, a2);
    } catch (const std::runtime_error& e) {
        threw = std::string(e.what()).rfind("cannot open checkpoint", 0) == 0;
    }
    require(threw, "missing file error");
    std::printf("ckpt ok V=%zu\n", V);
    return 0;
}

int run_render() {
    const auto tree = SparseOctree::build(occupancy_points(64, 0.02, 7), grid(64, 0));
    write_tree(tree);
    const SvlfModel model = init_model(tree, 0);
    dump("params.f32", flat(model));
    const Camera cam = c1_camera(200);
    FrameBuffers exact, fast;
    RenderStats st;
    render_frame_ref(model, cam, exact, &st);
    b200::set_render_precision(b200::Precision::FP16);
    render_frame(model, cam, fast, &st);
    dump("exact_rgb.f32", exact.rgb);
    dump("exact_alpha.f32", exact.alpha);
    dump("exact_depth.f32", exact.depth);
    dump("fast_rgb.f32", fast.rgb);
    dump("fast_alpha.f32", fast.alpha);
    dump("fast_depth.f32", fast.depth);
    const long long s[5] = {st.rays, st.rays_with_hits, st.traversal_hits, st.thickness_queries, st.color_queries};
    dump("stats.i64", std::vector<long long>(s, s + 5));

    // DeviceModel fast path renders the same bits as the drop-in
    b200::DeviceModel dm(model);
    FrameBuffers again;
    b200::set_render_precision(b200::Precision::FP32);
    dm.render(cam, again);
    require(again.rgb == exact.rgb && again.depth == exact.depth, "DeviceModel render");

    // a changed host model must be re-uploaded by the cache
    SvlfModel edited = model;
    for (auto& b : edited.dec_color.biases.back()) b += 0.5f;
    FrameBuffers e1, e2;
    render_frame_ref(edited, cam, e1);
    edited.dec_color.biases.back()[0] -= 1.0f;
    render_frame_ref(edited, cam, e2);
    require(e1.rgb != e2.rgb, "cache invalidation");

    // traversal through the C++ API (GPU) for the camera's centre ray
    const auto hits = tree.traverse(cam.pixel_ray(100, 100));
    std::vector<double> h;
    for (const auto& x : hits) {
        h.push_back(double(x.voxel_id));
        h.push_back(x.t_in);
        h.push_back(x.t_out);
    }
    dump("centre_hits.f64", h);
    std::printf("render ok hits=%lld\n", st.traversal_hits);
    return 0;
}

int run_train() {
    const auto tree = SparseOctree::build(occupancy_points(32, 0.03, 5), grid(32, 1));
    write_tree(tree);
    SvlfModel model = init_model(tree, 0);
    const SvlfModel teacher = init_model(tree, 9);
    const uint32_t W = 64;
    const Camera cam = c1_camera(W);
    FrameBuffers gt;
    render_frame_ref(teacher, cam, gt);
    std::vector<RaySupervision> batch(size_t(W) * W);
    std::vector<double> rays;
    std::vector<float> cgt;
    std::vector<double> depth;
    std::vector<uint8_t> alpha;
    for (uint32_t i = 0; i < W * W; ++i) {
        RaySupervision& s = batch[i];
        s.ray = cam.pixel_ray(i % W, i / W);
        for (int c = 0; c < 3; ++c) s.c_gt[c] = gt.rgb[3 * i + c];
        s.alpha_gt = gt.alpha[i] > 0.5f;
        s.depth_gt = s.alpha_gt ? gt.depth[i] : 0.0;
        const double r6[6] = {s.ray.origin.x, s.ray.origin.y, s.ray.origin.z, s.ray.dir.x, s.ray.dir.y, s.ray.dir.z};
        rays.insert(rays.end(), r6, r6 + 6);
        cgt.insert(cgt.end(), s.c_gt, s.c_gt + 3);
        depth.push_back(s.depth_gt);
        alpha.push_back(s.alpha_gt);
    }
    dump("rays.f64", rays);
    dump("cgt.f32", cgt);
    dump("depth.f64", depth);
    dump("alpha.u8", alpha);
    dump("params0.f32", flat(model));

    ModelGrads g;
    LossStats ls;
    const double l0 = loss_grads(model, batch, LossMode::Volumetric, false, LossWeights{}, &g, &ls);
    std::vector<float> gf(g.feat_thickness);
    gf.insert(gf.end(), g.feat_color.begin(), g.feat_color.end());
    for (const auto* d : {&g.dec_thickness, &g.dec_color})
        for (size_t l = 0; l < d->weights.size(); ++l) {
            gf.insert(gf.end(), d->weights[l].begin(), d->weights[l].end());
            gf.insert(gf.end(), d->biases[l].begin(), d->biases[l].end());
        }
    dump("grads.f32", gf);

    ModelAdam adam = ModelAdam::like(model);
    std::vector<double> losses{l0};
    for (int k = 0; k < 2; ++k) losses.push_back(train_step(model, adam, batch, LossMode::Volumetric, false, 1e-3f));
    dump("losses.f64", losses);
    dump("params2.f32", flat(model));
    const long long st[3] = {ls.rays, ls.skipped_rays, ls.eta_skipped};
    dump("loss_stats.i64", std::vector<long long>(st, st + 3));
    require(adam.feat_thickness.step == 2 && adam.dec_color[7].step == 2, "adam steps");

    // DeviceModel path: same two steps with the device copy authoritative
    SvlfModel fresh = init_model(tree, 0);
    b200::DeviceModel dm(fresh, ModelAdam::like(fresh));
    for (int k = 0; k < 2; ++k) dm.train_step(batch, LossMode::Volumetric, false, 1e-3f);
    SvlfModel synced;
    dm.sync_to(synced);
    dump("params2_device.f32", flat(synced));

    // the same two steps with the 3xTF32 tensor-core GEMMs (same fp32 gates)
    b200::set_train_precision(b200::TrainPrecision::TF32X3);
    {
        SvlfModel m3 = init_model(tree, 0);
        ModelAdam a3 = ModelAdam::like(m3);
        std::vector<double> l3;
        for (int k = 0; k < 2; ++k) l3.push_back(train_step(m3, a3, batch, LossMode::Volumetric, false, 1e-3f));
        dump("losses_x3.f64", l3);
        dump("params2_x3.f32", flat(m3));
    }
    b200::set_train_precision(b200::TrainPrecision::FP32);

    // checkpoint of the trained state reloads into an identical render
    save_checkpoint(g_out + "/trained.ckpt", model, adam);
    SvlfModel back;
    ModelAdam back_adam;
    load_checkpoint(g_out + "/trained.ckpt", back, back_adam);
    FrameBuffers f1, f2;
    render_frame_ref(model, cam, f1);
    render_frame_ref(back, cam, f2);
    require(f1.rgb == f2.rgb && f1.depth == f2.depth, "checkpoint render");
    std::printf("train ok loss %.6f -> %.6f\n", losses.front(), losses.back());
    return 0;
}

// ds.bin: u32 n, w, h, then per view: 20 f64 camera record (fx fy cx cy c2w[16]),
// i32 split (0 train, 1 val), rgb w*h*3 f32, depth w*h f32, mask w*h f32.
// argv: trainloop <dir> e1 e2 e3 grid
int run_trainloop(int argc, char** argv) {
    std::ifstream f(g_out + "/ds.bin", std::ios::binary);
    uint32_t hdr[3];
    f.read(reinterpret_cast<char*>(hdr), sizeof hdr);
    SceneDataset ds;
    ds.width = hdr[1];
    ds.height = hdr[2];
    for (uint32_t i = 0; i < hdr[0]; ++i) {
        double rec[20];
        int32_t split;
        f.read(reinterpret_cast<char*>(rec), sizeof rec);
        f.read(reinterpret_cast<char*>(&split), 4);
        DatasetFrame fr;
        fr.name = std::to_string(i);
        fr.split = split == 1 ? "val" : "train";
        fr.camera.fx = rec[0];
        fr.camera.fy = rec[1];
        fr.camera.cx = rec[2];
        fr.camera.cy = rec[3];
        std::copy(rec + 4, rec + 20, fr.camera.camera_to_world.begin());
        fr.camera.width = ds.width;
        fr.camera.height = ds.height;
        fr.rgb = Image::make(ds.width, ds.height, 3);
        fr.depth = Image::make(ds.width, ds.height, 1);
        fr.mask = Image::make(ds.width, ds.height, 1);
        for (Image* im : {&fr.rgb, &fr.depth, &fr.mask})
            f.read(reinterpret_cast<char*>(im->px.data()), std::streamsize(im->px.size() * 4));
        ds.frames.push_back(std::move(fr));
    }
    require(bool(f), "dataset file");
    TrainConfig cfg;
    cfg.epochs = {std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5])};
    cfg.grid_resolution = uint32_t(std::atoi(argv[6]));
    cfg.dilation = 1;
    cfg.seed = 0;
    cfg.out_dir = g_out + "/run";
    (void)argc;
    const TrainResult r = train(cfg, ds);
    std::vector<double> log;
    for (const EpochLog& e : r.log) {
        const double row[5] = {double(e.stage), double(e.epoch), e.mean_loss, e.val_psnr, e.seconds};
        log.insert(log.end(), row, row + 5);
    }
    dump("train_log.f64", log);
    dump("trained.f32", flat(r.model));
    write_tree(r.model.octree);
    dump("skipped.i64", std::vector<long long>{r.skipped_rays});
    require(!r.diverged, "diverged");
    require(!r.checkpoints[3].empty(), "final checkpoint");
    std::printf("trainloop ok: %zu epochs, final loss %.6f\n", r.log.size(), r.log.empty() ? 0.0 : r.log.back().mean_loss);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s ckpt|render|train|trainloop <outdir> [...]\n", argv[0]);
        return 2;
    }
    g_out = argv[2];
    try {
        const std::string mode = argv[1];
        if (mode == "ckpt") return run_ckpt();
        if (mode == "render") return run_render();
        if (mode == "train") return run_train();
        if (mode == "trainloop" && argc == 7) return run_trainloop(argc, argv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 2;
}
