// C++ API over the C ABI: session, model init, checkpoints, render_frame,
// train_step, loss_grads, DeviceModel (include/svlf/{model,render,train,b200}.hpp).
//
// Reference interfaces mirrored: init_model / ModelAdam::like /
// save_checkpoint / load_checkpoint (src/model.cpp:15-235), MlpSpec
// (src/mlp.cpp:10-34), render_frame / render_frame_ref
// (src/render.cpp:209-247), the train() step body (src/train.cpp:443-479)
// and the public per-ray losses (include/svlf/train.hpp:60-71).
//
// Device copies: the drop-in functions take host models; a small cache keyed
// by the SvlfModel object holds its device model and a 64-bit fingerprint of
// the host tensors, so repeated renders of an unchanged model upload nothing.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <list>
#include <memory>

#include "session.hpp"
#include "svlf/b200.hpp"
#include "svlf/model.hpp"
#include "svlf/render.hpp"
#include "svlf/train.hpp"

namespace svlf {

// ---- session ---------------------------------------------------------------
namespace detail {

struct Session {
    std::recursive_mutex mu;
    svlf_ctx* ctx = nullptr;
    int device = -1;
    b200::Precision precision = b200::Precision::FP16;
};

Session& session() {
    static Session* s = new Session();  // never destroyed: CUDA teardown order at exit is not ours
    return *s;
}

std::recursive_mutex& session_mutex() { return session().mu; }

svlf_precision to_c(b200::Precision p) {
    switch (p) {
        case b200::Precision::FP32: return SVLF_PRECISION_FP32;
        case b200::Precision::BF16: return SVLF_PRECISION_BF16;
        default: return SVLF_PRECISION_FP16;
    }
}

}  // namespace detail

namespace b200 {

void set_device(int device) {
    auto& s = detail::session();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    if (s.ctx && device != s.device) throw std::logic_error("svlf::b200::set_device after the session started");
    s.device = device;
}

void set_render_precision(Precision p) { detail::session().precision = p; }
Precision render_precision() { return detail::session().precision; }

svlf_ctx* session_context() {
    auto& s = detail::session();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    if (!s.ctx) {
        if (s.device < 0) {
            const char* e = std::getenv("SVLF_DEVICE");
            s.device = e ? std::atoi(e) : 0;
        }
        detail::check(svlf_ctx_create(s.device, &s.ctx));
    }
    return s.ctx;
}

void set_train_precision(TrainPrecision p) {
    auto& s = detail::session();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    detail::check(svlf_ctx_set_train_precision(session_context(), static_cast<svlf_precision>(int(p))));
}

}  // namespace b200

// ---- decoder specs ---------------------------------------------------------
void MlpSpec::validate() const {
    if (input_dim < 1 || hidden_dim < 1 || output_dim < 1) throw std::invalid_argument("mlp dims must be >= 1");
    if (head.size() != output_dim) throw std::invalid_argument("head size must match output_dim");
}

MlpSpec MlpSpec::thickness_decoder(uint32_t feat_dim, uint32_t hidden) {
    return MlpSpec{6 + 2 * feat_dim, hidden, 1, 2, {Activation::Relu, Activation::Sigmoid}};
}

MlpSpec MlpSpec::color_decoder(uint32_t feat_dim, uint32_t hidden) {
    return MlpSpec{6 + feat_dim, hidden, 3, 3, {Activation::Sigmoid, Activation::Sigmoid, Activation::Sigmoid}};
}

// ---- flat <-> structured tensors --------------------------------------------
namespace {

// The library's flat decoder layout is the reference's per-layer [W, b] order.
MlpParams shaped(const MlpSpec& spec, const float* flat) {
    MlpParams p;
    p.spec = spec;
    for (uint32_t l = 0; l < spec.layer_count(); ++l) {
        const size_t nw = size_t(spec.layer_out(l)) * spec.layer_in(l), nb = spec.layer_out(l);
        p.weights.emplace_back(flat, flat + nw);
        flat += nw;
        p.biases.emplace_back(flat, flat + nb);
        flat += nb;
    }
    return p;
}

std::vector<float> flat_of(const MlpParams& p) {
    std::vector<float> f;
    f.reserve(p.param_count());
    for (size_t l = 0; l < p.weights.size(); ++l) {
        f.insert(f.end(), p.weights[l].begin(), p.weights[l].end());
        f.insert(f.end(), p.biases[l].begin(), p.biases[l].end());
    }
    return f;
}

void require_layout(const SvlfModel& m) {
    const size_t V = m.octree.vertex_count();
    if (!m.octree.handle()) throw std::invalid_argument("model has no octree");
    if (m.feat_thickness.dim != kThicknessFeatDim || m.feat_color.dim != kColorFeatDim ||
        m.feat_thickness.data.size() != V * kThicknessFeatDim || m.feat_color.data.size() != V * kColorFeatDim)
        throw std::invalid_argument("feature volumes do not match the octree");
    if (m.dec_thickness.param_count() != SVLF_DEC_T_SIZE || m.dec_color.param_count() != SVLF_DEC_C_SIZE)
        throw std::invalid_argument("decoder shapes differ from f_T 134-128-2 / f_C 38-128-128-128-3");
}

// 64-bit fingerprint of a byte range (multiply-xorshift over 8-byte words)
uint64_t fold(uint64_t h, const void* p, size_t bytes) {
    const auto* b = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = (h ^ w) * 0x9e3779b97f4a7c15ULL;
        h ^= h >> 29;
    }
    for (; i < bytes; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
    return h ^ bytes;
}

template <typename V>
uint64_t fold_vec(uint64_t h, const V& v) {
    return fold(h, v.data(), v.size() * sizeof(typename V::value_type));
}

uint64_t fingerprint(const SvlfModel& m) {
    uint64_t h = 0x243f6a8885a308d3ULL;
    h = fold_vec(h, m.feat_thickness.data);
    h = fold_vec(h, m.feat_color.data);
    for (const auto* d : {&m.dec_thickness, &m.dec_color})
        for (size_t l = 0; l < d->weights.size(); ++l) h = fold_vec(fold_vec(h, d->weights[l]), d->biases[l]);
    return h;
}

// ModelAdam tensor order of the library: feat_t, feat_c, f_T [W,b]..., f_C [W,b]...
std::vector<const AdamState*> adam_tensors(const ModelAdam& a) {
    std::vector<const AdamState*> v{&a.feat_thickness, &a.feat_color};
    for (const auto& s : a.dec_thickness) v.push_back(&s);
    for (const auto& s : a.dec_color) v.push_back(&s);
    return v;
}

uint64_t fingerprint(const ModelAdam& a) {
    uint64_t h = 0x13198a2e03707344ULL;
    for (const AdamState* s : adam_tensors(a)) {
        h = fold_vec(fold_vec(h, s->m), s->v);
        h = fold(h, &s->step, 8);
        h = fold(fold(fold(h, &s->beta1, 4), &s->beta2, 4), &s->eps, 4);
    }
    return h;
}

void upload_params(svlf_model* dm, const SvlfModel& m) {
    const auto dt = flat_of(m.dec_thickness), dc = flat_of(m.dec_color);
    detail::check(svlf_model_set_params(dm, m.feat_thickness.data.data(), m.feat_color.data.data(), dt.data(),
                                        dc.data()));
}

void download_params(svlf_model* dm, SvlfModel& m) {
    const size_t V = m.octree.vertex_count();
    m.feat_thickness.dim = kThicknessFeatDim;
    m.feat_color.dim = kColorFeatDim;
    m.feat_thickness.data.resize(V * kThicknessFeatDim);
    m.feat_color.data.resize(V * kColorFeatDim);
    m.feat_thickness.grad.assign(m.feat_thickness.data.size(), 0.f);
    m.feat_color.grad.assign(m.feat_color.data.size(), 0.f);
    std::vector<float> dt(SVLF_DEC_T_SIZE), dc(SVLF_DEC_C_SIZE);
    detail::check(svlf_model_get_params(dm, m.feat_thickness.data.data(), m.feat_color.data.data(), dt.data(),
                                        dc.data()));
    m.dec_thickness = shaped(MlpSpec::thickness_decoder(kThicknessFeatDim), dt.data());
    m.dec_color = shaped(MlpSpec::color_decoder(kColorFeatDim), dc.data());
}

void upload_adam(svlf_model* dm, const ModelAdam& a, size_t total) {
    const auto ts = adam_tensors(a);
    if (ts.size() != 14) throw std::invalid_argument("ModelAdam does not match the model");
    std::vector<float> m, v;
    m.reserve(total);
    v.reserve(total);
    uint64_t steps[14];
    float b1[14], b2[14], eps[14];
    for (size_t i = 0; i < 14; ++i) {
        m.insert(m.end(), ts[i]->m.begin(), ts[i]->m.end());
        v.insert(v.end(), ts[i]->v.begin(), ts[i]->v.end());
        steps[i] = ts[i]->step;
        b1[i] = ts[i]->beta1;
        b2[i] = ts[i]->beta2;
        eps[i] = ts[i]->eps;
    }
    if (m.size() != total || v.size() != total) throw std::invalid_argument("ModelAdam does not match the model");
    detail::check(svlf_model_set_adam(dm, m.data(), v.data(), steps));
    detail::check(svlf_model_set_adam_hyper(dm, b1, b2, eps));
}

void download_adam(svlf_model* dm, const SvlfModel& model, ModelAdam& a) {
    const size_t total = svlf_model_param_count(dm);
    std::vector<float> m(total), v(total);
    uint64_t steps[14];
    float b1[14], b2[14], eps[14];
    detail::check(svlf_model_get_adam(dm, m.data(), v.data(), steps));
    detail::check(svlf_model_get_adam_hyper(dm, b1, b2, eps));
    a = ModelAdam::like(model);
    std::vector<AdamState*> ts{&a.feat_thickness, &a.feat_color};
    for (auto& s : a.dec_thickness) ts.push_back(&s);
    for (auto& s : a.dec_color) ts.push_back(&s);
    size_t off = 0;
    for (size_t i = 0; i < ts.size(); ++i) {
        const size_t n = ts[i]->m.size();
        std::copy_n(m.begin() + off, n, ts[i]->m.begin());
        std::copy_n(v.begin() + off, n, ts[i]->v.begin());
        ts[i]->step = steps[i];
        ts[i]->beta1 = b1[i];
        ts[i]->beta2 = b2[i];
        ts[i]->eps = eps[i];
        off += n;
    }
}

// ---- device-model cache for the drop-in (host-model) entry points ---------
struct CacheEntry {
    const void* key = nullptr;
    std::shared_ptr<void> octree_owner;  // keeps the octree alive while cached
    svlf_octree* octree = nullptr;
    svlf_model* dm = nullptr;
    uint64_t params_fp = 0;
    bool params_valid = false;
    uint64_t adam_fp = 0;
    bool adam_valid = false;
    ~CacheEntry() {
        if (dm) svlf_model_destroy(dm);
    }
};

std::list<CacheEntry>& cache() {
    static auto* c = new std::list<CacheEntry>();
    return *c;
}
constexpr size_t kCacheSlots = 4;

CacheEntry& entry_for(const SvlfModel& m) {
    require_layout(m);
    auto& c = cache();
    for (auto it = c.begin(); it != c.end(); ++it)
        if (it->key == &m) {
            if (it->octree != m.octree.handle()) {
                c.erase(it);
                break;
            }
            c.splice(c.begin(), c, it);  // most recently used first
            return c.front();
        }
    while (c.size() >= kCacheSlots) c.pop_back();
    c.emplace_front();
    CacheEntry& e = c.front();
    e.key = &m;
    e.octree = m.octree.handle();
    e.octree_owner = std::make_shared<SparseOctree>(m.octree);
    detail::check(svlf_model_create(b200::session_context(), e.octree, &e.dm));
    return e;
}

CacheEntry& device_params(const SvlfModel& m) {
    CacheEntry& e = entry_for(m);
    const uint64_t fp = fingerprint(m);
    if (!e.params_valid || fp != e.params_fp) {
        upload_params(e.dm, m);
        e.params_fp = fp;
        e.params_valid = true;
    }
    return e;
}

svlf_camera to_c(const Camera& c) {
    svlf_camera r{};
    r.fx = c.fx;
    r.fy = c.fy;
    r.cx = c.cx;
    r.cy = c.cy;
    std::copy(c.camera_to_world.begin(), c.camera_to_world.end(), r.camera_to_world);
    r.width = c.width;
    r.height = c.height;
    return r;
}

void add(RenderStats* s, const svlf_render_stats& r) {
    if (!s) return;
    s->rays += r.rays;
    s->rays_with_hits += r.rays_with_hits;
    s->traversal_hits += r.traversal_hits;
    s->thickness_queries += r.thickness_queries;
    s->color_queries += r.color_queries;
}

void render_with(svlf_model* dm, const Camera& camera, FrameBuffers& out, RenderStats* stats, const float* bg,
                 svlf_precision prec) {
    if (camera.width == 0 || camera.height == 0) throw std::invalid_argument("zero-size image");
    out.resize(camera.width, camera.height);
    const svlf_camera c = to_c(camera);
    svlf_render_stats st{};
    detail::check(svlf_render_frame(b200::session_context(), dm, &c, bg, prec, out.rgb.data(), out.alpha.data(),
                                    out.depth.data(), &st));
    add(stats, st);
}

struct PackedBatch {
    std::vector<double> rays, depth;
    std::vector<float> c_gt;
    std::vector<uint8_t> alpha;
    explicit PackedBatch(std::span<const RaySupervision> b)
        : rays(b.size() * 6), depth(b.size()), c_gt(b.size() * 3), alpha(b.size()) {
        for (size_t i = 0; i < b.size(); ++i) {
            const Ray& r = b[i].ray;
            const double v[6] = {r.origin.x, r.origin.y, r.origin.z, r.dir.x, r.dir.y, r.dir.z};
            std::copy(v, v + 6, rays.begin() + 6 * i);
            std::copy(b[i].c_gt, b[i].c_gt + 3, c_gt.begin() + 3 * i);
            depth[i] = b[i].depth_gt;
            alpha[i] = b[i].alpha_gt ? 1 : 0;
        }
    }
};

svlf_loss_weights to_c(const LossWeights& w) { return svlf_loss_weights{w.eta, w.tau, w.empty, w.alpha}; }

void add(LossStats* s, const svlf_loss_stats& r) {
    if (!s) return;
    s->rays += r.rays;
    s->skipped_rays += r.skipped_rays;
    s->eta_skipped += r.eta_skipped;
}

double step_with(svlf_model* dm, std::span<const RaySupervision> batch, LossMode mode, bool frozen, float lr,
                 const LossWeights& lw, LossStats* stats) {
    const PackedBatch p(batch);
    const svlf_loss_weights w = to_c(lw);
    svlf_loss_stats st{};
    double loss = 0;
    detail::check(svlf_train_step(b200::session_context(), dm, p.rays.data(), p.c_gt.data(), p.depth.data(),
                                  p.alpha.data(), batch.size(),
                                  mode == LossMode::Surface ? SVLF_LOSS_SURFACE : SVLF_LOSS_VOLUMETRIC, frozen ? 1 : 0,
                                  lr, &w, &st, &loss));
    add(stats, st);
    return loss;
}

}  // namespace

// ---- model -----------------------------------------------------------------
SvlfModel init_model(SparseOctree octree, uint64_t seed) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    if (!octree.handle()) throw std::invalid_argument("init_model: empty octree");
    svlf_model* dm = nullptr;
    detail::check(svlf_model_create(b200::session_context(), octree.handle(), &dm));
    SvlfModel m;
    m.octree = std::move(octree);
    try {
        detail::check(svlf_model_init(dm, seed));
        download_params(dm, m);
    } catch (...) {
        svlf_model_destroy(dm);
        throw;
    }
    svlf_model_destroy(dm);
    return m;
}

ModelAdam ModelAdam::like(const SvlfModel& m) {
    ModelAdam a;
    a.feat_thickness = AdamState::like(m.feat_thickness.data.size());
    a.feat_color = AdamState::like(m.feat_color.data.size());
    for (size_t l = 0; l < m.dec_thickness.weights.size(); ++l) {
        a.dec_thickness.push_back(AdamState::like(m.dec_thickness.weights[l].size()));
        a.dec_thickness.push_back(AdamState::like(m.dec_thickness.biases[l].size()));
    }
    for (size_t l = 0; l < m.dec_color.weights.size(); ++l) {
        a.dec_color.push_back(AdamState::like(m.dec_color.weights[l].size()));
        a.dec_color.push_back(AdamState::like(m.dec_color.biases[l].size()));
    }
    return a;
}

svlf_model* detail::device_model(const SvlfModel& m) { return device_params(m).dm; }

// ---- render ----------------------------------------------------------------
void render_frame(const SvlfModel& model, const Camera& camera, FrameBuffers& out, RenderStats* stats,
                  const float* background) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    render_with(device_params(model).dm, camera, out, stats, background, detail::to_c(b200::render_precision()));
}

void render_frame_ref(const SvlfModel& model, const Camera& camera, FrameBuffers& out, RenderStats* stats,
                      const float* background) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    render_with(device_params(model).dm, camera, out, stats, background, SVLF_PRECISION_FP32);
}

void render_rays(const SvlfModel& model, std::span<const Ray> rays, std::vector<float>& rgb,
                 std::vector<float>& alpha, std::vector<float>& depth, RenderStats* stats, const float* background) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const size_t n = rays.size();
    std::vector<double> r6(n * 6);
    for (size_t i = 0; i < n; ++i) {
        const double v[6] = {rays[i].origin.x, rays[i].origin.y, rays[i].origin.z,
                             rays[i].dir.x,    rays[i].dir.y,    rays[i].dir.z};
        std::copy(v, v + 6, r6.begin() + 6 * i);
    }
    rgb.assign(n * 3, 0.f);
    alpha.assign(n, 0.f);
    depth.assign(n, 0.f);
    svlf_render_stats st{};
    detail::check(svlf_render_rays(b200::session_context(), device_params(model).dm, r6.data(), n, background,
                                   detail::to_c(b200::render_precision()), rgb.data(), alpha.data(), depth.data(),
                                   &st));
    add(stats, st);
}

// ---- train -----------------------------------------------------------------
double train_step(SvlfModel& model, ModelAdam& adam, std::span<const RaySupervision> batch, LossMode mode,
                  bool color_frozen, float lr, const LossWeights& lw, LossStats* stats) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    CacheEntry& e = device_params(model);
    const uint64_t afp = fingerprint(adam);
    if (!e.adam_valid || afp != e.adam_fp) upload_adam(e.dm, adam, svlf_model_param_count(e.dm));
    e.adam_valid = false;
    e.params_valid = false;
    const double loss = step_with(e.dm, batch, mode, color_frozen, lr, lw, stats);
    // the reference mutates the host model and optimizer state: copy back
    download_params(e.dm, model);
    download_adam(e.dm, model, adam);
    e.params_fp = fingerprint(model);
    e.params_valid = true;
    e.adam_fp = fingerprint(adam);
    e.adam_valid = true;
    return loss;
}

double loss_grads(const SvlfModel& model, std::span<const RaySupervision> batch, LossMode mode, bool color_frozen,
                  const LossWeights& lw, ModelGrads* grads, LossStats* stats) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    CacheEntry& e = device_params(model);
    const PackedBatch p(batch);
    const svlf_loss_weights w = to_c(lw);
    svlf_loss_stats st{};
    double loss = 0;
    detail::check(svlf_loss_grads(b200::session_context(), e.dm, p.rays.data(), p.c_gt.data(), p.depth.data(),
                                  p.alpha.data(), batch.size(),
                                  mode == LossMode::Surface ? SVLF_LOSS_SURFACE : SVLF_LOSS_VOLUMETRIC,
                                  color_frozen ? 1 : 0, &w, &st, &loss));
    add(stats, st);
    if (grads) {
        if (grads->feat_thickness.empty()) *grads = ModelGrads::like(model);
        std::vector<float> ft(model.feat_thickness.data.size()), fc(model.feat_color.data.size());
        std::vector<float> dt(SVLF_DEC_T_SIZE), dc(SVLF_DEC_C_SIZE);
        detail::check(svlf_model_get_grads(e.dm, ft.data(), fc.data(), dt.data(), dc.data()));
        ModelGrads g;
        g.feat_thickness = std::move(ft);
        g.feat_color = std::move(fc);
        const MlpParams st_ = shaped(MlpSpec::thickness_decoder(kThicknessFeatDim), dt.data());
        const MlpParams sc_ = shaped(MlpSpec::color_decoder(kColorFeatDim), dc.data());
        g.dec_thickness.weights = st_.weights;
        g.dec_thickness.biases = st_.biases;
        g.dec_color.weights = sc_.weights;
        g.dec_color.biases = sc_.biases;
        grads->add(g);
    }
    return loss;
}

// ---- checkpoints (container of src/model.cpp:182-235) -----------------------
namespace {

constexpr char kMagic[8] = {'S', 'V', 'L', 'F', '0', '0', '0', '1'};

class Sink {
  public:
    explicit Sink(const std::string& path) : f_(path, std::ios::binary), path_(path) {
        if (!f_) throw std::runtime_error("cannot open checkpoint for writing: " + path);
    }
    template <typename T>
    void pod(T v) {
        f_.write(reinterpret_cast<const char*>(&v), sizeof(T));
    }
    template <typename T>
    void vec(const std::vector<T>& v) {
        pod<uint64_t>(v.size());
        f_.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(T)));
    }
    void raw(const char* p, size_t n) { f_.write(p, std::streamsize(n)); }
    void finish() {
        f_.flush();
        if (!f_) throw std::runtime_error("checkpoint write failed: " + path_);
    }

  private:
    std::ofstream f_;
    std::string path_;
};

class Source {
  public:
    explicit Source(const std::string& path) : f_(path, std::ios::binary) {
        if (!f_) throw std::runtime_error("cannot open checkpoint: " + path);
    }
    void raw(char* p, size_t n) {
        f_.read(p, std::streamsize(n));
        if (!f_) throw std::runtime_error("truncated checkpoint");
    }
    template <typename T>
    T pod() {
        T v;
        raw(reinterpret_cast<char*>(&v), sizeof(T));
        return v;
    }
    template <typename T>
    std::vector<T> vec() {
        const uint64_t n = pod<uint64_t>();
        if (n > (uint64_t(1) << 40) / sizeof(T)) throw std::runtime_error("truncated checkpoint");
        std::vector<T> v(n);
        raw(reinterpret_cast<char*>(v.data()), n * sizeof(T));
        return v;
    }

  private:
    std::ifstream f_;
};

void put(Sink& s, const MlpParams& p) {
    for (uint32_t d : {p.spec.input_dim, p.spec.hidden_dim, p.spec.hidden_layers, p.spec.output_dim}) s.pod(d);
    for (Activation a : p.spec.head) s.pod(uint32_t(a));
    for (size_t l = 0; l < p.weights.size(); ++l) {
        s.vec(p.weights[l]);
        s.vec(p.biases[l]);
    }
}

MlpParams get_mlp(Source& s) {
    MlpParams p;
    p.spec.input_dim = s.pod<uint32_t>();
    p.spec.hidden_dim = s.pod<uint32_t>();
    p.spec.hidden_layers = s.pod<uint32_t>();
    p.spec.output_dim = s.pod<uint32_t>();
    p.spec.head.resize(p.spec.output_dim);
    for (auto& a : p.spec.head) a = Activation(s.pod<uint32_t>());
    for (uint32_t l = 0; l < p.spec.layer_count(); ++l) {
        p.weights.push_back(s.vec<float>());
        p.biases.push_back(s.vec<float>());
    }
    return p;
}

void put(Sink& s, const AdamState& a) {
    s.pod(a.step);
    s.pod(a.beta1);
    s.pod(a.beta2);
    s.pod(a.eps);
    s.vec(a.m);
    s.vec(a.v);
}

AdamState get_adam(Source& s) {
    AdamState a;
    a.step = s.pod<uint64_t>();
    a.beta1 = s.pod<float>();
    a.beta2 = s.pod<float>();
    a.eps = s.pod<float>();
    a.m = s.vec<float>();
    a.v = s.vec<float>();
    return a;
}

FeatureVolume get_features(Source& s) {
    FeatureVolume f;
    f.dim = s.pod<uint32_t>();
    f.data = s.vec<float>();
    f.grad.assign(f.data.size(), 0.f);
    return f;
}

}  // namespace

void save_checkpoint(const std::string& path, const SvlfModel& model, const ModelAdam& adam) {
    Sink s(path);
    s.raw(kMagic, 8);
    const GridConfig& g = model.octree.config();
    s.pod(g.resolution);
    s.pod(g.dilation);
    for (const Vec3* v : {&g.scene_aabb.lo, &g.scene_aabb.hi})
        for (int a = 0; a < 3; ++a) s.pod((*v)[a]);
    s.vec(model.octree.leaf_codes());
    for (const FeatureVolume* f : {&model.feat_thickness, &model.feat_color}) {
        s.pod(f->dim);
        s.vec(f->data);
    }
    put(s, model.dec_thickness);
    put(s, model.dec_color);
    put(s, adam.feat_thickness);
    put(s, adam.feat_color);
    for (const auto* group : {&adam.dec_thickness, &adam.dec_color}) {
        s.pod(uint32_t(group->size()));
        for (const AdamState& a : *group) put(s, a);
    }
    s.finish();
}

void load_checkpoint(const std::string& path, SvlfModel& model, ModelAdam& adam) {
    Source s(path);
    char magic[8];
    s.raw(magic, 8);
    if (std::memcmp(magic, kMagic, 8) != 0) throw std::runtime_error("bad checkpoint magic");
    GridConfig g;
    g.resolution = s.pod<uint32_t>();
    g.dilation = s.pod<uint32_t>();
    double b[6];
    for (double& x : b) x = s.pod<double>();
    g.scene_aabb = Aabb{Vec3(b[0], b[1], b[2]), Vec3(b[3], b[4], b[5])};
    model.octree = SparseOctree::from_leaves(s.vec<uint64_t>(), g);
    model.feat_thickness = get_features(s);
    model.feat_color = get_features(s);
    model.dec_thickness = get_mlp(s);
    model.dec_color = get_mlp(s);
    adam.feat_thickness = get_adam(s);
    adam.feat_color = get_adam(s);
    for (auto* group : {&adam.dec_thickness, &adam.dec_color}) {
        group->resize(s.pod<uint32_t>());
        for (AdamState& a : *group) a = get_adam(s);
    }
}

// ---- DeviceModel (explicit fast path) ---------------------------------------
namespace b200 {

DeviceModel::DeviceModel(const SvlfModel& model) : octree_(model.octree) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    require_layout(model);
    detail::check(svlf_model_create(session_context(), octree_.handle(), &m_));
    upload(model);
}

DeviceModel::DeviceModel(const SvlfModel& model, const ModelAdam& adam) : DeviceModel(model) { upload(adam); }

// a staged batch: its packed host arrays stay alive until the slot is stepped
struct DeviceModel::StagedBatch {
    PackedBatch batch;
    size_t n;
    int slot = 0;
    explicit StagedBatch(std::span<const RaySupervision> b) : batch(b), n(b.size()) {}
};

DeviceModel::~DeviceModel() {
    for (auto& sb : staged_) svlf_train_batch_discard(session_context(), sb->slot);
    if (m_) svlf_model_destroy(m_);
}

void DeviceModel::stage_batch(std::span<const RaySupervision> batch) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    auto sb = std::make_unique<StagedBatch>(batch);
    detail::check(svlf_train_batch_stage(session_context(), sb->batch.rays.data(), sb->batch.c_gt.data(),
                                         sb->batch.depth.data(), sb->batch.alpha.data(), sb->n, &sb->slot));
    staged_.push_back(std::move(sb));
}

double DeviceModel::train_staged(LossMode mode, bool color_frozen, float lr, const LossWeights& lw,
                                 LossStats* stats) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    if (staged_.empty()) throw std::logic_error("no batch staged");
    const std::unique_ptr<StagedBatch> sb = std::move(staged_.front());
    staged_.pop_front();
    const svlf_loss_weights w = to_c(lw);
    svlf_loss_stats st{};
    double loss = 0;
    detail::check(svlf_train_step_staged(session_context(), m_, sb->slot,
                                         mode == LossMode::Surface ? SVLF_LOSS_SURFACE : SVLF_LOSS_VOLUMETRIC,
                                         color_frozen ? 1 : 0, lr, &w, &st, &loss));
    add(stats, st);
    return loss;
}

void DeviceModel::upload(const SvlfModel& model) {
    if (model.octree.handle() != octree_.handle()) throw std::invalid_argument("model belongs to another octree");
    require_layout(model);
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    upload_params(m_, model);
}

void DeviceModel::upload(const ModelAdam& adam) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    upload_adam(m_, adam, svlf_model_param_count(m_));
}

void DeviceModel::sync_to(SvlfModel& model) const {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    model.octree = octree_;
    download_params(m_, model);
}

void DeviceModel::sync_to(ModelAdam& adam) const {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    SvlfModel shape;
    shape.octree = octree_;
    shape.feat_thickness.data.resize(size_t(octree_.vertex_count()) * kThicknessFeatDim);
    shape.feat_color.data.resize(size_t(octree_.vertex_count()) * kColorFeatDim);
    std::vector<float> dt(SVLF_DEC_T_SIZE), dc(SVLF_DEC_C_SIZE);
    shape.dec_thickness = shaped(MlpSpec::thickness_decoder(kThicknessFeatDim), dt.data());
    shape.dec_color = shaped(MlpSpec::color_decoder(kColorFeatDim), dc.data());
    download_adam(m_, shape, adam);
}

void DeviceModel::render(const Camera& camera, FrameBuffers& out, RenderStats* stats, const float* bg) const {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    render_with(m_, camera, out, stats, bg, detail::to_c(render_precision()));
}

void DeviceModel::render_ref(const Camera& camera, FrameBuffers& out, RenderStats* stats, const float* bg) const {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    render_with(m_, camera, out, stats, bg, SVLF_PRECISION_FP32);
}

double DeviceModel::train_step(std::span<const RaySupervision> batch, LossMode mode, bool color_frozen, float lr,
                               const LossWeights& lw, LossStats* stats) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    return step_with(m_, batch, mode, color_frozen, lr, lw, stats);
}

}  // namespace b200
}  // namespace svlf
