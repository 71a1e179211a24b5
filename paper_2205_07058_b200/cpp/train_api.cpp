// C++ API: the training stage driver (include/svlf/train.hpp: train()), PSNR
// and PFMX I/O (include/svlf/{metrics,image}.hpp).
//
// Reference: train() src/train.cpp:364-527, make_supervision :334-343,
// TrainConfig::validate :22-28, psnr src/metrics.cpp:57-68, PFMX
// src/image.cpp:108-132. Every optimizer step is svlf_train_step on the GPU
// (through b200::DeviceModel, device copy authoritative); the host side is the
// reference's control flow: views, shuffle, logging, checkpoints.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <stdexcept>

#include "svlf/b200.hpp"
#include "svlf/metrics.hpp"
#include "svlf/rng.hpp"
#include "svlf/train.hpp"

namespace svlf {

void TrainConfig::validate() const {
    if (epochs[0] < 0 || epochs[1] < 0 || epochs[2] < 0) throw std::invalid_argument("epochs must be >= 0");
    if (lr_main <= 0 || lr_finetune <= 0) throw std::invalid_argument("learning rates must be > 0");
    if (lambda_eta < 0 || lambda_tau < 0 || lambda_empty < 0 || lambda_alpha < 0)
        throw std::invalid_argument("loss weights must be >= 0");
}

double psnr(const Image& pred, const Image& gt) {
    if (pred.width != gt.width || pred.height != gt.height || pred.channels != gt.channels ||
        pred.px.size() != gt.px.size())
        throw std::invalid_argument("image shapes differ");
    if (pred.px.empty()) throw std::invalid_argument("empty image");
    double se = 0;
    for (size_t i = 0; i < pred.px.size(); ++i) {
        const double d = double(pred.px[i]) - double(gt.px[i]);
        se += d * d;
    }
    const double mse = se / double(pred.px.size());
    if (mse == 0.0) return kPsnrCap;
    return std::min(kPsnrCap, 10.0 * std::log10(1.0 / mse));
}

void write_pfmx(const std::string& path, const Image& img) {
    if (img.channels != 1) throw std::invalid_argument("pfmx stores single-channel data");
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open for writing: " + path);
    const uint32_t head[3] = {img.width, img.height, 0};
    f.write("PFMX", 4);
    f.write(reinterpret_cast<const char*>(head), sizeof head);
    f.write(reinterpret_cast<const char*>(img.px.data()), std::streamsize(img.px.size() * 4));
    if (!f) throw std::runtime_error("pfmx write failed: " + path);
}

Image read_pfmx(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open: " + path);
    char magic[4];
    uint32_t head[3];
    if (!f.read(magic, 4) || std::memcmp(magic, "PFMX", 4) != 0) throw std::runtime_error("bad pfmx magic in " + path);
    if (!f.read(reinterpret_cast<char*>(head), sizeof head)) throw std::runtime_error("truncated pfmx header");
    Image img = Image::make(head[0], head[1], 1);
    if (!f.read(reinterpret_cast<char*>(img.px.data()), std::streamsize(img.px.size() * 4)))
        throw std::runtime_error("truncated pfmx data in " + path);
    return img;
}

namespace {

// supervision rays of one view (src/train.cpp:334-343, :443-448)
void view_batch(const DatasetFrame& f, bool foreground_only, std::vector<RaySupervision>& out) {
    out.clear();
    for (uint32_t y = 0; y < f.rgb.height; ++y)
        for (uint32_t x = 0; x < f.rgb.width; ++x) {
            if (foreground_only && f.mask.at(x, y) <= 0.5f) continue;
            RaySupervision s;
            s.ray = f.camera.pixel_ray(x, y);
            for (int c = 0; c < 3; ++c) s.c_gt[c] = f.rgb.at(x, y, c);
            s.depth_gt = f.depth.at(x, y);
            s.alpha_gt = f.mask.at(x, y) > 0.5f;
            out.push_back(s);
        }
}

}  // namespace

TrainResult train(const TrainConfig& config, const SceneDataset& dataset) {
    namespace fs = std::filesystem;
    config.validate();
    if (config.train_res != 0 && (config.train_res != dataset.width || config.train_res != dataset.height))
        throw std::invalid_argument("train_res must match the dataset resolution (no resampling)");
    const auto train_idx = dataset.split_indices("train");
    const auto val_idx = dataset.split_indices("val");
    if (train_idx.empty()) throw std::invalid_argument("dataset has no training frames");

    // occupancy: back-projected foreground depth of every training view
    std::vector<Vec3> points;
    for (size_t fi : train_idx) {
        const DatasetFrame& fr = dataset.frames[fi];
        for (uint32_t y = 0; y < fr.depth.height; ++y)
            for (uint32_t x = 0; x < fr.depth.width; ++x) {
                const float d = fr.depth.at(x, y);
                if (d <= 0.f) continue;
                points.push_back(fr.camera.pixel_ray(x, y).at(d));
            }
    }
    GridConfig grid;
    grid.resolution = config.grid_resolution;
    grid.dilation = config.dilation;
    SparseOctree octree = SparseOctree::build(points, grid);

    TrainResult result;
    result.dropped_points = static_cast<long long>(octree.dropped_points());
    result.model = init_model(std::move(octree), config.seed);
    result.adam = ModelAdam::like(result.model);
    result.stage_lrs = {config.lr_main, config.lr_main, config.lr_finetune};
    const LossWeights lw{config.lambda_eta, config.lambda_tau, config.lambda_empty, config.lambda_alpha};
    b200::DeviceModel dev(result.model, result.adam);

    std::ofstream log_file;
    if (!config.out_dir.empty()) {
        fs::create_directories(config.out_dir);
        log_file.open(fs::path(config.out_dir) / "train.log");
    }
    auto save_stage = [&](int stage_num, const std::string& name) {
        if (config.out_dir.empty()) return std::string();
        dev.sync_to(result.model);
        dev.sync_to(result.adam);
        const std::string path = (fs::path(config.out_dir) / name).string();
        save_checkpoint(path, result.model, result.adam);
        if (stage_num >= 0) result.checkpoints[size_t(stage_num)] = path;
        return path;
    };

    std::vector<RaySupervision> sups;
    LossStats stats_total;
    int global_epoch = 0;
    for (int stage = 0; stage < 3 && !result.diverged; ++stage) {
        const LossMode mode = stage == 0 ? LossMode::Surface : LossMode::Volumetric;
        const bool frozen = stage == 1;
        const float lr = static_cast<float>(result.stage_lrs[size_t(stage)]);
        for (int epoch = 1; epoch <= config.epochs[size_t(stage)]; ++epoch, ++global_epoch) {
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<size_t> order(train_idx);
            Rng shuffle = Rng(config.seed).sub(kStreamEpochShuffle).sub(uint64_t(global_epoch) + 1);
            for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[shuffle.below(i)]);

            double loss_sum = 0.0;
            long long ray_count = 0;
            // frame k + 1's batch uploads (copy stream) while frame k's step runs
            auto stage_frame = [&](size_t k) {
                view_batch(dataset.frames[order[k]], mode == LossMode::Surface, sups);
                dev.stage_batch(sups);
                ray_count += static_cast<long long>(sups.size());
            };
            if (!order.empty()) stage_frame(0);
            for (size_t k = 0; k < order.size(); ++k) {
                if (k + 1 < order.size()) stage_frame(k + 1);
                loss_sum += dev.train_staged(mode, frozen, lr, lw, &stats_total);
            }
            const double mean_loss = ray_count > 0 ? loss_sum / double(ray_count) : 0.0;
            if (!std::isfinite(mean_loss)) {
                result.diverged = true;
                save_stage(-1, "checkpoint_diverged.svlf");
                break;
            }
            double val_psnr = 0.0;
            if (!val_idx.empty()) {
                FrameBuffers fb;
                for (size_t vi : val_idx) {
                    const DatasetFrame& fr = dataset.frames[vi];
                    dev.render_ref(fr.camera, fb);
                    Image rendered;
                    rendered.width = fb.width;
                    rendered.height = fb.height;
                    rendered.channels = 3;
                    rendered.px = fb.rgb;
                    val_psnr += psnr(rendered, fr.rgb);
                }
                val_psnr /= double(val_idx.size());
            }
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            result.log.push_back({stage + 1, epoch, mean_loss, val_psnr, secs});
            if (log_file) {
                char line[160];
                std::snprintf(line, sizeof line, "%d\t%d\t%.8f\t%.4f\t%.3f\n", stage + 1, epoch, mean_loss, val_psnr,
                              secs);
                log_file << line;
                log_file.flush();
            }
        }
        save_stage(stage, "checkpoint_stage" + std::to_string(stage + 1) + ".svlf");
    }
    result.skipped_rays = stats_total.skipped_rays;
    if (!result.diverged) result.checkpoints[3] = save_stage(3, "checkpoint_final.svlf");
    dev.sync_to(result.model);
    dev.sync_to(result.adam);
    return result;
}

}  // namespace svlf
