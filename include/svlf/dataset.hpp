// svlf/dataset.hpp — in-memory training/validation views (reference
// include/svlf/dataset.hpp:11-27). Loading the on-disk layout (PNG + JSON
// manifest) is the reference's tooling and not provided here; callers fill
// SceneDataset directly.
#pragma once

#include <string>
#include <vector>

#include "svlf/camera.hpp"
#include "svlf/image.hpp"

namespace svlf {

struct DatasetFrame {
    std::string name;
    std::string split;  // train | val | test
    Camera camera;
    Image rgb;    // 3 channels
    Image depth;  // 1 channel, Euclidean ray distance, 0 = background
    Image mask;   // 1 channel, 0/1
};

struct SceneDataset {
    uint32_t width = 0, height = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    std::vector<DatasetFrame> frames;

    std::vector<size_t> split_indices(const std::string& split) const {
        std::vector<size_t> idx;
        for (size_t i = 0; i < frames.size(); ++i)
            if (frames[i].split == split) idx.push_back(i);
        return idx;
    }
};

}  // namespace svlf
