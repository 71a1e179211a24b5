// svlf/mlp.hpp — decoder specs, parameter tensors and Adam state (reference
// include/svlf/mlp.hpp:32-128). The forward/backward kernels are the B200
// library's (tcgen05 / CUDA-core decoders, csrc/decode_tc.cu, csrc/train.cu);
// this header carries the host tensors in the reference's layout:
// per layer W row-major [out][in], then b.
#pragma once

#include <cstdint>
#include <vector>

namespace svlf {

enum class Activation : uint8_t { Relu = 0, Sigmoid = 1 };

struct MlpSpec {
    uint32_t input_dim = 0;
    uint32_t hidden_dim = 128;
    uint32_t hidden_layers = 1;
    uint32_t output_dim = 0;
    std::vector<Activation> head;  // per output unit

    uint32_t layer_count() const { return hidden_layers + 1; }
    uint32_t layer_in(uint32_t l) const { return l ? hidden_dim : input_dim; }
    uint32_t layer_out(uint32_t l) const { return l == hidden_layers ? output_dim : hidden_dim; }
    void validate() const;

    static MlpSpec thickness_decoder(uint32_t feat_dim = 64, uint32_t hidden = 128);  // 6+2F -> H -> (relu, sigmoid)
    static MlpSpec color_decoder(uint32_t feat_dim = 32, uint32_t hidden = 128);      // 6+F -> H,H,H -> 3 sigmoid
};

template <typename T>
struct MlpParamsT {
    MlpSpec spec;
    std::vector<std::vector<T>> weights;  // [layer] row-major [out][in]
    std::vector<std::vector<T>> biases;   // [layer][out]

    size_t param_count() const {
        size_t n = 0;
        for (size_t l = 0; l < weights.size(); ++l) n += weights[l].size() + biases[l].size();
        return n;
    }
    template <typename U>
    static MlpParamsT from(const MlpParamsT<U>& o) {
        MlpParamsT r;
        r.spec = o.spec;
        for (const auto& w : o.weights) r.weights.emplace_back(w.begin(), w.end());
        for (const auto& b : o.biases) r.biases.emplace_back(b.begin(), b.end());
        return r;
    }
};

template <typename T>
struct MlpGradsT {
    std::vector<std::vector<T>> weights, biases;

    static MlpGradsT like(const MlpParamsT<T>& p) {
        MlpGradsT g;
        for (const auto& w : p.weights) g.weights.emplace_back(w.size(), T(0));
        for (const auto& b : p.biases) g.biases.emplace_back(b.size(), T(0));
        return g;
    }
    void clear() {
        for (auto& w : weights) std::fill(w.begin(), w.end(), T(0));
        for (auto& b : biases) std::fill(b.begin(), b.end(), T(0));
    }
    void add(const MlpGradsT& o) {
        for (size_t l = 0; l < weights.size(); ++l) {
            for (size_t i = 0; i < weights[l].size(); ++i) weights[l][i] += o.weights[l][i];
            for (size_t i = 0; i < biases[l].size(); ++i) biases[l][i] += o.biases[l][i];
        }
    }
};

using MlpParams = MlpParamsT<float>;
using MlpGrads = MlpGradsT<float>;

struct AdamState {
    std::vector<float> m, v;
    uint64_t step = 0;
    float beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f;

    static AdamState like(size_t n) {
        AdamState s;
        s.m.assign(n, 0.f);
        s.v.assign(n, 0.f);
        return s;
    }
};

}  // namespace svlf
