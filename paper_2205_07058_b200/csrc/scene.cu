// Ground truth and metrics on the GPU:
//   k_render_gt   generate_dataset's pixel loop (src/dataset.cpp:61-83): the
//                 analytic scene's raycast (closed-form spheres, slab boxes,
//                 src/scene.cpp:56-77) and shade (hard shadow ray, ambient,
//                 clamp, :79-90) per pixel -> rgb, Euclidean depth, mask; fp64
//                 in the reference's operand order (bit-exact with the
//                 reference built without FMA contraction)
//   k_backproject train()'s occupancy (src/train.cpp:376-386): foreground
//                 pixels -> ray.at(double(depth)), compacted with an atomic
//                 cursor (the octree build sorts, so order is irrelevant)
//   k_sq_err      psnr (src/metrics.cpp:57-68) and depth RMSE/MAE over the
//                 gt mask (:115-136): per-block fp64 partial sums in a fixed
//                 order, summed on the host in block order (deterministic)
//   k_ssim_h/_v   ssim (src/metrics.cpp:70-113): separable valid-region
//                 Gaussian in fp64 (horizontal, then vertical + SSIM map and
//                 block partial sums), per channel
#include <cmath>

#include "device.cuh"

namespace svlfb {

namespace {

struct SceneDev {
    const double* spheres;  // 7 per sphere: c xyz, r, albedo rgb
    uint32_t n_spheres;
    const double* boxes;    // 9 per box: lo xyz, hi xyz, albedo rgb
    uint32_t n_boxes;
    double light_dir[3], light_rgb[3], ambient[3], background[3];
};

constexpr double kRayEps = 1e-9;

struct Surf {
    double t;
    double p[3], n[3], alb[3];
};

__device__ bool raycast(const SceneDev& S, const double* o, const double* d, Surf& best) {
    bool have = false;
    for (uint32_t i = 0; i < S.n_spheres; ++i) {
        const double* s = S.spheres + 7 * size_t(i);
        const double oc[3] = {dsub(o[0], s[0]), dsub(o[1], s[1]), dsub(o[2], s[2])};
        const double b = dot3(oc, d);
        const double c = dsub(dot3(oc, oc), dmul(s[3], s[3]));
        const double disc = dsub(dmul(b, b), c);
        if (disc < 0) continue;
        const double sq = __dsqrt_rn(disc);
        double t = dsub(-b, sq);
        if (!(t > kRayEps)) {
            t = dadd(-b, sq);
            if (!(t > kRayEps)) continue;
        }
        if (have && !(t < best.t)) continue;
        have = true;
        best.t = t;
        double v[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            best.p[a] = dadd(o[a], dmul(d[a], t));
            v[a] = dsub(best.p[a], s[a]);
        }
        const double nv = __dsqrt_rn(dot3(v, v));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            best.n[a] = ddiv(v[a], nv);
            best.alb[a] = s[4 + a];
        }
    }
    RayPre pre;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        pre.r.o[a] = o[a];
        pre.r.d[a] = d[a];
        pre.inv[a] = d[a] == 0.0 ? 0.0 : ddiv(1.0, d[a]);
    }
    for (uint32_t i = 0; i < S.n_boxes; ++i) {
        const double* bx = S.boxes + 9 * size_t(i);
        double t0, t1;
        if (!slab_test(pre, bx, bx + 3, t0, t1)) continue;
        const double t = t0 > kRayEps ? t0 : (t1 > kRayEps ? t1 : -1.0);
        if (!(t > 0) || (have && !(t < best.t))) continue;
        have = true;
        best.t = t;
#pragma unroll
        for (int a = 0; a < 3; ++a) best.p[a] = dadd(o[a], dmul(d[a], t));
        // face with the smallest distance to the point, first minimum wins
        const double dist[6] = {dsub(best.p[0], bx[0]), dsub(bx[3], best.p[0]), dsub(best.p[1], bx[1]),
                                dsub(bx[4], best.p[1]), dsub(best.p[2], bx[2]), dsub(bx[5], best.p[2])};
        int k = 0;
        for (int f = 1; f < 6; ++f)
            if (dist[f] < dist[k]) k = f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            best.n[a] = a == k / 2 ? (k & 1 ? 1.0 : -1.0) : 0.0;
            best.alb[a] = bx[6 + a];
        }
    }
    return have;
}

__global__ void k_render_gt(SceneDev S, DevCamera cam, float* rgb, float* depth, float* mask) {
    const uint32_t n = cam.width * cam.height;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const Ray r = pixel_ray(cam, i % cam.width, i / cam.width);
        Surf h;
        if (!raycast(S, r.o, r.d, h)) {
#pragma unroll
            for (int a = 0; a < 3; ++a) rgb[3 * size_t(i) + a] = float(S.background[a]);
            depth[i] = 0.f;
            mask[i] = 0.f;
            continue;
        }
        const double nl[3] = {-S.light_dir[0], -S.light_dir[1], -S.light_dir[2]};
        double direct = fmax(0.0, dot3(h.n, nl));
        if (direct > 0) {
            double so[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) so[a] = dadd(h.p[a], dmul(h.n[a], 1e-6));
            Surf sh;
            if (raycast(S, so, nl, sh)) direct = 0;  // hard shadow
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double c = dmul(h.alb[a], dadd(S.ambient[a], dmul(S.light_rgb[a], direct)));
            rgb[3 * size_t(i) + a] = float(fmin(fmax(c, 0.0), 1.0));
        }
        depth[i] = float(h.t);
        mask[i] = 1.f;
    }
}

__global__ void k_backproject(DevCamera cam, const float* __restrict__ depth, double* pts, unsigned long long cap,
                              unsigned long long* count) {
    const uint32_t n = cam.width * cam.height;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float dv = depth[i];
        if (!(dv > 0.f)) continue;
        const Ray r = pixel_ray(cam, i % cam.width, i / cam.width);
        const unsigned long long k = atomicAdd(count, 1ull);
        if (k >= cap) continue;
        const double t = double(dv);
#pragma unroll
        for (int a = 0; a < 3; ++a) pts[3 * k + a] = dadd(r.o[a], dmul(r.d[a], t));
    }
}

// part[b] = {sum (p-g)^2 over values, depth: sum e^2, sum |e|, count} per block
constexpr int kRedThreads = 256;
__global__ void k_sq_err(const float* __restrict__ pred, const float* __restrict__ gt, size_t n, double* part) {
    __shared__ double sh[kRedThreads];
    double acc = 0.0;
    for (size_t i = blockIdx.x * size_t(kRedThreads) + threadIdx.x; i < n; i += size_t(gridDim.x) * kRedThreads) {
        const double e = dsub(double(pred[i]), double(gt[i]));
        acc = dadd(acc, dmul(e, e));
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (int(threadIdx.x) < s) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_depth_err(const float* __restrict__ pd, const float* __restrict__ gd, const float* __restrict__ gm,
                            size_t n, double* part) {
    __shared__ double s2[kRedThreads], s1[kRedThreads], sc[kRedThreads];
    double a2 = 0.0, a1 = 0.0, c = 0.0;
    for (size_t i = blockIdx.x * size_t(kRedThreads) + threadIdx.x; i < n; i += size_t(gridDim.x) * kRedThreads) {
        if (gm[i] < 0.5f) continue;
        const double e = dsub(double(pd[i]), double(gd[i]));
        a2 = dadd(a2, dmul(e, e));
        a1 = dadd(a1, fabs(e));
        c += 1.0;
    }
    s2[threadIdx.x] = a2;
    s1[threadIdx.x] = a1;
    sc[threadIdx.x] = c;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (int(threadIdx.x) < s) {
            s2[threadIdx.x] = dadd(s2[threadIdx.x], s2[threadIdx.x + s]);
            s1[threadIdx.x] = dadd(s1[threadIdx.x], s1[threadIdx.x + s]);
            sc[threadIdx.x] += sc[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = s2[0];
        part[3 * blockIdx.x + 1] = s1[0];
        part[3 * blockIdx.x + 2] = sc[0];
    }
}

constexpr unsigned kRedBlocks = 296;

// ---- ssim (src/metrics.cpp:70-113): per channel, separable 11-tap Gaussian
// over the valid region in fp64 (horizontal pass, then vertical), the SSIM
// map, and its mean; channels averaged.
constexpr int kSsimWin = 11;
struct Gauss11 {
    double k[kSsimWin];
};

// tmp planes (vw x h each): blur_h of x, y, x^2, y^2, xy
__global__ void k_ssim_h(const float* __restrict__ pred, const float* __restrict__ gt, uint32_t w, uint32_t h,
                         uint32_t channels, uint32_t ch, Gauss11 g, double* __restrict__ tmp) {
    const uint32_t vw = w - kSsimWin + 1;
    const size_t plane = size_t(vw) * h;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < plane; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t x = uint32_t(i % vw), y = uint32_t(i / vw);
        double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < kSsimWin; ++t) {
            const size_t src = (size_t(y) * w + x + t) * channels + ch;
            const double xv = double(pred[src]), yv = double(gt[src]);
            const double v[5] = {xv, yv, dmul(xv, xv), dmul(yv, yv), dmul(xv, yv)};
#pragma unroll
            for (int q = 0; q < 5; ++q) a[q] = dadd(a[q], dmul(g.k[t], v[q]));
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) tmp[q * plane + i] = a[q];
    }
}

__global__ void k_ssim_v(const double* __restrict__ tmp, uint32_t vw, uint32_t h, Gauss11 g, double c1, double c2,
                         double* part) {
    __shared__ double sh[kRedThreads];
    const uint32_t vh = h - kSsimWin + 1;
    const size_t plane = size_t(vw) * h, n = size_t(vw) * vh;
    double acc = 0.0;
    for (size_t i = blockIdx.x * size_t(kRedThreads) + threadIdx.x; i < n; i += size_t(gridDim.x) * kRedThreads) {
        const uint32_t x = uint32_t(i % vw), y = uint32_t(i / vw);
        double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < kSsimWin; ++t) {
            const size_t src = size_t(y + t) * vw + x;
#pragma unroll
            for (int q = 0; q < 5; ++q) m[q] = dadd(m[q], dmul(g.k[t], tmp[q * plane + src]));
        }
        const double mu_x = m[0], mu_y = m[1];
        const double var_x = dsub(m[2], dmul(mu_x, mu_x)), var_y = dsub(m[3], dmul(mu_y, mu_y));
        const double cov = dsub(m[4], dmul(mu_x, mu_y));
        const double num = dmul(dadd(dmul(2.0, dmul(mu_x, mu_y)), c1), dadd(dmul(2.0, cov), c2));
        const double den = dmul(dadd(dadd(dmul(mu_x, mu_x), dmul(mu_y, mu_y)), c1), dadd(dadd(var_x, var_y), c2));
        acc = dadd(acc, num / den);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (int(threadIdx.x) < s) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

}  // namespace

size_t ssim_scratch_doubles(uint32_t w, uint32_t h) {
    return w < uint32_t(kSsimWin) ? 0 : size_t(5) * (w - kSsimWin + 1) * h;
}

double device_ssim(const float* pred, const float* gt, uint32_t w, uint32_t h, uint32_t channels, double* tmp,
                   double* part, double* h_part, cudaStream_t s) {
    Gauss11 g;  // gaussian_kernel (src/metrics.cpp:21-32)
    double sum = 0.0;
    for (int i = 0; i < kSsimWin; ++i) {
        const double d = i - kSsimWin / 2;
        g.k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += g.k[i];
    }
    for (double& v : g.k) v /= sum;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    const uint32_t vw = w - kSsimWin + 1, vh = h - kSsimWin + 1;
    double total = 0.0;
    for (uint32_t ch = 0; ch < channels; ++ch) {
        const size_t plane = size_t(vw) * h;
        k_ssim_h<<<unsigned(std::min<size_t>((plane + 255) / 256, 148 * 16)), 256, 0, s>>>(pred, gt, w, h, channels, ch,
                                                                                         g, tmp);
        k_ssim_v<<<kRedBlocks, kRedThreads, 0, s>>>(tmp, vw, h, g, c1, c2, part);
        note_launch(2);
        SVLF_CUDA(cudaMemcpyAsync(h_part, part, kRedBlocks * 8, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        double acc = 0.0;
        for (unsigned b = 0; b < kRedBlocks; ++b) acc += h_part[b];
        total += acc / double(size_t(vw) * vh);
    }
    return total / channels;
}

void launch_render_gt(const svlf_scene_desc& d, const double* d_spheres, const double* d_boxes, const DevCamera& cam,
                      float* rgb, float* depth, float* mask, cudaStream_t s) {
    SceneDev S{d_spheres, uint32_t(d.n_spheres), d_boxes, uint32_t(d.n_boxes), {}, {}, {}, {}};
    for (int a = 0; a < 3; ++a) {
        S.light_dir[a] = d.light_dir[a];
        S.light_rgb[a] = d.light_rgb[a];
        S.ambient[a] = d.ambient[a];
        S.background[a] = d.background[a];
    }
    const uint32_t n = cam.width * cam.height;
    k_render_gt<<<std::min<uint32_t>((n + 127) / 128, 148 * 16), 128, 0, s>>>(S, cam, rgb, depth, mask);
    note_launch();
}

void launch_backproject(const DevCamera& cam, const float* depth, double* pts, size_t cap, unsigned long long* count,
                        cudaStream_t s) {
    const uint32_t n = cam.width * cam.height;
    k_backproject<<<std::min<uint32_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(cam, depth, pts, cap, count);
    note_launch();
}

// Deterministic sums: partials per block, host adds them in block order.
double device_sq_err(const float* pred, const float* gt, size_t n, double* part, double* h_part, cudaStream_t s) {
    k_sq_err<<<kRedBlocks, kRedThreads, 0, s>>>(pred, gt, n, part);
    note_launch();
    SVLF_CUDA(cudaMemcpyAsync(h_part, part, kRedBlocks * 8, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    double se = 0.0;
    for (unsigned b = 0; b < kRedBlocks; ++b) se += h_part[b];
    return se;
}

void device_depth_err(const float* pd, const float* gd, const float* gm, size_t n, double* part, double* h_part,
                      double* sum2, double* sum1, double* count, cudaStream_t s) {
    k_depth_err<<<kRedBlocks, kRedThreads, 0, s>>>(pd, gd, gm, n, part);
    note_launch();
    SVLF_CUDA(cudaMemcpyAsync(h_part, part, kRedBlocks * 24, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    *sum2 = *sum1 = *count = 0.0;
    for (unsigned b = 0; b < kRedBlocks; ++b) {
        *sum2 += h_part[3 * b];
        *sum1 += h_part[3 * b + 1];
        *count += h_part[3 * b + 2];
    }
}

size_t reduction_partials() { return kRedBlocks * 3; }

}  // namespace svlfb
