// features.cu — the reference's feature pyramid extraction and patch crop
// (SURVEY.md §8f row 2), sm_100a.
//
// Reference: features.cpp:55-235 — pool_image (4x4 mean), whiten_features
// (5x5 local-mean residual, 3x3 binomial smoothing, 5x5 local-RMS
// normalisation, optional central-difference gradients), lift_neighborhood
// (5x5 neighbourhood stacked to 25 * base channels, unit-normalised),
// pool_features (level 1 = 4x4 mean of the base grid), crop_patch_features
// (Catmull-Rom samples at the patch pixels / 4 and / 16).
//
// Every stage is a stencil with one thread per output cell (or descriptor
// entry), evaluating the reference's expression in the reference's order and
// precision (float sums where the reference sums floats, double where it uses
// double, float products accumulated into double where it does that); the
// file is compiled with --fmad=false, so the pyramid is bit-identical to the
// CPU restatement (tests).  It replaces the host->device copy of a frame's
// pyramid by the copy of its image (the reference's input).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace pvo_dev {

namespace {

// pool_image (features.cpp:55-71): float sum in (dy, dx) order, / 16
__global__ void pool_image_kernel(const float* img, int iw, int w, int h, float* raw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    float sum = 0;
    for (int dy = 0; dy < 4; ++dy)
        for (int dx = 0; dx < 4; ++dx) sum += img[(size_t)(4 * y + dy) * iw + 4 * x + dx];
    raw[i] = sum / 16.0f;
}

// residual against the 5x5 local mean, window clipped (features.cpp:105-121)
__global__ void rough_kernel(const float* raw, int w, int h, float* rough) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    double sum = 0;
    int count = 0;
    for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
            const int xi = x + dx, yi = y + dy;
            if (xi < 0 || yi < 0 || xi >= w || yi >= h) continue;
            sum += raw[yi * w + xi];
            ++count;
        }
    rough[i] = raw[i] - static_cast<float>(sum / count);
}

// 3x3 binomial smoothing, renormalised at the border (features.cpp:123-141)
__global__ void smooth_kernel(const float* rough, int w, int h, float* residual) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    const double kernel[3] = {1, 2, 1};
    double sum = 0, weight = 0;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            const int xi = x + dx, yi = y + dy;
            if (xi < 0 || yi < 0 || xi >= w || yi >= h) continue;
            const double k = kernel[dx + 1] * kernel[dy + 1];
            sum += k * rough[yi * w + xi];
            weight += k;
        }
    residual[i] = static_cast<float>(sum / weight);
}

// local-RMS normalisation (features.cpp:143-160) into channel 0 of the base grid
__global__ void normalize_kernel(const float* residual, int w, int h, int bc, float* base) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    double sum_sq = 0;
    int count = 0;
    for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
            const int xi = x + dx, yi = y + dy;
            if (xi < 0 || yi < 0 || xi >= w || yi >= h) continue;
            const float r = residual[yi * w + xi];
            sum_sq += r * r;  // float product, double accumulation (as the reference)
            ++count;
        }
    const double rms = sqrt(sum_sq / count);
    base[(size_t)i * bc] = rms > 1e-6 ? residual[i] / static_cast<float>(rms) : 0.0f;
}

// central-difference gradients for base_channels = 3 (features.cpp:162-173)
__global__ void gradient_kernel(int w, int h, float* base) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    auto g0 = [&](int xi, int yi) { return base[((size_t)yi * w + xi) * 3]; };
    const float gx = 0.5f * (g0(min(x + 1, w - 1), y) - g0(max(x - 1, 0), y));
    const float gy = 0.5f * (g0(x, min(y + 1, h - 1)) - g0(x, max(y - 1, 0)));
    base[(size_t)i * 3 + 1] = gx;
    base[(size_t)i * 3 + 2] = gy;
}

// lift_neighborhood (features.cpp:177-200): 5x5 neighbourhood stacked in (dy, dx,
// c) order, zero outside, unit-normalised (double norm of float squares)
__global__ void lift_kernel(const float* base, int w, int h, int bc, float* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    const int C = 25 * bc;
    float* o = out + (size_t)i * C;
    int ch = 0;
    for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
            const int xi = x + dx, yi = y + dy;
            const bool inside = xi >= 0 && yi >= 0 && xi < w && yi < h;
            for (int c = 0; c < bc; ++c) o[ch++] = inside ? base[((size_t)yi * w + xi) * bc + c] : 0.0f;
        }
    double norm_sq = 0;
    for (int c = 0; c < C; ++c) norm_sq += o[c] * o[c];
    if (norm_sq > 1e-12) {
        const float inv = static_cast<float>(1.0 / sqrt(norm_sq));
        for (int c = 0; c < C; ++c) o[c] *= inv;
    }
}

// pool_features (features.cpp:73-89): float 4x4 sums per channel, / 16
__global__ void pool_features_kernel(const float* grid, int gw, int bc, int w, int h, float* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h * bc) return;
    const int c = i % bc, cell = i / bc;
    const int x = cell % w, y = cell / w;
    float sum = 0;
    for (int dy = 0; dy < 4; ++dy)
        for (int dx = 0; dx < 4; ++dx) sum += grid[((size_t)(4 * y + dy) * gw + 4 * x + dx) * bc + c];
    out[i] = sum / 16.0f;
}

// crop_patch_features (features.cpp:204-224) with sample_cubic (:23-52): one
// thread per (patch, level, pixel, channel)
__global__ void crop_kernel(int n, const double* px, const double* py, const float* l0, int w0, int h0,
                            const float* l1, int w1, int h1, int C, float* out) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (size_t)n * 2 * 9 * C) return;
    const int c = (int)(t % C);
    const int k = (int)((t / C) % 9);
    const int level = (int)((t / ((size_t)C * 9)) % 2);
    const int p = (int)(t / ((size_t)C * 18));
    const double stride = level == 0 ? 4.0 : 16.0;
    const float* grid = level ? l1 : l0;
    const int W = level ? w1 : w0, H = level ? h1 : h0;
    const double x = px[9 * (size_t)p + k] / stride, y = py[9 * (size_t)p + k] / stride;
    const int x0 = (int)floor(x), y0 = (int)floor(y);
    const double tx = x - x0, ty = y - y0;
    double wx[4], wy[4];
    wx[0] = ((-0.5 * tx + 1.0) * tx - 0.5) * tx;
    wx[1] = (1.5 * tx - 2.5) * tx * tx + 1.0;
    wx[2] = ((-1.5 * tx + 2.0) * tx + 0.5) * tx;
    wx[3] = (0.5 * tx - 0.5) * tx * tx;
    wy[0] = ((-0.5 * ty + 1.0) * ty - 0.5) * ty;
    wy[1] = (1.5 * ty - 2.5) * ty * ty + 1.0;
    wy[2] = ((-1.5 * ty + 2.0) * ty + 0.5) * ty;
    wy[3] = (0.5 * ty - 0.5) * ty * ty;
    double v = 0;
    for (int j = 0; j < 4; ++j) {
        const int yi = y0 - 1 + j;
        if (yi < 0 || yi >= H) continue;
        double row = 0;
        for (int i = 0; i < 4; ++i) {
            const int xi = x0 - 1 + i;
            if (xi < 0 || xi >= W) continue;
            row += wx[i] * grid[((size_t)yi * W + xi) * C + c];
        }
        v += wy[j] * row;
    }
    out[t] = static_cast<float>(v);
}

unsigned nb(size_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t launch_extract_features(const float* image, int iw, int ih, int base_channels, float* scratch,
                                    float* level0, float* level1, cudaStream_t s) {
    const int w = iw / 4, h = ih / 4, bc = base_channels;
    const int w1 = w / 4, h1 = h / 4;
    float* raw = scratch;
    float* rough = raw + (size_t)w * h;
    float* residual = rough + (size_t)w * h;
    float* base = residual + (size_t)w * h;        // [h][w][bc]
    float* pooled = base + (size_t)w * h * bc;     // [h1][w1][bc]
    const size_t n = (size_t)w * h;
    pool_image_kernel<<<nb(n), 256, 0, s>>>(image, iw, w, h, raw);
    rough_kernel<<<nb(n), 256, 0, s>>>(raw, w, h, rough);
    smooth_kernel<<<nb(n), 256, 0, s>>>(rough, w, h, residual);
    normalize_kernel<<<nb(n), 256, 0, s>>>(residual, w, h, bc, base);
    if (bc == 3) gradient_kernel<<<nb(n), 256, 0, s>>>(w, h, base);
    lift_kernel<<<nb(n), 256, 0, s>>>(base, w, h, bc, level0);
    if (w1 > 0 && h1 > 0) {
        pool_features_kernel<<<nb((size_t)w1 * h1 * bc), 256, 0, s>>>(base, w, bc, w1, h1, pooled);
        lift_kernel<<<nb((size_t)w1 * h1), 256, 0, s>>>(pooled, w1, h1, bc, level1);
    }
    return cudaGetLastError();
}

size_t extract_scratch_floats(int iw, int ih, int base_channels) {
    const size_t w = iw / 4, h = ih / 4;
    return w * h * (3 + base_channels) + (w / 4) * (h / 4) * base_channels + 16;
}

cudaError_t launch_crop_patches(int n, const double* px, const double* py, const float* l0, int w0, int h0,
                                const float* l1, int w1, int h1, int C, float* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    crop_kernel<<<nb((size_t)n * 18 * C), 256, 0, s>>>(n, px, py, l0, w0, h0, l1, w1, h1, C, out);
    return cudaGetLastError();
}

}  // namespace pvo_dev
