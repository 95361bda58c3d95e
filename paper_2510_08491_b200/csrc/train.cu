// train.cu -- the training step around K7: the L1 photometric loss
// and its gradient, and Adam ("Adam optimizer ... learning rate of 1e-3 for the
// MLP ... means 1.6e-4, scales 5e-3, quaternions 1e-3, SH 2.5e-3").  The paper's loss is
// 3DGS's L1 + D-SSIM plus a std(s) regulariser; D-SSIM is out of scope (SURVEY
// A14), the regulariser is offered with a caller-chosen weight.
#include <math.h>

#include <algorithm>

#include "snp_internal.cuh"

namespace snp {
namespace {

// L = sum |out_rgb - target_rgb| / (3 n); grad_rgba = dL/d(out) (alpha channel 0).
__global__ void k_l1(const float4 *__restrict__ out, const float *__restrict__ target, int64_t n,
                     float4 *__restrict__ grad, float *loss) {
    const float inv = 1.0f / (3.0f * (float)n);
    float acc = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 o = out[i];
        const float d0 = o.x - target[3 * i], d1 = o.y - target[3 * i + 1], d2 = o.z - target[3 * i + 2];
        acc += fabsf(d0) + fabsf(d1) + fabsf(d2);
        grad[i] = make_float4(d0 > 0.f ? inv : (d0 < 0.f ? -inv : 0.f), d1 > 0.f ? inv : (d1 < 0.f ? -inv : 0.f),
                              d2 > 0.f ? inv : (d2 < 0.f ? -inv : 0.f), 0.f);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(loss, acc * inv);
}

// std(s) regulariser: R = w * mean_i std(s_i) (population std of the 3 semi-axes);
// adds dR/ds to grad_s and R to *loss.
__global__ void k_scale_reg(const float *__restrict__ s, int64_t n, float w, float *grad_s, float *loss) {
    float acc = 0.f;
    const float inv_n = 1.0f / (float)n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float a = s[3 * i], b = s[3 * i + 1], c = s[3 * i + 2];
        const float m = (a + b + c) / 3.0f;
        const float var = ((a - m) * (a - m) + (b - m) * (b - m) + (c - m) * (c - m)) / 3.0f;
        const float sd = sqrtf(var);
        acc += sd;
        if (sd > 0.f) {
            const float k = w * inv_n / (3.0f * sd);
            grad_s[3 * i] += k * (a - m);
            grad_s[3 * i + 1] += k * (b - m);
            grad_s[3 * i + 2] += k * (c - m);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(loss, w * acc * inv_n);
}

// Adam (Kingma & Ba) with bias correction.  log_space: the parameter is exp(theta) (the
// semi-axes, positive): the step is taken on theta = log s with dL/dtheta = s dL/ds.
__global__ void k_adam(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                       float *__restrict__ v, int64_t count, float lr, float b1, float b2, float eps, float bc1,
                       float bc2, int log_space) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float pi = p[i];
        const float gi = log_space ? g[i] * pi : g[i];
        const float mi = fmaf(b1, m[i], (1.0f - b1) * gi);
        const float vi = fmaf(b2, v[i], (1.0f - b2) * gi * gi);
        m[i] = mi;
        v[i] = vi;
        const float step = lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
        p[i] = log_space ? pi * expf(-step) : pi - step;
    }
}

unsigned grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace

cudaError_t launch_l1(const float *out_rgba, const float *target_rgb, int64_t n, float *grad_rgba, float *loss,
                      cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_l1<<<grid_for(n), 256, 0, st>>>(reinterpret_cast<const float4 *>(out_rgba), target_rgb, n,
                                      reinterpret_cast<float4 *>(grad_rgba), loss);
    return cudaGetLastError();
}

cudaError_t launch_scale_reg(const float *s, int64_t n, float w, float *grad_s, float *loss, cudaStream_t st) {
    if (n == 0 || w == 0.f) return cudaSuccess;
    k_scale_reg<<<grid_for(n), 256, 0, st>>>(s, n, w, grad_s, loss);
    return cudaGetLastError();
}

cudaError_t launch_adam(float *p, const float *g, float *m, float *v, int64_t count, float lr, float b1, float b2,
                        float eps, int step, bool log_space, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const float bc1 = 1.0f - powf(b1, (float)step), bc2 = 1.0f - powf(b2, (float)step);
    k_adam<<<grid_for(count), 256, 0, st>>>(p, g, m, v, count, lr, b1, b2, eps, bc1, bc2, log_space ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace snp
