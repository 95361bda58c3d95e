// train.cu -- the training step around K7: the photometric loss
// and its gradient, and Adam ("Adam optimizer ... learning rate of 1e-3 for the
// MLP ... means 1.6e-4, scales 5e-3, quaternions 1e-3, SH 2.5e-3").  The paper's loss is
// "the same loss function as 3DGS" plus a std(s) regulariser: L1 alone
// (snp_loss_l1) or 3DGS's (1 - lambda) L1 + lambda (1 - SSIM) (snp_loss_3dgs, reading
// R25: SSIM over 11x11 Gaussian windows, sigma 1.5, zero padding, C1 = 0.01^2,
// C2 = 0.03^2, per channel, averaged), the regulariser with a caller-chosen weight.
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

// ---- 3DGS loss: (1 - lambda) L1 + lambda (1 - SSIM) over [V][H][W] images (R25)
constexpr int kWin = 11, kHalf = 5;
struct Gauss {
    float w[kWin];
};
// maps are planar [V][planes][H][W]; separable blur with zero padding (dir 0: x, 1: y)
__global__ void k_blur(const float *__restrict__ in, float *__restrict__ out, int64_t planes, int H, int W, int dir,
                       Gauss g) {
    const int64_t total = planes * (int64_t)H * W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % W), y = (int)((i / W) % H);
        const float *row = in + (i - (dir ? (int64_t)y * W : x));   // start of the column (dir 1) / row (dir 0)
        float acc = 0.f;
#pragma unroll
        for (int k = -kHalf; k <= kHalf; ++k) {
            const int c = (dir ? y : x) + k;
            if (c >= 0 && c < (dir ? H : W)) acc = fmaf(g.w[k + kHalf], row[dir ? (int64_t)c * W : c], acc);
        }
        out[i] = acc;
    }
}
// the 5 moment maps per channel: x, y, x^2, y^2, x y  ->  m[V][5][3][H][W]
__global__ void k_ssim_moments(const float4 *__restrict__ out, const float *__restrict__ target, int V, int H, int W,
                               float *__restrict__ m) {
    const int64_t hw = (int64_t)H * W, total = (int64_t)V * hw;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / hw, p = i - v * hw;
        const float4 o = out[i];
        const float xs[3] = {o.x, o.y, o.z};
        float *b = m + v * 15 * hw + p;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float x = xs[c], y = target[3 * i + c];
            b[(0 * 3 + c) * hw] = x;
            b[(1 * 3 + c) * hw] = y;
            b[(2 * 3 + c) * hw] = x * x;
            b[(3 * 3 + c) * hw] = y * y;
            b[(4 * 3 + c) * hw] = x * y;
        }
    }
}
// per pixel and channel: SSIM s from the blurred moments mu[V][5][3][H][W]; its partial
// derivatives w.r.t. (mu_x, E[x^2], E[xy]) into d[V][3][3][H][W]; sum of s into *ssum
__global__ void k_ssim_map(const float *__restrict__ mu, int V, int H, int W, float *__restrict__ d, float *ssum) {
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    const int64_t hw = (int64_t)H * W, total = (int64_t)V * 3 * hw;
    float acc = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / (3 * hw), r = i - v * 3 * hw;   // r = c * hw + p
        const float *b = mu + v * 15 * hw + r;
        const float mx = b[0], my = b[3 * hw], exx = b[6 * hw], eyy = b[9 * hw], exy = b[12 * hw];
        const float n1 = 2.f * mx * my + C1, n2 = 2.f * (exy - mx * my) + C2;
        const float d1 = mx * mx + my * my + C1, d2 = (exx - mx * mx) + (eyy - my * my) + C2;
        const float sv = (n1 * n2) / (d1 * d2);
        acc += sv;
        float *o = d + v * 9 * hw + r;
        o[0] = sv * (2.f * my / n1 - 2.f * my / n2 - 2.f * mx / d1 + 2.f * mx / d2);   // ds/dmu_x
        o[3 * hw] = -sv / d2;                                                          // ds/dE[x^2]
        o[6 * hw] = 2.f * sv / n2;                                                     // ds/dE[xy]
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(ssum, acc);
}
// grad = (1 - lambda) dL1/dout - lambda / M (blur(ds/dmu) + 2 x blur(ds/dE[x^2]) + y blur(ds/dE[xy]));
// loss += (1 - lambda) L1 (k_l1 with that weight) + lambda (1 - ssum / M), M = 3 V H W
__global__ void k_ssim_grad(const float4 *__restrict__ out, const float *__restrict__ target, const float *__restrict__ bd,
                            int V, int H, int W, float lam, float4 *__restrict__ grad) {
    const int64_t hw = (int64_t)H * W, total = (int64_t)V * hw;
    const float inv = 1.0f / (3.0f * (float)total);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / hw, p = i - v * hw;
        const float4 o = out[i];
        const float xs[3] = {o.x, o.y, o.z};
        float g[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float x = xs[c], y = target[3 * i + c];
            const float *b = bd + v * 9 * hw + (int64_t)c * hw + p;
            const float dssim = b[0] + 2.f * x * b[3 * hw] + y * b[6 * hw];
            const float dl = x - y;
            const float l1 = dl > 0.f ? inv : (dl < 0.f ? -inv : 0.f);
            g[c] = (1.0f - lam) * l1 - lam * inv * dssim;
        }
        grad[i] = make_float4(g[0], g[1], g[2], 0.f);
    }
}
__global__ void k_ssim_loss(const float *ssum, float *l1sum, int64_t total, float lam, float *loss) {
    // (k_l1 accumulated the L1 mean into *l1sum)
    if (threadIdx.x == 0) atomicAdd(loss, (1.0f - lam) * l1sum[0] + lam * (1.0f - ssum[0] / (3.0f * (float)total)));
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

namespace snp {
size_t loss_3dgs_scratch_floats(int V, int H, int W) { return (size_t)V * H * W * (15 + 15 + 9 + 9) + 2; }

cudaError_t launch_loss_3dgs(const float *out_rgba, const float *target_rgb, int V, int H, int W, float lam,
                             float *grad_rgba, float *loss, float *scratch, cudaStream_t st) {
    const int64_t total = (int64_t)V * H * W;
    if (total == 0) return cudaSuccess;
    const int64_t hw = (int64_t)H * W;
    float *m = scratch, *t = m + 15 * total, *d = t + 15 * total, *t2 = d + 9 * total;
    float *sums = t2 + 9 * total;   // [0] = sum of SSIM, [1] = L1 mean
    Gauss g{};
    double gs[kWin], tot = 0.0;
    for (int k = 0; k < kWin; ++k) {
        gs[k] = exp(-(double)((k - kHalf) * (k - kHalf)) / (2.0 * 1.5 * 1.5));
        tot += gs[k];
    }
    for (int k = 0; k < kWin; ++k) g.w[k] = (float)(gs[k] / tot);
    cudaError_t e = cudaMemsetAsync(sums, 0, 2 * sizeof(float), st);
    if (e != cudaSuccess) return e;
    const unsigned gp = grid_for(total), g15 = grid_for(15 * total), g9 = grid_for(9 * total), g3 = grid_for(3 * total);
    k_ssim_moments<<<gp, 256, 0, st>>>(reinterpret_cast<const float4 *>(out_rgba), target_rgb, V, H, W, m);
    k_blur<<<g15, 256, 0, st>>>(m, t, 15 * (int64_t)V, H, W, 0, g);
    k_blur<<<g15, 256, 0, st>>>(t, m, 15 * (int64_t)V, H, W, 1, g);
    k_ssim_map<<<g3, 256, 0, st>>>(m, V, H, W, d, sums);
    k_blur<<<g9, 256, 0, st>>>(d, t2, 9 * (int64_t)V, H, W, 0, g);
    k_blur<<<g9, 256, 0, st>>>(t2, d, 9 * (int64_t)V, H, W, 1, g);
    // L1 mean into sums[1] (k_l1 writes a gradient we overwrite below)
    k_l1<<<gp, 256, 0, st>>>(reinterpret_cast<const float4 *>(out_rgba), target_rgb, total,
                             reinterpret_cast<float4 *>(grad_rgba), sums + 1);
    k_ssim_grad<<<gp, 256, 0, st>>>(reinterpret_cast<const float4 *>(out_rgba), target_rgb, d, V, H, W, lam,
                                    reinterpret_cast<float4 *>(grad_rgba));
    k_ssim_loss<<<1, 32, 0, st>>>(sums, sums + 1, total, lam, loss);
    (void)hw;
    return cudaGetLastError();
}
}  // namespace snp
