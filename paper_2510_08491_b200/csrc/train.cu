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
// Fused, tiled D-SSIM (R25): a CTA takes a kTx x kTy tile of one view, loads x (the
// render) and y (the target) of one channel at a time over the tile plus the 5-pixel
// halo (zero outside the image: conv2d's zero padding), blurs the five moments x, y, x^2,
// y^2, x y separably in shared memory (x pass over the halo rows, then y), and writes per
// pixel the SSIM s's partial derivatives w.r.t. (mu_x, E[x^2], E[xy]) -- three maps per
// channel -- while summing s and |x - y|.  k_ssim_back blurs those maps the same way and
// forms dL/d(out).  Two passes over HBM instead of 24 planar blur passes.
constexpr int kTx = 32, kTy = 16, kHx = kTx + 2 * kHalf, kHy = kTy + 2 * kHalf;
constexpr int kSsimThreads = 256;

__global__ void __launch_bounds__(kSsimThreads) k_ssim_fwd(const float4 *__restrict__ out,
                                                           const float *__restrict__ target, int H, int W, Gauss g,
                                                           float *__restrict__ d, float *sums) {
    __shared__ float sx3[3][kHy][kHx], sy3[3][kHy][kHx];
    __shared__ float hb[5][kHy][kTx];
    const int v = blockIdx.z, x0 = blockIdx.x * kTx - kHalf, y0 = blockIdx.y * kTy - kHalf;
    const int64_t hw = (int64_t)H * W;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    float ssum = 0.f, l1sum = 0.f;
    // the tile and its halo, all three channels at once (one 16-byte load per pixel)
    for (int i = threadIdx.x; i < kHx * kHy; i += kSsimThreads) {
        const int r = i / kHx, q = i - r * kHx, gy = y0 + r, gx = x0 + q;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        float t0 = 0.f, t1 = 0.f, t2 = 0.f;
        if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
            const int64_t pi = (int64_t)v * hw + (int64_t)gy * W + gx;
            o = out[pi];
            t0 = target[3 * pi];
            t1 = target[3 * pi + 1];
            t2 = target[3 * pi + 2];
        }
        sx3[0][r][q] = o.x; sx3[1][r][q] = o.y; sx3[2][r][q] = o.z;
        sy3[0][r][q] = t0; sy3[1][r][q] = t1; sy3[2][r][q] = t2;
    }
    __syncthreads();
    for (int c = 0; c < 3; ++c) {
        float(*sx)[kHx] = sx3[c];
        float(*sy)[kHx] = sy3[c];
        for (int i = threadIdx.x; i < kHy * kTx; i += kSsimThreads) {   // x pass
            const int r = i / kTx, q = i - r * kTx;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f;
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                const float xv = sx[r][q + k], yv = sy[r][q + k], w = g.w[k];
                a0 = fmaf(w, xv, a0);
                a1 = fmaf(w, yv, a1);
                a2 = fmaf(w, xv * xv, a2);
                a3 = fmaf(w, yv * yv, a3);
                a4 = fmaf(w, xv * yv, a4);
            }
            hb[0][r][q] = a0;
            hb[1][r][q] = a1;
            hb[2][r][q] = a2;
            hb[3][r][q] = a3;
            hb[4][r][q] = a4;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kTy * kTx; i += kSsimThreads) {   // y pass + SSIM
            const int r = i / kTx, q = i - r * kTx, gy = y0 + kHalf + r, gx = x0 + kHalf + q;
            if (gy >= H || gx >= W) continue;
            float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                const float w = g.w[k];
#pragma unroll
                for (int j = 0; j < 5; ++j) m[j] = fmaf(w, hb[j][r + k][q], m[j]);
            }
            const float mx = m[0], my = m[1], exx = m[2], eyy = m[3], exy = m[4];
            const float n1 = 2.f * mx * my + C1, n2 = 2.f * (exy - mx * my) + C2;
            const float d1 = mx * mx + my * my + C1, d2 = (exx - mx * mx) + (eyy - my * my) + C2;
            const float sv = (n1 * n2) / (d1 * d2);
            ssum += sv;
            l1sum += fabsf(sx[r + kHalf][q + kHalf] - sy[r + kHalf][q + kHalf]);
            float *o = d + ((int64_t)v * 9 + 3 * c) * hw + (int64_t)gy * W + gx;
            o[0] = sv * (2.f * my / n1 - 2.f * my / n2 - 2.f * mx / d1 + 2.f * mx / d2);   // ds/dmu_x
            o[hw] = -sv / d2;                                                              // ds/dE[x^2]
            o[2 * hw] = 2.f * sv / n2;                                                     // ds/dE[xy]
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        l1sum += __shfl_xor_sync(0xffffffffu, l1sum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(sums, ssum);
        atomicAdd(sums + 1, l1sum);
    }
}

// grad = (1 - lambda) dL1/dout - lambda / M (blur(ds/dmu) + 2 x blur(ds/dE[x^2]) + y blur(ds/dE[xy]))
// (the blur is self-adjoint: same Gaussian, zero padding), M = 3 V H W
__global__ void __launch_bounds__(kSsimThreads) k_ssim_back(const float4 *__restrict__ out,
                                                            const float *__restrict__ target,
                                                            const float *__restrict__ d, int H, int W, int64_t total,
                                                            float lam, Gauss g, float4 *__restrict__ grad) {
    __shared__ float sd[3][kHy][kHx];
    __shared__ float hb[3][kHy][kTx];
    const int v = blockIdx.z, x0 = blockIdx.x * kTx - kHalf, y0 = blockIdx.y * kTy - kHalf;
    const int64_t hw = (int64_t)H * W;
    const float inv = 1.0f / (3.0f * (float)total);
    float gacc[2][3];   // (2 output pixels per thread)
    float xo[2][3], yo[2][3];   // their render and target values (one 16-byte load per pixel)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int i = threadIdx.x + t * kSsimThreads;
        const int r = i / kTx, q = i - r * kTx, gy = y0 + kHalf + r, gx = x0 + kHalf + q;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        float t0 = 0.f, t1 = 0.f, t2 = 0.f;
        if (gy < H && gx < W) {
            const int64_t pi = (int64_t)v * hw + (int64_t)gy * W + gx;
            o = out[pi];
            t0 = target[3 * pi];
            t1 = target[3 * pi + 1];
            t2 = target[3 * pi + 2];
        }
        xo[t][0] = o.x; xo[t][1] = o.y; xo[t][2] = o.z;
        yo[t][0] = t0; yo[t][1] = t1; yo[t][2] = t2;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        for (int i = threadIdx.x; i < kHx * kHy; i += kSsimThreads) {
            const int r = i / kHx, q = i - r * kHx, gy = y0 + r, gx = x0 + q;
            const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
            const float *b = d + ((int64_t)v * 9 + 3 * c) * hw + (int64_t)gy * W + gx;
#pragma unroll
            for (int m = 0; m < 3; ++m) sd[m][r][q] = in ? b[m * hw] : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kHy * kTx; i += kSsimThreads) {
            const int r = i / kTx, q = i - r * kTx;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                const float w = g.w[k];
                a0 = fmaf(w, sd[0][r][q + k], a0);
                a1 = fmaf(w, sd[1][r][q + k], a1);
                a2 = fmaf(w, sd[2][r][q + k], a2);
            }
            hb[0][r][q] = a0;
            hb[1][r][q] = a1;
            hb[2][r][q] = a2;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int i = threadIdx.x + t * kSsimThreads;
            const int r = i / kTx, q = i - r * kTx, gy = y0 + kHalf + r, gx = x0 + kHalf + q;
            gacc[t][c] = 0.f;
            if (gy >= H || gx >= W) continue;
            float b0 = 0.f, b1 = 0.f, b2 = 0.f;
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                const float w = g.w[k];
                b0 = fmaf(w, hb[0][r + k][q], b0);
                b1 = fmaf(w, hb[1][r + k][q], b1);
                b2 = fmaf(w, hb[2][r + k][q], b2);
            }
            const float x = xo[t][c], y = yo[t][c];
            const float dssim = b0 + 2.f * x * b1 + y * b2;
            const float dl = x - y;
            const float l1 = dl > 0.f ? inv : (dl < 0.f ? -inv : 0.f);
            gacc[t][c] = (1.0f - lam) * l1 - lam * inv * dssim;
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int i = threadIdx.x + t * kSsimThreads;
        const int r = i / kTx, q = i - r * kTx, gy = y0 + kHalf + r, gx = x0 + kHalf + q;
        if (gy < H && gx < W)
            grad[(int64_t)v * hw + (int64_t)gy * W + gx] = make_float4(gacc[t][0], gacc[t][1], gacc[t][2], 0.f);
    }
}
static_assert(kTx * kTy == 2 * kSsimThreads, "k_ssim_back: two output pixels per thread");

__global__ void k_ssim_loss(const float *sums, int64_t part, int64_t total, float lam, float *loss) {
    // sums[0] = sum of SSIM, sums[1] = sum of |x - y| over this call's 3 V H W values (part
    // pixels of the step's total): its share of (1 - lam) mean|x - y| + lam (1 - mean SSIM)
    const float m = 3.0f * (float)total;
    if (threadIdx.x == 0)
        atomicAdd(loss, (1.0f - lam) * (sums[1] / m) + lam * (((float)part - sums[0] / 3.0f) * 3.0f / m));
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
size_t loss_3dgs_scratch_floats(int V, int H, int W) { return (size_t)V * H * W * 9 + 2; }

cudaError_t launch_loss_3dgs(const float *out_rgba, const float *target_rgb, int V, int H, int W, float lam,
                             float *grad_rgba, float *loss, float *scratch, int64_t norm_total, cudaStream_t st) {
    const int64_t total = (int64_t)V * H * W;
    if (total == 0) return cudaSuccess;
    float *d = scratch;                      // [V][3 channels][3 maps][H][W]
    float *sums = d + 9 * total;             // [0] = sum of SSIM, [1] = sum of |x - y|
    Gauss g{};
    double gs[kWin], tot = 0.0;
    for (int k = 0; k < kWin; ++k) {
        gs[k] = exp(-(double)((k - kHalf) * (k - kHalf)) / (2.0 * 1.5 * 1.5));
        tot += gs[k];
    }
    for (int k = 0; k < kWin; ++k) g.w[k] = (float)(gs[k] / tot);
    cudaError_t e = cudaMemsetAsync(sums, 0, 2 * sizeof(float), st);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)((W + kTx - 1) / kTx), (unsigned)((H + kTy - 1) / kTy), (unsigned)V);
    k_ssim_fwd<<<grid, kSsimThreads, 0, st>>>(reinterpret_cast<const float4 *>(out_rgba), target_rgb, H, W, g, d,
                                              sums);
    k_ssim_back<<<grid, kSsimThreads, 0, st>>>(reinterpret_cast<const float4 *>(out_rgba), target_rgb, d, H, W,
                                               norm_total, lam, g, reinterpret_cast<float4 *>(grad_rgba));
    k_ssim_loss<<<1, 32, 0, st>>>(sums, total, norm_total, lam, loss);
    return cudaGetLastError();
}
}  // namespace snp
