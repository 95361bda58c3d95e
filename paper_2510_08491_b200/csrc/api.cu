// api.cu -- the C ABI of include/snp.h: argument checks, scene-owned device
// memory, stage ordering and kernel orchestration on the caller's stream.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "snp_internal.cuh"

using namespace snp;

namespace {
// NVTX range per API call (SURVEY §5 "Tracing / profiling"): visible in Nsight Systems /
// Compute timelines; a no-op without an attached tool
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

thread_local std::string g_err;

snp_status fail(snp_status st, const std::string &msg) {
    g_err = msg;
    return st;
}

#define SNP_CUDA(expr)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return fail(_e == cudaErrorMemoryAllocation ? SNP_ERR_OUT_OF_MEMORY : SNP_ERR_CUDA,     \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                        \
    } while (0)

enum State { kCreated = 0, kProjected = 1, kBinned = 2 };
// K5 emits after every exact round when the tile lists average more keys than this, or
// the visible primitives more keys (tiles) each than kEagerKeysPerVisible -- large
// footprints, deep overlapping lists (DESIGN.md "K5 design" 7: C5 221 keys/tile and 2.9
// keys/primitive, C2 4.5 and C1 3.1 keys/primitive -> eager; C3 90 and 1.9 -> default)
constexpr double kEagerKeysPerTile = 150.0;
constexpr double kEagerKeysPerVisible = 2.5;

// Device buffer that only grows.
template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t cap = 0;  // elements
    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = n ? n : 1;
        cudaError_t e = cudaMalloc((void **)&p, want * sizeof(T));
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

struct snp_scene_s {
    int device = 0;
    int64_t n = 0;
    int32_t sh_degree = 3;
    int32_t n_hidden = kHidden;
    float omega = 30.f;
    // parameters (SoA)
    DevBuf<float> params;
    float *centers = nullptr, *rotations = nullptr, *scales = nullptr, *w1 = nullptr, *b1 = nullptr,
          *w2 = nullptr, *b2 = nullptr, *sh = nullptr;
    // projection
    int state = kCreated;
    int32_t n_views = 0, W = 0, H = 0, tiles_x = 0, tiles_y = 0, tile_bits = 0, view_bits = 0;
    std::vector<CamBatch> cams;
    DevBuf<short4> rects;
    DevBuf<uint32_t> depth;
    DevBuf<float4> records;
    DevBuf<float> w_t;               // temporal weights [n][N] (temporal scenes only)
    size_t param_off[8] = {};        // byte offsets of the 8 parameter arrays in `params`
    int64_t param_count[8] = {};     // floats per array
    DevBuf<float> adam_m, adam_v;    // Adam moments, same layout as `params` (training only)
    DevBuf<uint32_t> bw_queue;       // K7: pixels with more hits than its first (second) pass holds
    DevBuf<unsigned char> bw_scratch;  // K7: hit arrays of the global-memory pass
    DevBuf<float> loss_scratch;        // snp_loss_3dgs: moment / SSIM-derivative maps
    DevBuf<uint32_t> bw_skip;          // K7: composited hits K5's grad mode already emitted, per pixel
    DevBuf<float> bw_fwd;              // K7: the forward image when the caller does not pass it
    DevBuf<FwdEntry> rec_entries;      // snp_set_record: the forward's composited hits (K5 record mode)
    bool record_mode = false;
    bool recorded = false;             // the last render recorded them (this projection, one camera batch)
    int32_t rec_colour = 0;            //   in this colour mode
    float rec_floor = 0.f;             //   with this transmittance floor (its stop rule)
    int64_t rec_chunks = 0;            //   in this many entry chunks
    DevBuf<float4> tight;              // K1a -> K2, tight binning (SNP_BIN_*): per item, see tight_geom
    DevBuf<float4> intr;               //   per view (1/fx, 1/fy, cx, cy)
    int32_t bin_flags = 0;             // snp_set_binning (applies from the next snp_project)
    int32_t projected_bin_flags = 0;   // the flags of the current projection
    DevBuf<GradEntry> grad_entries;    // K5 grad mode -> K7f
    DevBuf<int32_t> grad_fill;         //   entries used per chunk
    DevBuf<uint32_t> grad_keys;        //   per slot: vloc * n + primitive
    DevBuf<uint32_t> grad_count;       //   entries per key -> offsets (K7s counting sort)
    DevBuf<uint32_t> es_bsum;
    DevBuf<uint32_t> es_sorted;
    DevBuf<unsigned long long> es_cnt;
    DevBuf<float4> gc_acc;             // K7f, primitive colour mode: summed dL/dc per (view, primitive)
    float *grad_w_t = nullptr;       // where snp_render_backward adds dL/dW_t (caller-owned, device)
    bool temporal = false;
    // binning
    int32_t row_begin = 0, row_stride = 1, stripe_rows = 0;
    DevBuf<uint64_t> keys0, keys1;
    DevBuf<uint32_t> vals0, vals1;
    int64_t key_capacity = 0;
    int64_t known_ndup = 0;    // key count seen by the last sync_check (sizes the sort grid only)
    DevBuf<unsigned long long> dup_status;   // K2 block look-back states + ticket (zero between frames)
    DevBuf<uint32_t> sort_scratch;
    int64_t sort_max_partitions = 0;
    int sorted_idx = 0;
    DevBuf<uint32_t> ranges;
    // render
    DevBuf<unsigned long long> fallback;
    int64_t fallback_capacity = 0;
    DevBuf<uint32_t> tile_order;     // K5's tile order, per camera batch (kCamsPerLaunch x stripe tiles each)
    DevBuf<float> host_out_staging;
    int32_t pending_limit = 16;
    // counters
    DevBuf<unsigned long long> counters;
    unsigned long long *h_counters = nullptr;  // pinned
    DevBuf<int> flag;
    int *h_flag = nullptr;                     // pinned
    // K1b (render records) runs on a side stream forked from the caller's stream
    // after K1a and joined at the end of snp_bin_sort (also under stream capture)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_bw_fork = nullptr, ev_bw_join = nullptr;   // backward: K7s beside the per-pixel K7
    bool join_pending = false;
    bool render_dirty = false;       // a render has used the counters since the last binning
    // K5's eager mid-batch emission: set by a synchronising snp_bin_sort when the tile
    // lists are long (more than kEagerKeysPerTile keys per tile on average), where the
    // pending lists overflow into K6 otherwise (a function of the binning only, so the
    // same frame always renders the same way)
    bool eager_emit = false;
};

namespace snp {
int greatest_priority() {
    static int prio = 1;   // 1 = not queried yet (priorities are <= 0)
    if (prio == 1) {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) hi = 0;
        prio = hi;
    }
    return prio;
}
}  // namespace snp

namespace {

int bits_for(int64_t n) {
    int b = 0;
    while (((int64_t)1 << b) < n) ++b;
    return b;
}

void fill_args(snp_scene s, ProjectArgs &a) {
    a.n = s->n;
    a.n_hidden = s->n_hidden;
    a.sh_degree = s->sh_degree;
    a.omega = s->omega;
    a.centers = s->centers; a.rotations = s->rotations; a.scales = s->scales;
    a.w1 = s->w1; a.b1 = s->b1; a.w2 = s->w2; a.b2 = s->b2; a.sh = s->sh;
    a.w_t = s->temporal ? s->w_t.p : nullptr;
    a.tiles_x = s->tiles_x; a.tiles_y = s->tiles_y;
    a.rects = s->rects.p; a.depth = s->depth.p; a.records = s->records.p;
    a.tight = s->bin_flags ? s->tight.p : nullptr;
    a.intr = s->bin_flags ? s->intr.p : nullptr;
    a.counters = s->counters.p;
}

snp_status check_scene(snp_scene s) {
    if (!s) return fail(SNP_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    cudaError_t e = cudaSetDevice(s->device);
    if (e != cudaSuccess) return fail(SNP_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return SNP_OK;
}

}  // namespace

extern "C" {

const char *snp_version(void) { return "snp 0.1.0 (sm_100a)"; }

const char *snp_last_error(void) { return g_err.c_str(); }

// Copies the parameters into the scene's device buffers and validates them on
// the device (one reduction kernel + one stream synchronisation).
static snp_status upload_and_validate(snp_scene s, const snp_scene_desc *d, cudaStream_t st) {
    const int64_t N = s->n_hidden;
    const int64_t per[8] = {3, 4, 3, 3 * N, N, N, 1, 48};
    const float *src[8] = {d->centers, d->rotations, d->scales, d->w1, d->b1, d->w2, d->b2, d->sh};
    float *dst[8] = {s->centers, s->rotations, s->scales, s->w1, s->b1, s->w2, s->b2, s->sh};
    const int64_t n = s->n;
    if (n == 0) return SNP_OK;
    const cudaMemcpyKind kind = d->memory == SNP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    for (int k = 0; k < 8; ++k) SNP_CUDA(cudaMemcpyAsync(dst[k], src[k], sizeof(float) * per[k] * n, kind, st));
    const int init[2] = {0, 0x7fffffff};
    SNP_CUDA(cudaMemcpyAsync(s->flag.p, init, sizeof init, cudaMemcpyHostToDevice, st));
    ProjectArgs a{};
    fill_args(s, a);
    SNP_CUDA(launch_validate(a, s->flag.p, st));
    SNP_CUDA(cudaMemcpyAsync(s->h_flag, s->flag.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    SNP_CUDA(cudaStreamSynchronize(st));
    const int bad = s->h_flag[0], idx = s->h_flag[1];
    if (bad & 2) return fail(SNP_ERR_INVALID_ARGUMENT, "zero quaternion at primitive " + std::to_string(idx));
    if (bad & 4) return fail(SNP_ERR_INVALID_ARGUMENT, "non-positive scale at primitive " + std::to_string(idx));
    if (bad) return fail(SNP_ERR_INVALID_ARGUMENT, "non-finite parameter at primitive " + std::to_string(idx));
    return SNP_OK;
}

static snp_status check_desc(const snp_scene_desc *d) {
    if (!d) return fail(SNP_ERR_INVALID_ARGUMENT, "desc is NULL");
    if (d->n < 0) return fail(SNP_ERR_INVALID_ARGUMENT, "n < 0");
    if (!hidden_supported(d->n_hidden))
        return fail(SNP_ERR_UNSUPPORTED, "n_hidden must be 4, 8 (P:394), 16 or 32");
    if (d->sh_degree < 0 || d->sh_degree > 3) return fail(SNP_ERR_INVALID_ARGUMENT, "sh_degree must be 0..3");
    if (!(d->omega > 0.f) || !std::isfinite(d->omega)) return fail(SNP_ERR_INVALID_ARGUMENT, "omega must be > 0");
    if (d->memory != SNP_MEM_HOST && d->memory != SNP_MEM_DEVICE)
        return fail(SNP_ERR_INVALID_ARGUMENT, "memory must be SNP_MEM_HOST or SNP_MEM_DEVICE");
    if (d->n > kMaxPrims) return fail(SNP_ERR_UNSUPPORTED, "n must be < 2^24 (K5's pending entries pack the id in 24 bits)");
    const float *src[8] = {d->centers, d->rotations, d->scales, d->w1, d->b1, d->w2, d->b2, d->sh};
    if (d->n > 0)
        for (int k = 0; k < 8; ++k)
            if (!src[k]) return fail(SNP_ERR_INVALID_ARGUMENT, "a parameter array is NULL");
    return SNP_OK;
}

snp_status snp_create_scene(const snp_scene_desc *d, int device, void *cuda_stream, snp_scene *out) {
    g_err.clear();
    if (!out) return fail(SNP_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    snp_status r = check_desc(d);
    if (r != SNP_OK) return r;
    const int64_t n = d->n;
    const int64_t N = d->n_hidden;
    const int64_t per[8] = {3, 4, 3, 3 * N, N, N, 1, 48};
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(SNP_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    snp_scene s = new snp_scene_s();
    s->device = device;
    s->n = n;
    s->n_hidden = d->n_hidden;
    s->sh_degree = d->sh_degree;
    s->omega = d->omega;
    // one allocation, each array 256-byte aligned
    size_t off[8];
    size_t tot = 0;
    for (int k = 0; k < 8; ++k) {
        off[k] = tot;
        tot += ((size_t)(per[k] * n) * sizeof(float) + 255) / 256 * 256;
    }
    cudaError_t ce = s->params.ensure(tot / sizeof(float) + 64);
    if (ce == cudaSuccess) ce = s->counters.ensure(kNumCounters);
    if (ce == cudaSuccess) ce = s->flag.ensure(2);
    if (ce == cudaSuccess) ce = cudaMallocHost((void **)&s->h_counters, sizeof(unsigned long long) * kNumCounters);
    if (ce == cudaSuccess) ce = cudaMallocHost((void **)&s->h_flag, 2 * sizeof(int));
    if (ce == cudaSuccess) ce = cudaMemsetAsync(s->counters.p, 0, sizeof(unsigned long long) * kNumCounters, st);
    // K1b's side stream keeps the default (lowest) priority: the K2-K4 chain it overlaps
    // is launched with the greatest priority and takes SM slots first (launch_hi)
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&s->ev_bw_fork, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&s->ev_bw_join, cudaEventDisableTiming);
    if (ce != cudaSuccess) {
        snp_destroy(s);
        return fail(ce == cudaErrorMemoryAllocation ? SNP_ERR_OUT_OF_MEMORY : SNP_ERR_CUDA,
                    std::string("allocation: ") + cudaGetErrorString(ce));
    }
    float **dst[8] = {&s->centers, &s->rotations, &s->scales, &s->w1, &s->b1, &s->w2, &s->b2, &s->sh};
    for (int k = 0; k < 8; ++k) *dst[k] = reinterpret_cast<float *>(reinterpret_cast<char *>(s->params.p) + off[k]);
    for (int k = 0; k < 8; ++k) {
        s->param_off[k] = off[k];
        s->param_count[k] = per[k] * n;
    }
    r = upload_and_validate(s, d, st);
    if (r != SNP_OK) {
        std::string msg = g_err;
        snp_destroy(s);
        g_err = msg;
        return r;
    }
    *out = s;
    return SNP_OK;
}

snp_status snp_update_scene(snp_scene s, const snp_scene_desc *d, void *cuda_stream) {
    NvtxRange nvtx_("snp_update_scene");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    r = check_desc(d);
    if (r != SNP_OK) return r;
    if (d->n != s->n) return fail(SNP_ERR_INVALID_ARGUMENT, "snp_update_scene: n differs from the scene's");
    if (d->n_hidden != s->n_hidden)
        return fail(SNP_ERR_INVALID_ARGUMENT, "snp_update_scene: n_hidden differs from the scene's");
    s->sh_degree = d->sh_degree;
    s->omega = d->omega;
    if (s->join_pending) {   // K1b may still read the parameters being replaced
        SNP_CUDA(cudaStreamWaitEvent((cudaStream_t)cuda_stream, s->ev_join, 0));
        s->join_pending = false;
    }
    s->recorded = false;
    r = upload_and_validate(s, d, (cudaStream_t)cuda_stream);
    if (r != SNP_OK) return r;
    s->state = kCreated;   // parameters changed: project again
    return SNP_OK;
}

snp_status snp_project(snp_scene s, const snp_camera *cams, int32_t n_views, void *cuda_stream) {
    return snp_project_at(s, cams, n_views, nullptr, cuda_stream);
}

snp_status snp_set_temporal(snp_scene s, const float *w_t, int32_t memory, void *cuda_stream) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (memory != SNP_MEM_HOST && memory != SNP_MEM_DEVICE)
        return fail(SNP_ERR_INVALID_ARGUMENT, "memory must be SNP_MEM_HOST or SNP_MEM_DEVICE");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (s->join_pending) {   // K1b may still read the weights being replaced
        SNP_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
        s->join_pending = false;
    }
    s->state = kCreated;   // the records change: project again
    if (!w_t) {
        s->temporal = false;
        return SNP_OK;
    }
    const int64_t count = s->n * s->n_hidden;
    SNP_CUDA(s->w_t.ensure((size_t)std::max<int64_t>(count, 4)));
    SNP_CUDA(cudaMemcpyAsync(s->w_t.p, w_t, sizeof(float) * count,
                             memory == SNP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    const int init[2] = {0, 0x7fffffff};
    SNP_CUDA(cudaMemcpyAsync(s->flag.p, init, sizeof init, cudaMemcpyHostToDevice, st));
    SNP_CUDA(launch_validate_finite(s->w_t.p, count, s->flag.p, st));
    SNP_CUDA(cudaMemcpyAsync(s->h_flag, s->flag.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    SNP_CUDA(cudaStreamSynchronize(st));
    if (s->h_flag[0]) {
        s->temporal = false;
        return fail(SNP_ERR_INVALID_ARGUMENT,
                    "non-finite temporal weight at primitive " + std::to_string(s->h_flag[1] / s->n_hidden));
    }
    s->temporal = true;
    return SNP_OK;
}

snp_status snp_set_temporal_grad(snp_scene s, float *grad_w_t) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    s->grad_w_t = grad_w_t;
    return SNP_OK;
}

snp_status snp_project_at(snp_scene s, const snp_camera *cams, int32_t n_views, const float *xi_t,
                          void *cuda_stream) {
    NvtxRange nvtx_("snp_project_at");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!cams) return fail(SNP_ERR_INVALID_ARGUMENT, "cams is NULL");
    if (n_views < 1 || n_views > 4096) return fail(SNP_ERR_INVALID_ARGUMENT, "n_views must be 1..4096");
    const int32_t W = cams[0].width, H = cams[0].height;
    if (W < 1 || H < 1 || W > 32767 || H > 32767) return fail(SNP_ERR_INVALID_ARGUMENT, "width/height must be 1..32767");
    for (int v = 0; v < n_views; ++v) {
        const snp_camera &c = cams[v];
        if (c.width != W || c.height != H) return fail(SNP_ERR_INVALID_ARGUMENT, "all views must share width/height");
        bool ok = c.fx > 0.f && c.fy > 0.f && std::isfinite(c.fx) && std::isfinite(c.fy) && std::isfinite(c.cx) &&
                  std::isfinite(c.cy) && c.t_near >= 0.f && c.t_far > c.t_near && std::isfinite(c.t_far);
        for (int k = 0; k < 9; ++k) ok = ok && std::isfinite(c.R_wc[k]);
        for (int k = 0; k < 3; ++k) ok = ok && std::isfinite(c.C_w[k]);
        if (xi_t) ok = ok && std::isfinite(xi_t[v]);
        if (!ok) return fail(SNP_ERR_INVALID_ARGUMENT, "invalid camera " + std::to_string(v));
    }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    s->n_views = n_views;
    s->W = W;
    s->H = H;
    s->tiles_x = (W + kTile - 1) / kTile;
    s->tiles_y = (H + kTile - 1) / kTile;
    s->tile_bits = bits_for((int64_t)s->tiles_x * s->tiles_y);
    s->view_bits = bits_for(n_views);
    if (kDepthBits + s->tile_bits + s->view_bits > 64) return fail(SNP_ERR_UNSUPPORTED, "key exceeds 64 bits");
    const size_t items = (size_t)n_views * (size_t)s->n;
    SNP_CUDA(s->rects.ensure(items + 2));   // (+2: K1b bulk-copies rect rows rounded up to 16 bytes)
    SNP_CUDA(s->depth.ensure(items));
    if (s->bin_flags) {
        SNP_CUDA(s->tight.ensure(items * 4));
        SNP_CUDA(s->intr.ensure((size_t)n_views));
    }
    SNP_CUDA(s->records.ensure(items * rec_f4(s->n_hidden)));
    s->cams.clear();
    for (int v0 = 0; v0 < n_views; v0 += kCamsPerLaunch) {
        CamBatch cb{};
        cb.view0 = v0;
        cb.nv = std::min(kCamsPerLaunch, n_views - v0);
        for (int k = 0; k < cb.nv; ++k) {
            const snp_camera &c = cams[v0 + k];
            DevCam &dc = cb.cams[k];
            std::memcpy(dc.R, c.R_wc, sizeof dc.R);
            std::memcpy(dc.C, c.C_w, sizeof dc.C);
            dc.fx = c.fx; dc.fy = c.fy; dc.cx = c.cx; dc.cy = c.cy;
            dc.ifx = 1.0 / (double)c.fx;
            dc.ify = 1.0 / (double)c.fy;
            dc.W = c.width; dc.H = c.height;
            dc.t_near = c.t_near; dc.t_far = c.t_far;
            dc.xi_t = xi_t ? xi_t[v0 + k] : 0.f;
        }
        s->cams.push_back(cb);
    }
    if (s->join_pending) {   // a previous K1b (project without bin_sort) must finish first
        SNP_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
        s->join_pending = false;
    }
    // (no memset: K2 moves K1a's visible count out of its accumulator and clears it; a
    // projection that was never binned leaves it to clear here)
    if (s->state == kProjected)
        SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntVisibleAcc, 0, sizeof(unsigned long long), st));
    ProjectArgs a{};
    fill_args(s, a);
    s->projected_bin_flags = s->bin_flags;
    for (const CamBatch &cb : s->cams) SNP_CUDA(launch_bin_geom(a, cb, st));
    // fork: K1b on the side stream, overlapping K2-K4 (which need only K1a's output)
    SNP_CUDA(cudaEventRecord(s->ev_fork, st));
    SNP_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    for (const CamBatch &cb : s->cams) SNP_CUDA(launch_records(a, cb, std::getenv("SNP_SERIAL_K1B") ? st : s->side));
    SNP_CUDA(cudaEventRecord(s->ev_join, s->side));
    s->join_pending = true;
    s->state = kProjected;
    s->recorded = false;
    return SNP_OK;
}

snp_status snp_bin_sort(snp_scene s, const snp_render_opts *opts, void *cuda_stream) {
    NvtxRange nvtx_("snp_bin_sort");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!opts) return fail(SNP_ERR_INVALID_ARGUMENT, "opts is NULL");
    if (s->state < kProjected) return fail(SNP_ERR_BAD_STATE, "snp_bin_sort before snp_project");
    if (opts->tile_row_stride < 1 || opts->tile_row_begin < 0)
        return fail(SNP_ERR_INVALID_ARGUMENT, "tile_row_stride must be >= 1 and tile_row_begin >= 0");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    s->row_begin = opts->tile_row_begin;
    s->row_stride = opts->tile_row_stride;
    s->stripe_rows = s->row_begin < s->tiles_y ? (s->tiles_y - 1 - s->row_begin) / s->row_stride + 1 : 0;
    const int64_t items = (int64_t)s->n_views * s->n;
    const int64_t nblk = bin_scan_blocks(items);
    if (!s->dup_status.p || s->dup_status.cap < (size_t)nblk + 1) {
        SNP_CUDA(s->dup_status.ensure((size_t)nblk + 1));
        SNP_CUDA(cudaMemsetAsync(s->dup_status.p, 0, sizeof(unsigned long long) * s->dup_status.cap, st));
    }
    if (s->key_capacity == 0) {
        // first guess: 4 keys per (view, primitive); sync_check resizes exactly
        s->key_capacity = std::max<int64_t>(4 * items, 1024);
    }
    BinArgs b{};
    b.n = s->n;
    b.n_views = s->n_views;
    b.tiles_x = s->tiles_x;
    b.tiles_y = s->tiles_y;
    b.tile_bits = s->tile_bits;
    b.row_begin = s->row_begin;
    b.row_stride = s->row_stride;
    b.rects = s->rects.p;
    b.depth = s->depth.p;
    b.bin_flags = s->projected_bin_flags;
    b.tight = s->projected_bin_flags ? s->tight.p : nullptr;
    b.intr = s->projected_bin_flags ? s->intr.p : nullptr;
    b.dup_status = s->dup_status.p;
    b.counters = s->counters.p;
    auto alloc_keys = [&](int64_t cap) -> cudaError_t {
        cudaError_t e;
        if ((e = s->keys0.ensure((size_t)cap)) != cudaSuccess) return e;
        if ((e = s->keys1.ensure((size_t)cap)) != cudaSuccess) return e;
        if ((e = s->vals0.ensure((size_t)cap)) != cudaSuccess) return e;
        if ((e = s->vals1.ensure((size_t)cap)) != cudaSuccess) return e;
        return cudaSuccess;
    };
    SNP_CUDA(alloc_keys(s->key_capacity));
    b.capacity = s->key_capacity;
    // K3 scratch: onesweep over the significant bits only; the digit histograms are
    // accumulated by the duplication kernel itself (zero on entry, cleared again by K4);
    // the look-back regions are cleared by the passes themselves (region 0 is clean on entry)
    const int bits = kDepthBits + s->tile_bits + s->view_bits;
    const int passes = (bits + 7) / 8;
    auto ensure_sort_scratch = [&]() -> cudaError_t {
        const int64_t maxp = (s->key_capacity + sort_partition_size() - 1) / sort_partition_size();
        if (maxp <= s->sort_max_partitions && s->sort_scratch.p) return cudaSuccess;
        cudaError_t e = s->sort_scratch.ensure(sort_scratch_words(8, maxp));
        if (e != cudaSuccess) return e;
        s->sort_max_partitions = maxp;
        return cudaMemsetAsync(s->sort_scratch.p, 0, sizeof(uint32_t) * sort_scratch_words(8, maxp), st);
    };
    SNP_CUDA(ensure_sort_scratch());
    const int64_t slots = (int64_t)s->n_views * s->tiles_x * s->tiles_y;
    SNP_CUDA(s->ranges.ensure((size_t)slots * 2));
    b.hist = s->sort_scratch.p;
    b.passes = passes;
    b.ranges = s->ranges.p;
    b.n_slots = slots;
    b.keys = s->keys0.p;
    b.vals = s->vals0.p;
    SNP_CUDA(launch_dup(b, st));
    if (opts->sync_check) {
        static_assert(kCntVisible + 1 == kCntDup, "one copy reads both counters");
        SNP_CUDA(cudaMemcpyAsync(s->h_counters + kCntVisible, s->counters.p + kCntVisible,
                                 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        SNP_CUDA(cudaStreamSynchronize(st));
        s->eager_emit = (double)s->h_counters[kCntDup] > kEagerKeysPerTile * (double)slots ||
                        (double)s->h_counters[kCntDup] > kEagerKeysPerVisible * (double)s->h_counters[kCntVisible];
        const int64_t ndup = (int64_t)s->h_counters[kCntDup];
        s->known_ndup = ndup;
        if (ndup > s->key_capacity) {
            // grow exactly once, then duplicate again (the first pass's keys were cut at
            // the old capacity; its histograms and block states are cleared)
            s->key_capacity = ndup + ndup / 4 + 1024;
            SNP_CUDA(alloc_keys(s->key_capacity));
            SNP_CUDA(ensure_sort_scratch());
            SNP_CUDA(cudaMemsetAsync(s->sort_scratch.p, 0, sizeof(uint32_t) * 8 * 256, st));
            SNP_CUDA(cudaMemsetAsync(s->dup_status.p, 0, sizeof(unsigned long long) * s->dup_status.cap, st));
            SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntDeadKeysAcc, 0, sizeof(unsigned long long), st));
            b.capacity = s->key_capacity;
            b.hist = s->sort_scratch.p;
            b.keys = s->keys0.p;
            b.vals = s->vals0.p;
            SNP_CUDA(launch_dup(b, st));
        }
    }
    SortScratch sc{};
    sc.hist = s->sort_scratch.p;
    sc.lookback = s->sort_scratch.p + 8 * 256;
    sc.tickets = s->sort_scratch.p + 8 * 256 + (size_t)8 * s->sort_max_partitions * 256;
    sc.max_partitions = s->sort_max_partitions;
    int final_idx = 0;
    SNP_CUDA(launch_onesweep(s->keys0.p, s->vals0.p, s->keys1.p, s->vals1.p, s->key_capacity, s->counters.p,
                             passes, sc, s->known_ndup + s->known_ndup / 8, st, &final_idx));
    s->sorted_idx = final_idx;
    const uint64_t *sk = final_idx ? s->keys1.p : s->keys0.p;
    // K4
    SNP_CUDA(launch_tile_ranges(sk, s->counters.p, s->key_capacity, s->tile_bits, s->tiles_x * s->tiles_y,
                                s->ranges.p, b, st));
    // K5's tile orders (longest tile list first), one per camera batch; they run while
    // K1b may still be busy on the side stream
    {
        const size_t order_stride = (size_t)kCamsPerLaunch * (size_t)(s->tiles_x * s->stripe_rows);
        SNP_CUDA(s->tile_order.ensure(std::max<size_t>(1, order_stride * s->cams.size())));
        RenderArgs ra{};
        ra.tiles_x = s->tiles_x;
        ra.tiles_y = s->tiles_y;
        ra.tiles_per_view = s->tiles_x * s->tiles_y;
        ra.row_begin = s->row_begin;
        ra.row_stride = s->row_stride;
        ra.stripe_rows = s->stripe_rows;
        ra.ranges = s->ranges.p;
        for (size_t k = 0; k < s->cams.size(); ++k)
            SNP_CUDA(launch_tile_order(ra, s->cams[k], s->tile_order.p + k * order_stride, st));
    }
    // join K1b: everything after bin_sort on the caller's stream sees the records
    if (s->join_pending) {
        SNP_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
        s->join_pending = false;
    }
    s->state = kBinned;
    s->render_dirty = false;
    return SNP_OK;
}

// Common render arguments of a binned scene (K5, K6w, K6, K7).
static RenderArgs render_args(snp_scene s, const snp_render_opts *opts) {
    RenderArgs a{};
    a.n_hidden = s->n_hidden;
    a.colour_ray = opts->colour_mode == SNP_COLOUR_RAY ? 1 : 0;
    a.eager_emit = s->eager_emit ? 1 : 0;
    if (const char *ee = std::getenv("SNP_EAGER_EMIT")) a.eager_emit = std::atoi(ee) != 0;   // A/B override
    a.sh = s->sh;
    a.sh_degree = s->sh_degree;
    a.centers = s->centers;
    a.scales = s->scales;
    a.rotations = s->rotations;
    a.tiles_x = s->tiles_x;
    a.tiles_y = s->tiles_y;
    a.tiles_per_view = s->tiles_x * s->tiles_y;
    a.tile_bits = s->tile_bits;
    a.row_begin = s->row_begin;
    a.row_stride = s->row_stride;
    a.stripe_rows = s->stripe_rows;
    a.n = s->n;
    a.records = s->records.p;
    a.keys = s->sorted_idx ? s->keys1.p : s->keys0.p;
    a.vals = s->sorted_idx ? s->vals1.p : s->vals0.p;
    a.ranges = s->ranges.p;
    for (int c = 0; c < 3; ++c) a.bg[c] = opts->background[c];
    a.t_floor = opts->transmittance_floor;
    a.pending_limit = s->pending_limit;
    {
        const char *dbg = std::getenv("SNP_DEBUG");
        a.debug_flags = dbg ? std::atoi(dbg) : 0;
    }
    a.counters = s->counters.p;
    return a;
}

// K5 (+ K6w, K6) into a device image: the body of snp_render.
static snp_status render_device(snp_scene s, const snp_render_opts *opts, float *dout, cudaStream_t st) {
    const int64_t fb_cap = std::min<int64_t>((int64_t)s->n_views * s->W * s->H, (int64_t)1 << 22);
    if (s->fallback_capacity < fb_cap) {
        SNP_CUDA(s->fallback.ensure((size_t)(2 * fb_cap)));
        SNP_CUDA(cudaMemsetAsync(s->fallback.p, 0, sizeof(unsigned long long) * (size_t)(2 * fb_cap), st));
        s->fallback_capacity = fb_cap;
    }
    // stats, fallback queue, tile queue: K4 cleared them for the first render of this
    // binning; a further render clears them with one memset (contiguous counters)
    if (s->render_dirty)
        SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntTested, 0,
                                 sizeof(unsigned long long) * (kCntRenderLast - kCntTested + 1), st));
    s->render_dirty = true;
    RenderArgs a = render_args(s, opts);
    a.out = dout;
    a.fallback = s->fallback.p;
    a.fallback_capacity = s->fallback_capacity;
    // record mode (training): K5 also writes its composited hits for the next backward;
    // one camera batch, the whole image
    const bool rec = s->record_mode && s->cams.size() == 1 && s->n > 0 && s->stripe_rows > 0 &&
                     s->row_begin == 0 && s->row_stride == 1;
    s->recorded = false;
    if (rec) {
        const int64_t npix_batch = (int64_t)s->cams[0].nv * s->W * s->H;
        int dev_sms = 148;
        SNP_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, s->device));
        const int64_t chunks = (12 * npix_batch + kGradChunk - 1) / kGradChunk + 2 * 8 * (int64_t)dev_sms;
        SNP_CUDA(s->rec_entries.ensure((size_t)(chunks * kGradChunk)));
        SNP_CUDA(s->grad_fill.ensure((size_t)chunks));
        SNP_CUDA(s->grad_keys.ensure((size_t)(chunks * kGradChunk)));
        SNP_CUDA(s->bw_queue.ensure((size_t)std::max<int64_t>(1, 3 * npix_batch)));
        SNP_CUDA(s->bw_skip.ensure((size_t)std::max<int64_t>(1, npix_batch)));
        SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntBwdQueue, 0, sizeof(unsigned long long), st));
        SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntGradEntries, 0, 2 * sizeof(unsigned long long), st));
        a.record = 1;
        a.rec_entries = s->rec_entries.p;
        a.grad_fill = s->grad_fill.p;
        a.grad_chunks = chunks;
        a.grad_keys = s->grad_keys.p;
        a.bw_queue = s->bw_queue.p;
        a.bw_skip = s->bw_skip.p;
        s->rec_chunks = chunks;
        s->rec_colour = opts->colour_mode;
        s->rec_floor = opts->transmittance_floor;
    }
    const size_t order_stride = (size_t)kCamsPerLaunch * (size_t)(s->tiles_x * s->stripe_rows);
    a.k5_grid = render_grid(s->n_hidden, a.colour_ray != 0, a.eager_emit != 0,
                            s->tiles_x * s->stripe_rows * (s->cams.empty() ? 0 : s->cams[0].nv));
    if (s->stripe_rows > 0) {
        // (an empty scene has empty tile ranges: every pixel gets the background)
        for (size_t k = 0; k < s->cams.size(); ++k) {
            a.tile_order = s->tile_order.p + k * order_stride;
            SNP_CUDA(launch_render(a, s->cams[k], k > 0, st));
        }
        // (SNP_DEBUG bit 2 skips K6: timing experiments only, overflowed pixels stay unwritten)
        if (s->n > 0 && !(a.debug_flags & 2)) SNP_CUDA(launch_fallback(a, s->cams.data(), (int)s->cams.size(), st));
    }
    s->recorded = rec;
    return SNP_OK;
}

snp_status snp_render(snp_scene s, const snp_render_opts *opts, float *out_rgba, void *cuda_stream) {
    NvtxRange nvtx_("snp_render");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!opts || !out_rgba) return fail(SNP_ERR_INVALID_ARGUMENT, "opts or out_rgba is NULL");
    if (s->state < kBinned) return fail(SNP_ERR_BAD_STATE, "snp_render before snp_bin_sort");
    if (!(opts->transmittance_floor >= 0.f) || !(opts->transmittance_floor < 1.f))
        return fail(SNP_ERR_INVALID_ARGUMENT, "transmittance_floor must be in [0, 1)");
    if (opts->out_memory != SNP_MEM_HOST && opts->out_memory != SNP_MEM_DEVICE &&
        opts->out_memory != SNP_MEM_HOST_ASYNC)
        return fail(SNP_ERR_INVALID_ARGUMENT, "out_memory must be SNP_MEM_HOST, SNP_MEM_DEVICE or SNP_MEM_HOST_ASYNC");
    if (opts->colour_mode != SNP_COLOUR_PRIMITIVE && opts->colour_mode != SNP_COLOUR_RAY)
        return fail(SNP_ERR_INVALID_ARGUMENT, "colour_mode must be SNP_COLOUR_PRIMITIVE or SNP_COLOUR_RAY");
    const bool host_out = opts->out_memory != SNP_MEM_DEVICE;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const size_t out_floats = (size_t)s->n_views * s->W * s->H * 4;
    float *dout = out_rgba;
    if (host_out) {
        SNP_CUDA(s->host_out_staging.ensure(out_floats));
        dout = s->host_out_staging.p;
        // pixels outside the stripe come back as 0 (every pixel is written otherwise)
        if (s->row_begin != 0 || s->row_stride != 1)
            SNP_CUDA(cudaMemsetAsync(dout, 0, out_floats * sizeof(float), st));
    }
    r = render_device(s, opts, dout, st);
    if (r != SNP_OK) return r;
    if (host_out) {
        SNP_CUDA(cudaMemcpyAsync(out_rgba, dout, out_floats * sizeof(float), cudaMemcpyDeviceToHost, st));
        if (opts->out_memory == SNP_MEM_HOST) SNP_CUDA(cudaStreamSynchronize(st));
    }
    return SNP_OK;
}

snp_status snp_render_backward_ex(snp_scene s, const snp_render_opts *opts, const float *fwd_rgba,
                                  const float *grad_rgba, float *grad_w1, float *grad_b1, float *grad_w2,
                                  float *grad_b2, float *grad_sh, float *grad_centers, float *grad_rotations,
                                  float *grad_scales, void *cuda_stream) {
    NvtxRange nvtx_("snp_render_backward_ex");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!opts || !grad_rgba || !grad_w1 || !grad_b1 || !grad_w2 || !grad_b2 || !grad_sh)
        return fail(SNP_ERR_INVALID_ARGUMENT, "opts or a gradient pointer is NULL");
    if ((grad_centers == nullptr) != (grad_rotations == nullptr) || (grad_centers == nullptr) != (grad_scales == nullptr))
        return fail(SNP_ERR_INVALID_ARGUMENT, "grad_centers, grad_rotations, grad_scales: all NULL or all set");
    if (s->state < kBinned) return fail(SNP_ERR_BAD_STATE, "snp_render_backward before snp_bin_sort");
    if (s->row_begin != 0 || s->row_stride != 1)
        return fail(SNP_ERR_UNSUPPORTED, "snp_render_backward needs the whole image (tile rows 0, 1)");
    if (opts->colour_mode != SNP_COLOUR_PRIMITIVE && opts->colour_mode != SNP_COLOUR_RAY)
        return fail(SNP_ERR_INVALID_ARGUMENT, "colour_mode must be SNP_COLOUR_PRIMITIVE or SNP_COLOUR_RAY");
    if (!(opts->transmittance_floor >= 0.f) || !(opts->transmittance_floor < 1.f))
        return fail(SNP_ERR_INVALID_ARGUMENT, "transmittance_floor must be in [0, 1)");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int64_t npix_all = (int64_t)s->n_views * s->W * s->H;
    const int64_t npix_batch = (int64_t)std::min<int>(s->n_views, kCamsPerLaunch) * s->W * s->H;
    SNP_CUDA(s->bw_queue.ensure((size_t)std::max<int64_t>(1, 3 * npix_batch)));
    SNP_CUDA(s->bw_skip.ensure((size_t)std::max<int64_t>(1, npix_batch)));
    SNP_CUDA(s->bw_scratch.ensure(backward_scratch_bytes()));
    SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntBwdSkipped, 0, sizeof(unsigned long long), st));
    BackwardGrads g{grad_w1, grad_b1, grad_w2, grad_b2, grad_sh, grad_centers, grad_rotations, grad_scales,
                    s->temporal ? s->grad_w_t : nullptr, false};
    {
        auto al = [](const void *p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; };
        g.vec = al(grad_w1) && al(grad_b1) && al(grad_w2) && al(grad_sh) && al(grad_rotations) && al(g.wt);
    }
    const bool legacy = [] {   // A/B: the per-pixel K7 for every pixel (round-1 path)
        const char *e = std::getenv("SNP_BWD_LEGACY");
        return e && std::atoi(e) != 0;
    }();
    if (legacy) {
        RenderArgs a = render_args(s, opts);
        a.bw_queue = s->bw_queue.p;
        for (const CamBatch &cb : s->cams)
            SNP_CUDA(launch_backward(a, cb, grad_rgba, g, s->omega, s->bw_scratch.p, false, nullptr, st, st));
        return SNP_OK;
    }
    // the forward result the gradients refer to (the caller's, or rendered here)
    const float *fwd = fwd_rgba;
    if (!fwd) {
        SNP_CUDA(s->bw_fwd.ensure((size_t)std::max<int64_t>(1, npix_all * 4)));
        r = render_device(s, opts, s->bw_fwd.p, st);
        if (r != SNP_OK) return r;
        fwd = s->bw_fwd.p;
    }
    // the forward recorded its composited hits (snp_set_record, one camera batch, this
    // colour mode): no gradient-mode traversal; K7s forms dL/dI and dL/dc from them
    const bool from_fwd = s->recorded && s->rec_colour == opts->colour_mode &&
                          s->rec_floor == opts->transmittance_floor && s->cams.size() == 1 &&
                          !std::getenv("SNP_K7F_UNSORTED");
    // K5 in grad mode: one GradEntry per composited hit, in per-warp chunks (12 per pixel
    // of a camera batch, plus a partly filled chunk per resident consumer warp, before the
    // path falls back to the per-pixel K7 for every pixel)
    int dev_sms = 148;
    SNP_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, s->device));
    const int64_t chunks = from_fwd ? s->rec_chunks
                                    : (12 * npix_batch + kGradChunk - 1) / kGradChunk + 2 * 8 * (int64_t)dev_sms;
    if (!from_fwd) SNP_CUDA(s->grad_entries.ensure((size_t)(chunks * kGradChunk)));
    SNP_CUDA(s->grad_fill.ensure((size_t)chunks));
    RenderArgs a = render_args(s, opts);
    a.bw_queue = s->bw_queue.p;
    a.bw_skip = s->bw_skip.p;
    a.grad_in = reinterpret_cast<const float4 *>(grad_rgba);
    a.fwd = reinterpret_cast<const float4 *>(fwd);
    a.grad_entries = s->grad_entries.p;
    a.grad_fill = s->grad_fill.p;
    a.grad_chunks = chunks;
    a.rec_entries = s->rec_entries.p;
    a.from_fwd = from_fwd ? 1 : 0;
    // K7s (default; SNP_K7F_UNSORTED=1: K7f in slot order, A/B)
    const bool unsorted = [] {
        const char *e = std::getenv("SNP_K7F_UNSORTED");
        return e && std::atoi(e) != 0;
    }();
    EntrySort es{};
    int nv_max = 1;
    for (const CamBatch &cb : s->cams) nv_max = std::max(nv_max, cb.nv);
    if (!unsorted) {
        const int64_t slots = chunks * kGradChunk, nk = (int64_t)nv_max * std::max<int64_t>(1, s->n);
        SNP_CUDA(s->grad_keys.ensure((size_t)slots));
        SNP_CUDA(s->grad_count.ensure((size_t)nk));
        SNP_CUDA(s->es_bsum.ensure((size_t)((nk + 4095) / 4096)));
        SNP_CUDA(s->es_sorted.ensure((size_t)slots));
        SNP_CUDA(s->es_cnt.ensure(64));
        a.grad_keys = s->grad_keys.p;
        a.grad_count = s->grad_count.p;
        es.bsum = s->es_bsum.p;
        es.sorted = s->es_sorted.p;
        es.cnt = s->es_cnt.p;
    }
    if (!a.colour_ray) {
        SNP_CUDA(s->gc_acc.ensure((size_t)nv_max * (size_t)std::max<int64_t>(1, s->n)));
        a.gc_acc = s->gc_acc.p;
    }
    const size_t order_stride = (size_t)kCamsPerLaunch * (size_t)(s->tiles_x * s->stripe_rows);
    for (size_t k = 0; k < s->cams.size(); ++k) {
        if (!a.colour_ray)
            SNP_CUDA(cudaMemsetAsync(a.gc_acc, 0, (size_t)s->cams[k].nv * (size_t)s->n * sizeof(float4), st));
        if (a.grad_count)
            SNP_CUDA(cudaMemsetAsync(a.grad_count, 0, (size_t)s->cams[k].nv * (size_t)s->n * sizeof(uint32_t), st));
        a.tile_order = s->tile_order.p + k * order_stride;
        if (!from_fwd) {
            SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntBwdQueue, 0, sizeof(unsigned long long), st));
            SNP_CUDA(cudaMemsetAsync(s->counters.p + kCntGradEntries, 0, 2 * sizeof(unsigned long long), st));
            if (s->n > 0) SNP_CUDA(launch_render_grad(a, s->cams[k], st));
        }
        // K7s over the entries, and beside it (side stream) the per-pixel K7 for the pixels
        // K5 queued (latency-bound long pixels: they overlap K7s; joined before the next
        // batch reuses the queue)
        SNP_CUDA(cudaEventRecord(s->ev_bw_fork, st));
        SNP_CUDA(cudaStreamWaitEvent(s->side, s->ev_bw_fork, 0));
        SNP_CUDA(launch_backward(a, s->cams[k], grad_rgba, g, s->omega, s->bw_scratch.p, true, unsorted ? nullptr : &es,
                                 st, s->side));
        SNP_CUDA(cudaEventRecord(s->ev_bw_join, s->side));
        SNP_CUDA(cudaStreamWaitEvent(st, s->ev_bw_join, 0));
    }
    return SNP_OK;
}

snp_status snp_render_backward(snp_scene s, const snp_render_opts *opts, const float *grad_rgba, float *grad_w1,
                               float *grad_b1, float *grad_w2, float *grad_b2, float *grad_sh, float *grad_centers,
                               float *grad_rotations, float *grad_scales, void *cuda_stream) {
    return snp_render_backward_ex(s, opts, nullptr, grad_rgba, grad_w1, grad_b1, grad_w2, grad_b2, grad_sh,
                                  grad_centers, grad_rotations, grad_scales, cuda_stream);
}

snp_status snp_loss_l1(const float *out_rgba, const float *target_rgb, int64_t n_pixels, float *grad_rgba, float *loss,
                       void *cuda_stream) {
    g_err.clear();
    if (n_pixels < 0) return fail(SNP_ERR_INVALID_ARGUMENT, "n_pixels < 0");
    if (n_pixels > 0 && (!out_rgba || !target_rgb || !grad_rgba || !loss))
        return fail(SNP_ERR_INVALID_ARGUMENT, "a pointer is NULL");
    SNP_CUDA(launch_l1(out_rgba, target_rgb, n_pixels, grad_rgba, loss, (cudaStream_t)cuda_stream));
    return SNP_OK;
}

snp_status snp_loss_3dgs(snp_scene s, const float *out_rgba, const float *target_rgb, int32_t n_views, int32_t height,
                         int32_t width, float lambda_dssim, float *grad_rgba, float *loss, void *cuda_stream) {
    return snp_loss_3dgs_part(s, out_rgba, target_rgb, n_views, height, width, n_views, lambda_dssim, grad_rgba, loss,
                              cuda_stream);
}

snp_status snp_loss_3dgs_part(snp_scene s, const float *out_rgba, const float *target_rgb, int32_t n_views,
                              int32_t height, int32_t width, int32_t step_views, float lambda_dssim, float *grad_rgba,
                              float *loss, void *cuda_stream) {
    NvtxRange nvtx_("snp_loss_3dgs_part");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (n_views < 0 || height < 0 || width < 0) return fail(SNP_ERR_INVALID_ARGUMENT, "negative image size");
    if (step_views < n_views) return fail(SNP_ERR_INVALID_ARGUMENT, "step_views < n_views");
    if (!(lambda_dssim >= 0.f && lambda_dssim <= 1.f))
        return fail(SNP_ERR_INVALID_ARGUMENT, "lambda_dssim must be in [0, 1]");
    const int64_t total = (int64_t)n_views * height * width;
    if (total == 0) return SNP_OK;
    if (!out_rgba || !target_rgb || !grad_rgba || !loss) return fail(SNP_ERR_INVALID_ARGUMENT, "a pointer is NULL");
    SNP_CUDA(s->loss_scratch.ensure(loss_3dgs_scratch_floats(n_views, height, width)));
    SNP_CUDA(launch_loss_3dgs(out_rgba, target_rgb, n_views, height, width, lambda_dssim, grad_rgba, loss,
                              s->loss_scratch.p, (int64_t)step_views * height * width, (cudaStream_t)cuda_stream));
    return SNP_OK;
}

snp_status snp_scale_regularizer(snp_scene s, float weight, float *grad_scales, float *loss, void *cuda_stream) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!grad_scales || !loss) return fail(SNP_ERR_INVALID_ARGUMENT, "a pointer is NULL");
    if (!(weight >= 0.f) || !std::isfinite(weight)) return fail(SNP_ERR_INVALID_ARGUMENT, "weight must be >= 0");
    SNP_CUDA(launch_scale_reg(s->scales, s->n, weight, grad_scales, loss, (cudaStream_t)cuda_stream));
    return SNP_OK;
}

snp_status snp_adam_step(snp_scene s, const float *const *grads, const float *lr, float beta1, float beta2, float eps,
                         int32_t step, void *cuda_stream) {
    NvtxRange nvtx_("snp_adam_step");
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!grads || !lr) return fail(SNP_ERR_INVALID_ARGUMENT, "grads or lr is NULL");
    if (step < 1) return fail(SNP_ERR_INVALID_ARGUMENT, "step must be >= 1");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && eps > 0.f))
        return fail(SNP_ERR_INVALID_ARGUMENT, "need 0 <= beta1, beta2 < 1 and eps > 0");
    for (int k = 0; k < 8; ++k)
        if (!grads[k] || !(lr[k] >= 0.f)) return fail(SNP_ERR_INVALID_ARGUMENT, "a gradient is NULL or lr < 0");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (s->join_pending) {   // K1b may still read the parameters being updated
        SNP_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
        s->join_pending = false;
    }
    if (!s->adam_m.p || s->adam_m.cap < s->params.cap) {
        SNP_CUDA(s->adam_m.ensure(s->params.cap));
        SNP_CUDA(s->adam_v.ensure(s->params.cap));
        SNP_CUDA(cudaMemsetAsync(s->adam_m.p, 0, sizeof(float) * s->adam_m.cap, st));
        SNP_CUDA(cudaMemsetAsync(s->adam_v.p, 0, sizeof(float) * s->adam_v.cap, st));
    }
    float *dst[8] = {s->centers, s->rotations, s->scales, s->w1, s->b1, s->w2, s->b2, s->sh};
    for (int k = 0; k < 8; ++k) {
        const size_t o = s->param_off[k] / sizeof(float);
        // the semi-axes (k = 2) stay positive: their step is taken on log s
        SNP_CUDA(launch_adam(dst[k], grads[k], s->adam_m.p + o, s->adam_v.p + o, s->param_count[k], lr[k], beta1,
                             beta2, eps, step, k == 2, st));
    }
    s->state = kCreated;   // parameters changed: project again
    return SNP_OK;
}

snp_status snp_get_params(snp_scene s, float *const *dst, int32_t memory, void *cuda_stream) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!dst) return fail(SNP_ERR_INVALID_ARGUMENT, "dst is NULL");
    if (memory != SNP_MEM_HOST && memory != SNP_MEM_DEVICE)
        return fail(SNP_ERR_INVALID_ARGUMENT, "memory must be SNP_MEM_HOST or SNP_MEM_DEVICE");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const float *src[8] = {s->centers, s->rotations, s->scales, s->w1, s->b1, s->w2, s->b2, s->sh};
    for (int k = 0; k < 8; ++k) {
        if (!dst[k]) return fail(SNP_ERR_INVALID_ARGUMENT, "a destination is NULL");
        SNP_CUDA(cudaMemcpyAsync(dst[k], src[k], sizeof(float) * s->param_count[k],
                                 memory == SNP_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    }
    if (memory == SNP_MEM_HOST) SNP_CUDA(cudaStreamSynchronize(st));
    return SNP_OK;
}

snp_status snp_render_views(snp_scene s, const snp_camera *cams, int32_t n_views, const snp_render_opts *opts,
                            float *out_rgba, void *cuda_stream) {
    snp_status r = snp_project(s, cams, n_views, cuda_stream);
    if (r != SNP_OK) return r;
    r = snp_bin_sort(s, opts, cuda_stream);
    if (r != SNP_OK) return r;
    return snp_render(s, opts, out_rgba, cuda_stream);
}

snp_status snp_destroy(snp_scene s) {
    if (!s) return SNP_OK;
    cudaSetDevice(s->device);
    cudaDeviceSynchronize();
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->ev_bw_fork) cudaEventDestroy(s->ev_bw_fork);
    if (s->ev_bw_join) cudaEventDestroy(s->ev_bw_join);
    if (s->side) cudaStreamDestroy(s->side);
    s->params.release();
    s->rects.release();
    s->depth.release();
    s->records.release();
    s->w_t.release();
    s->adam_m.release();
    s->bw_queue.release();
    s->bw_scratch.release();
    s->loss_scratch.release();
    s->bw_skip.release();
    s->bw_fwd.release();
    s->grad_entries.release();
    s->rec_entries.release();
    s->tight.release();
    s->intr.release();
    s->grad_fill.release();
    s->grad_keys.release();
    s->grad_count.release();
    s->es_bsum.release();
    s->es_sorted.release();
    s->es_cnt.release();
    s->gc_acc.release();
    s->adam_v.release();
    s->keys0.release();
    s->keys1.release();
    s->vals0.release();
    s->vals1.release();
    s->dup_status.release();
    s->sort_scratch.release();
    s->ranges.release();
    s->fallback.release();
    s->tile_order.release();
    s->host_out_staging.release();
    s->counters.release();
    s->flag.release();
    if (s->h_counters) cudaFreeHost(s->h_counters);
    if (s->h_flag) cudaFreeHost(s->h_flag);
    delete s;
    return SNP_OK;
}

snp_status snp_get_binning(snp_scene s, int32_t *rects, uint32_t *depth_keys, uint64_t *sorted_keys,
                           uint32_t *sorted_ids, int64_t capacity, int64_t *n_dup, uint32_t *tile_ranges,
                           void *cuda_stream) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (s->state < kProjected) return fail(SNP_ERR_BAD_STATE, "nothing projected yet");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    SNP_CUDA(cudaStreamSynchronize(st));
    const size_t items = (size_t)s->n_views * s->n;
    if (rects && items) {
        std::vector<short4> tmp(items);
        SNP_CUDA(cudaMemcpy(tmp.data(), s->rects.p, items * sizeof(short4), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < items; ++i) {
            rects[4 * i] = tmp[i].x; rects[4 * i + 1] = tmp[i].y;
            rects[4 * i + 2] = tmp[i].z; rects[4 * i + 3] = tmp[i].w;
        }
    }
    if (depth_keys && items) SNP_CUDA(cudaMemcpy(depth_keys, s->depth.p, items * 4, cudaMemcpyDeviceToHost));
    if (s->state >= kBinned) {
        unsigned long long nd = 0;
        SNP_CUDA(cudaMemcpy(&nd, s->counters.p + kCntDup, sizeof nd, cudaMemcpyDeviceToHost));
        if (n_dup) *n_dup = (int64_t)nd;
        int64_t m = std::min<int64_t>(std::min<int64_t>((int64_t)nd, capacity), s->key_capacity);
        const uint64_t *sk = s->sorted_idx ? s->keys1.p : s->keys0.p;
        const uint32_t *sv = s->sorted_idx ? s->vals1.p : s->vals0.p;
        if (sorted_keys && m > 0) SNP_CUDA(cudaMemcpy(sorted_keys, sk, (size_t)m * 8, cudaMemcpyDeviceToHost));
        if (sorted_ids && m > 0) SNP_CUDA(cudaMemcpy(sorted_ids, sv, (size_t)m * 4, cudaMemcpyDeviceToHost));
        const size_t slots = (size_t)s->n_views * s->tiles_x * s->tiles_y;
        if (tile_ranges) SNP_CUDA(cudaMemcpy(tile_ranges, s->ranges.p, slots * 8, cudaMemcpyDeviceToHost));
    } else if (n_dup) {
        *n_dup = -1;
    }
    return SNP_OK;
}

snp_status snp_get_stats(snp_scene s, snp_stats *out, void *cuda_stream) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!out) return fail(SNP_ERR_INVALID_ARGUMENT, "out is NULL");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    SNP_CUDA(cudaMemcpyAsync(s->h_counters, s->counters.p, sizeof(unsigned long long) * kNumCounters,
                             cudaMemcpyDeviceToHost, st));
    SNP_CUDA(cudaStreamSynchronize(st));
    const unsigned long long *c = s->h_counters;
    out->n_visible = c[kCntVisible];
    out->n_dup = c[kCntDup];
    out->key_capacity = (uint64_t)s->key_capacity;
    out->tested_pairs = c[kCntTested];
    out->candidate_pairs = c[kCntCandidate];
    out->hit_pairs = c[kCntHit];
    out->composited = c[kCntComposited];
    out->overflow_pixels = c[kCntOverflow];
    out->capacity_overflow = c[kCntCapOverflow];
    out->backward_skipped = c[kCntBwdSkipped];
    out->dead_keys = c[kCntDeadKeys];
    return SNP_OK;
}

snp_status snp_get_debug_counters(snp_scene s, uint64_t *out, int32_t n, void *cuda_stream) {
    g_err.clear();
    snp_status r = check_scene(s);
    if (r != SNP_OK) return r;
    if (!out || n < 0 || n > kNumCounters) return fail(SNP_ERR_INVALID_ARGUMENT, "out is NULL or n out of range");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    SNP_CUDA(cudaMemcpyAsync(s->h_counters, s->counters.p, sizeof(unsigned long long) * kNumCounters,
                             cudaMemcpyDeviceToHost, st));
    SNP_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i) out[i] = s->h_counters[i];
    // the instrumented slots accumulate until read: clear them for the next measurement
    SNP_CUDA(cudaMemsetAsync(s->counters.p + 16, 0, sizeof(unsigned long long) * (kCntBwdQueue2 - 16), st));
    SNP_CUDA(cudaStreamSynchronize(st));
    return SNP_OK;
}

snp_status snp_set_record(snp_scene s, int32_t on) {
    g_err.clear();
    if (!s) return fail(SNP_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    s->record_mode = on != 0;
    if (!s->record_mode) s->recorded = false;
    return SNP_OK;
}

snp_status snp_set_binning(snp_scene s, int32_t flags) {
    g_err.clear();
    if (!s) return fail(SNP_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    if (flags & ~(SNP_BIN_CONIC_TILES | SNP_BIN_TILE_DEPTH)) return fail(SNP_ERR_INVALID_ARGUMENT, "unknown binning flag");
    s->bin_flags = flags;
    return SNP_OK;
}

snp_status snp_set_pending_limit(snp_scene s, int32_t k) {
    if (!s) return fail(SNP_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    if (k < 0 || k > 16) return fail(SNP_ERR_INVALID_ARGUMENT, "pending limit must be 0..16");
    s->pending_limit = k == 0 ? 16 : k;
    return SNP_OK;
}

}  // extern "C"
