// snp_internal.cuh -- shared definitions of the CUDA path (product code).
// Nothing here is shared with oracle/: the two sides are independent.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/snp.h"

// Device-side invariant checks, compiled in only for the checked A/B build
// (tools/ab_build.py checked -DSNP_CHECKS): index bounds of every shared-memory ring,
// queue and global array the kernels address, plus protocol invariants.  A failed
// check traps with file/line.  (compute-sanitizer is not available on the GPU pool.)
#ifdef SNP_CHECKS
#include <assert.h>
#define SNP_CHECK(cond) assert(cond)
#else
#define SNP_CHECK(cond) ((void)0)
#endif

namespace snp {

// Launch with the device's greatest scheduling priority.  Used for the K2-K4 chain
// (latency-bound, on the frame's critical path) so that its CTAs take SM slots
// ahead of the concurrently running K1b (side stream, default priority).
// The launch is also a programmatic dependent launch: the kernel may be scheduled
// while its predecessor in the stream still runs, so every kernel launched this way
// starts with pdl_prologue() before touching global memory.
int greatest_priority();
__device__ __forceinline__ void pdl_prologue() {
    // wait for the predecessor grid (complete, memory visible), then let the next
    // grid in the stream be scheduled (it waits in its own prologue)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
cudaError_t launch_hi(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = greatest_priority();
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr int kTile = 16;                 // BASELINE north_star: 16x16 tiles (R18)
constexpr int kHidden = 8;                // N_sigma = 8, the paper's width
// Supported widths N_sigma: every N-dependent kernel is a template
// instantiated for these; N = 8 is the measured configuration.
__host__ __device__ constexpr bool hidden_supported(int N) { return N == 4 || N == 8 || N == 16 || N == 32; }
constexpr int kCamsPerLaunch = 32;        // cameras passed by value per launch
// Largest scene: K5's pending entries carry the primitive id in 24 bits beside an
// 8-bit code of t_in's low part (render.cu, tin_code).
constexpr int64_t kMaxPrims = (1 << 24) - 1;
// float4 per render record: 6 (conic, colour, centre, whitening) + N units + N/4 for W2
// = 11 / 16 / 26 / 46 for N = 4 / 8 / 16 / 32 (256 B at N = 8)
__host__ __device__ constexpr int rec_f4(int N) { return 6 + N + N / 4; }
// Key = view << (tile_bits + 19) | tile << 19 | (bits(L) >> 12): the depth code is
// the fp32 lower bound L truncated to 11 mantissa bits (still a lower bound, R19).
constexpr int kDepthBits = 19;
constexpr int kDepthDrop = 12;
constexpr uint64_t kDeadKey = ~0ull;   // K2, tight binning: a key of a tile the silhouette misses
__host__ __device__ __forceinline__ float key_depth(uint64_t key) {
    const uint32_t c = ((uint32_t)key & ((1u << kDepthBits) - 1u)) << kDepthDrop;
#ifdef __CUDA_ARCH__
    return __uint_as_float(c);
#else
    float f;
    __builtin_memcpy(&f, &c, 4);
    return f;
#endif
}

// Camera as the kernels see it (by value in the launch parameters).
struct DevCam {
    float R[9];      // world-from-camera, row-major
    float C[3];
    float fx, fy, cx, cy;
    int32_t W, H;
    float t_near, t_far;
    double ifx, ify;  // 1 / fx, 1 / fy (host-computed: no FP64 division per pixel ray)
    float xi_t;       // timestamp of this view (temporal scenes, R24)
};

struct CamBatch {
    int32_t view0;   // global index of cams[0]
    int32_t nv;      // cameras in this launch
    DevCam cams[kCamsPerLaunch];
};

// Render record of one (view, primitive), 16 float4:
//  f4[0]  = x0, y0, a, 2b        silhouette conic, pixel space, margin folded in:
//  f4[1]  = c, r, g, b           candidate iff a dx^2 + 2b dx dy + c dy^2 <= 1
//  f4[2]  = mh.x, mh.y, mh.z, b2 m = mu - C (world) as hi + lo floats
//  f4[3]  = ml.x, ml.y, ml.z, Wh00
//  f4[4]  = Wh01, Wh02, Wh10, Wh11   Wh = diag(1/s) R^T (world -> unit-sphere frame)
//  f4[5]  = Wh12, Wh20, Wh21, Wh22
//  f4[6+k]= W1'_k.x, W1'_k.y, W1'_k.z, omega*b1_k   W1'_k = omega W1_k / ||s||_inf  (k < N)
//  f4[6+N+j] = W2_{4j..4j+3}                        (j < N/4)
// (N hidden units; rec_f4(N) float4 in all)
enum RecordSlot { kRecConic = 0, kRecConicRgb = 1, kRecMh = 2, kRecMl = 3, kRecWh0 = 4,
                  kRecWh1 = 5, kRecUnits = 6 };
__host__ __device__ constexpr int rec_w2(int N) { return kRecUnits + N; }

// Device-side counters (one 64-bit slot each), see snp_stats.
// The render counters kCntTested..kCntRenderLast are contiguous: K4 clears them for the
// first render after a binning (a further render of the same binning clears them with
// one memset).  kCntVisibleAcc is K1a's accumulator, moved to kCntVisible (and cleared)
// by K2's last block.  No memset node in a project -> bin_sort -> render frame.
enum Counter { kCntVisible = 0, kCntDup = 1, kCntCapOverflow = 2, kCntTested = 3, kCntCandidate = 4, kCntHit = 5,
               kCntComposited = 6, kCntOverflow = 7, kCntFallbackQueue = 8, kCntTileQueue = 9,
               kCntFallbackClaim = 10, kCntK5Done = 11, kCntBigQueue = 12, kCntRenderLast = kCntBigQueue,
               kCntVisibleAcc = 13, kCntBwdSkipped = 14, kCntBwdQueue = 15,
               kCntGraze = 48,          // cumulative until the debug readback
               kCntBwdQueue2 = 49,      // K7: pixels for its second (2048-hit) pass
               kCntBwdQueue3 = 50,      // K7: pixels for the global-memory pass
               kCntGradEntries = 51,    // K5 grad mode: entry chunks reserved
               kCntGradOverflow = 52,   // K5 grad mode: the entry buffer overflowed
               kCntDeadKeysAcc = 53,    // K2, tight binning: keys of tiles the silhouette misses
               kCntDeadKeys = 54,       //   (moved here by K4, which clears the accumulator)
               kNumCounters = 56 };     // 16..47: instrumented (A/B) builds only, cleared by the debug readback

struct ProjectArgs {
    int64_t n;
    int32_t n_hidden;       // N_sigma (hidden_supported)
    int32_t sh_degree;
    float omega;
    const float *centers, *rotations, *scales, *w1, *b1, *w2, *b2, *sh;
    const float *w_t;       // [n][N] temporal weights, or nullptr (static scene)
    int32_t tiles_x, tiles_y;
    short4 *rects;          // [V*n] tile rect or (-1,-1,-1,-1)
    uint32_t *depth;        // [V*n] fp32 bits of the depth lower bound
    float4 *tight;          // [V*n][4] tight binning data (nullptr: rect binning), see k_bin_geom
    float4 *intr;           // [V] (1/fx, 1/fy, cx, cy) for K2's per-tile depth bounds (with tight)
    float4 *records;        // [V*n*16]
    unsigned long long *counters;
};

// ---- host-side launchers (each .cu owns its kernels) ----
cudaError_t launch_validate(const ProjectArgs &a, int *d_bad, cudaStream_t st);
cudaError_t launch_validate_finite(const float *v, int64_t count, int *d_bad, cudaStream_t st);
// K1a: cull + tile rect + depth key (critical path).  K1b: render records of the
// visible pairs (reads K1a's rects; may run concurrently with K2-K4).
cudaError_t launch_bin_geom(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st);
cudaError_t launch_records(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st);

struct BinArgs {
    int64_t n;              // primitives per view
    int32_t n_views;
    int32_t tiles_x, tiles_y, tile_bits;
    int32_t row_begin, row_stride;
    const short4 *rects;    // [V*n]
    const uint32_t *depth;  // [V*n]
    const float4 *tight;    // [V*n][4] or nullptr (SURVEY 8(f)3 tight binning, bin_flags)
    const float4 *intr;     // [V] (1/fx, 1/fy, cx, cy)
    int32_t bin_flags;      // SNP_BIN_CONIC_TILES | SNP_BIN_TILE_DEPTH
    uint64_t *keys;         // [capacity]
    uint32_t *vals;         // [capacity]
    int64_t capacity;
    unsigned long long *dup_status;   // [num_blocks + 1]: look-back states of the K2 blocks + ticket;
                                      // zero on entry, cleared again by K4
    unsigned long long *counters;
    uint32_t *hist;         // [passes][256] digit histograms accumulated during duplication
                            // (zero on entry, cleared again by K4)
    int32_t passes;
    uint32_t *ranges;       // [n_slots][2] tile ranges, zeroed by K2 (filled by K4)
    int64_t n_slots;
};
int64_t bin_scan_blocks(int64_t items);
// K2, one pass: keys + values (up to capacity), digit histograms, counters[kCntDup]
cudaError_t launch_dup(const BinArgs &a, cudaStream_t st);
// K4 (also clears b.dup_status and b.hist for the next frame)
cudaError_t launch_tile_ranges(const uint64_t *keys, const unsigned long long *counters, int64_t capacity,
                               int32_t tile_bits, int32_t tiles, uint32_t *ranges, const BinArgs &b,
                               cudaStream_t st);

struct SortScratch {
    uint32_t *hist;         // [passes][256]
    uint32_t *lookback;     // [8][max_partitions][256]; region 0 is zero on entry, pass p
                            // zeroes region (p+1) % passes (region 0 again after the last pass)
    uint32_t *tickets;      // [passes]
    int64_t max_partitions;
};
int64_t sort_partition_size();
size_t sort_scratch_words(int passes, int64_t max_partitions);
// Sorts keys/vals (n read from counters[kCntDup], clamped to capacity) by bits
// [0, 8*passes).  Ping-pongs between (k0,v0) and (k1,v1); returns in *final_idx
// which buffer (0 or 1) holds the result.  expected_n (the last host-known key
// count, or 0) only sizes the persistent grid.
cudaError_t launch_onesweep(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1, int64_t capacity,
                            const unsigned long long *counters, int passes, SortScratch scratch,
                            int64_t expected_n, cudaStream_t st, int *final_idx);

// K5 grad mode (the backward's forward traversal): one entry per composited hit, its
// dL/dI and dL/dc, from which K7f computes the parameter gradients
// K5 grad mode: a consumer warp writes its entries to a chunk of this many, reserved with
// one global atomic (>= the 32 x kPend entries one emission call can produce)
constexpr int kGradChunk = 1024;

// K5 record mode (training: the forward render also records its composited hits, so that
// the backward needs no second traversal): per hit the transmittance in front of it, its
// kappa and the colour accumulated up to and including it
struct FwdEntry {
    uint32_t pix;      // view within the camera batch << 24 | y * W + x
    uint32_t id;       // primitive
    float T, kap, cr, cg, cb, pad;
};

struct GradEntry {
    uint32_t pix;      // view within the camera batch << 24 | y * W + x
    uint32_t id;       // primitive
    float gI, gc0, gc1, gc2;
};

struct RenderArgs {
    int32_t n_hidden;              // N_sigma (hidden_supported): selects the kernel instantiation
    int32_t colour_ray;            // 1: SH colour at each pixel's ray direction (SNP_COLOUR_RAY)
    int32_t eager_emit;            // K5 blends after every exact round (not only near-full lists)
    const float *sh;               // scene SH coefficients [n][16][3] (per-ray colour)
    int32_t sh_degree;
    const float *centers;          // scene centres [n][3] (FP64 grazing branch)
    const float *scales;           // scene semi-axes [n][3] (FP64 grazing branch, backward)
    const float *rotations;        // scene quaternions [n][4] (FP64 grazing branch, backward)
    uint32_t *bw_queue;            // [3][V*H*W] K7's pixel queues (K5 grad overflow, > 256, > 2048 hits)
    uint32_t *bw_skip;             // [V*H*W] composited hits of a pixel K5's grad mode already emitted
    const float4 *grad_in;         // K5 grad mode: dL/d(out RGBA) [V][H][W]
    const float4 *fwd;             // K5 grad mode: the forward's out RGBA [V][H][W]
    GradEntry *grad_entries;       // K5 grad mode: entry buffer, grad_chunks chunks of kGradChunk
    int32_t *grad_fill;            //   entries used per chunk
    uint32_t *grad_keys;           //   per slot: vloc * n + primitive (K7s)
    FwdEntry *rec_entries;         // K5 record mode: entry buffer (same chunks, fills and keys)
    int32_t record;                // K5: record the composited hits (forward render)
    int32_t from_fwd;              // K7s: the entries are rec_entries (no grad-mode traversal)
    uint32_t *grad_count;          //   [nv * n] entries per key -> offsets (K7s; zeroed per batch)
    int64_t grad_chunks;
    float4 *gc_acc;                // K7f, primitive colour mode: [batch views][n] summed dL/dc
    int32_t tiles_x, tiles_y, tiles_per_view;
    int32_t tile_bits;
    int32_t row_begin, row_stride, stripe_rows;
    int64_t n;                     // primitives per view (record index = view*n + id)
    const float4 *records;
    const uint64_t *keys;          // sorted
    const uint32_t *vals;          // sorted primitive ids
    const uint32_t *ranges;        // [V*T][2]
    float bg[3];
    float t_floor;
    int32_t pending_limit;
    int32_t debug_flags;           // SNP_DEBUG env bits (1: no sub-tile culling); 0 in production
    float *out;                    // [V][H][W][4]
    unsigned long long *fallback;  // [2 x capacity] overflowed pixels: 1 << 63 | view << 32 | pixel; 0 = empty
                                   // (K6w clears every entry it consumes: all zero between renders); the
                                   // second half lists the pixels with more hits than K6w holds (count in
                                   // counters[kCntBigQueue]) for the block-wide K6
    int64_t fallback_capacity;
    const uint32_t *tile_order;    // K5 claims tiles in this order (heaviest list first)
    int32_t k5_grid;               // K5's CTA count (K6 overlapping K5 waits for that many exits)
    unsigned long long *counters;
};
// LPT order of one camera batch's (view, stripe tile) slots into order[]: descending
// tile-list length (8 buckets per octave), so that K5's dynamic queue ends on light tiles
cudaError_t launch_tile_order(const RenderArgs &a, const CamBatch &cams, uint32_t *order, cudaStream_t st);
// reset_queue: zero the tile queue first (needed for every camera batch after the
// first; the caller zeroes all render counters once per snp_render)
cudaError_t launch_render(const RenderArgs &a, const CamBatch &cams, bool reset_queue, cudaStream_t st);
// K6.  With one camera batch it overlaps K5: its CTAs start on the SMs K5's finished
// CTAs leave, take overflowed pixels as K5 queues them and end once every K5 CTA has
// exited.  With several batches it runs after all of them.
cudaError_t launch_fallback(const RenderArgs &a, const CamBatch *cams, int n_batches, cudaStream_t st);
int render_grid(int n_hidden, bool colour_ray, bool eager, int tiles);
// K7 (backward.cu): adds dL/d{W1, b1, W2, b2, SH} for grad = dL/d(out RGBA) of one camera
// batch, re-deriving each pixel's forward (whole image; counters[kCntBwdSkipped] counts
// pixels with more hits than the kernel holds)
struct BackwardGrads {
    float *w1, *b1, *w2, *b2, *sh;
    float *mu, *q, *s;             // geometry gradients, or all nullptr (not computed)
    float *wt;                     // temporal weights' gradient [n][N], or nullptr
    bool vec;                      // every array 16-byte aligned: vector (float4) atomics
};
// K7s: the K5-path entries grouped by key vloc * n + primitive (a counting sort over
// RenderArgs::grad_keys, which K5 writes, with RenderArgs::grad_count)
struct EntrySort {
    uint32_t *bsum;                // [ceil(nv n / 4096)] scan block sums
    uint32_t *sorted;              // [grad_chunks * kGradChunk] entry slots in key order
    unsigned long long *cnt;       // cnt[kCntDup] = entries
};
// k5: K7f (es: sorted, K7s; nullptr: in slot order) over the K5 entries on st, and the
// per-pixel K7 for the pixels K5 queued on st_pix (the caller forks and joins; st_pix may
// be st); !k5: the per-pixel K7 for every pixel (on st_pix)
cudaError_t launch_backward(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                            float omega, void *scratch, bool k5, const EntrySort *es, cudaStream_t st,
                            cudaStream_t st_pix);
// K5 in grad mode over one camera batch (render.cu): the forward traversal emitting
// GradEntry per composited hit; overflowing pixels go to bw_queue with their skip count
cudaError_t launch_render_grad(const RenderArgs &a, const CamBatch &cams, cudaStream_t st);
size_t backward_scratch_bytes();   // K7's global-memory pass (pixels with > 2048 hits)
// train.cu: L1 loss + gradient, std(s) regulariser, Adam
cudaError_t launch_l1(const float *out_rgba, const float *target_rgb, int64_t n, float *grad_rgba, float *loss,
                      cudaStream_t st);
cudaError_t launch_scale_reg(const float *s, int64_t n, float w, float *grad_s, float *loss, cudaStream_t st);
size_t loss_3dgs_scratch_floats(int V, int H, int W);
// (norm_total: the pixel count the means divide by -- V H W, or the whole step's when the
//  step's views are taken in parts)
cudaError_t launch_loss_3dgs(const float *out_rgba, const float *target_rgb, int V, int H, int W, float lam,
                             float *grad_rgba, float *loss, float *scratch, int64_t norm_total, cudaStream_t st);
cudaError_t launch_adam(float *p, const float *g, float *m, float *v, int64_t count, float lr, float b1, float b2,
                        float eps, int step, bool log_space, cudaStream_t st);   // K5's persistent grid for `tiles` work units

}  // namespace snp
