// sort.cu -- K3: hand-written onesweep LSD radix sort of (u64 key, u32 value)
// pairs, 8-bit digits, stable (BASELINE north_star: "a hand-written onesweep
// LSD radix sort over 64-bit tile|depth keys").  Realises the tile-granular
// part of "depth-sorted"; the exact per-ray order is restored in K5.
//
// Structure: the digit histograms of every pass are accumulated by K2 while it
// duplicates the keys; then one k_pass launch per 8-bit digit (LSD first):
//   k_pass : persistent CTAs (grid <= resident CTAs, partition c, c + G, ... in
//            order, so every partition a look-back waits on is resident); per
//            partition of kPart keys: stable warp ranking from 8 ballots, per-digit
//            decoupled look-back over the earlier partitions (windows of 24 loads),
//            shuffle into block-sorted order in shared memory, coalesced-run scatter.
//            Each pass also clears the look-back region of the next one.
#include "snp_internal.cuh"

namespace snp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef SNP_SORT_IPT
#define SNP_SORT_IPT 12
#endif
constexpr int kIpt = SNP_SORT_IPT;           // keys per thread
constexpr int kPart = kThreads * kIpt;       // 3072 keys per partition
constexpr int kWarpKeys = kPart / kWarps;    // 384 keys per warp (warp-striped)
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1u;

__device__ __forceinline__ int64_t sort_n(const unsigned long long *counters, int64_t capacity) {
    int64_t n = (int64_t)counters[kCntDup];
    return n > capacity ? capacity : n;
}

#ifdef SNP_SORT_INSTRUMENT
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
    return *reinterpret_cast<const volatile uint32_t *>(p);
}

__global__ void __launch_bounds__(kThreads) k_pass(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                   uint64_t *__restrict__ kout, uint32_t *__restrict__ vout,
                                                   int64_t capacity, const unsigned long long *counters, int pass,
                                                   const uint32_t *hist, uint32_t *lookback, uint32_t *zero_next,
                                                   int64_t zero_words) {
    pdl_prologue();
    __shared__ uint64_t s_keys[kPart];
    __shared__ uint32_t s_vals[kPart];
    __shared__ uint32_t s_wh[kWarps][256];     // per-warp digit counts -> per-warp exclusive offsets
    __shared__ uint32_t s_goff[256];           // global start of digit (over all keys)
    __shared__ uint32_t s_bstart[256];         // block-local start of digit
    __shared__ uint32_t s_excl[256];           // keys of this digit in earlier partitions
    __shared__ uint32_t s_scan[kWarps];

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int shift = 8 * pass;
    // clear the look-back region of the next pass (no memset node between passes)
    for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < zero_words; j += (int64_t)gridDim.x * kThreads)
        zero_next[j] = 0u;
    const int64_t n = sort_n(counters, capacity);
    const int64_t nparts = (n + kPart - 1) / kPart;
    // Persistent: CTA c takes partitions c, c + G, ... in increasing order; the grid
    // never exceeds the co-resident CTA count, so every partition a look-back waits
    // on is owned by a running CTA that never waits on a later one (no deadlock).
#ifdef SNP_SORT_INSTRUMENT
    unsigned long long _t0 = gtimer(), _t1 = 0, _t2 = 0, _t3 = 0;
    if (threadIdx.x == 0) atomicMax(const_cast<unsigned long long *>(counters) + 16 + 3 * pass, ~_t0);
#endif
    for (int64_t part = blockIdx.x; part < nparts; part += gridDim.x) {
    for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) (&s_wh[0][0])[i] = 0;
    const int64_t pbase = part * kPart;

    // ---- load (warp-striped: item k of lane l is key pbase + wid*384 + k*32 + l)
    uint64_t key[kIpt];
    uint32_t val[kIpt];
    uint32_t rank[kIpt];
#pragma unroll
    for (int k = 0; k < kIpt; ++k) {
        const int64_t idx = pbase + wid * kWarpKeys + k * 32 + lane;
        if (idx < n) {
            key[k] = kin[idx];
            val[k] = vin[idx];
        } else {
            key[k] = ~0ull;  // digit 255, placed after every valid key of this partition
            val[k] = 0;
        }
    }
    __syncthreads();   // s_wh zeroed (and the previous partition's smem reads are done)
#ifdef SNP_SORT_INSTRUMENT
    _t1 = gtimer();
#endif
    // ---- stable warp ranking: peers with the same digit from 8 ballots (no MATCH)
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kIpt; ++k) {
        const uint32_t d = (uint32_t)(key[k] >> shift) & 255u;
        uint32_t peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bal : ~bal;
        }
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader) {
            base = s_wh[wid][d];
            s_wh[wid][d] = base + __popc(peers);
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        rank[k] = base + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();
#ifdef SNP_SORT_INSTRUMENT
    _t2 = gtimer();
#endif
    // ---- per digit: exclusive over warps, block count, block-local digit start
    const int d = threadIdx.x;  // kThreads == 256 == radix
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        uint32_t c = s_wh[w][d];
        s_wh[w][d] = cnt;
        cnt += c;
    }
    // invalid tail keys (digit 255) must not be published
    if (d == 255) {
        const int64_t valid = n - pbase < kPart ? n - pbase : kPart;
        cnt -= (uint32_t)(kPart - valid);
    }
    // publish aggregate early, then decoupled look-back
    uint32_t *lb = lookback;   // this pass's look-back words [partition][digit]
    if (part == 0) {
        atomicExch(lb + d, kFlagInc | cnt);
        s_excl[d] = 0;
    } else {
        atomicExch(lb + part * 256 + d, kFlagAgg | cnt);
        // look back over windows of kWin predecessors (kWin independent loads per L2 round trip)
        constexpr int kWin = 24;
        uint32_t sum = 0;
        int64_t q = part - 1;
        bool found = false;
        while (!found) {
            uint32_t v[kWin];
#pragma unroll
            for (int w = 0; w < kWin; ++w) v[w] = (q - w >= 0) ? ld_volatile(lb + (q - w) * 256 + d) : kFlagInc;
            int w = 0;
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                if (w != k) continue;                    // stopped earlier in this window
                if ((v[k] & ~kValMask) == 0) break;      // not yet published: re-poll from here
                sum += v[k] & kValMask;
                ++w;
                if (v[k] & kFlagInc) { found = true; break; }
            }
            q -= w;
        }
        atomicExch(lb + part * 256 + d, kFlagInc | (sum + cnt));
        s_excl[d] = sum;
    }
#ifdef SNP_SORT_INSTRUMENT
    __syncthreads();
    _t3 = gtimer();
#endif
    // block-wide exclusive scan of cnt over digits (d = threadIdx.x); the tail
    // correction above only shrinks digit 255, the last, so starts are unaffected
    {
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_scan[wid] = x;
        __syncthreads();
        uint32_t before = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) before += (w < wid) ? s_scan[w] : 0u;
        s_bstart[d] = before + x - cnt;
        // global digit offsets: exclusive scan of hist[pass][*]
        const uint32_t hv = hist[pass * 256 + d];
        uint32_t y2 = hv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t z = __shfl_up_sync(0xffffffffu, y2, o);
            if (lane >= o) y2 += z;
        }
        __syncthreads();
        if (lane == 31) s_scan[wid] = y2;
        __syncthreads();
        uint32_t b2 = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) b2 += (w < wid) ? s_scan[w] : 0u;
        s_goff[d] = b2 + y2 - hv;
    }
    __syncthreads();
    // ---- shuffle into block-sorted order in shared memory
#pragma unroll
    for (int k = 0; k < kIpt; ++k) {
        const uint32_t dd = (uint32_t)(key[k] >> shift) & 255u;
        const uint32_t pos = s_bstart[dd] + s_wh[wid][dd] + rank[k];
        s_keys[pos] = key[k];
        s_vals[pos] = val[k];
    }
    __syncthreads();
    // ---- scatter runs of equal digits to their global positions
    const int valid = (int)(n - pbase < kPart ? n - pbase : kPart);
    for (int i = threadIdx.x; i < valid; i += kThreads) {
        const uint64_t kk = s_keys[i];
        const uint32_t dd = (uint32_t)(kk >> shift) & 255u;
        const uint32_t dest = s_goff[dd] + s_excl[dd] + (uint32_t)i - s_bstart[dd];
        SNP_CHECK((int64_t)dest < n);
        kout[dest] = kk;
        vout[dest] = s_vals[i];
    }
    __syncthreads();   // smem reuse by the next partition of this CTA
#ifdef SNP_SORT_INSTRUMENT
    if (threadIdx.x == 0) {
        unsigned long long *c = const_cast<unsigned long long *>(counters);
        const unsigned long long t4 = gtimer();
        atomicAdd(c + 28, _t1 - _t0);
        atomicAdd(c + 29, _t2 - _t1);
        atomicAdd(c + 30, _t3 - _t2);
        atomicAdd(c + 31, t4 - _t3);
        atomicMax(c + 17 + 3 * pass, t4);
        atomicMax(c + 18 + 3 * pass, 1ull);
        _t0 = t4;
    }
#endif
    }
}

}  // namespace

int64_t sort_partition_size() { return kPart; }

size_t sort_scratch_words(int passes, int64_t max_partitions) {
    return (size_t)passes * 256 + (size_t)passes * (size_t)max_partitions * 256 + (size_t)passes;
}

cudaError_t launch_onesweep(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1, int64_t capacity,
                            const unsigned long long *counters, int passes, SortScratch sc,
                            int64_t expected_n, cudaStream_t st, int *final_idx) {
    *final_idx = 0;
    if (capacity == 0 || passes == 0) return cudaSuccess;
    const int64_t maxp = (capacity + kPart - 1) / kPart;
    if (maxp > sc.max_partitions) return cudaErrorInvalidValue;
    static int res[64] = {};   // per device
    int dev = 0;
    cudaGetDevice(&dev);
    int &resident = res[dev < 64 ? dev : 0];
    if (!resident) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass, kThreads, 0);
        resident = (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 1);
    }
    cudaError_t e;
    // persistent partitions: any grid size is correct; size it for the expected key
    // count so that idle CTAs do not hold SM slots that concurrent work (K1b) could use
    int64_t want = expected_n > 0 ? (expected_n + kPart - 1) / kPart : maxp;
    if (want > maxp) want = maxp;
    const unsigned grid = (unsigned)(want < resident ? want : resident);
    const size_t region = (size_t)sc.max_partitions * 256;   // look-back words per pass (fixed layout)
    uint64_t *kin = k0, *kout = k1;
    uint32_t *vin = v0, *vout = v1;
    for (int p = 0; p < passes; ++p) {
        e = launch_hi(k_pass, dim3(grid), dim3(kThreads), 0, st, kin, vin, kout, vout, capacity, counters, p, sc.hist,
                      sc.lookback + (size_t)p * region, sc.lookback + (size_t)((p + 1) % passes) * region,
                      (int64_t)region);
        if (e != cudaSuccess) return e;
        uint64_t *tk = kin; kin = kout; kout = tk;
        uint32_t *tv = vin; vin = vout; vout = tv;
    }
    *final_idx = passes & 1;
    return cudaGetLastError();
}

}  // namespace snp
