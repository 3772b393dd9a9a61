// Stable LSD radix sort of (u64 key, i32 value) pairs and the run-length
// segmentation of a sorted key array: the grouping steps of the voxel map and
// the sliding window (voxmap.py:213-230 groups scan points by leaf with a
// stable lexsort; window.py:136-143 / initialize.py group and de-duplicate
// keys), on the device with no library sort.
//
// Radix sort, 8-bit digits, one pass per digit of the key bits in use:
//   k_rs_hist    per RS_TILE-element tile: the digit histogram (shared-memory
//                atomics) -> hist[digit][tile]
//   k_rs_scan    one CTA: exclusive scan of hist in digit-major order, so
//                tile t's digit-d elements go to offset[d][t] onwards
//   k_rs_scatter per tile, 8 warps x 32 RS_ITEMS consecutive elements: each warp
//                walks its chunk 32 elements at a time in order; an element's
//                rank among equal digits is the popcount of its
//                __match_any_sync peers below it plus the warp's running
//                digit count, so the pass is stable; the warp counts are
//                then prefix-summed across the tile's warps per digit.
// Segments: a flag per element where the key changes, a three-phase exclusive
// scan of the flags (tile sums, one-CTA scan, tile add) and the compaction
// of the segment starts.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lsb.h"

namespace lsb {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef LSB_RS_ITEMS
#define LSB_RS_ITEMS 4
#endif
// elements per thread: 1024-element tiles, so a scan's 100k keys spread over
// ~100 CTAs (the passes are latency-bound at these sizes, not bandwidth-bound)
constexpr int RS_ITEMS = LSB_RS_ITEMS;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;     // 1024
constexpr int RS_RADIX = 256;

__device__ __forceinline__ unsigned digit_of(uint64_t k, int shift) { return (unsigned)(k >> shift) & 0xffu; }

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                       int ntiles, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[RS_RADIX];
    for (int i = threadIdx.x; i < RS_RADIX; i += RS_THREADS) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
        const int64_t g = base + i;
        if (g < n) atomicAdd(&h[digit_of(keys[g], shift)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

// Exclusive scan of `len` counts in place (one CTA of 1024 threads; each
// thread owns a contiguous run).
constexpr int SC_THREADS = 1024;
__global__ void __launch_bounds__(SC_THREADS) k_scan_one_cta(uint32_t* __restrict__ a, int64_t len,
                                                             uint32_t* __restrict__ total) {
    __shared__ uint32_t ws[SC_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t per = (len + SC_THREADS - 1) / SC_THREADS;
    const int64_t b = tid * per, e = b + per < len ? b + per : len;
    uint32_t s = 0;
    for (int64_t i = b; i < e; ++i) s += a[i];
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < SC_THREADS / 32 ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        ws[lane] = v;
    }
    __syncthreads();
    uint32_t run = x - s + (warp ? ws[warp - 1] : 0u);
    for (int64_t i = b; i < e; ++i) {
        const uint32_t c = a[i];
        a[i] = run;
        run += c;
    }
    if (tid == SC_THREADS - 1 && total) *total = run;
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint64_t* __restrict__ kin,
                                                          const int32_t* __restrict__ vin, uint64_t* __restrict__ kout,
                                                          int32_t* __restrict__ vout, int64_t n, int shift, int ntiles,
                                                          const uint32_t* __restrict__ offs) {
    __shared__ uint32_t wc[RS_WARPS][RS_RADIX];     // per-warp digit counts, then per-warp bases
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&wc[0][0])[i] = 0;
    __syncthreads();
    const int64_t wbase = (int64_t)blockIdx.x * RS_TILE + (int64_t)warp * (32 * RS_ITEMS);
    uint64_t k[RS_ITEMS];
    int32_t v[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t g = wbase + r * 32 + lane;
        const bool ok = g < n;
        k[r] = ok ? kin[g] : 0ull;
        v[r] = ok ? (vin ? vin[g] : (int32_t)g) : 0;
        const unsigned d = digit_of(k[r], shift);
        const unsigned act = __ballot_sync(0xffffffffu, ok);
        const unsigned peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u + 0u) & act;
        const uint32_t before = wc[warp][d & 0xffu];
        __syncwarp();
        rank[r] = before + __popc(peers & lt);
        const int leader = 31 - __clz(peers ? peers : 1u);       // highest peer lane updates the count
        if (ok && lane == leader) wc[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: prefix of the warp counts (warps in order) + the tile's global offset
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) {
        uint32_t run = offs[(int64_t)d * ntiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const uint32_t c = wc[w][d];
            wc[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t g = wbase + r * 32 + lane;
        if (g >= n) continue;
        const uint32_t pos = wc[warp][digit_of(k[r], shift)] + rank[r];
        kout[pos] = k[r];
        vout[pos] = v[r];
    }
}

size_t sort_temp_bytes(int64_t n) {
    const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    const size_t a = ((size_t)(n > 0 ? n : 1) * 8 + 255) & ~(size_t)255;
    const size_t b = ((size_t)(n > 0 ? n : 1) * 4 + 255) & ~(size_t)255;
    const size_t h = ((size_t)RS_RADIX * (ntiles > 0 ? ntiles : 1) * 4 + 255) & ~(size_t)255;
    return a + b + h + 256;
}

// keys_out / vals_out receive the sorted pairs; vals_in NULL means 0..n-1.
cudaError_t launch_sort_pairs(const uint64_t* keys_in, const int32_t* vals_in, uint64_t* keys_out, int32_t* vals_out,
                              int64_t n, int key_bits, void* temp, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
    const int ntiles = (int)((n + RS_TILE - 1) / RS_TILE);
    char* t = (char*)temp;
    uint64_t* kb = (uint64_t*)t;
    t += ((size_t)n * 8 + 255) & ~(size_t)255;
    int32_t* vb = (int32_t*)t;
    t += ((size_t)n * 4 + 255) & ~(size_t)255;
    uint32_t* hist = (uint32_t*)t;
    // ping-pong so that the last pass writes keys_out / vals_out
    const uint64_t* ksrc = keys_in;
    const int32_t* vsrc = vals_in;
    for (int p = 0; p < passes; ++p) {
        const bool to_out = ((passes - 1 - p) & 1) == 0;
        uint64_t* kd = to_out ? keys_out : kb;
        int32_t* vd = to_out ? vals_out : vb;
        k_rs_hist<<<ntiles, RS_THREADS, 0, st>>>(ksrc, n, 8 * p, ntiles, hist);
        k_scan_one_cta<<<1, SC_THREADS, 0, st>>>(hist, (int64_t)RS_RADIX * ntiles, nullptr);
        k_rs_scatter<<<ntiles, RS_THREADS, 0, st>>>(ksrc, vsrc, kd, vd, n, 8 * p, ntiles, hist);
        ksrc = kd;
        vsrc = vd;
    }
    return cudaGetLastError();
}

// ---- segments of a sorted key array ------------------------------------------
constexpr int SG_TILE = 1024;
__global__ void __launch_bounds__(RS_THREADS) k_seg_count(const uint64_t* __restrict__ k, int64_t n,
                                                         uint32_t* __restrict__ tile_cnt) {
    __shared__ uint32_t c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    uint32_t mine = 0;
    const int64_t base = (int64_t)blockIdx.x * SG_TILE;
    for (int i = threadIdx.x; i < SG_TILE; i += RS_THREADS) {
        const int64_t g = base + i;
        if (g < n && (g == 0 || k[g] != k[g - 1])) ++mine;
    }
    atomicAdd(&c, mine);
    __syncthreads();
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = c;
}

__global__ void __launch_bounds__(RS_THREADS) k_seg_emit(const uint64_t* __restrict__ k, int64_t n,
                                                        const uint32_t* __restrict__ tile_off,
                                                        int64_t* __restrict__ starts) {
    // ordered compaction inside the tile: warps take 32-element rounds in order
    __shared__ uint32_t wsum[RS_WARPS];
    __shared__ uint32_t run_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) run_base = tile_off[blockIdx.x];
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SG_TILE;
    for (int r0 = 0; r0 < SG_TILE; r0 += RS_THREADS) {
        const int64_t g = base + r0 + threadIdx.x;
        const bool f = g < n && (g == 0 || k[g] != k[g - 1]);
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[warp] = __popc(b);
        __syncthreads();
        uint32_t off = run_base;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        if (f) starts[off + __popc(b & ((1u << lane) - 1u))] = g;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < RS_WARPS; ++w) t += wsum[w];
            run_base += t;
        }
        __syncthreads();
    }
}

cudaError_t launch_segments(const uint64_t* keys, int64_t n, int64_t* starts, int64_t* nseg, void* temp,
                            cudaStream_t st) {
    if (n <= 0) return cudaMemsetAsync(nseg, 0, sizeof(int64_t), st);
    const int ntiles = (int)((n + SG_TILE - 1) / SG_TILE);
    uint32_t* cnt = (uint32_t*)temp;
    uint32_t* total = cnt + ntiles;
    k_seg_count<<<ntiles, RS_THREADS, 0, st>>>(keys, n, cnt);
    k_scan_one_cta<<<1, SC_THREADS, 0, st>>>(cnt, ntiles, total);
    k_seg_emit<<<ntiles, RS_THREADS, 0, st>>>(keys, n, cnt, starts);
    // nseg (int64) from the u32 total
    cudaError_t e = cudaMemsetAsync(nseg, 0, sizeof(int64_t), st);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(nseg, total, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
}

}  // namespace lsb
