// Sliding-window maintenance on the device (window.py:136-276): the live
// window stays in HBM as the f32 SoA arena the renderer reads, the global
// map's Gaussians live in a device row store indexed by the leaf's gid
// (lsb_voxmap.gslot), and a maintain step is a handful of kernels:
//
//   hash_build  window hash: packed key -> slot, rebuilt from the live keys
//   mark        FoV keys probe it: live ∩ FoV marks `keep`, the rest are adds
//   plan        one CTA: deleted slots (ascending) and the compaction moves —
//               the reference's rear-pointer loop (window.py:151-181) has the
//               closed form "the i-th deleted slot below the new live count
//               takes the i-th live slot at or above it, counted from the
//               rear", so every move is independent
//   to_map      write-back of deleted rows into the map store (window.py:145)
//   move        the compaction moves
//   leaf_gids   map lookup of the (sorted, capacity-trimmed) adds
//   from_map    ordered append of the adds that hold a Gaussian (window.py:183)
//
// Window keys are "order keys": ((ix+2^20) << 42) | ((iy+2^20) << 21) |
// (iz+2^20), so integer order is the reference's sorted VoxelKey order.
#include <cuda_runtime.h>

#include "common.cuh"
#include "voxkey.cuh"

namespace lsb {

__device__ __forceinline__ void okey_unpack(long long k, long long& ix, long long& iy, long long& iz) {
    ix = ((k >> (2 * KB)) & (long long)KMASK) - KOFF;
    iy = ((k >> KB) & (long long)KMASK) - KOFF;
    iz = (k & (long long)KMASK) - KOFF;
}

__device__ __forceinline__ unsigned long long whash(unsigned long long k, unsigned long long mask) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k & mask;
}

#define GRID_STRIDE(i, n) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_win_hash_build(const int64_t* __restrict__ wkeys, int64_t n, unsigned long long* hk, int32_t* hs,
                                 int64_t hcap) {
    const unsigned long long mask = (unsigned long long)hcap - 1;
    GRID_STRIDE(s, n) {
        const unsigned long long k = (unsigned long long)wkeys[s];
        unsigned long long h = whash(k, mask);
        for (int64_t probe = 0; probe < hcap; ++probe) {
            const unsigned long long prev = atomicCAS(&hk[h], EMPTY, k);
            if (prev == EMPTY || prev == k) {
                hs[h] = (int32_t)s;
                break;
            }
            h = (h + 1) & mask;
        }
    }
}

__global__ void k_win_mark(const unsigned long long* __restrict__ hk, const int32_t* __restrict__ hs, int64_t hcap,
                           const int64_t* __restrict__ fov, int64_t m, uint8_t* keep, uint8_t* is_add) {
    const unsigned long long mask = (unsigned long long)hcap - 1;
    GRID_STRIDE(i, m) {
        const unsigned long long k = (unsigned long long)fov[i];
        unsigned long long h = whash(k, mask);
        int32_t slot = -1;
        for (int64_t probe = 0; probe < hcap; ++probe) {
            const unsigned long long cur = hk[h];
            if (cur == k) {
                slot = hs[h];
                break;
            }
            if (cur == EMPTY) break;
            h = (h + 1) & mask;
        }
        if (slot >= 0) keep[slot] = 1;
        is_add[i] = slot < 0 ? 1 : 0;
    }
}

// Block-wide exclusive scan of one int per thread (1024 threads).

// The compaction plan as three multi-CTA passes over tiles of PLAN_TILE
// slots (a one-CTA pass over the whole window was bound by one SM: ~160 us
// per maintain): per tile the count of deleted slots, one CTA's exclusive
// scan of the tile counts (k = their total), and per tile the emission:
// dels = deleted slots ascending (k of them; the first h lie below the new
// live count nk = n - k and are the holes), movers[r] = the r-th live slot
// >= nk counted from the rear, counts = [k, h] with h = deleted slots below
// nk (added per tile: integer atomics, order-free).
constexpr int PLAN_TILE = 1024;
constexpr int APPEND_TILE = 256;

// Exclusive block scan for any block size that is a multiple of 32 (<= 1024).
__device__ __forceinline__ int block_scan_n(int v, int* s_w, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int y = lane < nw ? s_w[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        s_w[lane] = y;
    }
    __syncthreads();
    const int excl = x - v + (warp > 0 ? s_w[warp - 1] : 0);
    total = s_w[nw - 1];
    __syncthreads();
    return excl;
}

// per tile: how many of its slots are deleted (keep == 0)
__global__ void __launch_bounds__(PLAN_TILE) k_plan_count(const uint8_t* __restrict__ keep, int64_t n,
                                                          int32_t* __restrict__ tile_cnt) {
    __shared__ int s_w[32];
    const int64_t s = (int64_t)blockIdx.x * PLAN_TILE + threadIdx.x;
    int tot;
    (void)block_scan_n(s < n && !keep[s] ? 1 : 0, s_w, tot);
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

// per tile: valid adds (gid >= 0)
__global__ void __launch_bounds__(APPEND_TILE) k_append_count(const int32_t* __restrict__ gids, int64_t cnt,
                                                              int32_t* __restrict__ tile_cnt) {
    __shared__ int s_w[32];
    const int64_t i = (int64_t)blockIdx.x * APPEND_TILE + threadIdx.x;
    int tot;
    (void)block_scan_n(i < cnt && gids[i] >= 0 ? 1 : 0, s_w, tot);
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

// one CTA: tile_off = exclusive scan of tile_cnt; *total = the sum (and
// *zero, when given, = 0: the h counter the emission adds to)
__global__ void __launch_bounds__(1024) k_tiles_scan(const int32_t* __restrict__ tile_cnt, int64_t ntiles,
                                                     int32_t* __restrict__ tile_off, int64_t* total, int64_t* zero) {
    __shared__ int s_w[32];
    int base = 0;
    for (int64_t b = 0; b < ntiles; b += 1024) {
        const int64_t t = b + threadIdx.x;
        int tot;
        const int ex = block_scan_n(t < ntiles ? tile_cnt[t] : 0, s_w, tot);
        if (t < ntiles) tile_off[t] = base + ex;
        base += tot;
    }
    if (threadIdx.x == 0) {
        *total = base;
        if (zero) *zero = 0;
    }
}

__global__ void __launch_bounds__(PLAN_TILE) k_plan_emit(const uint8_t* __restrict__ keep, int64_t n,
                                                         const int32_t* __restrict__ tile_off, int64_t* counts,
                                                         int32_t* dels, int32_t* movers) {
    __shared__ int s_w[32];
    const int64_t s = (int64_t)blockIdx.x * PLAN_TILE + threadIdx.x;
    const int64_t kk = counts[0], nk = n - kk;
    const int d = s < n && !keep[s] ? 1 : 0;
    int tot;
    const int64_t Ds = tile_off[blockIdx.x] + block_scan_n(d, s_w, tot);   // deleted slots in [0, s)
    if (s < n) {
        if (d)
            dels[Ds] = (int32_t)s;
        else if (s >= nk)
            movers[(n - 1 - s) - (kk - Ds)] = (int32_t)s;    // rank = live slots in (s, n)
    }
    int below;
    (void)block_scan_n(d && s < nk ? 1 : 0, s_w, below);
    if (threadIdx.x == 0 && below) atomicAdd((unsigned long long*)&counts[1], (unsigned long long)below);
}

struct Arena {
    float* means;   // (cap, 3)
    float* rots;    // (cap, 9)
    float* scales;  // (cap, 3)
    float* opac;    // (cap)
    float* shs;     // (cap, K, 3)
    int K;
};

// Map row layout (the reference's _Arena row, window.py:58-60):
// mean 3 | rot 9 | scale 3 | opacity 1 | sh 3K
__device__ __forceinline__ void row_copy_out(const Arena& a, int64_t s, float* row) {
    for (int c = 0; c < 3; ++c) row[c] = a.means[3 * s + c];
    for (int c = 0; c < 9; ++c) row[3 + c] = a.rots[9 * s + c];
    for (int c = 0; c < 3; ++c) row[12 + c] = a.scales[3 * s + c];
    row[15] = a.opac[s];
    for (int c = 0; c < 3 * a.K; ++c) row[16 + c] = a.shs[3 * a.K * s + c];
}

__device__ __forceinline__ void row_copy_in(const Arena& a, int64_t s, const float* row) {
    for (int c = 0; c < 3; ++c) a.means[3 * s + c] = row[c];
    for (int c = 0; c < 9; ++c) a.rots[9 * s + c] = row[3 + c];
    for (int c = 0; c < 3; ++c) a.scales[3 * s + c] = row[12 + c];
    a.opac[s] = row[15];
    for (int c = 0; c < 3 * a.K; ++c) a.shs[3 * a.K * s + c] = row[16 + c];
}

__device__ __forceinline__ int32_t leaf_gid(const lsb_voxmap& m, long long okey) {
    long long ix, iy, iz;
    okey_unpack(okey, ix, iy, iz);
    if (!in_range(ix) || !in_range(iy) || !in_range(iz)) return -1;
    const long long t = find(m, ix, iy, iz);
    return t < 0 ? -1 : m.gslot[t];
}

__global__ void k_win_to_map(lsb_voxmap m, Arena a, const int64_t* __restrict__ wkeys,
                             const int32_t* __restrict__ dels, int64_t k, float* store) {
    const int R = 16 + 3 * a.K;
    GRID_STRIDE(i, k) {
        const int32_t s = dels[i];
        const int32_t gid = leaf_gid(m, wkeys[s]);
        if (gid < 0) {
            atomicOr((unsigned long long*)m.flags, 2ull);      // MissingVoxel: window key without a map leaf
            continue;
        }
        row_copy_out(a, s, store + (int64_t)gid * R);
    }
}

__global__ void k_win_move(Arena a, int64_t* wkeys, const int32_t* __restrict__ dels,
                           const int32_t* __restrict__ movers, int64_t h, int64_t nk, int64_t n) {
    GRID_STRIDE(r, h) {
        const int32_t src = movers[r], dst = dels[r];
        float row[16 + 3 * 16];
        row_copy_out(a, src, row);
        row_copy_in(a, dst, row);
        wkeys[dst] = wkeys[src];
    }
}

__global__ void k_win_clear_keys(int64_t* wkeys, int64_t from, int64_t to) {
    GRID_STRIDE(i, to - from) wkeys[from + i] = -1;
}

__global__ void k_win_leaf_gids(lsb_voxmap m, const int64_t* __restrict__ okeys, int64_t cnt, int32_t* gids) {
    GRID_STRIDE(i, cnt) gids[i] = leaf_gid(m, okeys[i]);
}

// Distance from the voxel centre to the sensor, as numpy evaluates
// np.linalg.norm(voxel_center(k) - origin) (window.py:266-269; the length-3
// dot product is an FMA chain, checked bit-exact against numpy).
__global__ void k_win_dist(const int64_t* __restrict__ okeys, int64_t cnt, double edge, double ox, double oy,
                           double oz, double* out) {
    GRID_STRIDE(i, cnt) {
        long long ix, iy, iz;
        okey_unpack(okeys[i], ix, iy, iz);
        const double dx = ((double)ix + 0.5) * edge - ox;
        const double dy = ((double)iy + 0.5) * edge - oy;
        const double dz = ((double)iz + 0.5) * edge - oz;
        out[i] = sqrt(__fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx)));
    }
}

// Ordered append: the adds (sorted keys) that hold a Gaussian go to slots
// first_slot, first_slot + 1, ... in key order (tile counts, one-CTA scan,
// then every tile copies its rows in parallel).
__global__ void __launch_bounds__(APPEND_TILE) k_win_from_map(Arena a, int64_t* wkeys, const int64_t* __restrict__ okeys,
                                                              const int32_t* __restrict__ gids, int64_t cnt,
                                                              const float* __restrict__ store, int64_t first_slot,
                                                              const int32_t* __restrict__ tile_off) {
    __shared__ int s_w[32];
    const int R = 16 + 3 * a.K;
    const int64_t i = (int64_t)blockIdx.x * APPEND_TILE + threadIdx.x;
    const int g = i < cnt ? gids[i] : -1;
    int tot;
    const int ex = block_scan_n(g >= 0 ? 1 : 0, s_w, tot);
    if (g >= 0) {
        const int64_t s = first_slot + tile_off[blockIdx.x] + ex;
        row_copy_in(a, s, store + (int64_t)g * R);
        wkeys[s] = okeys[i];
    }
}

static Arena arena_of(const lsb_params& p) {
    return Arena{(float*)p.means, (float*)p.rots, (float*)p.scales, (float*)p.opacities, (float*)p.shs, p.sh_coeffs};
}

static int grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

cudaError_t launch_win_mark(const int64_t* wkeys, int64_t n, uint64_t* hkeys, int32_t* hslots, int64_t hcap,
                            const int64_t* fov, int64_t m, uint8_t* keep, uint8_t* is_add, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(hkeys, 0xFF, sizeof(uint64_t) * hcap, st);
    if (e == cudaSuccess && n) e = cudaMemsetAsync(keep, 0, n, st);
    if (e != cudaSuccess) return e;
    if (n) k_win_hash_build<<<grid_for(n), 256, 0, st>>>(wkeys, n, (unsigned long long*)hkeys, hslots, hcap);
    if (m)
        k_win_mark<<<grid_for(m), 256, 0, st>>>((const unsigned long long*)hkeys, hslots, hcap, fov, m, keep, is_add);
    return cudaGetLastError();
}

int64_t win_plan_tiles(int64_t n) { return 2 * ((n + PLAN_TILE - 1) / PLAN_TILE) + 2; }
int64_t win_append_tiles(int64_t cnt) { return 2 * ((cnt + APPEND_TILE - 1) / APPEND_TILE) + 2; }

cudaError_t launch_win_plan(const uint8_t* keep, int64_t n, int32_t* dels, int32_t* movers, int64_t* counts,
                            int32_t* tiles, cudaStream_t st) {
    const int64_t nt = (n + PLAN_TILE - 1) / PLAN_TILE;
    if (nt == 0) {
        cudaError_t e = cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st);
        return e;
    }
    k_plan_count<<<(unsigned)nt, PLAN_TILE, 0, st>>>(keep, n, tiles);
    k_tiles_scan<<<1, 1024, 0, st>>>(tiles, nt, tiles + nt, counts, counts + 1);
    k_plan_emit<<<(unsigned)nt, PLAN_TILE, 0, st>>>(keep, n, tiles + nt, counts, dels, movers);
    return cudaGetLastError();
}

cudaError_t launch_win_compact(const lsb_voxmap& m, const lsb_params& arena, int64_t* wkeys, const int32_t* dels,
                               int64_t k, const int32_t* movers, int64_t h, int64_t n, float* store, cudaStream_t st) {
    const Arena a = arena_of(arena);
    if (k) k_win_to_map<<<grid_for(k), 256, 0, st>>>(m, a, wkeys, dels, k, store);
    if (h) k_win_move<<<grid_for(h), 256, 0, st>>>(a, wkeys, dels, movers, h, n - k, n);
    if (k) k_win_clear_keys<<<grid_for(k), 256, 0, st>>>(wkeys, n - k, n);
    return cudaGetLastError();
}

cudaError_t launch_win_leaf_gids(const lsb_voxmap& m, const int64_t* okeys, int64_t cnt, int32_t* gids,
                                 cudaStream_t st) {
    if (cnt) k_win_leaf_gids<<<grid_for(cnt), 256, 0, st>>>(m, okeys, cnt, gids);
    return cudaGetLastError();
}

cudaError_t launch_win_dist(const int64_t* okeys, int64_t cnt, double edge, const double* origin, double* out,
                            cudaStream_t st) {
    if (cnt) k_win_dist<<<grid_for(cnt), 256, 0, st>>>(okeys, cnt, edge, origin[0], origin[1], origin[2], out);
    return cudaGetLastError();
}

cudaError_t launch_win_append(const lsb_params& arena, int64_t* wkeys, const int64_t* okeys, const int32_t* gids,
                              int64_t cnt, const float* store, int64_t first_slot, int64_t* n_added, int32_t* tiles,
                              cudaStream_t st) {
    const int64_t nt = (cnt + APPEND_TILE - 1) / APPEND_TILE;
    if (nt == 0) return cudaMemsetAsync(n_added, 0, sizeof(int64_t), st);
    k_append_count<<<(unsigned)nt, APPEND_TILE, 0, st>>>(gids, cnt, tiles);
    k_tiles_scan<<<1, 1024, 0, st>>>(tiles, nt, tiles + nt, n_added, nullptr);
    k_win_from_map<<<(unsigned)nt, APPEND_TILE, 0, st>>>(arena_of(arena), wkeys, okeys, gids, cnt, store, first_slot,
                                                         tiles + nt);
    return cudaGetLastError();
}

}  // namespace lsb
