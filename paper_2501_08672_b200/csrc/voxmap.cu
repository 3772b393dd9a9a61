// K8 voxel map: a GPU open-addressing hash of octree leaves
// (voxmap.py:21-65, 99-251).
//
// The reference keeps a dict of root voxels, each an 8-ary octree down to
// max_level, with leaf statistics in a flat dict.  An internal node exists
// iff some leaf below it was created, so the whole octree is determined by
// its set of leaf keys: the device table stores leaves only, keyed by the
// packed leaf key (ix, iy, iz at max_level), and parents/roots are derived by
// arithmetic shifts (floor division, voxmap.py:33-38).  The probe start is
// the reference's prime-XOR hash (voxmap.py:27-28) passed through a 64-bit
// finaliser; linear probing; insertion by atomicCAS on the key word.
//
// Keys are floor(p / edge) with TRUE division in f64 (voxmap.py:50,64), so
// the integer keys are bit-exact with the reference.  Leaf statistics
// (count, sum p, sum p p^T) are exact fixed-point group sums (deterministic,
// lsb_voxmap_accumulate below).  The map also keeps the packed keys of its
// Gaussian leaves in an append-only list, which the FoV enumeration walks.
#include <cuda_runtime.h>

#include "common.cuh"
#include "voxkey.cuh"

namespace lsb {

__device__ __forceinline__ void floor_key(const double* p, double edge, long long* k) {
    k[0] = (long long)floor(p[0] / edge);
    k[1] = (long long)floor(p[1] / edge);
    k[2] = (long long)floor(p[2] / edge);
}

// keys_of_points (voxmap.py:59-65): floor(p / edge), true division.
__global__ void k_keys(const double* __restrict__ pts, int64_t n, double edge, int64_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        long long k[3];
        floor_key(pts + 3 * i, edge, k);
        out[3 * i] = k[0];
        out[3 * i + 1] = k[1];
        out[3 * i + 2] = k[2];
    }
}

// accumulate_points / group_by_leaf + ensure_leaf + add_leaf_stats
// (voxmap.py:184-230): one thread per point.
__global__ void k_insert_points(lsb_voxmap m, const double* __restrict__ pts, int64_t n, int accumulate,
                                int64_t* __restrict__ slots) {
    const double edge = m.root_len / (double)(1ll << m.max_level);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double* p = pts + 3 * i;
        long long k[3];
        floor_key(p, edge, k);
        long long s = -1;
        if (in_range(k[0]) && in_range(k[1]) && in_range(k[2])) s = find_or_insert(m, k[0], k[1], k[2]);
        if (slots) slots[i] = s;
        if (s < 0) {
            atomicExch((unsigned long long*)m.flags, 1ull);   // table full or key out of range
            continue;
        }
        if (!accumulate) continue;
        atomicAdd((unsigned long long*)&m.count[s], 1ull);
        const double x = p[0], y = p[1], z = p[2];
        atomicAdd(&m.sum[3 * s], x);
        atomicAdd(&m.sum[3 * s + 1], y);
        atomicAdd(&m.sum[3 * s + 2], z);
        double* o = m.outer + 6 * s;     // xx xy xz yy yz zz
        atomicAdd(&o[0], x * x);
        atomicAdd(&o[1], x * y);
        atomicAdd(&o[2], x * z);
        atomicAdd(&o[3], y * y);
        atomicAdd(&o[4], y * z);
        atomicAdd(&o[5], z * z);
    }
}

// try_insert with leaf_capacity 1 (voxmap.py:171-182): the first Gaussian of
// the batch (lowest index) landing in an empty leaf wins, as in the
// reference's sequential loop.  Pass 1 claims with atomicMin, pass 2 writes.
__global__ void k_claim(lsb_voxmap m, const double* __restrict__ means, int64_t n, int64_t* __restrict__ slots) {
    const double edge = m.root_len / (double)(1ll << m.max_level);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        long long k[3];
        floor_key(means + 3 * i, edge, k);
        long long s = -1;
        if (in_range(k[0]) && in_range(k[1]) && in_range(k[2])) s = find_or_insert(m, k[0], k[1], k[2]);
        slots[i] = s;
        if (s < 0) {
            atomicExch((unsigned long long*)m.flags, 1ull);
            continue;
        }
        if (m.gslot[s] < 0) atomicMin(&m.claim[s], (int)i);
    }
}

__global__ void k_commit(lsb_voxmap m, const int64_t* __restrict__ slots, int64_t n, int32_t first_gid,
                         int32_t* __restrict__ status) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const long long s = slots[i];
        int st = 0;
        if (s >= 0 && m.gslot[s] < 0 && m.claim[s] == (int)i) st = 1;
        status[i] = st;
    }
}

__global__ void k_commit2(lsb_voxmap m, const int64_t* __restrict__ slots, int64_t n, int32_t first_gid,
                          const int32_t* __restrict__ status) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const long long s = slots[i];
        if (status[i]) {
            m.gslot[s] = first_gid + (int32_t)i;
            if (m.gkeys) m.gkeys[atomicAdd((unsigned long long*)m.n_gkeys, 1ull)] = m.keys[s];   // a new Gaussian leaf
        }
        if (s >= 0) m.claim[s] = 0x7fffffff;
    }
}

// Batched get_leaf (voxmap.py:162-166): slot or -1 per leaf key.
__global__ void k_lookup(lsb_voxmap m, const int64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const long long ix = keys[3 * i], iy = keys[3 * i + 1], iz = keys[3 * i + 2];
        out[i] = (in_range(ix) && in_range(iy) && in_range(iz)) ? find(m, ix, iy, iz) : -1;
    }
}

// FoV: root keys of the scan points go into a small root set (same hashing),
// then every occupied leaf holding a Gaussian whose root is in the set is
// emitted (leaf_keys_under_roots, voxmap.py:232-251, over
// keys_of_points(p, root_len, 0), pipeline.py:190-191).
__global__ void k_fov_roots(const double* __restrict__ pts, int64_t n, double root_len, unsigned long long* rset,
                            int64_t rcap) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        long long k[3];
        floor_key(pts + 3 * i, root_len, k);
        if (!(in_range(k[0]) && in_range(k[1]) && in_range(k[2]))) continue;
        // root set: plain find-or-insert without the used counter
        const unsigned long long key = pack_key(k[0], k[1], k[2]);
        const unsigned long long mask = (unsigned long long)rcap - 1;
        unsigned long long s = slot_of(k[0], k[1], k[2], 0, mask);
        for (long long probe = 0; probe < rcap; ++probe) {
            const unsigned long long cur = rset[s];
            if (cur == key) break;
            if (cur == EMPTY) {
                const unsigned long long prev = atomicCAS(&rset[s], EMPTY, key);
                if (prev == EMPTY || prev == key) break;
            }
            s = (s + 1) & mask;
        }
    }
}

__global__ void k_fov_leaves(lsb_voxmap m, const unsigned long long* __restrict__ rset, int64_t rcap,
                             int64_t* __restrict__ out, unsigned long long* __restrict__ n_out, int64_t out_cap) {
    const int L = m.max_level;
    const unsigned lane = threadIdx.x & 31;
    // warp-uniform trip count (every block's threads share `base`), so the
    // ballots below see the whole warp converged
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m.cap; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = base + threadIdx.x;
        // gslot first: 4 bytes per slot streamed, the key only for the leaves
        // that hold a Gaussian (gslot >= 0 implies an occupied slot)
        bool hit = false;
        long long ix = 0, iy = 0, iz = 0;
        const unsigned long long key = (s < m.cap && m.gslot[s] >= 0) ? (unsigned long long)m.keys[s] : EMPTY;
        if (key != EMPTY) {
            unpack_key(key, ix, iy, iz);
            const long long rx = ix >> L, ry = iy >> L, rz = iz >> L;   // floor division by 2^L
            const unsigned long long rkey = pack_key(rx, ry, rz);
            const unsigned long long mask = (unsigned long long)rcap - 1;
            unsigned long long q = slot_of(rx, ry, rz, 0, mask);
            for (long long probe = 0; probe < rcap; ++probe) {
                const unsigned long long cur = rset[q];
                if (cur == rkey) { hit = true; break; }
                if (cur == EMPTY) break;
                q = (q + 1) & mask;
            }
        }
        // warp-aggregated output slot: one atomic per warp instead of per leaf
        __syncwarp();
        const unsigned hits = __ballot_sync(0xffffffffu, hit);
        if (!hits) continue;
        const int leader = __ffs(hits) - 1;
        unsigned long long ob = 0;
        if ((int)lane == leader) ob = atomicAdd(n_out, (unsigned long long)__popc(hits));
        ob = __shfl_sync(0xffffffffu, ob, leader);
        if (!hit) continue;
        const unsigned long long o = ob + __popc(hits & ((1u << lane) - 1u));
        if ((int64_t)o < out_cap) {
            out[3 * o] = ix;
            out[3 * o + 1] = iy;
            out[3 * o + 2] = iz;
        }
    }
}

// The same over the list of Gaussian leaves (gkeys): n_gkeys entries instead
// of the whole table's cap slots.
__global__ void k_fov_gleaves(lsb_voxmap m, const unsigned long long* __restrict__ rset, int64_t rcap,
                              int64_t* __restrict__ out, unsigned long long* __restrict__ n_out, int64_t out_cap) {
    const int L = m.max_level;
    const unsigned lane = threadIdx.x & 31;
    const int64_t ng = (int64_t)*m.n_gkeys;           // the same for every thread: warp-uniform trip count
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ng; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = base + threadIdx.x;
        bool hit = false;
        long long ix = 0, iy = 0, iz = 0;
        if (j < ng) {
            unpack_key(m.gkeys[j], ix, iy, iz);
            const long long rx = ix >> L, ry = iy >> L, rz = iz >> L;   // floor division by 2^L
            const unsigned long long rkey = pack_key(rx, ry, rz);
            const unsigned long long mask = (unsigned long long)rcap - 1;
            unsigned long long q = slot_of(rx, ry, rz, 0, mask);
            for (long long probe = 0; probe < rcap; ++probe) {
                const unsigned long long cur = rset[q];
                if (cur == rkey) { hit = true; break; }
                if (cur == EMPTY) break;
                q = (q + 1) & mask;
            }
        }
        __syncwarp();
        const unsigned hits = __ballot_sync(0xffffffffu, hit);
        if (!hits) continue;
        const int leader = __ffs(hits) - 1;
        unsigned long long ob = 0;
        if ((int)lane == leader) ob = atomicAdd(n_out, (unsigned long long)__popc(hits));
        ob = __shfl_sync(0xffffffffu, ob, leader);
        if (!hit) continue;
        const unsigned long long o = ob + __popc(hits & ((1u << lane) - 1u));
        if ((int64_t)o < out_cap) {
            out[3 * o] = ix;
            out[3 * o + 1] = iy;
            out[3 * o + 2] = iz;
        }
    }
}

// Dump occupied leaves (keys, counts, sums, outers, gslot) for export.
__global__ void k_dump(lsb_voxmap m, int64_t* __restrict__ keys, int64_t* __restrict__ slots,
                       unsigned long long* __restrict__ n_out, int64_t out_cap) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m.cap; s += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = (unsigned long long)m.keys[s];
        if (key == EMPTY) continue;
        const unsigned long long o = atomicAdd(n_out, 1ull);
        if ((int64_t)o >= out_cap) continue;
        long long ix, iy, iz;
        unpack_key(key, ix, iy, iz);
        keys[3 * o] = ix;
        keys[3 * o + 1] = iy;
        keys[3 * o + 2] = iz;
        slots[o] = s;
    }
}

__global__ void k_rehash(lsb_voxmap src, lsb_voxmap dst) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < src.cap; s += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = (unsigned long long)src.keys[s];
        if (key == EMPTY) continue;
        long long ix, iy, iz;
        unpack_key(key, ix, iy, iz);
        const long long d = find_or_insert(dst, ix, iy, iz);
        if (d < 0) {
            atomicExch((unsigned long long*)dst.flags, 1ull);
            continue;
        }
        dst.count[d] = src.count[s];
        for (int k = 0; k < 3; ++k) dst.sum[3 * d + k] = src.sum[3 * s + k];
        for (int k = 0; k < 6; ++k) dst.outer[6 * d + k] = src.outer[6 * s + k];
        dst.gslot[d] = src.gslot[s];
    }
}

static int grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

cudaError_t launch_vox_keys(const double* pts, int64_t n, double edge, int64_t* out, cudaStream_t st) {
    if (n > 0) k_keys<<<grid_for(n), 256, 0, st>>>(pts, n, edge, out);
    return cudaGetLastError();
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// ---- deterministic leaf statistics: exact fixed-point group sums -------------
// add_leaf_stats (voxmap.py:204-211) adds each leaf group's (count, sum p,
// sum p p^T) once per call.  Floating-point atomics would make the sums
// depend on the arrival order; here every per-point term is converted
// exactly (to 2^-60, far below f64 resolution at these magnitudes) into a
// signed 128-bit fixed-point value split over three 64-bit limbs
// (a 2^64 + b 2^32 + c, b and c < 2^32), and the limbs are added with
// integer atomics, which are associative: the group sum is the same exact
// integer whatever the order, converted to f64 once and added to the leaf's
// statistics once.  Three kernels (local leaf index per touched slot, the
// atomic adds, the fold) instead of a sort of the points by leaf.
constexpr int ACC_FRAC = 60;                 // fixed-point fraction bits
constexpr int ACC_W = 1 + 9 * 3;             // count + 9 values x 3 limbs

__device__ __forceinline__ void fixed_limbs(double v, long long& a, unsigned long long& b, unsigned long long& c) {
    a = 0;
    b = c = 0;
    if (v == 0.0) return;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const int e = (int)((bits >> 52) & 0x7ff);
    unsigned long long m = bits & ((1ull << 52) - 1);
    if (e) m |= 1ull << 52;
    const int k = (e ? e : 1) - 1075 + ACC_FRAC;          // y = m 2^k
    unsigned long long lo, hi;                             // |y| as a 128-bit (hi, lo)
    if (k >= 0) {
        lo = k >= 64 ? 0ull : m << k;
        hi = k == 0 ? 0ull : (k >= 64 ? m << (k - 64) : m >> (64 - k));
    } else {
        const int r = -k;
        lo = r >= 64 ? 0ull : (m + (1ull << (r - 1))) >> r;   // round half up on the magnitude
        hi = 0;
    }
    if (bits >> 63) {                                      // negate the 128-bit value
        lo = ~lo + 1ull;
        hi = ~hi + (lo == 0ull ? 1ull : 0ull);
    }
    c = lo & 0xffffffffull;
    b = lo >> 32;
    a = (long long)hi;
}

__device__ __forceinline__ double fixed_value(long long a, unsigned long long b, unsigned long long c) {
    b += c >> 32;
    c &= 0xffffffffull;
    a += (long long)(b >> 32);
    b &= 0xffffffffull;
    const double hi = (double)a * 18446744073709551616.0;                 // a 2^64 (exact: |a| < 2^53)
    const double lo = (double)((b << 32) | c);
    return (hi + lo) * 0x1p-60;
}

__global__ void k_acc_local(lsb_voxmap m, const int64_t* __restrict__ slots, int64_t n, int64_t* __restrict__ loc_slot,
                            unsigned long long* __restrict__ nloc, unsigned long long* __restrict__ acc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = slots[i];
        if (s < 0 || s >= m.cap) continue;
        if (atomicCAS(&m.claim[s], 0x7fffffff, -2) != 0x7fffffff) continue;
        const unsigned long long j = atomicAdd(nloc, 1ull);
        loc_slot[j] = s;
        for (int q = 0; q < ACC_W; ++q) acc[j * ACC_W + q] = 0ull;
        m.claim[s] = (int)j;
    }
}

__global__ void k_acc_add(lsb_voxmap m, const double* __restrict__ pts, const int64_t* __restrict__ slots, int64_t n,
                          unsigned long long* __restrict__ acc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = slots[i];
        if (s < 0 || s >= m.cap) continue;
        unsigned long long* r = acc + (int64_t)m.claim[s] * ACC_W;
        const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
        const double v[9] = {x, y, z, x * x, x * y, x * z, y * y, y * z, z * z};
        atomicAdd(r, 1ull);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            long long a;
            unsigned long long b, c;
            fixed_limbs(v[q], a, b, c);
            if (a) atomicAdd(r + 1 + 3 * q, (unsigned long long)a);
            if (b) atomicAdd(r + 2 + 3 * q, b);
            if (c) atomicAdd(r + 3 + 3 * q, c);
        }
    }
}

__global__ void k_acc_fold(lsb_voxmap m, const int64_t* __restrict__ loc_slot, const unsigned long long* __restrict__ nloc,
                           const unsigned long long* __restrict__ acc) {
    const int64_t nl = (int64_t)*nloc;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = loc_slot[j];
        const unsigned long long* r = acc + j * ACC_W;
        double g[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) g[q] = fixed_value((long long)r[1 + 3 * q], r[2 + 3 * q], r[3 + 3 * q]);
        // one group per leaf per call: the only writer of this leaf's statistics
        m.count[s] += r[0];
        m.sum[3 * s] += g[0];
        m.sum[3 * s + 1] += g[1];
        m.sum[3 * s + 2] += g[2];
        double* o = m.outer + 6 * s;
#pragma unroll
        for (int q = 0; q < 6; ++q) o[q] += g[3 + q];
        m.claim[s] = 0x7fffffff;
    }
}

size_t vox_accumulate_temp_bytes(int64_t n) {
    const size_t nn = (size_t)(n > 0 ? n : 1);
    return al256(8 * nn) * 2 + al256(8) + al256(8 * ACC_W * nn);
}

cudaError_t launch_vox_insert(const lsb_voxmap& m, const double* pts, int64_t n, int accumulate, int64_t* slots,
                              cudaStream_t st);

cudaError_t launch_vox_accumulate(const lsb_voxmap& m, const double* pts, int64_t n, int64_t* slots, void* temp,
                                  cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const size_t nn = (size_t)n;
    char* t = (char*)temp;
    int64_t* sl = (int64_t*)t;
    t += al256(8 * nn);
    int64_t* loc_slot = (int64_t*)t;
    t += al256(8 * nn);
    unsigned long long* nloc = (unsigned long long*)t;
    t += al256(8);
    unsigned long long* acc = (unsigned long long*)t;
    if (!slots) slots = sl;
    cudaError_t e = launch_vox_insert(m, pts, n, 0, slots, st);      // find / create every point's leaf
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(nloc, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    k_acc_local<<<grid_for(n), 256, 0, st>>>(m, slots, n, loc_slot, nloc, acc);
    k_acc_add<<<grid_for(n), 256, 0, st>>>(m, pts, slots, n, acc);
    k_acc_fold<<<grid_for(n), 256, 0, st>>>(m, loc_slot, nloc, acc);
    return cudaGetLastError();
}

cudaError_t launch_vox_insert(const lsb_voxmap& m, const double* pts, int64_t n, int accumulate, int64_t* slots,
                              cudaStream_t st) {
    if (n > 0) k_insert_points<<<grid_for(n), 256, 0, st>>>(m, pts, n, accumulate, slots);
    return cudaGetLastError();
}

cudaError_t launch_vox_try_insert(const lsb_voxmap& m, const double* means, int64_t n, int32_t first_gid,
                                  int64_t* slots, int32_t* status, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_claim<<<grid_for(n), 256, 0, st>>>(m, means, n, slots);
    k_commit<<<grid_for(n), 256, 0, st>>>(m, slots, n, first_gid, status);
    k_commit2<<<grid_for(n), 256, 0, st>>>(m, slots, n, first_gid, status);
    return cudaGetLastError();
}

cudaError_t launch_vox_lookup(const lsb_voxmap& m, const int64_t* keys, int64_t n, int64_t* out, cudaStream_t st) {
    if (n > 0) k_lookup<<<grid_for(n), 256, 0, st>>>(m, keys, n, out);
    return cudaGetLastError();
}

cudaError_t launch_vox_fov(const lsb_voxmap& m, const double* pts, int64_t n, unsigned long long* rset, int64_t rcap,
                           int64_t* out, unsigned long long* n_out, int64_t out_cap, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(rset, 0xff, sizeof(unsigned long long) * rcap, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(n_out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (n > 0) k_fov_roots<<<grid_for(n), 256, 0, st>>>(pts, n, m.root_len, rset, rcap);
    if (m.gkeys && m.n_gkeys)
        k_fov_gleaves<<<148 * 8, 256, 0, st>>>(m, rset, rcap, out, n_out, out_cap);
    else
        k_fov_leaves<<<grid_for(m.cap), 256, 0, st>>>(m, rset, rcap, out, n_out, out_cap);
    return cudaGetLastError();
}

cudaError_t launch_vox_rehash(const lsb_voxmap& src, const lsb_voxmap& dst, cudaStream_t st) {
    k_rehash<<<grid_for(src.cap), 256, 0, st>>>(src, dst);
    return cudaGetLastError();
}

cudaError_t launch_vox_dump(const lsb_voxmap& m, int64_t* keys, int64_t* slots, unsigned long long* n_out,
                            int64_t out_cap, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(n_out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    k_dump<<<grid_for(m.cap), 256, 0, st>>>(m, keys, slots, n_out, out_cap);
    return cudaGetLastError();
}

// ---- plane fits and the LiDAR point-to-plane measurement (§8(f) rank 2) ----
// fit_planes / estimate_normal (voxmap.py:255-335): the leaf's and its 6 face
// neighbours' statistics summed in the reference's order, scatter = outer/n -
// mean mean^T, the smallest-eigenvalue eigenvector (f64 cyclic Jacobi: the
// symmetric 3x3 problem numpy hands to LAPACK's dsyevd), flipped to face the
// sensor; rejected with fewer than 3 points or rank < 2
// (w1 <= 1e-12 + 1e-6 max(w2, 0)).  The anchor is the leaf's own centroid.

__device__ void eig3_jacobi(double A[3][3], double w[3], double V[3][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) V[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 32; ++sweep) {
        const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
        const double dia = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
        if (off <= 1e-34 * dia || off == 0.0) break;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int p = r == 2 ? 1 : 0, q = r == 0 ? 1 : 2;
            const double apq = A[p][q];
            if (apq == 0.0) continue;
            const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
            const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
            for (int k = 0; k < 3; ++k) {           // A <- J^T A J
                const double akp = A[k][p], akq = A[k][q];
                A[k][p] = c * akp - s * akq;
                A[k][q] = s * akp + c * akq;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double apk = A[p][k], aqk = A[q][k];
                A[p][k] = c * apk - s * aqk;
                A[q][k] = s * apk + c * aqk;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {           // V <- V J
                const double vkp = V[k][p], vkq = V[k][q];
                V[k][p] = c * vkp - s * vkq;
                V[k][q] = s * vkp + c * vkq;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = A[i][i];
}

__device__ bool plane_fit(const lsb_voxmap& m, long long ix, long long iy, long long iz, const double* origin,
                          double* normal, double* anchor) {
    const long long self = find(m, ix, iy, iz);
    if (self < 0 || m.count[self] == 0) return false;
    const long long nb[7][3] = {{0, 0, 0}, {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
    unsigned long long n_tot = 0;
    double s[3] = {0.0, 0.0, 0.0}, so[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < 7; ++k) {
        const long long t = find(m, ix + nb[k][0], iy + nb[k][1], iz + nb[k][2]);
        if (t < 0 || m.count[t] == 0) continue;          // leaf_stats holds leaves that saw points
        n_tot += m.count[t];
        for (int c = 0; c < 3; ++c) s[c] = s[c] + m.sum[3 * t + c];
        for (int c = 0; c < 6; ++c) so[c] = so[c] + m.outer[6 * t + c];
    }
    if (n_tot < 3) return false;
    const double n = (double)n_tot;
    const double mean[3] = {s[0] / n, s[1] / n, s[2] / n};
    double A[3][3];
    const int ij[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    for (int c = 0; c < 6; ++c) {
        const int i = ij[c][0], j = ij[c][1];
        A[i][j] = A[j][i] = so[c] / n - mean[i] * mean[j];
    }
    double w[3], V[3][3];
    eig3_jacobi(A, w, V);
    int o[3] = {0, 1, 2};                     // ascending eigenvalues (eigh's order)
    if (w[o[1]] < w[o[0]]) { const int x = o[0]; o[0] = o[1]; o[1] = x; }
    if (w[o[2]] < w[o[1]]) { const int x = o[1]; o[1] = o[2]; o[2] = x; }
    if (w[o[1]] < w[o[0]]) { const int x = o[0]; o[0] = o[1]; o[1] = x; }
    const int i0 = o[0], i1 = o[1], i2 = o[2];
    if (!(w[i1] > 1e-12 + 1e-6 * fmax(w[i2], 0.0))) return false;
    double nv[3] = {V[0][i0], V[1][i0], V[2][i0]};
    const double dot = nv[0] * (origin[0] - mean[0]) + nv[1] * (origin[1] - mean[1]) + nv[2] * (origin[2] - mean[2]);
    if (dot < 0.0)
        for (int c = 0; c < 3; ++c) nv[c] = -nv[c];
    const double cnt = (double)m.count[self];
    for (int c = 0; c < 3; ++c) {
        normal[c] = nv[c];
        anchor[c] = m.sum[3 * self + c] / cnt;
    }
    return true;
}

__global__ void k_fit_planes(lsb_voxmap m, const int64_t* __restrict__ keys, int64_t k, double ox, double oy,
                             double oz, double* normals, double* anchors, uint8_t* valid) {
    const double origin[3] = {ox, oy, oz};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        double nv[3], an[3];
        const long long ix = keys[3 * i], iy = keys[3 * i + 1], iz = keys[3 * i + 2];
        const bool ok = in_range(ix) && in_range(iy) && in_range(iz) && plane_fit(m, ix, iy, iz, origin, nv, an);
        valid[i] = ok ? 1 : 0;
        for (int c = 0; c < 3; ++c) {
            normals[3 * i + c] = ok ? nv[c] : __longlong_as_double(0x7ff8000000000000ll);
            anchors[3 * i + c] = ok ? an[c] : __longlong_as_double(0x7ff8000000000000ll);
        }
    }
}

struct LidarArgs {
    double R_il[9], t_il[3], R_wi[9], t_wi[3], origin[3];
    double leaf_len, gate;
};

// x @ R^T + t as numpy/OpenBLAS evaluates it (k = 3 FMA chain, then + t).
__device__ __forceinline__ void apply_rt(const double* R, const double* t, const double* x, double* y) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
        y[r] = __dadd_rn(__fma_rn(R[3 * r + 2], x[2], __fma_rn(R[3 * r + 1], x[1], __dmul_rn(R[3 * r], x[0]))), t[r]);
}

// lidar_measurement (estimator.py:190-238), one thread per scan point:
// rows = -H[:, :6] (the convention of Measurement.rows_dev / lsb_hb_reduce),
// z = n . (p_w - anchor), keep = plane found && |z| <= gate.
__global__ void k_lidar_rows(lsb_voxmap m, const double* __restrict__ pts, int64_t n, LidarArgs a, double* rows,
                             double* z, uint8_t* keep) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double pi[3], pw[3];
        apply_rt(a.R_il, a.t_il, pts + 3 * i, pi);
        apply_rt(a.R_wi, a.t_wi, pi, pw);
        const long long ix = (long long)floor(__ddiv_rn(pw[0], a.leaf_len));
        const long long iy = (long long)floor(__ddiv_rn(pw[1], a.leaf_len));
        const long long iz = (long long)floor(__ddiv_rn(pw[2], a.leaf_len));
        double nv[3], an[3];
        bool ok = in_range(ix) && in_range(iy) && in_range(iz) && plane_fit(m, ix, iy, iz, a.origin, nv, an);
        double r = 0.0;
        if (ok) {
            r = nv[0] * (pw[0] - an[0]) + nv[1] * (pw[1] - an[1]) + nv[2] * (pw[2] - an[2]);
            ok = fabs(r) <= a.gate;
        }
        keep[i] = ok ? 1 : 0;
        z[i] = r;
        double h[6] = {0, 0, 0, 0, 0, 0};
        if (ok) {
            double nR[3];      // n^T R_wi
            for (int c = 0; c < 3; ++c) nR[c] = nv[0] * a.R_wi[c] + nv[1] * a.R_wi[3 + c] + nv[2] * a.R_wi[6 + c];
            h[0] = -(nR[1] * pi[2] - nR[2] * pi[1]);
            h[1] = -(nR[2] * pi[0] - nR[0] * pi[2]);
            h[2] = -(nR[0] * pi[1] - nR[1] * pi[0]);
            h[3] = nv[0];
            h[4] = nv[1];
            h[5] = nv[2];
        }
        for (int c = 0; c < 6; ++c) rows[6 * i + c] = -h[c];
    }
}

cudaError_t launch_fit_planes(const lsb_voxmap& m, const int64_t* keys, int64_t k, const double* origin,
                              double* normals, double* anchors, uint8_t* valid, cudaStream_t st) {
    if (k) k_fit_planes<<<grid_for(k), 256, 0, st>>>(m, keys, k, origin[0], origin[1], origin[2], normals, anchors, valid);
    return cudaGetLastError();
}

cudaError_t launch_lidar_rows(const lsb_voxmap& m, const double* pts, int64_t n, const double* R_il,
                              const double* t_il, const double* R_wi, const double* t_wi, double leaf_len,
                              double gate, double* rows, double* z, uint8_t* keep, cudaStream_t st) {
    LidarArgs a;
    for (int c = 0; c < 9; ++c) {
        a.R_il[c] = R_il[c];
        a.R_wi[c] = R_wi[c];
    }
    for (int c = 0; c < 3; ++c) {
        a.t_il[c] = t_il[c];
        a.t_wi[c] = t_wi[c];
    }
    // T_WL = T_WI T_IL: its translation R_wi t_il + t_wi (SE3 compose, numpy
    // matmul order) is the sensor origin of the normal flip
    for (int r = 0; r < 3; ++r)
        a.origin[r] = (R_wi[3 * r] * t_il[0] + R_wi[3 * r + 1] * t_il[1] + R_wi[3 * r + 2] * t_il[2]) + t_wi[r];
    a.leaf_len = leaf_len;
    a.gate = gate;
    if (n) k_lidar_rows<<<grid_for(n), 256, 0, st>>>(m, pts, n, a, rows, z, keep);
    return cudaGetLastError();
}

// ---- batched Gaussian initialisation (§8(f) rank 3) ------------------------
// pipeline.py:99-137 + initialize.py:22-124, one thread per new leaf group
// (sorted keys, the scan's centroid of the leaf): skip leaves that already
// hold a Gaussian; observability pre-check (z > near, 1 <= u <= W-2,
// 1 <= v <= H-2); plane normal (plane_fit), else the unit view direction;
// bilinear colour (area weights, pixel centres at integers) -> the degree-0
// SH coefficient (c - 0.5) / SH_C0; slab frame (n, u, n x u) with
// u = e_x x n / |e_x x n| (e_y if |e_x x n| < 1e-6); scale (delta, s, s),
// s = kappa * root_len / 2^max_level.  status[i] = 1 if a row was made.

struct InitArgs {
    double R_cw[9], t_cw[3], origin[3];
    double fx, fy, cx, cy;
    int W, H, K;
    double near, kappa, delta, opacity, root_len;
};

__device__ __forceinline__ double norm3(double x, double y, double z) {
    return sqrt(__fma_rn(z, z, __fma_rn(y, y, x * x)));      // numpy's length-3 norm
}

__global__ void k_init_gaussians(lsb_voxmap m, const int64_t* __restrict__ keys, const double* __restrict__ cent,
                                 int64_t k, const float* __restrict__ image, InitArgs a, float* rows,
                                 uint8_t* status) {
    const int R = 16 + 3 * a.K;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        status[i] = 0;
        const long long ix = keys[3 * i], iy = keys[3 * i + 1], iz = keys[3 * i + 2];
        if (!in_range(ix) || !in_range(iy) || !in_range(iz)) continue;
        const long long t = find(m, ix, iy, iz);
        if (t < 0 || m.gslot[t] >= 0) continue;                    // missing leaf or already full
        const double c[3] = {cent[3 * i], cent[3 * i + 1], cent[3 * i + 2]};
        double pc[3];
        for (int r = 0; r < 3; ++r)
            pc[r] = __dadd_rn(__fma_rn(a.R_cw[3 * r + 2], c[2], __fma_rn(a.R_cw[3 * r + 1], c[1], __dmul_rn(a.R_cw[3 * r], c[0]))),
                              a.t_cw[r]);
        if (!(pc[2] > a.near)) continue;
        const double u = __dadd_rn(__ddiv_rn(__dmul_rn(a.fx, pc[0]), pc[2]), a.cx);
        const double v = __dadd_rn(__ddiv_rn(__dmul_rn(a.fy, pc[1]), pc[2]), a.cy);
        if (!(1.0 <= u && u <= (double)(a.W - 2) && 1.0 <= v && v <= (double)(a.H - 2))) continue;
        double n[3], anc[3];
        if (!plane_fit(m, ix, iy, iz, a.origin, n, anc)) {
            const double vx = a.origin[0] - c[0], vy = a.origin[1] - c[1], vz = a.origin[2] - c[2];
            const double nv = norm3(vx, vy, vz);
            if (nv == 0.0) continue;
            n[0] = vx / nv;
            n[1] = vy / nv;
            n[2] = vz / nv;
        }
        // bilinear colour (initialize.py:64-93)
        const int x0 = (int)floor(u), y0 = (int)floor(v);
        const double fxw = u - x0, fyw = v - y0;
        const double wgt[4] = {(1.0 - fxw) * (1.0 - fyw), fxw * (1.0 - fyw), (1.0 - fxw) * fyw, fxw * fyw};
        const int px[4] = {x0, x0 + 1, x0, x0 + 1}, py[4] = {y0, y0, y0 + 1, y0 + 1};
        double col[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < 4; ++q)
            for (int ch = 0; ch < 3; ++ch)
                col[ch] = __dadd_rn(col[ch], __dmul_rn(wgt[q], (double)image[3 * ((int64_t)py[q] * a.W + px[q]) + ch]));
        // slab frame (initialize.py:30-61)
        double ux = 0.0 * n[2] - 0.0 * n[1], uy = 0.0 * n[0] - 1.0 * n[2], uz = 1.0 * n[1] - 0.0 * n[0];
        double nu = norm3(ux, uy, uz);
        if (nu < 1e-6) {
            ux = 1.0 * n[2] - 0.0 * n[1];
            uy = 0.0 * n[0] - 0.0 * n[2];
            uz = 0.0 * n[1] - 1.0 * n[0];
            nu = norm3(ux, uy, uz);
            if (nu < 1e-6) continue;                                // Degenerate
        }
        ux /= nu;
        uy /= nu;
        uz /= nu;
        const double wx = n[1] * uz - n[2] * uy, wy = n[2] * ux - n[0] * uz, wz = n[0] * uy - n[1] * ux;   // n x u
        float* o = rows + i * R;
        for (int ch = 0; ch < 3; ++ch) o[ch] = (float)c[ch];
        const double rot[9] = {n[0], ux, wx, n[1], uy, wy, n[2], uz, wz};
        for (int q = 0; q < 9; ++q) o[3 + q] = (float)rot[q];
        const double s = a.kappa * (a.root_len / (double)(1ll << m.max_level));
        o[12] = (float)a.delta;
        o[13] = (float)s;
        o[14] = (float)s;
        o[15] = (float)a.opacity;
        for (int q = 0; q < 3 * a.K; ++q) o[16 + q] = 0.f;
        for (int ch = 0; ch < 3; ++ch) o[16 + ch] = (float)((col[ch] - 0.5) / 0.28209479177387814);
        status[i] = 1;
    }
}

cudaError_t launch_init_gaussians(const lsb_voxmap& m, const int64_t* keys, const double* cent, int64_t k,
                                  const float* image, int W, int H, const double* R_cw, const double* t_cw,
                                  const double* cam4, const double* origin, double near, double kappa, double delta,
                                  double opacity, int K, float* rows, uint8_t* status, cudaStream_t st) {
    InitArgs a;
    for (int q = 0; q < 9; ++q) a.R_cw[q] = R_cw[q];
    for (int q = 0; q < 3; ++q) {
        a.t_cw[q] = t_cw[q];
        a.origin[q] = origin[q];
    }
    a.fx = cam4[0];
    a.fy = cam4[1];
    a.cx = cam4[2];
    a.cy = cam4[3];
    a.W = W;
    a.H = H;
    a.K = K;
    a.near = near;
    a.kappa = kappa;
    a.delta = delta;
    a.opacity = opacity;
    a.root_len = m.root_len;
    if (k) k_init_gaussians<<<grid_for(k), 128, 0, st>>>(m, keys, cent, k, image, a, rows, status);
    return cudaGetLastError();
}

// Per group g (points perm[start_g .. start_g + count_g) in scan order): the
// mean as numpy's axis-0 mean evaluates it (row-by-row sums, then / count).
__global__ void k_segment_mean(const double* __restrict__ pts, const int64_t* __restrict__ perm,
                               const int64_t* __restrict__ starts, const int64_t* __restrict__ counts, int64_t k,
                               double* out) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < k; g += (int64_t)gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        const int64_t b = starts[g], n = counts[g];
        for (int64_t j = 0; j < n; ++j) {
            const int64_t p = perm[b + j];
            s0 = __dadd_rn(s0, pts[3 * p]);
            s1 = __dadd_rn(s1, pts[3 * p + 1]);
            s2 = __dadd_rn(s2, pts[3 * p + 2]);
        }
        out[3 * g] = s0 / (double)n;
        out[3 * g + 1] = s1 / (double)n;
        out[3 * g + 2] = s2 / (double)n;
    }
}

cudaError_t launch_segment_mean(const double* pts, const int64_t* perm, const int64_t* starts, const int64_t* counts,
                                int64_t k, double* out, cudaStream_t st) {
    if (k) k_segment_mean<<<grid_for(k), 128, 0, st>>>(pts, perm, starts, counts, k, out);
    return cudaGetLastError();
}

}  // namespace lsb

