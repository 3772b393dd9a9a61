// Packed leaf keys and the open-addressing probe of the voxel map (shared by
// voxmap.cu and window.cu).
#pragma once
#include "common.cuh"

namespace lsb {

constexpr unsigned long long EMPTY = ~0ull;
constexpr int KB = 21;                       // bits per packed coordinate
constexpr long long KOFF = 1ll << (KB - 1);  // signed offset
constexpr unsigned long long KMASK = (1ull << KB) - 1;

__device__ __forceinline__ unsigned long long pack_key(long long ix, long long iy, long long iz) {
    return ((unsigned long long)(ix + KOFF) & KMASK) | (((unsigned long long)(iy + KOFF) & KMASK) << KB) |
           (((unsigned long long)(iz + KOFF) & KMASK) << (2 * KB));
}

__device__ __forceinline__ void unpack_key(unsigned long long k, long long& ix, long long& iy, long long& iz) {
    ix = (long long)(k & KMASK) - KOFF;
    iy = (long long)((k >> KB) & KMASK) - KOFF;
    iz = (long long)((k >> (2 * KB)) & KMASK) - KOFF;
}

__device__ __forceinline__ unsigned long long slot_of(long long ix, long long iy, long long iz, int level,
                                                      unsigned long long mask) {
    // VoxelKey.__hash__ (voxmap.py:27-28), then a murmur3 finaliser for the low bits
    unsigned long long h = (unsigned long long)((ix * 73856093ll) ^ (iy * 19349669ll) ^ (iz * 83492791ll) ^ level);
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h & mask;
}

__device__ __forceinline__ bool in_range(long long v) { return v >= -KOFF && v < KOFF; }

// Find or create the slot of a leaf key; -1 if the table is full.
__device__ __forceinline__ long long find_or_insert(const lsb_voxmap& m, long long ix, long long iy, long long iz) {
    const unsigned long long key = pack_key(ix, iy, iz);
    const unsigned long long mask = (unsigned long long)m.cap - 1;
    unsigned long long s = slot_of(ix, iy, iz, m.max_level, mask);
    for (long long probe = 0; probe < m.cap; ++probe) {
        const unsigned long long cur = (unsigned long long)m.keys[s];
        if (cur == key) return (long long)s;
        if (cur == EMPTY) {
            const unsigned long long prev = atomicCAS((unsigned long long*)&m.keys[s], EMPTY, key);
            if (prev == EMPTY) {
                atomicAdd((unsigned long long*)m.n_used, 1ull);
                return (long long)s;
            }
            if (prev == key) return (long long)s;
        }
        s = (s + 1) & mask;
    }
    return -1;
}

__device__ __forceinline__ long long find(const lsb_voxmap& m, long long ix, long long iy, long long iz) {
    const unsigned long long key = pack_key(ix, iy, iz);
    const unsigned long long mask = (unsigned long long)m.cap - 1;
    unsigned long long s = slot_of(ix, iy, iz, m.max_level, mask);
    for (long long probe = 0; probe < m.cap; ++probe) {
        const unsigned long long cur = (unsigned long long)m.keys[s];
        if (cur == key) return (long long)s;
        if (cur == EMPTY) return -1;
        s = (s + 1) & mask;
    }
    return -1;
}

}  // namespace lsb
