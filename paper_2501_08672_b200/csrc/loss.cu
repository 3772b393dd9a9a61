// Photometric loss (optimize.py:48-74): masked L1 / L2 value, MSE and the
// image gradient, fused in one HBM-bound pass.  The gradient is written
// per element; the two sums are reduced deterministically (fixed grid, block
// partials, last-block ticket).
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

constexpr int LOSS_BLOCKS = 296;
constexpr int LOSS_THREADS = 256;

__global__ void __launch_bounds__(LOSS_THREADS)
k_loss(const float* __restrict__ rend, const void* __restrict__ obs, bool obs_u8, const uint8_t* __restrict__ mask,
       int64_t npx, int kind, float gscale, float* __restrict__ grad, double* scratch) {
    __shared__ double s_r[LOSS_THREADS / 32][2];
    __shared__ bool s_last;
    double acc0 = 0.0, acc1 = 0.0;
    const int64_t n = 3 * npx;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const bool m = mask ? (mask[i / 3] != 0) : true;
        const double dd = (double)rend[i] - obs_value(obs, obs_u8, i);
        float gv = 0.f;
        if (m) {
            acc1 += dd * dd;
            if (kind == 0) {
                acc0 += fabs(dd);
                gv = (dd > 0.0) ? gscale : ((dd < 0.0) ? -gscale : 0.f);
            } else {
                acc0 += dd * dd;
                gv = (float)(2.0 * dd * (double)gscale);
            }
        }
        if (grad) grad[i] = gv;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
        acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
    }
    if (lane == 0) {
        s_r[warp][0] = acc0;
        s_r[warp][1] = acc1;
    }
    __syncthreads();
    double* part = scratch + 4;
    unsigned long long* ticket = (unsigned long long*)(scratch + 2);
    if (threadIdx.x < 2) {
        double v = 0.0;
        for (int k = 0; k < LOSS_THREADS / 32; ++k) v += s_r[k][threadIdx.x];
        part[2 * blockIdx.x + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1ull) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
        __threadfence();
        if (threadIdx.x < 2) {
            double v = 0.0;
            for (int b = 0; b < (int)gridDim.x; ++b) v += ((volatile double*)part)[2 * b + threadIdx.x];
            scratch[threadIdx.x] = v;
        }
        if (threadIdx.x == 0) *ticket = 0;
    }
}

cudaError_t launch_loss(const float* rend, const void* obs, const uint8_t* mask, int64_t npx,
                        int kind, float gscale, float* grad, double* scratch, cudaStream_t st) {
    k_loss<<<LOSS_BLOCKS, LOSS_THREADS, 0, st>>>(rend, obs, (kind & LSB_OBS_U8) != 0, mask, npx, kind & 0xff, gscale,
                                                 grad, scratch);
    return cudaGetLastError();
}

int loss_scratch_doubles() { return 4 + 2 * LOSS_BLOCKS; }

}  // namespace lsb
