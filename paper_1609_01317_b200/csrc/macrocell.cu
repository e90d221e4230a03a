// macrocell.cu -- min/max macrocell grid + per-window occupancy.
//
// GPU replacement for the reference's min/max octree (octree.py:52-136).
// Macrocell (mx, my, mz) covers the interpolation cells whose lower
// corner is in [8m, 8m+7] on every axis, i.e. voxels [8m, 8m+8] -- the
// same "pad by one voxel" rule the octree uses for its skip ranges
// (octree.py:4-8), because a trilinear sample in a cell reads the cell's
// upper corners.  Every trilinear / linear / nearest sample taken in such
// a cell lies within [min, max] of those voxels (a float64 lerp with
// t in [0,1] never leaves its endpoints' range), so a macrocell whose
// range misses the threshold window holds no in-window sample.
#include <cfloat>

#include "vc_internal.h"

namespace vc {

template <typename T>
__global__ void macrocell_minmax_kernel(const T* __restrict__ vol, int nx, int ny, int nz, float2* mm,
                                        int mx, int my, int mz) {
    // one warp per macrocell; lanes stride over the (<=9)^3 voxel box
    const int warps = (blockDim.x >> 5) * gridDim.x;
    const int lane = threadIdx.x & 31;
    const int total = mx * my * mz;
    for (int m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; m < total; m += warps) {
        const int cx = m % mx, cy = (m / mx) % my, cz = m / (mx * my);
        const int xa = cx * 8, ya = cy * 8, za = cz * 8;
        const int xb = min(xa + 8, nx - 1), yb = min(ya + 8, ny - 1), zb = min(za + 8, nz - 1);
        const int ex = xb - xa + 1, ey = yb - ya + 1, ez = zb - za + 1;
        float lo = FLT_MAX, hi = -FLT_MAX;
        for (int e = lane; e < ex * ey * ez; e += 32) {
            const int ix = e % ex, iy = (e / ex) % ey, iz = e / (ex * ey);
            const float v = (float)vol[((size_t)(za + iz) * ny + (ya + iy)) * nx + (xa + ix)];
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) mm[m] = make_float2(lo, hi);
    }
}

__global__ void occupancy_kernel(const float2* __restrict__ mm, int count, double lo, double hi,
                                 uint8_t* occ) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const float2 r = mm[i];
        occ[i] = ((double)r.x <= hi && (double)r.y >= lo) ? 1 : 0;
    }
}

cudaError_t launch_macrocell_minmax(int dtype, const void* data, int nx, int ny, int nz, float2* mm,
                                    int mx, int my, int mz, cudaStream_t s) {
    const int threads = 256;
    const int total = mx * my * mz;
    int blocks = (total * 32 + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    switch (dtype) {
        case VC_U8:
            macrocell_minmax_kernel<<<blocks, threads, 0, s>>>(static_cast<const uint8_t*>(data), nx, ny,
                                                               nz, mm, mx, my, mz);
            break;
        case VC_U16:
            macrocell_minmax_kernel<<<blocks, threads, 0, s>>>(static_cast<const uint16_t*>(data), nx, ny,
                                                               nz, mm, mx, my, mz);
            break;
        default:
            macrocell_minmax_kernel<<<blocks, threads, 0, s>>>(static_cast<const float*>(data), nx, ny, nz,
                                                               mm, mx, my, mz);
    }
    return cudaGetLastError();
}

cudaError_t launch_occupancy(const float2* mm, int count, double lo, double hi, uint8_t* occ,
                             cudaStream_t s) {
    int blocks = (count + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    occupancy_kernel<<<blocks, 256, 0, s>>>(mm, count, lo, hi, occ);
    return cudaGetLastError();
}

}  // namespace vc
