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
        const int xa = cx * MC_EDGE, ya = cy * MC_EDGE, za = cz * MC_EDGE;
        const int xb = min(xa + MC_EDGE, nx - 1), yb = min(ya + MC_EDGE, ny - 1), zb = min(za + MC_EDGE, nz - 1);
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

// occupancy of the window [lo, hi]: 0 = may hold an in-window sample,
// DIST_CAP = empty.  Empty cells start at the cap, not at infinity: after
// DIST_PASSES relaxation passes every cell within DIST_PASSES of an
// occupied one holds its exact distance, and every other cell keeps
// DIST_CAP = DIST_PASSES + 1, a valid lower bound of its distance.
constexpr uint8_t DIST_CAP = DIST_PASSES + 1;

__global__ void occupancy_kernel(const float2* __restrict__ mm, int count, double lo, double hi,
                                 uint8_t* dist) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const float2 r = mm[i];
        dist[i] = ((double)r.x <= hi && (double)r.y >= lo) ? 0 : DIST_CAP;
    }
}

// One relaxation pass of the Chebyshev (L-infinity) distance transform of
// the occupancy over the 26-neighbourhood.  Macrocells outside the grid
// hold no in-range sample and count as empty.  Shortest 26-neighbour paths
// have exactly the Chebyshev length, so dist[m] = d >= 1 guarantees that
// every macrocell within Chebyshev distance d - 1 of m is empty.
__global__ void chebyshev_pass_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int mx,
                                      int my, int mz) {
    const int count = mx * my * mz;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const int x = i % mx, y = (i / mx) % my, z = i / (mx * my);
        int best = in[i];
        if (best != 0) {
            for (int dz = -1; dz <= 1; dz++) {
                const int zz = z + dz;
                if (zz < 0 || zz >= mz) continue;
                for (int dy = -1; dy <= 1; dy++) {
                    const int yy = y + dy;
                    if (yy < 0 || yy >= my) continue;
                    for (int dx = -1; dx <= 1; dx++) {
                        const int xx = x + dx;
                        if (xx < 0 || xx >= mx) continue;
                        const int v = in[(zz * my + yy) * mx + xx] + 1;
                        if (v < best) best = v;
                    }
                }
            }
        }
        out[i] = (uint8_t)best;
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

cudaError_t launch_occupancy(const float2* mm, int mx, int my, int mz, double lo, double hi, uint8_t* dist,
                             uint8_t* scratch, cudaStream_t s) {
    const int count = mx * my * mz;
    int blocks = (count + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    occupancy_kernel<<<blocks, 256, 0, s>>>(mm, count, lo, hi, dist);
    // distances up to DIST_PASSES + 1 macrocells (8 voxels each); an even
    // pass count leaves the result in `dist`
    for (int p = 0; p < DIST_PASSES; p += 2) {
        chebyshev_pass_kernel<<<blocks, 256, 0, s>>>(dist, scratch, mx, my, mz);
        chebyshev_pass_kernel<<<blocks, 256, 0, s>>>(scratch, dist, mx, my, mz);
    }
    return cudaGetLastError();
}

}  // namespace vc
