// macrocell.cu -- min/max macrocell grid + per-window occupancy.
//
// GPU replacement for the reference's min/max octree (octree.py:52-136).
// Macrocell (mx, my, mz) covers the interpolation cells whose lower
// corner is in [E m, E m + E - 1] on every axis (E = MC_EDGE = 4), i.e.
// voxels [E m, E m + E] -- the
// same "pad by one voxel" rule the octree uses for its skip ranges
// (octree.py:4-8), because a trilinear sample in a cell reads the cell's
// upper corners.  Every trilinear / linear / nearest sample taken in such
// a cell lies within [min, max] of those voxels (a float64 lerp with
// t in [0,1] never leaves its endpoints' range), so a macrocell whose
// range misses the threshold window holds no in-window sample.
#include <cfloat>

#include "vc_internal.h"

namespace vc {

// One thread per macrocell column (cx, cy) and chunk of MC_ZCHUNK
// macrocells along z: it sweeps the planes of its chunk once, reducing the
// (MC_EDGE+1)^2 voxel patch of each plane, and closes a macrocell on its
// last plane -- which is also the first plane of the next one (the boxes
// overlap by one voxel).  A warp reads 32 adjacent patches of a row, so
// every plane is read with coalesced loads and each voxel about
// ((E+1)/E)^2 times from L1 (the warp-per-macrocell version re-gathered
// every box with scattered loads: 1.6 ms at 512^3, 20x slower).
constexpr int MC_ZCHUNK = 8;

template <typename T>
__global__ void __launch_bounds__(128) macrocell_minmax_kernel(const T* __restrict__ vol, int nx, int ny,
                                                               int nz, float2* mm, int mx, int my, int mz) {
    const int cx = blockIdx.x * blockDim.x + threadIdx.x;
    const int cy = blockIdx.y * blockDim.y + threadIdx.y;
    if (cx >= mx || cy >= my) return;
    int cz = blockIdx.z * MC_ZCHUNK;
    const int cz1 = min(cz + MC_ZCHUNK, mz);
    const int xa = cx * MC_EDGE, ya = cy * MC_EDGE;
    // clamped patch coordinates (a repeated edge voxel leaves min / max unchanged)
    int xs[MC_EDGE + 1], ys[MC_EDGE + 1];
#pragma unroll
    for (int d = 0; d <= MC_EDGE; d++) {
        xs[d] = min(xa + d, nx - 1);
        ys[d] = min(ya + d, ny - 1);
    }
    float lo = FLT_MAX, hi = -FLT_MAX;
    int zb = min(cz * MC_EDGE + MC_EDGE, nz - 1);
    for (int z = cz * MC_EDGE;; z++) {
        const T* plane = vol + (size_t)z * nx * ny;
        float pl = FLT_MAX, ph = -FLT_MAX;
#pragma unroll
        for (int dy = 0; dy <= MC_EDGE; dy++) {
            const T* row = plane + (size_t)ys[dy] * nx;
#pragma unroll
            for (int dx = 0; dx <= MC_EDGE; dx++) {
                const float v = (float)__ldg(row + xs[dx]);
                pl = fminf(pl, v);
                ph = fmaxf(ph, v);
            }
        }
        lo = fminf(lo, pl);
        hi = fmaxf(hi, ph);
        if (z == zb) {  // last plane of macrocell cz: also the first of cz + 1
            mm[((size_t)cz * my + cy) * mx + cx] = make_float2(lo, hi);
            if (++cz >= cz1) break;
            zb = min(cz * MC_EDGE + MC_EDGE, nz - 1);
            lo = pl;
            hi = ph;
        }
    }
}

// occupancy of the window [lo, hi]: 0 = may hold an in-window sample,
// DIST_CAP = empty.  Distances are capped at DIST_CAP = DIST_PASSES + 1
// (the largest jump, in macrocells), a valid lower bound beyond it.
constexpr uint8_t DIST_CAP = DIST_PASSES + 1;

__global__ void occupancy_kernel(const float2* __restrict__ mm, int count, double lo, double hi,
                                 uint8_t* dist) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const float2 r = mm[i];
        dist[i] = ((double)r.x <= hi && (double)r.y >= lo) ? 0 : DIST_CAP;
    }
}

// Chebyshev (L-infinity) distance transform of the occupancy, capped at
// DIST_CAP, in three separable 1-D passes:
//   D(c) = min_c' max(|dx|, |dy|, |dz|) = min_dz max(|dz|, min_dy max(|dy|,
//          min_dx max(|dx|, occ(c + d))))
// each pass over a window of +-DIST_CAP cells along one axis (outside the
// grid counts as empty).  dist[m] = d >= 1 guarantees that every macrocell
// within Chebyshev distance d - 1 of m is empty.  The result equals
// DIST_PASSES relaxation passes over the 26-neighbourhood (exact up to
// DIST_PASSES, DIST_CAP beyond) in 3 launches instead of 16.
__global__ void chebyshev_axis_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int mx,
                                      int my, int mz, int axis) {
    const int count = mx * my * mz;
    const int n = axis == 0 ? mx : (axis == 1 ? my : mz);
    const int stride = axis == 0 ? 1 : (axis == 1 ? mx : mx * my);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const int c = axis == 0 ? i % mx : (axis == 1 ? (i / mx) % my : i / (mx * my));
        int best = in[i];
        for (int d = 1; d < best; d++) {  // max(d, .) >= d: nothing at distance >= best can improve
            int v = DIST_CAP;
            if (c - d >= 0) v = min(v, (int)in[i - d * stride]);
            if (c + d < n) v = min(v, (int)in[i + d * stride]);
            best = min(best, max(d, v));
        }
        out[i] = (uint8_t)best;
    }
}

cudaError_t launch_macrocell_minmax(int dtype, const void* data, int nx, int ny, int nz, float2* mm,
                                    int mx, int my, int mz, cudaStream_t s) {
    const dim3 threads(32, 4);
    const dim3 blocks((mx + 31) / 32, (my + 3) / 4, (mz + MC_ZCHUNK - 1) / MC_ZCHUNK);
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
    occupancy_kernel<<<blocks, 256, 0, s>>>(mm, count, lo, hi, scratch);
    chebyshev_axis_kernel<<<blocks, 256, 0, s>>>(scratch, dist, mx, my, mz, 0);
    chebyshev_axis_kernel<<<blocks, 256, 0, s>>>(dist, scratch, mx, my, mz, 1);
    chebyshev_axis_kernel<<<blocks, 256, 0, s>>>(scratch, dist, mx, my, mz, 2);
    return cudaGetLastError();
}

}  // namespace vc
