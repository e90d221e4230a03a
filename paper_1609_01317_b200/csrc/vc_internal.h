// vc_internal.h -- launchers shared between the C-ABI layer and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "vc_device.cuh"

namespace vc {

// macrocell edge = 2^MC_SHIFT voxels (cells [m*E, m*E + E-1], voxels [m*E, m*E + E])
#ifndef VC_MC_SHIFT
#define VC_MC_SHIFT 2
#endif
constexpr int MC_SHIFT = VC_MC_SHIFT;
constexpr int MC_EDGE = 1 << MC_SHIFT;

// device copy of the level-grid octree (vc_octree_desc); levels == 0: none
struct OctDev {
    int levels;
    const int* dims;
    const int* amap;
    const int* ivl_off;
    const int* ivl;
    const long long* box_off;
    const uint8_t* state;
    const double* srange;
};

struct RenderLaunch {
    const vc_render_params* p;
    int dtype;
    const void* data;
    int nx, ny, nz;
    double amax;          // max |voxel value| (float32 pre-test bound)
    const void* grad;     // packed float4 gradient volume or nullptr (taps)
    RayPos rp;            // spacing / reciprocal / pow2 filled in; o, d per pixel
    const uint8_t* occ;   // macrocell occupancy for the current window
    int mx, my;
    int skip_on;
    int seg_walk;         // first hit replays the reference's octree-segment walk
    uint8_t* out;         // local_rows x width x 4 (npeers == 0)
    void* const* peers;   // device array of npeers full-frame buffers (fused gather)
    int npeers;
    int peer_self, peer_dest;  // this rank's own buffer in peers; receiving rank (-1: all)
    unsigned* tile_cnt;        // 8x4 tile completion counters (peer tile pushes) or nullptr
    int local_rows;
    uint64_t* counters;   // VC_NUM_COUNTERS or nullptr
    void* work;           // frame work counters (FrameWork, zeroed per launch)
    void* hits;           // first-hit queue, >= local_rows * width entries
    unsigned seq;         // this render's hit-entry tag (never 0, unique per scratch until it wraps)
    int overlap_stages;   // launch the shade kernel with programmatic stream serialization
    cudaEvent_t ev[3];    // optional: recorded before stage 1, between, after stage 2
    OctDev oct;           // adaptive stepping (levels == 0 when unused)
    // VC_SAMPLER_TEXTURE: tex3D objects over cudaArray copies of the grid
    // (normalized-float read for integer grids, tex_scale undoes it) and of
    // the float4 gradient volume (0 when grad == nullptr)
    cudaTextureObject_t tex_value, tex_grad;
    float tex_scale;
    // VC_CHECKED builds: the [lo, hi) byte ranges the launch may touch
    const unsigned long long* regions;
    int nregions;
};

#ifdef VC_CHECKED
cudaError_t vc_set_regions_raycast(const unsigned long long* lohi, int n, cudaStream_t s);
unsigned long long vc_take_violations_raycast(unsigned long long* first);
cudaError_t vc_set_regions_points(const unsigned long long* lohi, int n, cudaStream_t s);
unsigned long long vc_take_violations_points(unsigned long long* first);
#endif

cudaError_t launch_raycast(const RenderLaunch& L, cudaStream_t s);
size_t hit_entry_bytes();
size_t frame_work_bytes();

// Kernel 1 (gradient_prepass.cu)
cudaError_t launch_gradient_prepass(int dtype, const void* data, int nx, int ny, int nz, int op,
                                    float4* out, cudaStream_t s);

// macrocells (macrocell.cu)
cudaError_t launch_macrocell_minmax(int dtype, const void* data, int nx, int ny, int nz, float2* mm,
                                    int mx, int my, int mz, cudaStream_t s);
// occupancy of [lo, hi] + its Chebyshev distance field (dist: 0 = occupied)
#ifndef VC_DIST_PASSES
#define VC_DIST_PASSES 16
#endif
constexpr int DIST_PASSES = VC_DIST_PASSES;  // max jump = (DIST_PASSES + 1) macrocells
cudaError_t launch_occupancy(const float2* mm, int mx, int my, int mz, double lo, double hi, uint8_t* dist,
                             uint8_t* scratch, cudaStream_t s);

// device completion flags of the peer gather (peer.cu)
cudaError_t launch_signal_flags(uint32_t* const* blocks, int n, int dest, int slot, uint32_t seq, cudaStream_t s);
cudaError_t launch_wait_flags(const uint32_t* block, int first, int count, uint32_t seq, uint32_t timeout_us,
                              int32_t* status, cudaStream_t s);

// point queries (points.cu)
cudaError_t launch_sample_points(int dtype, const void* data, int nx, int ny, int nz, int interp,
                                 const double* pts, int64_t n, double* out, cudaStream_t s);
cudaError_t launch_gradient_points(int dtype, const void* data, int nx, int ny, int nz, int op,
                                   const double* pts, int64_t n, double* out, cudaStream_t s);
cudaError_t launch_box_rays(const double* rays, int64_t n, const double* lohi, double* out,
                            cudaStream_t s);
cudaError_t launch_first_hit_rays(int dtype, const void* data, int nx, int ny, int nz, RayPos rp,
                                  const double* rays, int64_t n, double coarse, double fine,
                                  double t_low, double t_high, int interp, double* out,
                                  unsigned long long* samples, cudaStream_t s);
cudaError_t launch_bisect_rays(int dtype, const void* data, int nx, int ny, int nz, RayPos rp,
                               const double* rays, int64_t n, double t_low, double t_high, int iters,
                               int interp, double* out, unsigned long long* samples, cudaStream_t s);

}  // namespace vc
