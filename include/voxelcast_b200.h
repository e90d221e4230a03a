/*
 * voxelcast_b200.h -- C ABI of the B200-native per-pixel volume raycaster.
 *
 * Drop-in boundary for the hot path of the reference package `voxelcast`
 * (/root/reference/pkg/src/voxelcast).  The reference has no FFI: its
 * "kernel contract" is the numba function _kernels.render_tile
 * (_kernels.py:582-627) driven by raycast.render_frame (raycast.py:431-514),
 * plus _kernels.grad_raw (_kernels.py:140-177) behind gradients.gradient
 * (gradients.py:101-104).  Each entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - return value: VC_OK (0) or a vc_status error; the message is in
 *     vc_last_error() (thread-local).  Invalid parameters -> VC_ERR_INVALID
 *     (the Python layer raises ValueError, like the reference's dataclass
 *     validation, raycast.py:66-74, :195-215); CUDA failures ->
 *     VC_ERR_CUDA (RuntimeError).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - `d_` pointers are device (HBM) pointers, `h_` pointers host memory.
 *   - volumes are flat, x fastest: value(i,j,k) = data[i + nx*(j + ny*k)]
 *     (volume.py:51-52); world position of voxel (i,j,k) is
 *     ((i+0.5)*sx, ...), continuous voxel coords = world/spacing - 0.5
 *     (volume.py:3-7, _kernels.py:414-416).
 */
#ifndef VOXELCAST_B200_H
#define VOXELCAST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VC_API __attribute__((visibility("default")))
#else
#define VC_API
#endif

#define VC_ABI_VERSION 4
#define VC_MAX_LUT 64

typedef enum {
    VC_OK = 0,
    VC_ERR_INVALID = 1,
    VC_ERR_CUDA = 2,
    VC_ERR_NOMEM = 3,
    VC_ERR_UNSUPPORTED = 4
} vc_status;

/* voxel storage type.  The reference Volume is uint16 (volume.py:71); its
 * kernels are type-generic, so u8 and f32 grids are
 * accepted as well. */
typedef enum { VC_U8 = 0, VC_U16 = 1, VC_F32 = 2 } vc_dtype;

/* integer codes identical to _kernels.py:14-23 */
typedef enum { VC_OP_CENTRAL = 0, VC_OP_SOBEL3D = 1, VC_OP_ZUCKER_HUMMEL = 2 } vc_op;
typedef enum { VC_NEAREST = 0, VC_LINEAR = 1, VC_TRILINEAR = 2 } vc_interp;
typedef enum { VC_SURFACE = 0, VC_COMPOSITED = 1 } vc_mode;

/* where the shading gradient comes from */
typedef enum {
    /* the reference's 6/26 trilinear taps evaluated at the shade point,
     * reference term order, float64 (bit-faithful) */
    VC_GRAD_TAPS = 0,
    /* trilinear interpolation (float64) of the packed float4 lattice
     * gradient volume built by vc_gradient_prepass; taps in the 1-voxel
     * boundary band where the two differ */
    VC_GRAD_VOLUME = 1
} vc_grad_source;

/* how the scalar field (and, with VC_GRAD_VOLUME, the gradient) is
 * reconstructed at a ray sample */
typedef enum {
    /* the reference's float64 7-lerp cascade from 8 voxel loads
     * (_kernels.py:104-115): in-window decisions bit-exact */
    VC_SAMPLER_SOFTWARE = 0,
    /* hardware trilinear filtering of 3-D textures (tex3D on a cudaArray
     * copy of the grid and of the float4 gradient volume): 8-bit filter
     * weights, so decisions near the thresholds can differ from the
     * reference; tolerance stated in DESIGN.md.  Trilinear only. */
    VC_SAMPLER_TEXTURE = 1
} vc_sampler;

typedef struct vc_volume vc_volume;

/* Scalars of _kernels.render_tile (_kernels.py:583-627) in one POD block.
 * The camera basis is computed on the host exactly like
 * raycast.camera_basis (raycast.py:238-268); clip_lo/hi are already
 * intersected with the volume box (raycast.py:448-452).
 *
 * Image-plane partition (multi-GPU tiles): the image is cut into bands of
 * band_rows rows; this call renders bands b = band_first, band_first +
 * band_step, ... and writes them packed, in band order, into d_rgba
 * (rows x width x 4 uint8).  band_first = 0, band_step = 1,
 * band_rows = height renders the whole (height, width, 4) image. */
typedef struct vc_render_params {
    double eye[3];
    double right[3];
    double up[3];
    double forward[3];
    double half_w, half_h;
    int32_t width, height;
    int32_t band_rows, band_first, band_step;
    int32_t lut_n;
    double clip_lo[3], clip_hi[3];
    double light_pos[3], light_col[3];
    double t_low, t_high;               /* ThresholdWindow (raycast.py:113-124) */
    double lut_hu[VC_MAX_LUT];          /* TransferFunction.tables() (raycast.py:150-153) */
    double lut_rgba[VC_MAX_LUT][4];
    double mu_water;
    int32_t op, interp, mode, refine_iters;
    double coarse, fine;
    double bg[4];
    int32_t skip_empty;                 /* use_octree (raycast.py:187): macrocell empty-space
                                           skipping, output-neutral; with 0 inside
                                           [t_low, t_high] (or use_adaptive) the first hit
                                           replays the reference's octree-segment walk
                                           instead, which can skip in-window border samples
                                           as the reference does (needs vc_volume_set_octree) */
    int32_t grad_source;                /* vc_grad_source */
    /* adaptive stride (use_adaptive, _kernels.py:437-463): after an
     * out-of-window first-hit sample inside an octree leaf whose padded
     * range spans < detail_eps, advance up to adapt_jump lattice steps
     * (never past the leaf).  Needs vc_volume_set_octree; forces
     * skip_empty off (the stride depends on the exact lattice sequence). */
    int32_t use_adaptive, adapt_jump;
    double detail_eps;
    int32_t sampler;                    /* vc_sampler (ABI 2) */
    int32_t row_end;                    /* ABI 3: image rows >= row_end are not rendered
                                           (0 = none).  render_tile's [y0, y1) band
                                           (_kernels.py:582-627) is band_rows = 1,
                                           band_first = y0, band_step = 1, row_end = y1 */
} vc_render_params;

/* Min/max octree in level-grid form (see paper_1609_01317_b200/octree.py):
 * the boxes of depth L are the product of per-axis interval lists; per box
 * a state (0 absent, 1 internal, 2 leaf) and the padded value range.  All
 * arrays are host memory, copied by vc_volume_set_octree. */
typedef struct vc_octree_desc {
    int32_t levels;
    const int32_t *dims;     /* levels x 3: intervals per axis (x, y, z) */
    const int32_t *axis_map; /* levels x (nx + ny + nz): voxel index -> interval index */
    const int32_t *ivl_off;  /* levels x 3: offset of the axis' (lo, hi) pairs in ivl */
    const int32_t *ivl;      /* (lo, hi) voxel bounds of every interval, n_ivl ints */
    const int64_t *box_off;  /* levels: first box of the level in state / srange */
    const uint8_t *state;    /* per box, [bz][by][bx] within a level, n_boxes bytes */
    const double *srange;    /* per box (smin, smax), 2 x n_boxes doubles */
    int64_t n_ivl, n_boxes;
} vc_octree_desc;

/* counters written by vc_render (device, VC_NUM_COUNTERS x uint64):
 *   [0] volume samples taken by marching, fine scan, bisection and the
 *       composite loop (each one sample_any call in the reference)
 *   [1] shades (each _shade_sample call: 1 value sample + GRAD_SAMPLES taps)
 *   [2] empty-space skip events (jumps over empty macrocells, out-of-volume samples)
 *   [3] pixels whose ray hit the volume box
 *   [4] of [0], samples taken by the first-hit stage (march, fine scan, bisection)
 *   [5] of [0], samples taken by the shade stage (composite march)
 * The reference's FrameBuffer.sample_count (raycast.py:513) equals
 * c[0] + c[1] * (1 + GRAD_SAMPLES[op]) when skip_empty == 0. */
#define VC_NUM_COUNTERS 6

VC_API int vc_abi_version(void);
/* sizeof(vc_render_params), so bindings can check their struct mirror */
VC_API int vc_render_params_size(void);
VC_API const char *vc_last_error(void);
VC_API int vc_device_count(int *out);

/* Volume.from_array + upload (volume.py:61-80).  The device copy is
 * immutable after creation; also builds the macrocell
 * min/max grid used by empty-space skipping. */
VC_API int vc_volume_create(int device, const void *h_data, int dtype, int nx, int ny, int nz,
                     const double spacing[3], vc_volume **out);
/* same, from data already resident in HBM on `device` (copied): the
 * device side of the raw-slice ingest (load_raw_slices, volume.py:197-242). */
VC_API int vc_volume_create_device(int device, const void *d_data, int dtype, int nx, int ny, int nz,
                            const double spacing[3], vc_volume **out);
VC_API int vc_volume_destroy(vc_volume *vol);
/* Attach the octree used by adaptive stepping (octree.py:52-136). */
VC_API int vc_volume_set_octree(vc_volume *vol, const vc_octree_desc *desc);
/* device pointer of the voxel array (read-only) */
VC_API int vc_volume_data(const vc_volume *vol, const void **d_data);

/* Kernel 1: gradient pre-pass.  Lattice gradients of operator `op`
 * (grad_raw at every integer point, _kernels.py:140-177, zero outside
 * the grid) packed as float4 (gx, gy, gz, value), x fastest, cached on
 * the volume.  New: the reference computes gradients on the fly only. */
VC_API int vc_gradient_prepass(vc_volume *vol, int op, void *stream);
/* device pointer of the cached packed gradient volume (NULL if not built) */
VC_API int vc_gradient_volume(const vc_volume *vol, int op, const void **d_grad);
/* run the pre-pass into a caller buffer of nx*ny*nz float4 (no caching) */
VC_API int vc_gradient_prepass_into(const vc_volume *vol, int op, void *d_out, void *stream);

/* Kernel 2: raycast.  Replaces the thread-pool fan-out of
 * _kernels.render_tile in raycast.render_frame (raycast.py:476-505).
 * d_counters may be NULL. */
VC_API int vc_render(vc_volume *vol, const vc_render_params *p, uint8_t *d_rgba, uint64_t *d_counters,
              void *stream);
/* Image-tile render fused with the gather (multi-GPU, one process per GPU).
 * Every rank owns one full (height, width, 4) frame buffer; d_frames is a
 * device array of all ranks' buffers (this rank's own at index self, the
 * others mapped over NVLink with vc_ipc_open).  The call renders the bands
 * of p (band_first / band_step) and delivers them into the frame buffer of
 * every receiving rank (dest = -1: all ranks, an all-gather; dest = r: rank
 * r only, a gather) from inside the raycast kernels: with band_rows a
 * multiple of 4 each finished 8x4 screen tile is pushed as 16-byte row
 * segments, otherwise pixel by pixel.  With d_done set, a signal follows on
 * the same stream: after a system-scope fence, d_done[r][self] = seq for
 * every receiving rank r (release).  A receiver waits for
 * d_done[own][0..n) >= seq with vc_wait_flags on its stream: no host
 * barrier per frame.  Replaces the separate NCCL all-gather of packed bands
 * (raycast.py:476-505 has one host, one pool). */
#define VC_MAX_PEERS 64
typedef struct vc_peer_frames {
    void *const *d_frames;     /* device array [n] of frame buffers */
    uint32_t *const *d_done;   /* device array [n] of "done" flag blocks (VC_MAX_PEERS slots), or NULL */
    uint64_t frame_bytes;      /* size of every frame buffer (>= height * width * 4) */
    int32_t n;                 /* ranks, 1..VC_MAX_PEERS */
    int32_t self;              /* this rank's index */
    int32_t dest;              /* -1: every rank receives the frame; r: only rank r */
    uint32_t seq;              /* this frame's sequence number (signalled into d_done) */
} vc_peer_frames;
VC_API int vc_render_to_peers(vc_volume *vol, const vc_render_params *p, const vc_peer_frames *peers,
                              uint64_t *d_counters, void *stream);
/* Flag signal / wait of the peer protocol (also the "buffer free again"
 * back-channel from receivers to senders).  vc_signal_flags: after a
 * system-scope fence, blocks[r][slot] = seq for r in [0, n) (only r = dest
 * when dest >= 0), stream-ordered.  vc_wait_flags: the stream waits until
 * block[first .. first+count) are all >= seq (acquire, sequence numbers
 * compared modulo 2^32); after timeout_us it gives up and writes 1 to
 * *d_status (0 on success; d_status may be NULL). */
VC_API int vc_signal_flags(uint32_t *const *d_blocks, int n, int dest, int slot, uint32_t seq, void *stream);
VC_API int vc_wait_flags(const uint32_t *d_block, int first, int count, uint32_t seq, uint32_t timeout_us,
                         int32_t *d_status, void *stream);
/* Frame buffers shared across processes must be whole allocations (an IPC
 * handle maps the allocation base): allocate them here. */
VC_API int vc_device_alloc(int device, size_t bytes, void **d_ptr);
VC_API int vc_device_free(void *d_ptr);
VC_API int vc_memcpy_to_host(void *h_dst, const void *d_src, size_t bytes, void *stream);
/* CUDA IPC helpers for vc_render_to_peers: 64-byte handle of a device
 * allocation, open a peer's handle on `device`, close it. */
#define VC_IPC_HANDLE_BYTES 64
VC_API int vc_ipc_handle(const void *d_ptr, void *handle_out);
VC_API int vc_ipc_open(int device, const void *handle, void **d_ptr);
VC_API int vc_ipc_close(void *d_ptr);
/* vc_render plus per-stage device time (synchronous): stage_ms[0] = the
 * first-hit stage (ray generation, march, fine scan, bisection), stage_ms[1]
 * = the shade / composite stage.  For profiling and the roofline report. */
VC_API int vc_render_profiled(vc_volume *vol, const vc_render_params *p, uint8_t *d_rgba,
                              uint64_t *d_counters, void *stream, float *stage_ms);
/* render_frame end to end: render, copy the frame to host memory h_rgba
 * (pinned or pageable), counters to h_counters (may be NULL); synchronous.
 * *ms (may be NULL) = device time of render + copy (CUDA events). */
VC_API int vc_render_host(vc_volume *vol, const vc_render_params *p, uint8_t *h_rgba,
                   uint64_t *h_counters, float *ms);

/* Frame egress (image_io.png_bytes, image_io.py:52-55): encode a device
 * RGBA frame (height x width x 4, row-major) as an 8-bit RGB PNG on the
 * device and copy only the compressed file into h_out (capacity h_cap);
 * *out_len = file size.  h_out == NULL: size query.  Synchronous on stream. */
VC_API int vc_encode_png(const uint8_t *d_rgba, int width, int height, void *stream, uint8_t *h_out,
                         size_t h_cap, size_t *out_len);

/* Measured ceiling of the march's unit of work on `device`: float64 ray
 * samples per second (Gsamples/s) with all data L1-resident and no
 * divergence -- the "sample roofline" reported beside the HBM one. */
VC_API int vc_sample_peak(int device, double *gsamples_per_s);
/* The same ceiling for the VC_SAMPLER_TEXTURE path: tex3D trilinear
 * fetches (u16 grid, normalized float read) of an L1-resident 3-D texture. */
VC_API int vc_sample_peak_texture(int device, double *gsamples_per_s);

/* Point queries backing the public sampling / gradient API, host arrays.
 *   vc_sample_points   -> volume.sample / _kernels.sample_any (volume.py:104-110)
 *   vc_gradient_points -> _kernels.grad_raw (gradients.py:79-83), raw (N,3)  */
VC_API int vc_sample_points(const vc_volume *vol, int interp, const double *h_pts, int64_t n,
                     double *h_out);
VC_API int vc_gradient_points(const vc_volume *vol, int op, const double *h_pts, int64_t n,
                       double *h_out);

/* Single-ray helpers of raycast.py on the device.
 *   vc_box_interval_rays -> intersect_clipbox / _kernels.box_interval (raycast.py:283-293)
 *       h_rays: n x {org[3], dir[3]}; h_out: n x {hit, t0, t1}
 *   vc_first_hit_rays    -> march_surface / _kernels.first_hit (raycast.py:332-382)
 *       h_rays: n x {org[3], dir[3], t_enter, t_exit};
 *       h_out: n x {found, t_hit, t_before, bracket}
 *   vc_bisect_rays       -> refine_hitpoint / _kernels.bisect_window (raycast.py:385-411)
 *       h_rays: n x {org[3], dir[3], t_before, t_after}; h_out: n refined t */
VC_API int vc_box_interval_rays(const double *h_rays, int64_t n, const double lo[3], const double hi[3],
                         double *h_out);
VC_API int vc_first_hit_rays(const vc_volume *vol, const double *h_rays, int64_t n, double coarse,
                      double fine, double t_low, double t_high, int interp, double *h_out,
                      uint64_t *h_samples);
VC_API int vc_bisect_rays(const vc_volume *vol, const double *h_rays, int64_t n, double t_low,
                   double t_high, int iters, int interp, double *h_out, uint64_t *h_samples);

#ifdef __cplusplus
}
#endif

#endif /* VOXELCAST_B200_H */
