// points.cu -- device kernels behind the point / single-ray public API.
//
// volume.sample          -> _kernels.sample_any        (_kernels.py:118-127)
// gradients.gradient     -> _kernels.grad_raw          (_kernels.py:140-177)
// raycast.intersect_clipbox -> _kernels.box_interval   (_kernels.py:215-224)
// raycast.march_surface  -> _kernels.first_hit         (_kernels.py:367-465)
// raycast.refine_hitpoint -> _kernels.bisect_window    (_kernels.py:468-487)
// One thread per point / ray; same float64 arithmetic as the renderer.
#include "vc_internal.h"

namespace vc {

template <typename T, int INTERP>
__global__ void sample_points_kernel(Vol<T> v, const double* __restrict__ pts, int64_t n, double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = sample_any<T, INTERP>(v, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

template <typename T, int OP>
__global__ void gradient_points_kernel(Vol<T> v, const double* __restrict__ pts, int64_t n, double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double g[3], center;
    if (!grad_raw_shared<T, OP>(v, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], g, center))
        grad_raw<T, OP>(v, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], g);
    out[3 * i] = g[0];
    out[3 * i + 1] = g[1];
    out[3 * i + 2] = g[2];
}

__global__ void box_rays_kernel(const double* __restrict__ rays, int64_t n, const double* lohi,
                                double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double t0 = 0.0, t1 = 0.0;
    const bool hit = box_interval(rays + 6 * i, rays + 6 * i + 3, lohi, lohi + 3, t0, t1);
    out[3 * i] = hit ? 1.0 : 0.0;
    out[3 * i + 1] = hit ? t0 : 0.0;
    out[3 * i + 2] = hit ? t1 : 0.0;
}

template <typename T, int INTERP>
__global__ void first_hit_kernel(Vol<T> v, RayPos rp, const double* __restrict__ rays, int64_t n,
                                 double coarse, double fine, double lo, double hi, double* out,
                                 unsigned long long* samples) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = rays + 8 * i;
    for (int a = 0; a < 3; a++) {
        rp.o[a] = r[a];
        rp.d[a] = r[3 + a];
    }
    const double t_enter = r[6], t_exit = r[7];
    unsigned long long cnt = 0;
    double res[4] = {0.0, 0.0, 0.0, 0.0};
    // _kernels.py:401-465 with the single segment [t_enter, t_exit]
    for (long long k = 0;; k++) {
        const double t = dadd(t_enter, dmul((double)k, coarse));
        if (t > dadd(t_exit, 1e-12)) break;
        double p[3];
        rp.at(t, p);
        cnt++;
        const double val = sample_any<T, INTERP>(v, p[0], p[1], p[2]);
        if (lo <= val && val <= hi) {
            for (long long j = 1;; j++) {
                const double tb = dsub(t, dmul((double)j, fine));
                if (tb < dsub(t_enter, 1e-12)) {
                    const double th = dsub(t, dmul((double)(j - 1), fine));
                    res[0] = 1.0;
                    res[1] = th;
                    res[2] = th;
                    res[3] = 0.0;
                    break;
                }
                double b[3];
                rp.at(tb, b);
                cnt++;
                const double vb = sample_any<T, INTERP>(v, b[0], b[1], b[2]);
                if (vb < lo || vb > hi) {
                    res[0] = 1.0;
                    res[1] = dsub(t, dmul((double)(j - 1), fine));
                    res[2] = tb;
                    res[3] = 1.0;
                    break;
                }
            }
            break;
        }
    }
    for (int c = 0; c < 4; c++) out[4 * i + c] = res[c];
    if (samples) atomicAdd(samples, cnt);
}

template <typename T, int INTERP>
__global__ void bisect_kernel(Vol<T> v, RayPos rp, const double* __restrict__ rays, int64_t n, double lo,
                              double hi, int iters, double* out, unsigned long long* samples) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = rays + 8 * i;
    for (int a = 0; a < 3; a++) {
        rp.o[a] = r[a];
        rp.d[a] = r[3 + a];
    }
    double tb = r[6], ta = r[7];
    for (int it = 0; it < iters; it++) {
        const double tm = dmul(0.5, dadd(tb, ta));
        double p[3];
        rp.at(tm, p);
        const double val = sample_any<T, INTERP>(v, p[0], p[1], p[2]);
        if (lo <= val && val <= hi) ta = tm;
        else tb = tm;
    }
    out[i] = ta;
    if (samples) atomicAdd(samples, (unsigned long long)iters);
}

static inline unsigned blocks_for(int64_t n) { return (unsigned)((n + 127) / 128); }

#define VC_DISPATCH_DTYPE(dtype, T, ...)            \
    switch (dtype) {                               \
        case VC_U8: {                              \
            using T = uint8_t;                     \
            __VA_ARGS__;                           \
        } break;                                   \
        case VC_U16: {                             \
            using T = uint16_t;                    \
            __VA_ARGS__;                           \
        } break;                                   \
        default: {                                 \
            using T = float;                       \
            __VA_ARGS__;                           \
        }                                          \
    }

#ifdef VC_CHECKED
VC_CHECKED_HOST_API(points)
#endif

cudaError_t launch_sample_points(int dtype, const void* data, int nx, int ny, int nz, int interp,
                                 const double* pts, int64_t n, double* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    VC_DISPATCH_DTYPE(dtype, T, {
        const Vol<T> v = make_vol(static_cast<const T*>(data), nx, ny, nz);
        if (interp == VC_NEAREST)
            sample_points_kernel<T, VC_NEAREST><<<blocks_for(n), 128, 0, s>>>(v, pts, n, out);
        else if (interp == VC_LINEAR)
            sample_points_kernel<T, VC_LINEAR><<<blocks_for(n), 128, 0, s>>>(v, pts, n, out);
        else
            sample_points_kernel<T, VC_TRILINEAR><<<blocks_for(n), 128, 0, s>>>(v, pts, n, out);
    })
    return cudaGetLastError();
}

cudaError_t launch_gradient_points(int dtype, const void* data, int nx, int ny, int nz, int op,
                                   const double* pts, int64_t n, double* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    VC_DISPATCH_DTYPE(dtype, T, {
        const Vol<T> v = make_vol(static_cast<const T*>(data), nx, ny, nz);
        if (op == VC_OP_CENTRAL)
            gradient_points_kernel<T, VC_OP_CENTRAL><<<blocks_for(n), 128, 0, s>>>(v, pts, n, out);
        else if (op == VC_OP_SOBEL3D)
            gradient_points_kernel<T, VC_OP_SOBEL3D><<<blocks_for(n), 128, 0, s>>>(v, pts, n, out);
        else
            gradient_points_kernel<T, VC_OP_ZUCKER_HUMMEL><<<blocks_for(n), 128, 0, s>>>(v, pts, n, out);
    })
    return cudaGetLastError();
}

cudaError_t launch_box_rays(const double* rays, int64_t n, const double* lohi, double* out,
                            cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    box_rays_kernel<<<blocks_for(n), 128, 0, s>>>(rays, n, lohi, out);
    return cudaGetLastError();
}

cudaError_t launch_first_hit_rays(int dtype, const void* data, int nx, int ny, int nz, RayPos rp,
                                  const double* rays, int64_t n, double coarse, double fine,
                                  double t_low, double t_high, int interp, double* out,
                                  unsigned long long* samples, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    VC_DISPATCH_DTYPE(dtype, T, {
        const Vol<T> v = make_vol(static_cast<const T*>(data), nx, ny, nz);
        if (interp == VC_NEAREST)
            first_hit_kernel<T, VC_NEAREST><<<blocks_for(n), 128, 0, s>>>(v, rp, rays, n, coarse, fine,
                                                                        t_low, t_high, out, samples);
        else if (interp == VC_LINEAR)
            first_hit_kernel<T, VC_LINEAR><<<blocks_for(n), 128, 0, s>>>(v, rp, rays, n, coarse, fine,
                                                                       t_low, t_high, out, samples);
        else
            first_hit_kernel<T, VC_TRILINEAR><<<blocks_for(n), 128, 0, s>>>(v, rp, rays, n, coarse, fine,
                                                                          t_low, t_high, out, samples);
    })
    return cudaGetLastError();
}

cudaError_t launch_bisect_rays(int dtype, const void* data, int nx, int ny, int nz, RayPos rp,
                               const double* rays, int64_t n, double t_low, double t_high, int iters,
                               int interp, double* out, unsigned long long* samples, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    VC_DISPATCH_DTYPE(dtype, T, {
        const Vol<T> v = make_vol(static_cast<const T*>(data), nx, ny, nz);
        if (interp == VC_NEAREST)
            bisect_kernel<T, VC_NEAREST><<<blocks_for(n), 128, 0, s>>>(v, rp, rays, n, t_low, t_high,
                                                                     iters, out, samples);
        else if (interp == VC_LINEAR)
            bisect_kernel<T, VC_LINEAR><<<blocks_for(n), 128, 0, s>>>(v, rp, rays, n, t_low, t_high,
                                                                    iters, out, samples);
        else
            bisect_kernel<T, VC_TRILINEAR><<<blocks_for(n), 128, 0, s>>>(v, rp, rays, n, t_low, t_high,
                                                                       iters, out, samples);
    })
    return cudaGetLastError();
}

}  // namespace vc
