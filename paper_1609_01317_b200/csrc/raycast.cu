// raycast.cu -- Kernel 2: one thread per pixel, warp-tiled screen blocks.
//
// Restates _kernels.render_tile (/root/reference/pkg/src/voxelcast/_kernels.py:582-797)
// for one pixel per thread: ray generation (:639-648), ray/AABB interval
// (:649, :188-224), coarse-lattice march + fine backward scan (first_hit,
// :367-465), bisection (:468-487), HU -> LUT -> diffuse shading
// (_shade_sample, :528-579) and the surface / front-to-back composite
// with early ray termination (:744-797).  All of it float64 with the
// reference's operation order (see vc_device.cuh).
//
// B200 mapping
//   * block = 128 threads = 4 warps, each warp an 8x4 pixel tile, the block
//     a 16x8 screen tile: neighbouring rays share voxel cache lines in L1.
//   * empty-space skipping over an 8^3 macrocell grid replaces the
//     reference's octree (octree.py, _kernels.py:227-364).  It only jumps
//     over lattice samples t_enter + k*coarse that provably lie in cells
//     whose 8 corners are all outside the threshold window, so the
//     evaluated samples -- and the image -- are those of the brute-force
//     march (the invariant of pkg/tests/test_render.py:125-139).
//   * the shading gradient comes either from the reference taps or from
//     the packed float4 volume of Kernel 1 (interior only; the 1-voxel
//     boundary band always uses the taps).
//   * warp-vote retirement: per-warp sample / shade counters are reduced
//     with __reduce_add_sync and committed with one atomic per warp.
#include <cfloat>

#include "vc_device.cuh"
#include "vc_internal.h"

namespace vc {

constexpr int MC_SHIFT = 3;  // 8^3 voxel macrocells

struct Skip {
    // per macrocell: 0 = may hold an in-window sample; d >= 1 = every
    // macrocell within Chebyshev distance d-1 is empty (distance field of
    // the occupancy, rebuilt only when the threshold window changes)
    const uint8_t* __restrict__ dist;
    int mx, my;        // macrocell grid dims (x, y)
    double ib[3];      // 1 / (ray direction in voxel units per unit t)
    double inv_coarse;
    bool on;
};

template <typename T>
struct Ctx {
    Vol<T> v;
    const float4* __restrict__ grad;  // packed lattice gradients (may be null)
    RayPos rp;
    Skip sk;
};

// ceil(x) for 0 <= x < 2^31 without the XU pipe
__device__ __forceinline__ double ceil_pos(double x) {
    const double t = __dadd_rn(x, TWO52);
    double r = __dsub_rn(t, TWO52);
    if (r < x) r = __dadd_rn(r, 1.0);
    return r;
}

// Lattice index of the first sample after k that may leave the empty box
// of macrocells [m - (d-1), m + (d-1)] around position p (cell indices c).
// Samples strictly between are inside that box shrunk by 1e-6 voxel, hence
// inside the real box after the reference's rounding (error ~1e-13 voxel):
// they read provably out-of-window values and are skipped.  Only this
// conservativeness matters here, not bit-exactness.
__device__ __forceinline__ double skip_to(double t, double k, double base, const Skip& sk,
                                          const double p[3], const int c[3], int d) {
    constexpr double EPS = 1e-6;
    const int r = (d - 1) << MC_SHIFT;
    double dt = DBL_MAX;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const int lo = (c[a] >> MC_SHIFT) << MC_SHIFT;
        const double ib = sk.ib[a];
        if (ib > 0.0) dt = fmin(dt, ((double)(lo + (1 << MC_SHIFT) + r) - EPS - p[a]) * ib);
        else if (ib < 0.0) dt = fmin(dt, ((double)(lo - r) + EPS - p[a]) * ib);
    }
    double kn = k + 1.0;
    if (dt > 0.0) {
        const double x = (t + dt - base) * sk.inv_coarse;
        if (x > kn) kn = x < 1.0e9 ? ceil_pos(x) : 1.0e9;
    }
    return kn;
}

// Is the lattice sample at position p skippable?  Returns true when it is
// provably outside the window (no fetch needed) and updates k.
template <typename T>
__device__ __forceinline__ bool try_skip(const Ctx<T>& C, const double p[3], double t, double& k,
                                         double base, unsigned& nskip) {
    if (!in_range(C.v, p[0], p[1], p[2])) {  // reads 0, and 0 is outside the window
        k += 1.0;
        nskip += 1;
        return true;
    }
    int c[3];
    double f;
    c[0] = cell(p[0], C.v.nx, C.v.cx, f);
    c[1] = cell(p[1], C.v.ny, C.v.cy, f);
    c[2] = cell(p[2], C.v.nz, C.v.cz, f);
    const uint32_t m = ((uint32_t)(c[2] >> MC_SHIFT) * (uint32_t)C.sk.my + (uint32_t)(c[1] >> MC_SHIFT)) *
                           (uint32_t)C.sk.mx + (uint32_t)(c[0] >> MC_SHIFT);
    const int d = __ldg(C.sk.dist + m);
    if (d == 0) return false;
    const double kn = skip_to(t, k, base, C.sk, p, c, d);
    nskip += (unsigned)__double2uint_rz(kn - k);
    k = kn;
    return true;
}

// Trilinear interpolation of the packed gradient volume at an interior
// point; also returns the trilinear value from the .w channel, which is
// bit-identical to sample_trilinear (same operands, same order).
__device__ __forceinline__ void grad_from_volume(const float4* __restrict__ G, int nx, int ny,
                                                 const double p[3], double g[3], double& value) {
    double fx, fy, fz;
    double r;  // interior point: no clamping
    const int i0 = floor_pos(p[0], r);
    fx = dsub(p[0], r);
    const int j0 = floor_pos(p[1], r);
    fy = dsub(p[1], r);
    const int k0 = floor_pos(p[2], r);
    fz = dsub(p[2], r);
    const uint32_t sy = (uint32_t)nx, sz = (uint32_t)nx * (uint32_t)ny;
    const float4* b = G + (((uint32_t)k0 * (uint32_t)ny + (uint32_t)j0) * (uint32_t)nx + (uint32_t)i0);
    const float4 c000 = __ldg(b), c100 = __ldg(b + 1), c010 = __ldg(b + sy), c110 = __ldg(b + sy + 1);
    const float4 c001 = __ldg(b + sz), c101 = __ldg(b + sz + 1), c011 = __ldg(b + sz + sy),
                 c111 = __ldg(b + sz + sy + 1);
#define VC_TRI(comp)                                                                   \
    lerp(lerp(lerp((double)c000.comp, (double)c100.comp, fx),                          \
              lerp((double)c010.comp, (double)c110.comp, fx), fy),                     \
         lerp(lerp((double)c001.comp, (double)c101.comp, fx),                          \
              lerp((double)c011.comp, (double)c111.comp, fx), fy),                     \
         fz)
    g[0] = VC_TRI(x);
    g[1] = VC_TRI(y);
    g[2] = VC_TRI(z);
    value = VC_TRI(w);
#undef VC_TRI
}

struct Rgba {
    double r, g, b, a;
};

// Raw gradient from the reference taps, out of line: it is the rare path
// when shading from the gradient volume (boundary band only) and keeping
// it out of the march loop keeps the hot code small (the first profile
// showed instruction-cache stalls).
template <typename T, int OP>
__device__ __noinline__ double3 grad_taps(Vol<T> v, double x, double y, double z) {
    double g[3];
    grad_raw<T, OP>(v, x, y, z, g);
    return make_double3(g[0], g[1], g[2]);
}

// _kernels.py:528-579
template <typename T, int OP, int INTERP>
__device__ __forceinline__ Rgba shade_sample(const Ctx<T>& C, const vc_render_params& P, double t) {
    const RayPos& r = C.rp;
    const double wx = dadd(r.o[0], dmul(t, r.d[0]));
    const double wy = dadd(r.o[1], dmul(t, r.d[1]));
    const double wz = dadd(r.o[2], dmul(t, r.d[2]));
    double p[3];
    p[0] = dsub(r.pow2 ? dmul(wx, r.rs[0]) : ddiv(wx, r.s[0]), 0.5);
    p[1] = dsub(r.pow2 ? dmul(wy, r.rs[1]) : ddiv(wy, r.s[1]), 0.5);
    p[2] = dsub(r.pow2 ? dmul(wz, r.rs[2]) : ddiv(wz, r.s[2]), 0.5);
    double val, g[3];
    const bool interior = p[0] >= 1.0 && p[0] <= dsub(C.v.mx, 1.0) && p[1] >= 1.0 &&
                          p[1] <= dsub(C.v.my, 1.0) && p[2] >= 1.0 && p[2] <= dsub(C.v.mz, 1.0);
    if (C.grad != nullptr && interior) {
        double gv;
        grad_from_volume(C.grad, C.v.nx, C.v.ny, p, g, gv);
        val = (INTERP == VC_TRILINEAR) ? gv : sample_any<T, INTERP>(C.v, p[0], p[1], p[2]);
    } else {
        val = sample_any<T, INTERP>(C.v, p[0], p[1], p[2]);
        const double3 gg = grad_taps<T, OP>(C.v, p[0], p[1], p[2]);
        g[0] = gg.x;
        g[1] = gg.y;
        g[2] = gg.z;
    }
    double u[3];
    normalize3(g, u);
    // field values rise toward the interior, the surface normal points away
    const double snx = -u[0], sny = -u[1], snz = -u[2];
    const double lx = dsub(P.light_pos[0], wx);
    const double ly = dsub(P.light_pos[1], wy);
    const double lz = dsub(P.light_pos[2], wz);
    const double ln = __dsqrt_rn(dadd(dadd(dmul(lx, lx), dmul(ly, ly)), dmul(lz, lz)));
    double illum = 0.0;
    if (ln > 0.0) illum = ddiv(dadd(dadd(dmul(lx, snx), dmul(ly, sny)), dmul(lz, snz)), ln);
    illum = clamp01(illum);
    const double hu = dmul(ddiv(dsub(val, P.mu_water), P.mu_water), 1000.0);
    double m[4];
    lut_eval(P, hu, m);
    Rgba out;
    out.r = clamp01(dmul(dmul(illum, P.light_col[0]), m[0]));
    out.g = clamp01(dmul(dmul(illum, P.light_col[1]), m[1]));
    out.b = clamp01(dmul(dmul(illum, P.light_col[2]), m[2]));
    out.a = m[3];
    return out;
}

__device__ __forceinline__ bool in_window(const vc_render_params& P, double v) {
    return P.t_low <= v && v <= P.t_high;
}

// One pixel as a single state machine, so the march loop and the shading
// code each appear once in the binary:
//   phase 0: march t_enter + k*coarse to the first in-window sample, fine
//            backward scan, bisection (first_hit + bisect_window)
//   phase 1: march t_star + m*coarse to the next in-window sample
//            (composite loop, _kernels.py:755-790)
// and one shading site.  Accumulation is arranged so the first shade's
// acc = a*c, remain = 1 - a come out bit-identical to the reference
// (1.0*a*c == a*c, 0.0 + x == x, 1.0*(1-a) == 1-a).
template <typename T, int OP, int INTERP>
__device__ __forceinline__ uchar4 trace_pixel(Ctx<T>& C, const vc_render_params& P, int px, int py,
                                              unsigned& nsamp, unsigned& nshade, unsigned& nskip,
                                              unsigned& nhit) {
    const uchar4 bgq = make_uchar4(quant(P.bg[0]), quant(P.bg[1]), quant(P.bg[2]), quant(P.bg[3]));
    // ray generation, _kernels.py:639-648
    const double v_ndc = dsub(1.0, ddiv(dmul(2.0, dadd((double)py, 0.5)), (double)P.height));
    const double u_ndc = dsub(ddiv(dmul(2.0, dadd((double)px, 0.5)), (double)P.width), 1.0);
    const double uw = dmul(u_ndc, P.half_w), vh = dmul(v_ndc, P.half_h);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; a++) d[a] = dadd(dadd(P.forward[a], dmul(uw, P.right[a])), dmul(vh, P.up[a]));
    const double dn = __dsqrt_rn(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
    for (int a = 0; a < 3; a++) {
        C.rp.d[a] = ddiv(d[a], dn);
        C.rp.o[a] = P.eye[a];
        C.sk.ib[a] = C.rp.d[a] == 0.0 ? 0.0 : C.rp.s[a] / C.rp.d[a];
    }
    C.sk.inv_coarse = 1.0 / P.coarse;
    double t_enter, t_exit;
    if (!box_interval(C.rp.o, C.rp.d, P.clip_lo, P.clip_hi, t_enter, t_exit)) return bgq;
    nhit++;
    const double coarse = P.coarse, fine = P.fine;
    const double lim = dadd(t_exit, 1e-12);

    double base = t_enter, k = 0.0;  // lattice base and index (exact doubles)
    bool composite = false;
    double tcur = 0.0;
    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, remain = 1.0;
    for (;;) {
        // ---- march the lattice base + k*coarse to the next in-window sample
        bool found = false;
        double t = 0.0;
        for (;;) {
            t = dadd(base, dmul(k, coarse));
            if (t > lim) break;
            double p[3];
            C.rp.at(t, p);
            if (C.sk.on && try_skip(C, p, t, k, base, nskip)) continue;
            nsamp++;
            const double val = sample_any<T, INTERP>(C.v, p[0], p[1], p[2]);
            k += 1.0;
            if (in_window(P, val)) {
                found = true;
                break;
            }
        }
        if (!found) {
            if (!composite) return bgq;
            break;
        }
        if (!composite) {
            // fine backward scan (_kernels.py:419-436)
            bool bracket = false;
            double t_in = t, t_before = t;
            const double floor_t = dsub(t_enter, 1e-12);
            for (double j = 1.0;; j += 1.0) {
                const double tb = dsub(t, dmul(j, fine));
                if (tb < floor_t) {
                    t_in = t_before = dsub(t, dmul(j - 1.0, fine));
                    break;
                }
                double b[3];
                C.rp.at(tb, b);
                nsamp++;
                const double vb = sample_any<T, INTERP>(C.v, b[0], b[1], b[2]);
                if (!in_window(P, vb)) {
                    t_in = dsub(t, dmul(j - 1.0, fine));
                    t_before = tb;
                    bracket = true;
                    break;
                }
            }
            // bisect_window (_kernels.py:468-487)
            tcur = t_in;
            if (bracket && P.refine_iters > 0) {
                double tb = t_before, ta = t_in;
                for (int it = 0; it < P.refine_iters; it++) {
                    const double tm = dmul(0.5, dadd(tb, ta));
                    double p[3];
                    C.rp.at(tm, p);
                    nsamp++;
                    const double val = sample_any<T, INTERP>(C.v, p[0], p[1], p[2]);
                    if (in_window(P, val)) ta = tm;
                    else tb = tm;
                }
                tcur = ta;
            }
            base = tcur;
            k = 1.0;
        } else {
            tcur = t;
        }
        // ---- shade (the one call site)
        const Rgba s = shade_sample<T, OP, INTERP>(C, P, tcur);
        nshade++;
        if (P.mode == VC_SURFACE) return make_uchar4(quant(s.r), quant(s.g), quant(s.b), 255);
        const double w = dmul(remain, s.a);
        acc_r = dadd(acc_r, dmul(w, s.r));
        acc_g = dadd(acc_g, dmul(w, s.g));
        acc_b = dadd(acc_b, dmul(w, s.b));
        remain = dmul(remain, dsub(1.0, s.a));
        if (s.a >= OPAQUE_ALPHA || remain < MIN_REMAINING) break;
        composite = true;
    }
    acc_r = dadd(acc_r, dmul(remain, P.bg[0]));
    acc_g = dadd(acc_g, dmul(remain, P.bg[1]));
    acc_b = dadd(acc_b, dmul(remain, P.bg[2]));
    return make_uchar4(quant(acc_r), quant(acc_g), quant(acc_b), 255);
}

template <typename T, int OP, int INTERP>
__global__ void __launch_bounds__(128, 4) raycast_kernel(const __grid_constant__ vc_render_params P, Vol<T> vol,
                                                      const float4* __restrict__ grad, RayPos rp0,
                                                      const uint8_t* __restrict__ occ, int mx, int my,
                                                      int skip_on, uchar4* __restrict__ out,
                                                      int local_rows, unsigned long long* counters) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
    const int lr = blockIdx.y * 8 + (warp >> 1) * 4 + (lane >> 3);
    unsigned nsamp = 0, nshade = 0, nskip = 0, nhit = 0;
    if (px < P.width && lr < local_rows) {
        const int band = lr / P.band_rows, within = lr - band * P.band_rows;
        const int py = (P.band_first + band * P.band_step) * P.band_rows + within;
        if (py < P.height) {
            Ctx<T> C;
            C.v = vol;
            C.grad = grad;
            C.rp = rp0;
            C.sk.dist = occ;
            C.sk.mx = mx;
            C.sk.my = my;
            C.sk.on = skip_on != 0;
            out[(size_t)lr * P.width + px] =
                trace_pixel<T, OP, INTERP>(C, P, px, py, nsamp, nshade, nskip, nhit);
        }
    }
    if (counters != nullptr) {
        nsamp = __reduce_add_sync(0xffffffffu, nsamp);
        nshade = __reduce_add_sync(0xffffffffu, nshade);
        nskip = __reduce_add_sync(0xffffffffu, nskip);
        nhit = __reduce_add_sync(0xffffffffu, nhit);
        if (lane == 0) {
            if (nsamp) atomicAdd(counters + 0, (unsigned long long)nsamp);
            if (nshade) atomicAdd(counters + 1, (unsigned long long)nshade);
            if (nskip) atomicAdd(counters + 2, (unsigned long long)nskip);
            if (nhit) atomicAdd(counters + 3, (unsigned long long)nhit);
        }
    }
}

}  // namespace vc

namespace vc {

template <typename T, int OP, int INTERP>
static cudaError_t launch_t(const RenderLaunch& L, cudaStream_t stream) {
    const Vol<T> vol = make_vol(static_cast<const T*>(L.data), L.nx, L.ny, L.nz);
    const dim3 block(128);
    const dim3 grid((L.p->width + 15) / 16, (L.local_rows + 7) / 8);
    raycast_kernel<T, OP, INTERP><<<grid, block, 0, stream>>>(
        *L.p, vol, static_cast<const float4*>(L.grad), L.rp, L.occ, L.mx, L.my, L.skip_on,
        reinterpret_cast<uchar4*>(L.out), L.local_rows, reinterpret_cast<unsigned long long*>(L.counters));
    return cudaGetLastError();
}

template <typename T, int OP>
static cudaError_t launch_op(const RenderLaunch& L, cudaStream_t s) {
    switch (L.p->interp) {
        case VC_NEAREST: return launch_t<T, OP, VC_NEAREST>(L, s);
        case VC_LINEAR: return launch_t<T, OP, VC_LINEAR>(L, s);
        default: return launch_t<T, OP, VC_TRILINEAR>(L, s);
    }
}

template <typename T>
static cudaError_t launch_dtype(const RenderLaunch& L, cudaStream_t s) {
    switch (L.p->op) {
        case VC_OP_CENTRAL: return launch_op<T, VC_OP_CENTRAL>(L, s);
        case VC_OP_SOBEL3D: return launch_op<T, VC_OP_SOBEL3D>(L, s);
        default: return launch_op<T, VC_OP_ZUCKER_HUMMEL>(L, s);
    }
}

cudaError_t launch_raycast(const RenderLaunch& L, cudaStream_t s) {
    switch (L.dtype) {
        case VC_U8: return launch_dtype<uint8_t>(L, s);
        case VC_U16: return launch_dtype<uint16_t>(L, s);
        default: return launch_dtype<float>(L, s);
    }
}

}  // namespace vc
