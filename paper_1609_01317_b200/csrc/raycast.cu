// raycast.cu -- Kernel 2: one ray per lane, warp-tiled screen blocks.
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
//   * two persistent kernels per frame (a wavefront split): firsthit_kernel
//     generates rays, marches to the first in-window lattice sample, refines
//     it and queues the hit; shade_kernel pulls hits, shades and composites
//     front to back with early ray termination.  Each sizes its grid to the
//     resident CTAs of 148 SMs and tunes its own register budget.
//   * work is handed out per lane through warp-aggregated atomic tickets in
//     8x4 screen tiles (a refilled warp traces a compact tile: L1 reuse), and
//     finished lanes are refilled at once (dynamic ray scheduling), so warps
//     stay full although rays march very different lengths; warp votes
//     decide when a warp leaves its march loop.
//   * empty-space skipping over a 4^3 macrocell grid replaces the
//     reference's octree (octree.py, _kernels.py:227-364).  It only jumps
//     over lattice samples t_enter + k*coarse that provably lie in cells
//     whose 8 corners are all outside the threshold window, so the
//     evaluated samples -- and the image -- are those of the brute-force
//     march (the invariant of pkg/tests/test_render.py:125-139).  Only
//     use_adaptive with use_octree replays the reference's octree-segment
//     walk (firsthit_seg_kernel, itself a wavefront over walk nodes and
//     lattice samples), because there the samples that exist decide the
//     pixel.
//   * the shading gradient comes either from the reference taps or from
//     the packed float4 volume of Kernel 1 (interior only; the 1-voxel
//     boundary band always uses the taps, and so do samples whose corner
//     gradients cancel, see grad_from_volume); the scalar field either from
//     the float64 software cascade or from tex3D (VC_SAMPLER_TEXTURE).
//   * per-warp sample / shade counters are reduced with __reduce_add_sync
//     and committed with one atomic per warp.
#include <cfloat>
#include <cmath>
#include <type_traits>

#include "vc_device.cuh"
#include "vc_internal.h"

namespace vc {


struct Skip {
    // per macrocell: 0 = may hold an in-window sample; d >= 1 = every
    // macrocell within Chebyshev distance d-1 is empty (distance field of
    // the occupancy, rebuilt only when the threshold window changes)
    const uint8_t* __restrict__ dist;
    int mx, my;        // macrocell grid dims (x, y)
    double ib[3];      // 1 / (ray direction in voxel units per unit t)
    double inv_coarse;
    float inv_coarse_f;
    bool on;
    WinF win;          // float32 pre-test thresholds of the window
};

// VC_SAMPLER_TEXTURE: the kernels take INTERP == VC_TEX (an internal code
// next to the reference's 0/1/2) and sample through the texture unit
constexpr int VC_TEX = 3;

struct TexArgs {
    cudaTextureObject_t v, g;  // scalar grid, float4 gradient volume (0: none)
    float scale;               // undoes the normalized-float read of integer grids
    float lo, hi;              // window thresholds rounded inward (exact test for a float value)
};

template <typename T>
struct Ctx {
    Vol<T> v;
    const float4* __restrict__ grad;  // packed lattice gradients (may be null)
    RayPos rp;
    Skip sk;
    TexArgs tx;
    double rmu;                       // rcp_for(mu_water): the HU division
    const SharedLut* lut;             // shade stage: transfer breakpoints in shared memory
};

// ceil(x) for 0 <= x < 2^31 without the XU pipe
__device__ __forceinline__ double ceil_pos(double x) {
    const double t = __dadd_rn(x, MAGIC_RND);
    double r = __dsub_rn(t, MAGIC_RND);
    if (r < x) r = __dadd_rn(r, 1.0);
    return r;
}

// Lattice index of the first sample after k that may leave the empty box
// of macrocells [m - (d-1), m + (d-1)] around position p (cell indices c).
// Samples strictly between are inside that box shrunk by 1e-6 voxel, hence
// inside the real box after the reference's rounding (error ~1e-13 voxel):
// they read provably out-of-window values and are skipped.  Only this
// conservativeness matters here, not bit-exactness.
// LAZY (shade stage, few skip events per ray): the reciprocal speeds are
// recomputed here from the direction instead of living in registers
// RN(1/x) pinned to where it is written: the compiler hoists a plain
// __drcp_rn of the (per-ray) direction out of the rare skip branch to every
// resolve step of the shade loop (ncu: three MUFU.RCP64H + Newton chains per
// shade).  Same instruction (rcp.rn.f64), same value.
__device__ __forceinline__ double drcp_rn_here(double x) {
    double r;
    asm volatile("rcp.rn.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

template <bool LAZY = false>
__device__ __forceinline__ double skip_to(double t, double k, double base, const Skip& sk, const RayPos& rp,
                                          const double p[3], const int c[3], int d) {
    constexpr double EPS = 1e-6;
    const int r = (d - 1) << MC_SHIFT;
    double dt = DBL_MAX;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const int lo = (c[a] >> MC_SHIFT) << MC_SHIFT;
        const double ib = LAZY ? (rp.d[a] == 0.0 ? 0.0 : dmul(rp.s[a], drcp_rn_here(rp.d[a]))) : sk.ib[a];
        // the box face ahead, in voxel units (branch-free: selects, one exact
        // int -> double on the FP64 pipe); a zero direction adds no limit
        const bool up = ib > 0.0;
        const int face = up ? lo + (1 << MC_SHIFT) + r : lo - r;
        const double cand = (biased2d((uint32_t)face + 0x80000000u) + (up ? -EPS : EPS) - p[a]) * ib;
        dt = ib != 0.0 ? fmin(dt, cand) : dt;
    }
    double kn = k + 1.0;
    if (dt > 0.0) {
        const double x = (t + dt - base) * sk.inv_coarse;
        if (x > kn) kn = x < 1.0e9 ? ceil_pos(x) : 1.0e9;
    }
    return kn;
}

__device__ __forceinline__ bool in_window(const vc_render_params& P, double v) {
    return P.t_low <= v && v <= P.t_high;
}

__device__ __forceinline__ uint32_t macro_index(const Skip& sk, const Loc& L) {
    return ((uint32_t)(L.k >> MC_SHIFT) * (uint32_t)sk.my + (uint32_t)(L.j >> MC_SHIFT)) * (uint32_t)sk.mx +
           (uint32_t)(L.i >> MC_SHIFT);
}

// texture-unit trilinear value at voxel-space p (texel centres at i + 0.5)
__device__ __forceinline__ float tex_value(const TexArgs& t, const double p[3]) {
    return tex3D<float>(t.v, __double2float_rn(p[0]) + 0.5f, __double2float_rn(p[1]) + 0.5f,
                        __double2float_rn(p[2]) + 0.5f) * t.scale;
}
__device__ __forceinline__ bool tex_in_window(const TexArgs& t, const double p[3]) {
    const float v = tex_value(t, p);
    return v >= t.lo && v <= t.hi;
}

// One lattice sample of the march: -1 when empty-space skipping proves it
// out of window (k has been advanced, no fetch), else whether the
// reference's sample_any at p lies in the threshold window (0 / 1).
template <typename T, int INTERP, bool LAZY = false>
__device__ __forceinline__ int march_sample(const Ctx<T>& C, const vc_render_params& P, const double p[3],
                                            double t, double& k, double base, unsigned& nskip) {
    if (INTERP != VC_TRILINEAR && INTERP != VC_TEX) {
        if (C.sk.on && !in_range(C.v, p[0], p[1], p[2])) {  // reads 0, outside the window
            k += 1.0;
            nskip += 1;
            return -1;
        }
        if (C.sk.on) {
            Loc L;
            locate(C.v, p, L);
            const int d = vc_ldg(C.sk.dist + macro_index(C.sk, L));
            if (d != 0) {
                const int c[3] = {L.i, L.j, L.k};
                const double kn = skip_to<LAZY>(t, k, base, C.sk, C.rp, p, c, d);
                nskip += 1;
                k = kn;
                return -1;
            }
        }
        return in_window(P, sample_any<T, INTERP>(C.v, p[0], p[1], p[2])) ? 1 : 0;
    }
    Loc L;
    const bool inr = locate(C.v, p, L);
    if (C.sk.on) {
        if (!inr) {  // reads 0, and 0 is outside the window when skipping is on
            k += 1.0;
            nskip += 1;
            return -1;
        }
        const int d = vc_ldg(C.sk.dist + macro_index(C.sk, L));
        if (d != 0) {
            const int c[3] = {L.i, L.j, L.k};
            const double kn = skip_to<LAZY>(t, k, base, C.sk, C.rp, p, c, d);
            nskip += 1;  // one empty-space jump (counting the samples it skips costs 3%)
            k = kn;
            return -1;
        }
    }
    if (!inr) return in_window(P, 0.0) ? 1 : 0;
    if (INTERP == VC_TEX) return tex_in_window(C.tx, p) ? 1 : 0;
    return in_window_trilinear(C.v, L, P.t_low, P.t_high, C.sk.win) ? 1 : 0;
}

// is sample_any at p in the window? (fine scan, bisection)
template <typename T, int INTERP>
__device__ __forceinline__ bool window_at(const Ctx<T>& C, const vc_render_params& P, const double p[3]) {
    if (INTERP == VC_TEX) {
        if (!in_range(C.v, p[0], p[1], p[2])) return in_window(P, 0.0);
        return tex_in_window(C.tx, p);
    }
    if (INTERP != VC_TRILINEAR) return in_window(P, sample_any<T, INTERP>(C.v, p[0], p[1], p[2]));
    Loc L;
    if (!locate(C.v, p, L)) return in_window(P, 0.0);
    return in_window_trilinear(C.v, L, P.t_low, P.t_high, C.sk.win);
}

// Trilinear interpolation of the packed gradient volume at an interior
// point.  The value comes from the .w channel in float64 and is
// bit-identical to sample_trilinear (same operands, same order), so the
// opacity, the transmittance and every early-termination decision stay the
// reference's.  The gradient only feeds the diffuse term; it is stored in
// float32 and interpolated in float32 (the float64 lerps of float32 data
// bought nothing: the stored values already carry the float32 rounding).
template <typename T>
__device__ __forceinline__ double w_to_double(float w) {
    if constexpr (std::is_integral<T>::value) {
        // .w holds an exact integer <= 65535: w + 2^23 has it as mantissa
        return u2d(__float_as_uint(__fadd_rn(w, 8388608.0f)) & 0x7fffffu);
    } else {
        return (double)w;
    }
}

// The suspect case of grad_from_volume, out of line (the corners are
// re-read from L1 rather than kept live on the hot path): the same corners
// re-interpolated in float64 -- exact inputs for CD / Sobel on integer
// grids, so only 2^-53 M rounding remains; for ZH and float grids the
// storage error 2^-24 M stays and |g| >= 1e-4 M is still required.
// .w = 0 when the reference taps are needed after all (that, or the
// EPS_GRADIENT band |g| < 2e-8).
template <typename T, int OP>
__device__ __noinline__ float4 gv_refine(const float4* __restrict__ b, uint32_t sy, uint32_t sz, double fx,
                                         double fy, double fz, float M) {
    const float4 c000 = vc_ldg(b), c100 = vc_ldg(b + 1), c010 = vc_ldg(b + sy), c110 = vc_ldg(b + sy + 1);
    const float4 c001 = vc_ldg(b + sz), c101 = vc_ldg(b + sz + 1), c011 = vc_ldg(b + sz + sy),
                 c111 = vc_ldg(b + sz + sy + 1);
    double h[3];
#define VC_TRID(comp)                                                                                        \
    lerp(lerp(lerp((double)c000.comp, (double)c100.comp, fx), lerp((double)c010.comp, (double)c110.comp, fx), \
              fy),                                                                                           \
         lerp(lerp((double)c001.comp, (double)c101.comp, fx), lerp((double)c011.comp, (double)c111.comp, fx), \
              fy),                                                                                           \
         fz)
    h[0] = VC_TRID(x);
    h[1] = VC_TRID(y);
    h[2] = VC_TRID(z);
#undef VC_TRID
    const double h2 = dadd(dadd(dmul(h[0], h[0]), dmul(h[1], h[1])), dmul(h[2], h[2]));
    constexpr bool exact_corners = std::is_integral<T>::value && OP != VC_OP_ZUCKER_HUMMEL;
    const bool ok = !(h2 < 4e-16 || (!exact_corners && h2 < 1e-8 * ((double)M * (double)M)));
    return make_float4((float)h[0], (float)h[1], (float)h[2], ok ? 1.0f : 0.0f);
}

// Trilinear interpolation of the packed gradient volume at an interior point
// p: value (float64, exact) and the gradient for the diffuse term, in
// float32.  Returns whether that gradient is suspect; `cell` and `M` feed
// gv_refine then.
//
// The float32 gradient's absolute error is at most about 13 * 2^-24 * M
// per component (M = largest corner component: the float32 storage of
// irrational / float corners, then three lerp levels each rounding b - a,
// the fraction and the fma), so its direction is good to the 1/255 bar
// whenever |g| >= 1e-3 M.  Below that the corners cancel (a zero crossing
// of the gradient field; ~0.08% of the C3 shades) and the sample is
// suspect, as is one near the reference's EPS_GRADIENT cutoff (|g| < 2e-8
// with nonzero corners), where the zero-normal decision could differ.
template <typename T, int OP>
__device__ __forceinline__ bool grad_from_volume(const float4* __restrict__ G, int nx, int ny,
                                                 const double p[3], float g[3], double& value,
                                                 const float4*& cell, float& M) {
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
    cell = b;
    const float4 c000 = vc_ldg(b), c100 = vc_ldg(b + 1), c010 = vc_ldg(b + sy), c110 = vc_ldg(b + sy + 1);
    const float4 c001 = vc_ldg(b + sz), c101 = vc_ldg(b + sz + 1), c011 = vc_ldg(b + sz + sy),
                 c111 = vc_ldg(b + sz + sy + 1);
    const float ffx = (float)fx, ffy = (float)fy, ffz = (float)fz;
#define VC_LF(a, b, t) fmaf((b) - (a), (t), (a))
#define VC_TRIF(comp)                                                                          \
    VC_LF(VC_LF(VC_LF(c000.comp, c100.comp, ffx), VC_LF(c010.comp, c110.comp, ffx), ffy),     \
          VC_LF(VC_LF(c001.comp, c101.comp, ffx), VC_LF(c011.comp, c111.comp, ffx), ffy), ffz)
    g[0] = VC_TRIF(x);
    g[1] = VC_TRIF(y);
    g[2] = VC_TRIF(z);
#undef VC_TRIF
#undef VC_LF
#define VC_W(c) w_to_double<T>(c.w)
    value = lerp(lerp(lerp(VC_W(c000), VC_W(c100), fx), lerp(VC_W(c010), VC_W(c110), fx), fy),
                 lerp(lerp(VC_W(c001), VC_W(c101), fx), lerp(VC_W(c011), VC_W(c111), fx), fy), fz);
#undef VC_W
#define VC_AM(c) fmaxf(fabsf(c.x), fmaxf(fabsf(c.y), fabsf(c.z)))
    M = fmaxf(fmaxf(fmaxf(VC_AM(c000), VC_AM(c100)), fmaxf(VC_AM(c010), VC_AM(c110))),
              fmaxf(fmaxf(VC_AM(c001), VC_AM(c101)), fmaxf(VC_AM(c011), VC_AM(c111))));
#undef VC_AM
    const float g2 = fmaf(g[0], g[0], fmaf(g[1], g[1], g[2] * g[2]));
    return g2 < 1e-6f * M * M || (g2 < 4e-16f && M > 0.0f);
}

#ifdef VC_DEBUG_TAPS
__device__ unsigned g_debug_taps;
}  // namespace vc
extern "C" __attribute__((visibility("default"))) unsigned vc_debug_taps() {
    unsigned h = 0, z = 0;
    cudaMemcpyFromSymbol(&h, vc::g_debug_taps, sizeof(unsigned));
    cudaMemcpyToSymbol(vc::g_debug_taps, &z, sizeof(unsigned));
    return h;
}
namespace vc {
#endif

struct Rgba {
    double r, g, b, a;
};

// Raw gradient from the reference taps, out of line: it is the rare path
// when shading from the gradient volume (boundary band only) and keeping
// it out of the march loop keeps the hot code small (the first profile
// showed instruction-cache stalls).
// .w of the result: sample_trilinear at the point when the shared-footprint
// path applied (NaN otherwise)
template <typename T, int OP, bool ROLL = false>
__device__ __noinline__ double4 grad_taps(Vol<T> v, double x, double y, double z) {
    double g[3], center;
    if (grad_raw_shared<T, OP>(v, x, y, z, g, center)) return make_double4(g[0], g[1], g[2], center);
    grad_raw<T, OP, ROLL>(v, x, y, z, g);
    return make_double4(g[0], g[1], g[2], __longlong_as_double(0x7ff8000000000000LL));
}

// _shade_sample's value and diffuse term from the reference taps
// (_kernels.py:549-571): (illum before clamping, value)
template <typename T, int OP, int SI, bool ROLL>
__device__ __forceinline__ double2 taps_illum_value_inl(const Vol<T>& v, double p0, double p1, double p2, double wx,
                                                        double wy, double wz, double lpx, double lpy, double lpz) {
    const double4 gg = grad_taps<T, OP, ROLL>(v, p0, p1, p2);
    double g[3] = {gg.x, gg.y, gg.z};
    // the footprint's centre is sample_trilinear(p) (bit-identical)
    const double val = (SI == VC_TRILINEAR && gg.w == gg.w) ? gg.w : sample_any<T, SI>(v, p0, p1, p2);
    double u[3];
    normalize3(g, u);
    // field values rise toward the interior, the surface normal points away
    const double snx = -u[0], sny = -u[1], snz = -u[2];
    const double lx = dsub(lpx, wx);
    const double ly = dsub(lpy, wy);
    const double lz = dsub(lpz, wz);
    const double ln = __dsqrt_rn(dadd(dadd(dmul(lx, lx), dmul(ly, ly)), dmul(lz, lz)));
    double illum = 0.0;
    if (ln > 0.0) illum = ddiv(dadd(dadd(dmul(lx, snx), dmul(ly, sny)), dmul(lz, snz)), ln);
    return make_double2(illum, val);
}
template <typename T, int OP, int SI, bool ROLL>
__device__ __noinline__ double2 taps_illum_value(Vol<T> v, double p0, double p1, double p2, double wx, double wy,
                                                 double wz, double lpx, double lpy, double lpz) {
    return taps_illum_value_inl<T, OP, SI, ROLL>(v, p0, p1, p2, wx, wy, wz, lpx, lpy, lpz);
}

// _kernels.py:528-579
// GV: shading gradient from the packed volume (C.grad != nullptr) -- a
// template parameter so the taps-only kernel carries none of that code
template <typename T, int OP, int INTERP, bool GV>
__device__ __forceinline__ Rgba shade_sample(const Ctx<T>& C, const vc_render_params& P, double t) {
    const RayPos& r = C.rp;
    const double wx = dadd(r.o[0], dmul(t, r.d[0]));
    const double wy = dadd(r.o[1], dmul(t, r.d[1]));
    const double wz = dadd(r.o[2], dmul(t, r.d[2]));
    double p[3];
    p[0] = dsub(r.vox(wx, 0), 0.5);
    p[1] = dsub(r.vox(wy, 1), 0.5);
    p[2] = dsub(r.vox(wz, 2), 0.5);
    double val, illum = 0.0;
    const bool interior = p[0] >= 1.0 && p[0] <= dsub(C.v.mx, 1.0) && p[1] >= 1.0 &&
                          p[1] <= dsub(C.v.my, 1.0) && p[2] >= 1.0 && p[2] <= dsub(C.v.mz, 1.0);
    bool taps = !(GV && interior);
    if (!taps) {
        // diffuse term in float32 from the stored float32 gradient:
        // illum = dot(L, -g) / (|L| |g|), 0 for |g| <= EPS_GRADIENT or |L| = 0
        float g[3];
        bool suspect = false;
        const float4* cell = nullptr;
        float M = 0.0f;
        if (INTERP == VC_TEX) {  // one filtered float4 fetch: gradient + value
            const float4 q = tex3D<float4>(C.tx.g, __double2float_rn(p[0]) + 0.5f,
                                           __double2float_rn(p[1]) + 0.5f, __double2float_rn(p[2]) + 0.5f);
            g[0] = q.x;
            g[1] = q.y;
            g[2] = q.z;
            val = (double)q.w;
        } else {
            double gv;
            suspect = grad_from_volume<T, OP>(C.grad, C.v.nx, C.v.ny, p, g, gv, cell, M);
            val = (INTERP == VC_TRILINEAR) ? gv : sample_any<T, INTERP>(C.v, p[0], p[1], p[2]);
        }
        const float lx = (float)dsub(P.light_pos[0], wx);
        const float ly = (float)dsub(P.light_pos[1], wy);
        const float lz = (float)dsub(P.light_pos[2], wz);
        const float g2 = fmaf(g[0], g[0], fmaf(g[1], g[1], g[2] * g[2]));
        const float l2 = fmaf(lx, lx, fmaf(ly, ly, lz * lz));
        if (g2 > 1e-16f && l2 > 0.0f) {
            const float d = -fmaf(lx, g[0], fmaf(ly, g[1], lz * g[2]));
            illum = (double)(d * rsqrtf(g2) * rsqrtf(l2));
        }
        if constexpr (INTERP != VC_TEX) {
            if (__builtin_expect(suspect, 0)) {  // cancelling corners (grad_from_volume)
                const uint32_t sy = (uint32_t)C.v.nx, sz = (uint32_t)C.v.nx * (uint32_t)C.v.ny;
                double r;
                floor_pos(p[0], r);
                const double fx = dsub(p[0], r);
                floor_pos(p[1], r);
                const double fy = dsub(p[1], r);
                floor_pos(p[2], r);
                const double fz = dsub(p[2], r);
                const float4 h = gv_refine<T, OP>(cell, sy, sz, fx, fy, fz, M);
                if (h.w == 0.0f) {
                    taps = true;
                } else {
                    illum = 0.0;
                    const float h2 = fmaf(h.x, h.x, fmaf(h.y, h.y, h.z * h.z));
                    if (h2 > 1e-16f && l2 > 0.0f) {
                        const float d = -fmaf(lx, h.x, fmaf(ly, h.y, lz * h.z));
                        illum = (double)(d * rsqrtf(h2) * rsqrtf(l2));
                    }
                }
            }
        }
    }
    if (taps) {
#ifdef VC_DEBUG_TAPS
        if (GV) atomicAdd(&g_debug_taps, 1u);
#endif
        constexpr int SI = INTERP == VC_TEX ? VC_TRILINEAR : INTERP;  // boundary band: software value
        // the general 26-tap loop rolled except in the integer-grid
        // gradient-volume kernels (grad_raw: register pressure vs icache);
        // central differences' 6 taps stay unrolled (small code)
        constexpr bool ROLL = (!GV || !std::is_integral<T>::value) && grad_samples(OP) > 6;
        if constexpr (GV) {  // the rare path of the gradient-volume kernel: out of line
            const double2 iv = taps_illum_value<T, OP, SI, ROLL>(C.v, p[0], p[1], p[2], wx, wy, wz, P.light_pos[0],
                                                                 P.light_pos[1], P.light_pos[2]);
            illum = iv.x;
            val = iv.y;
        } else {
            const double2 iv = taps_illum_value_inl<T, OP, SI, ROLL>(C.v, p[0], p[1], p[2], wx, wy, wz,
                                                                     P.light_pos[0], P.light_pos[1], P.light_pos[2]);
            illum = iv.x;
            val = iv.y;
        }
    }
    illum = clamp01(illum);
    const double hu = dmul(div_rcp(dsub(val, P.mu_water), P.mu_water, C.rmu), 1000.0);
    double m[4];
    lut_eval(*C.lut, hu, m);
    Rgba out;
    out.r = clamp01(dmul(dmul(illum, P.light_col[0]), m[0]));
    out.g = clamp01(dmul(dmul(illum, P.light_col[1]), m[1]));
    out.b = clamp01(dmul(dmul(illum, P.light_col[2]), m[2]));
    out.a = m[3];
    return out;
}

// Per-lane ray state of the persistent kernel.  A pixel is traced as a
// sequence of "events"; one event = march the lattice base + k*coarse to
// the next in-window sample (+ fine backward scan and bisection for the
// first one) and shade it.  The first event's lattice is t_enter + k*coarse
// (first_hit, _kernels.py:401-465 + bisect_window :468-487); later events
// march t_star + m*coarse (composite loop, :755-790).  Accumulation is
// arranged so the first shade's acc = a*c, remain = 1 - a come out
// bit-identical to the reference (1.0*a*c == a*c, 0.0 + x == x,
// 1.0*(1-a) == 1-a).
struct RayState {
    double t_enter, lim, base, k;
    double acc_r, acc_g, acc_b, remain;
    double t_hit;    // lattice parameter of the in-window sample found by the march
    bool found;      // march stopped on an in-window sample
    bool exhausted;  // march ran past t_exit
};

__device__ __forceinline__ uchar4 bg_pixel(const vc_render_params& P) {
    return make_uchar4(quant(P.bg[0]), quant(P.bg[1]), quant(P.bg[2]), quant(P.bg[3]));
}

// image row of local (packed) row lr under the band partition
__device__ __forceinline__ int image_row(const vc_render_params& P, int lr) {
    if (P.band_step == 1) return P.band_first * P.band_rows + lr;  // contiguous rows
    const int band = lr / P.band_rows, within = lr - band * P.band_rows;
    return (P.band_first + band * P.band_step) * P.band_rows + within;
}

// ray generation (_kernels.py:639-648) + box interval (:649); false = miss
template <typename T>
// rhw (optional): RN(1/width), RN(1/height) computed once per block
__device__ __forceinline__ bool start_ray(Ctx<T>& C, const vc_render_params& P, int px, int py,
                                          RayState& R, double* t_exit_out = nullptr,
                                          const double* rhw = nullptr) {
    const double H = (double)P.height, W = (double)P.width;  // integers: never an all-ones significand
    const double rW = rhw ? rhw[0] : __drcp_rn(W), rH = rhw ? rhw[1] : __drcp_rn(H);
    const double v_ndc = dsub(1.0, ddiv_rcp(dmul(2.0, dadd((double)py, 0.5)), H, rH));
    const double u_ndc = dsub(ddiv_rcp(dmul(2.0, dadd((double)px, 0.5)), W, rW), 1.0);
    const double uw = dmul(u_ndc, P.half_w), vh = dmul(v_ndc, P.half_h);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; a++) d[a] = dadd(dadd(P.forward[a], dmul(uw, P.right[a])), dmul(vh, P.up[a]));
    const double dn = __dsqrt_rn(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
    const double ydn = rcp_for(dn);
#pragma unroll
    for (int a = 0; a < 3; a++) C.rp.d[a] = div_rcp(d[a], dn, ydn);
    double t_enter, t_exit, inv[3];
    if (!box_interval(C.rp.o, C.rp.d, P.clip_lo, P.clip_hi, t_enter, t_exit, inv)) return false;
    // skip_to's reciprocal speed s / d from the slab test's RN(1 / d) (0 for
    // d == 0): only conservativeness matters (EPS margins)
#pragma unroll
    for (int a = 0; a < 3; a++) C.sk.ib[a] = dmul(C.rp.s[a], inv[a]);
    R.t_enter = t_enter;
    if (t_exit_out != nullptr) *t_exit_out = t_exit;
    R.lim = dadd(t_exit, 1e-12);
    R.base = t_enter;
    R.k = 0.0;
    R.acc_r = R.acc_g = R.acc_b = 0.0;
    R.remain = 1.0;
    R.t_hit = 0.0;
    R.found = false;
    R.exhausted = false;
    return true;
}

// Adaptive stride after an out-of-window first-hit sample at p with lattice
// index k (_kernels.py:437-463): leaf_for_point (:345-364) over the level
// grid, then _node_interval (:227-264) of the leaf when its padded range is
// below detail_eps.  Same float64 operations as the reference.  Out of line
// with by-value arguments: the mode is rare and inlining it into the march
// loop cost every other mode code size and registers.
struct StrideArgs {
    int nx, ny, nz, adapt_jump;
    double o[3], d[3], s[3];
    double detail_eps, coarse;
};

// _node_interval (_kernels.py:227-264) of box b of level L of the level grid
__device__ __forceinline__ bool oct_node_interval(const OctDev& o, int L, const int b[3], const double ov3[3],
                                                  const double d3[3], const double inv3[3], const double s3[3],
                                                  double& tmin, double& tmax) {
    tmin = -1e300;
    tmax = 1e300;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const int* iv = o.ivl + vc_ldg(o.ivl_off + 3 * L + a) + 2 * b[a];
        const double lo = dmul(u2d((uint32_t)vc_ldg(iv)), s3[a]);  // exact, FP64 pipe
        const double hi = dmul(u2d((uint32_t)vc_ldg(iv + 1)), s3[a]);
        const double ov = ov3[a], d = d3[a];
        if (d == 0.0) {
            if (ov < lo || ov > hi) return false;
        } else {
            const double inv = inv3[a];
            double ta = dmul(dsub(lo, ov), inv), tb = dmul(dsub(hi, ov), inv);
            if (ta > tb) {
                const double sw = ta;
                ta = tb;
                tb = sw;
            }
            if (ta > tmin) tmin = ta;
            if (tb < tmax) tmax = tb;
        }
    }
    return !(tmin > tmax);
}

__device__ __noinline__ double adaptive_stride(const OctDev o, const StrideArgs A, double p0, double p1,
                                               double p2, double k, double t_enter) {
    const double p[3] = {p0, p1, p2};
    const int n3[3] = {A.nx, A.ny, A.nz};
    int ic[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        double r;
        int i = floor_pos(p[a], r);
        i = i < 0 ? 0 : (i > n3[a] - 1 ? n3[a] - 1 : i);
        ic[a] = i;
    }
    const int stride_map = A.nx + A.ny + A.nz;
    int L = 0, b[3] = {0, 0, 0};
    long long leaf = 0;
    for (L = 0; L < o.levels; L++) {
        const int* m = o.amap + (size_t)L * stride_map;
        b[0] = vc_ldg(m + ic[0]);
        b[1] = vc_ldg(m + A.nx + ic[1]);
        b[2] = vc_ldg(m + A.nx + A.ny + ic[2]);
        leaf = vc_ldg(o.box_off + L) +
               ((long long)b[2] * vc_ldg(o.dims + 3 * L + 1) + b[1]) * vc_ldg(o.dims + 3 * L + 0) + b[0];
        if (vc_ldg(o.state + leaf) == 2) break;
    }
    if (L == o.levels) return 1.0;  // unreachable for a well-formed tree
    const double smin = vc_ldg(o.srange + 2 * leaf), smax = vc_ldg(o.srange + 2 * leaf + 1);
    if (!(dsub(smax, smin) < A.detail_eps)) return 1.0;
    double tmin, tmax;
    double inv[3];
#pragma unroll
    for (int a = 0; a < 3; a++) inv[a] = A.d[a] == 0.0 ? 0.0 : __drcp_rn(A.d[a]);  // = RN(1.0 / d)
    if (!oct_node_interval(o, L, b, A.o, A.d, inv, A.s, tmin, tmax)) return 1.0;
    double step = (double)A.adapt_jump;
    const double kex = floor(ddiv(dsub(tmax, t_enter), A.coarse)) + 1.0;
    if (dsub(kex, k) < step) step = dsub(kex, k);
    if (step < 1.0) step = 1.0;
    return step;
}

// One lattice step of the march base + k*coarse (first_hit's loop body,
// _kernels.py:410-436 / the composite loop :756-765).
template <typename T, int INTERP, bool LAZY = false>
__device__ __forceinline__ void march_step(const Ctx<T>& C, const vc_render_params& P, RayState& R,
                                           unsigned& nsamp, unsigned& nskip, const OctDev* oct = nullptr) {
    const double t = dadd(R.base, dmul(R.k, P.coarse));
    if (t > R.lim) {
        R.exhausted = true;
        return;
    }
    double p[3];
    C.rp.at(t, p);
    const int w = march_sample<T, INTERP, LAZY>(C, P, p, t, R.k, R.base, nskip);
    if (w < 0) return;
    nsamp++;
    if (oct != nullptr && !w) {  // first-hit stage, adaptive mode
        StrideArgs A;
        A.nx = C.v.nx;
        A.ny = C.v.ny;
        A.nz = C.v.nz;
        A.adapt_jump = P.adapt_jump;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            A.o[a] = C.rp.o[a];
            A.d[a] = C.rp.d[a];
            A.s[a] = C.rp.s[a];
        }
        A.detail_eps = P.detail_eps;
        A.coarse = P.coarse;
        R.k += adaptive_stride(*oct, A, p[0], p[1], p[2], R.k, R.t_enter);
        return;
    }
    R.k += 1.0;
    if (w) {
        R.found = true;
        R.t_hit = t;
    }
}

// fine backward scan (_kernels.py:419-436) + bisect_window (:468-487) from
// the first in-window lattice sample t; returns t_star
template <typename T, int INTERP>
__device__ __forceinline__ double refine_hit(const Ctx<T>& C, const vc_render_params& P, const RayState& R,
                                             double t, unsigned& nsamp) {
    const double fine = P.fine;
    bool bracket = false;
    double t_in = t, t_before = t;
    const double floor_t = dsub(R.t_enter, 1e-12);
    for (double j = 1.0;; j += 1.0) {
        const double tb = dsub(t, dmul(j, fine));
        if (tb < floor_t) {
            t_in = t_before = dsub(t, dmul(j - 1.0, fine));
            break;
        }
        double b[3];
        C.rp.at(tb, b);
        nsamp++;
        if (!window_at<T, INTERP>(C, P, b)) {
            t_in = dsub(t, dmul(j - 1.0, fine));
            t_before = tb;
            bracket = true;
            break;
        }
    }
    double tcur = t_in;
    if (bracket && P.refine_iters > 0) {
        double tb = t_before, ta = t_in;
        for (int it = 0; it < P.refine_iters; it++) {
            const double tm = dmul(0.5, dadd(tb, ta));
            double p[3];
            C.rp.at(tm, p);
            nsamp++;
            if (window_at<T, INTERP>(C, P, p)) ta = tm;
            else tb = tm;
        }
        tcur = ta;
    }
    return tcur;
}

// ---- fixed-point lattice walk (first hit, trilinear) -----------------------
// The reference forms every march position in float64 from scratch,
// p(k) = (o + (base + k*coarse) * d) / s - 0.5, and only uses it to pick a
// cell (floor), to test the cell's macrocell and to interpolate.  Here the
// walk runs on p(k) = P0 + k*DP in 24.40 fixed point (two integer adds per
// axis, no FP64 work) and is exact where it matters:
//   * deviation.  |p_fx(k) - p_ref(k)| <= 2*Eref + (k+1)*2^-41 where Eref
//     <= 2^-50 * ((|o| + 2T|d|) / s + |p| + 1) bounds the reference's own
//     float64 rounding (T = |lim| + |base| + coarse).  fx_setup admits a
//     ray only when Eref <= 2^-24, |p| <= 2^22 and k_last <= 2^19, so the
//     deviation stays below 2^-21 (fine scan: + j*2^-41, j <= 2^18;
//     bisection: each midpoint + 2^-41 + 2^-28, <= 64 of them): below
//     0.75 * 2^-20 everywhere;
//   * cells.  A coordinate whose fixed-point fraction lies within 2^-20 of
//     a cell face ("guard") -- and every sample of a ray fx_setup did not
//     admit -- takes the reference's float64 path; elsewhere floor(p_fx) ==
//     floor(p_ref), so the range test, the macrocell and the eight gathered
//     voxels are the reference's;
//   * values.  The float32 pre-test uses the fixed-point fractions
//     (truncated to 23 bits): error <= 2^-20 per fraction, <= 6 * amax *
//     2^-20 = 96 * 2^-24 * amax over the three lerp levels; with the
//     arithmetic's 34 * 2^-24 * amax that stays below the pre-test's E =
//     256 * 2^-24 * amax.  An ambiguous value is re-evaluated with the
//     reference's float64 position and cascade;
//   * the end.  k > k_last <=> t(k) > lim: k_last is found once per ray
//     with the march's own float64 t(k) (monotone in k);
//   * skips.  Empty-space jumps only need conservativeness: the box-exit
//     distance is formed in float32 from the cell, the fraction and a
//     2^-8 voxel margin (float32 error <= 5e-4 voxel over a 1016-voxel box).
constexpr double FX_ONE = 0x1p40;
#ifndef VC_FX_UNROLL2
#define VC_FX_UNROLL2 1
#endif

// Per-lane walk state.  It lives in shared memory (structure of arrays: a
// warp's accesses are conflict-free) and is loaded into registers at the
// top of each march phase; the march loop itself holds nothing else, so it
// runs without spills, and the rare float64 fallbacks run between march
// phases with the walk registers dead.  A ray fx_setup does not admit gets
// p0 = dp = 0: its fractions are 0, inside the guard band, so every one of
// its samples takes the float64 path.
struct FxRay {
    long long p0[3], dp[3];  // p(k) = p0 + k*dp, units of 2^-40 voxel
    float ibf[3];            // s / d per axis (voxel -> t), 0 for d == 0
    int klast;               // last lattice index with t(k) <= lim
};

struct FxLanes {
    long long p0[3][128], dp[3][128];
    float ibf[3][128];
    int klast[128];
    // direction and parameter bounds (fallbacks, refinement, hit entry)
    double d[3][128], base[128], lim[128], t_enter[128];
};

__device__ __forceinline__ FxRay fx_load(const FxLanes& S, int me) {
    FxRay F;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        F.p0[a] = S.p0[a][me];
        F.dp[a] = S.dp[a][me];
        F.ibf[a] = S.ibf[a][me];
    }
    F.klast = S.klast[me];
    return F;
}

// the lane's RayPos (direction from the shared state)
__device__ __forceinline__ RayPos fx_rp(const RayPos& rp0, const FxLanes& S, int me) {
    RayPos rp = rp0;
#pragma unroll
    for (int a = 0; a < 3; a++) rp.d[a] = S.d[a][me];
    return rp;
}

__device__ __forceinline__ long long to_fx(double v) { return __double2ll_rn(dmul(v, FX_ONE)); }

__device__ __forceinline__ int fx_cell(long long x) { return (int)(x >> 40); }

// p0 + k*dp for 0 <= k < 2^31 (two IMADs: unsigned wrap-around arithmetic)
__device__ __forceinline__ long long fx_at(long long p0, long long dp, int k) {
    return (long long)((unsigned long long)p0 + (unsigned long long)(unsigned)k * (unsigned long long)dp);
}

// fraction of a fixed-point coordinate, truncated to 23 bits; g |= within
// 2^-20 of a cell face
__device__ __forceinline__ float fx_frac(long long x, bool& g) {
    const unsigned m = __funnelshift_l((unsigned)x, (unsigned)(x >> 32), 15);  // bits 39..17
    const float F = __uint_as_float((m & 0x7fffffu) | 0x3f800000u);         // 1 + fraction
    g = g || fabsf(__fsub_rn(F, 1.5f)) > 0.5f - 0x1p-20f;
    return __fsub_rn(F, 1.0f);
}

// The admission bound for every ray of the frame at once: a ray's path
// parameter never exceeds T = 2*Dmax + coarse (Dmax: the eye's distance to
// the farthest clip-box corner; t_enter, t_exit <= Dmax), so per axis
// (|o| + 2T|d|)/s <= (|o| + 2T)/s bounds both the reference's rounding
// scale and the walk's reach; <= 2^21 leaves the per-ray conditions of the
// analysis above (2^24, 2^22) a 2x-8x margin.  Computed once per block.
__device__ __forceinline__ bool fx_frame_admits(const vc_render_params& P, const RayPos& rp) {
    double dmax = 0.0;
    for (int c = 0; c < 8; c++) {
        double q = 0.0;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const double w = ((c >> a) & 1) ? P.clip_hi[a] : P.clip_lo[a];
            q += (w - P.eye[a]) * (w - P.eye[a]);
        }
        dmax = fmax(dmax, sqrt(q));
    }
    const double T = 2.0 * dmax * (1.0 + 0x1p-20) + P.coarse + 1.0;
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; a++) ok = ok && (fabs(P.eye[a]) + 2.0 * T) * fabs(rp.rs[a]) <= 0x1p21;
    return ok;
}

template <typename T>
__device__ __forceinline__ void fx_setup(const Ctx<T>& C, const vc_render_params& P, const RayState& R, FxLanes& S,
                                         int me, bool frame_ok) {
    bool ok = true;
    double x = dmul(dsub(R.lim, R.base), C.sk.inv_coarse);
    if (!(x < 524288.0)) {
        ok = false;
        x = 0.0;
    }
    int kl = (int)x;
#pragma unroll 1
    while (kl > 0 && dadd(R.base, dmul((double)kl, P.coarse)) > R.lim) kl--;
#pragma unroll 1
    while (kl < 524288 && dadd(R.base, dmul((double)(kl + 1), P.coarse)) <= R.lim) kl++;
    S.klast[me] = kl;
    ok = ok && frame_ok;  // the frame-wide rounding / reach bound (fx_frame_admits)
    double pb[3];
    C.rp.at(R.base, pb);
#pragma unroll
    for (int a = 0; a < 3; a++) {
        S.p0[a][me] = ok ? to_fx(pb[a]) : 0;
        S.dp[a][me] = ok ? to_fx(dmul(dmul(P.coarse, C.rp.d[a]), C.rp.rs[a])) : 0;
        S.ibf[a][me] = __double2float_rn(C.sk.ib[a]);
        S.d[a][me] = C.rp.d[a];
    }
    S.base[me] = R.base;
    S.lim[me] = R.lim;
    S.t_enter[me] = R.t_enter;
}

__device__ __forceinline__ uint32_t macro_index3(const Skip& sk, int i, int j, int k) {
    return ((uint32_t)(k >> MC_SHIFT) * (uint32_t)sk.my + (uint32_t)(j >> MC_SHIFT)) * (uint32_t)sk.mx +
           (uint32_t)(i >> MC_SHIFT);
}

// skip_to for the fixed-point walk: float32 box-exit distance (see above)
__device__ __forceinline__ int skip_fx(int k, const int c[3], const float f[3], const float ibf[3], float inv_coarse,
                                       int d) {
    constexpr float EPSF = 0x1p-8f;
    const int r = (d - 1) << MC_SHIFT;
    float dt = FLT_MAX;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const int lo = (c[a] >> MC_SHIFT) << MC_SHIFT;
        const bool up = ibf[a] > 0.0f;
        const int rel = (up ? lo + (1 << MC_SHIFT) + r : lo - r) - c[a];  // face - cell, small
        const float relf = __fsub_rn(__int_as_float(0x4b400000 + rel), 12582912.0f);
        const float cand = __fmul_rn(__fsub_rn(__fadd_rn(relf, up ? -EPSF : EPSF), f[a]), ibf[a]);
        dt = ibf[a] != 0.0f ? fminf(dt, cand) : dt;
    }
    int kn = k + 1;
    if (dt > 0.0f) {
        const float xs = __fmul_rn(dt, inv_coarse);
        // ceil(xs) on the FMA pipe (F2I is an XU op): 2^23 + x rounded up has
        // ceil(x) as its integer part for 0 <= x <= 2^23; a jump clamped to
        // 2^23 lattice steps still passes klast (< 2^19), so the ray ends
        // exactly as with the full jump
        const float xc = fminf(xs, 0x1p23f);
        kn = max(kn, k + (__float_as_int(__fadd_ru(xc, 0x1p23f)) - 0x4b000000));
    }
    return kn;
}

// One lattice step of the fixed-point walk at index k.  Returns false,
// leaving k unchanged, when the sample needs the reference's float64 path
// (a coordinate within 2^-20 of a cell face, or an ambiguous pre-test):
// the lane then pauses until the warp's march phase ends (fx_exact_step).
template <typename T>
__device__ __forceinline__ bool march_step_fx(const Ctx<T>& C, const vc_render_params& P, RayState& R,
                                              const FxRay& F, int& k, unsigned& nsamp, unsigned& nskip) {
    if (k > F.klast) {
        R.exhausted = true;
        return true;
    }
    long long q[3];
#pragma unroll
    for (int a = 0; a < 3; a++) q[a] = fx_at(F.p0[a], F.dp[a], k);
    bool g = false;
    const int c[3] = {fx_cell(q[0]), fx_cell(q[1]), fx_cell(q[2])};
    const float f[3] = {fx_frac(q[0], g), fx_frac(q[1], g), fx_frac(q[2], g)};
    if (g) return false;
    const bool inr = (unsigned)c[0] < (unsigned)(C.v.nx - 1) && (unsigned)c[1] < (unsigned)(C.v.ny - 1) &&
                     (unsigned)c[2] < (unsigned)(C.v.nz - 1);
    if (C.sk.on) {
        if (!inr) {  // reads 0, outside the window when skipping is on
            k++;
            nskip++;
            return true;
        }
        const int d = vc_ldg(C.sk.dist + macro_index3(C.sk, c[0], c[1], c[2]));
        if (d != 0) {
            k = skip_fx(k, c, f, F.ibf, C.sk.inv_coarse_f, d);
            nskip++;
            return true;
        }
    }
    int w;
    if (!inr) {
        w = in_window(P, 0.0) ? 1 : 0;
    } else {
        w = window_cell_f<T>(C.v, c[0], c[1], c[2], f[0], f[1], f[2], C.sk.win);
        if (w < 0) return false;
    }
    nsamp++;
    k++;
    if (w) R.found = true;
    return true;
}

// the reference's float64 sample at lattice index k (march_sample, with its
// own empty-space jump)
template <typename T>
__device__ __forceinline__ void fx_exact_step(const Ctx<T>& C, const vc_render_params& P, RayState& R,
                                              const FxLanes& S, int me, int& k, unsigned& nsamp, unsigned& nskip) {
    Ctx<T> Cx = C;
    Cx.rp = fx_rp(C.rp, S, me);
    const double base = S.base[me];
    const double t = dadd(base, dmul((double)k, P.coarse));
    double p[3];
    Cx.rp.at(t, p);
    double kd = (double)k;
    const int w = march_sample<T, VC_TRILINEAR, true>(Cx, P, p, t, kd, base, nskip);
    if (w < 0) {
        k = (int)kd;
        return;
    }
    nsamp++;
    k++;
    if (w) R.found = true;
}

// window test of a fixed-point position whose float64 parameter is t
template <typename T>
__device__ __forceinline__ bool window_fx(const Ctx<T>& C, const vc_render_params& P, const FxLanes& S, int me,
                                          const long long q[3], double t, bool ok) {
    bool g = !ok;
    const int ci = fx_cell(q[0]), cj = fx_cell(q[1]), ck = fx_cell(q[2]);
    const float fx = fx_frac(q[0], g), fy = fx_frac(q[1], g), fz = fx_frac(q[2], g);
    int w = -1;
    if (!g) {
        const bool inr = (unsigned)ci < (unsigned)(C.v.nx - 1) && (unsigned)cj < (unsigned)(C.v.ny - 1) &&
                         (unsigned)ck < (unsigned)(C.v.nz - 1);
        if (!inr) return in_window(P, 0.0);
        w = window_cell_f<T>(C.v, ci, cj, ck, fx, fy, fz, C.sk.win);
    }
    if (w >= 0) return w != 0;
    const RayPos rp = fx_rp(C.rp, S, me);
    double p[3];
    rp.at(t, p);
    return window_at<T, VC_TRILINEAR>(C, P, p);
}

// window_fx through a cell cache (the bisection)
template <typename T>
__device__ __forceinline__ bool window_fx_cached(const Ctx<T>& C, const vc_render_params& P, const FxLanes& S,
                                                 int me, const long long q[3], double t, bool ok, CellCache& cc) {
    bool g = !ok;
    const int ci = fx_cell(q[0]), cj = fx_cell(q[1]), ck = fx_cell(q[2]);
    const float fx = fx_frac(q[0], g), fy = fx_frac(q[1], g), fz = fx_frac(q[2], g);
    int w = -1;
    if (!g) {
        const bool inr = (unsigned)ci < (unsigned)(C.v.nx - 1) && (unsigned)cj < (unsigned)(C.v.ny - 1) &&
                         (unsigned)ck < (unsigned)(C.v.nz - 1);
        if (!inr) return in_window(P, 0.0);
        w = window_cell_cached<T>(C.v, ci, cj, ck, fx, fy, fz, C.sk.win, cc);
    }
    if (w >= 0) return w != 0;
    const RayPos rp = fx_rp(C.rp, S, me);
    double p[3];
    rp.at(t, p);
    return window_at<T, VC_TRILINEAR>(C, P, p);
}

// refine_hit on the fixed-point walk from the hit at lattice index khit:
// the fine lattice t - j*fine is p_hit - j*DF, the bisection midpoints
// (qa + qb) >> 1; every t is still formed in float64 exactly as the
// reference does (the result t_star and the float64 fallbacks use it)
template <typename T>
__device__ __forceinline__ double refine_hit_fx(const Ctx<T>& C, const vc_render_params& P, const FxLanes& S,
                                                int me, int khit, unsigned& nsamp) {
    const double t = dadd(S.base[me], dmul((double)khit, P.coarse));
    const double fine = P.fine;
    long long q[3], df[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const long long dp = S.dp[a][me];
        q[a] = fx_at(S.p0[a][me], dp, khit);
        // dp == 0: a ray fx_setup did not admit (its fractions stay at 0)
        df[a] = dp != 0 ? to_fx(dmul(dmul(fine, S.d[a][me]), C.rp.rs[a])) : 0;
    }
    bool bracket = false;
    double t_in = t, t_before = t;
    const double floor_t = dsub(S.t_enter[me], 1e-12);
    int jj = 0;
    for (double j = 1.0;; j += 1.0) {
        const double tb = dsub(t, dmul(j, fine));
        if (tb < floor_t) {
            t_in = t_before = dsub(t, dmul(j - 1.0, fine));
            break;
        }
#pragma unroll
        for (int a = 0; a < 3; a++) q[a] -= df[a];
        jj++;
        nsamp++;
        if (!window_fx<T>(C, P, S, me, q, tb, jj < (1 << 18))) {
            t_in = dsub(t, dmul(j - 1.0, fine));
            t_before = tb;
            bracket = true;
            break;
        }
    }
    double tcur = t_in;
    if (bracket && P.refine_iters > 0) {
        const bool okb = P.refine_iters <= 64;
        long long qa[3];  // q: the out-of-window end, qa: the in-window end
#pragma unroll
        for (int a = 0; a < 3; a++) qa[a] = q[a] + df[a];
        double tb = t_before, ta = t_in;
        CellCache cc;
        cc.i = -1;
        cc.j = cc.k = 0;
        for (int it = 0; it < P.refine_iters; it++) {
            const double tm = dmul(0.5, dadd(tb, ta));
            long long qm[3];
#pragma unroll
            for (int a = 0; a < 3; a++) qm[a] = (qa[a] + q[a]) >> 1;
            nsamp++;
            const bool in = window_fx_cached<T>(C, P, S, me, qm, tm, okb, cc);
#pragma unroll
            for (int a = 0; a < 3; a++) {
                qa[a] = in ? qm[a] : qa[a];
                q[a] = in ? q[a] : qm[a];
            }
            if (in) ta = tm;
            else tb = tm;
        }
        tcur = ta;
    }
    return tcur;
}

__device__ __forceinline__ uchar4 composite_pixel(const vc_render_params& P, const RayState& R) {
    return make_uchar4(quant(dadd(R.acc_r, dmul(R.remain, P.bg[0]))),
                       quant(dadd(R.acc_g, dmul(R.remain, P.bg[1]))),
                       quant(dadd(R.acc_b, dmul(R.remain, P.bg[2]))), 255);
}

// Shade at tcur and composite front to back.  Accumulation is arranged so
// the first shade's acc = a*c, remain = 1 - a come out bit-identical to the
// reference (_kernels.py:744-754: 1.0*a*c == a*c, 0.0 + x == x,
// 1.0*(1-a) == 1-a).  Returns true when the pixel is finished.
template <typename T, int OP, int INTERP, bool GV>
__device__ __forceinline__ bool shade_and_composite(const Ctx<T>& C, const vc_render_params& P, RayState& R,
                                                    double tcur, uchar4& out, unsigned& nshade) {
    const Rgba s = shade_sample<T, OP, INTERP, GV>(C, P, tcur);
    nshade++;
    if (P.mode == VC_SURFACE) {
        out = make_uchar4(quant(s.r), quant(s.g), quant(s.b), 255);
        return true;
    }
    const double w = dmul(R.remain, s.a);
    R.acc_r = dadd(R.acc_r, dmul(w, s.r));
    R.acc_g = dadd(R.acc_g, dmul(w, s.g));
    R.acc_b = dadd(R.acc_b, dmul(w, s.b));
    R.remain = dmul(R.remain, dsub(1.0, s.a));
    if (s.a >= OPAQUE_ALPHA || R.remain < MIN_REMAINING) {
        out = composite_pixel(P, R);
        return true;
    }
    return false;
}

// a warp leaves the march loop when READY_NUM / READY_DEN of its live lanes
// have a hit (or an exhausted ray) to resolve (first-hit / shade kernel)
#ifndef VC_FH_READY
#define VC_FH_READY 32
#endif
#ifndef VC_SH_READY
#define VC_SH_READY 8
#endif
#ifndef VC_SH_REFILL  // shade stage: idle lanes before a refill
#define VC_SH_REFILL 24
#endif
#ifndef VC_SHV_READY  // shade stage, gradient-volume kernel
#define VC_SHV_READY 1
#endif
constexpr int READY_DEN = 32;

// Where finished pixels go: the packed local rows of this rank (npeers == 0)
// or, fused with the image-tile gather, the full frame buffers of the ranks
// (npeers > 0: a device table of every rank's frame, this rank's own local,
// the others mapped over NVLink).  With tile counters (band_rows a multiple
// of 4, so an 8x4 screen tile never straddles two bands) a pixel goes to the
// rank's own frame first; the lane that completes a tile -- its pixels come
// from both kernels, in any order -- pushes the tile's four 32-byte rows to
// the receiving ranks as 16-byte stores (two per row per receiver) instead
// of one 4-byte remote store per pixel per receiver.  dest >= 0 sends to one
// rank only (a gather to that rank), -1 to every rank.
struct PixelSink {
    uchar4* out;
    uchar4* const* peers;
    int npeers;
    int self, dest;
    unsigned* tile_cnt;  // zeroed per frame; nullptr: per-pixel remote stores
    int tiles_x, local_rows;
};

__device__ __forceinline__ bool sink_receives(const PixelSink& s, int r) { return s.dest < 0 || r == s.dest; }

// the completed tile (local rows lr0.., columns x0..) from this rank's frame to
// the receiving ranks; its pixels were written and fenced by any thread of
// either kernel, so they are read through L2 (ld.global.cg)
__device__ __noinline__ void push_tile(const PixelSink s, const vc_render_params& P, int lr0, int x0) {
    const int W = P.width;
    const int nr = min(4, s.local_rows - lr0), nc = min(8, W - x0);
    const uchar4* own = vc_ld(s.peers + s.self);
    const bool vec = nc == 8 && (W & 3) == 0;  // 16-byte aligned 32-byte rows
    for (int r = 0; r < nr; r++) {
        const size_t base = (size_t)image_row(P, lr0 + r) * W + x0;
        if (vec) {
            const uint4* src = reinterpret_cast<const uint4*>(own + base);
            const uint4 a = __ldcg(src), b = __ldcg(src + 1);
            for (int q = 0; q < s.npeers; q++) {
                if (q == s.self || !sink_receives(s, q)) continue;
                uint4* dst = reinterpret_cast<uint4*>(vc_ld(s.peers + q) + base);
                if (vc_st_ok(dst, 32)) {
                    dst[0] = a;
                    dst[1] = b;
                }
            }
        } else {
            for (int c = 0; c < nc; c++) {
                const unsigned v = __ldcg(reinterpret_cast<const unsigned*>(own + base + c));
                for (int q = 0; q < s.npeers; q++) {
                    if (q == s.self || !sink_receives(s, q)) continue;
                    unsigned* dst = reinterpret_cast<unsigned*>(vc_ld(s.peers + q) + base + c);
                    if (vc_st_ok(dst, 4)) *dst = v;
                }
            }
        }
    }
}

__device__ __forceinline__ void put_pixel(const PixelSink& s, const vc_render_params& P, int lr, int px,
                                          uchar4 o) {
    if (s.npeers == 0) {
        uchar4* d = s.out + (size_t)lr * P.width + px;
        if (vc_st_ok(d, sizeof(uchar4))) *d = o;
        return;
    }
    const size_t idx = (size_t)image_row(P, lr) * P.width + px;
    if (s.tile_cnt == nullptr) {  // one store per pixel per receiving rank
        for (int r = 0; r < s.npeers; r++) {
            if (r != s.self && !sink_receives(s, r)) continue;
            uchar4* d = vc_ld(s.peers + r) + idx;
            if (vc_st_ok(d, sizeof(uchar4))) *d = o;
        }
        return;
    }
    uchar4* d = vc_ld(s.peers + s.self) + idx;
    if (vc_st_ok(d, sizeof(uchar4))) *d = o;
    __threadfence();  // the pixel is visible before it is counted
    const int lr0 = lr & ~3, x0 = px & ~7;
    const unsigned need = (unsigned)(min(8, P.width - x0) * min(4, s.local_rows - lr0));
    unsigned* cnt = s.tile_cnt + (size_t)(lr0 >> 2) * s.tiles_x + (x0 >> 3);
    if (vc_st_ok(cnt, sizeof(unsigned)) && atomicAdd(cnt, 1u) + 1u == need) {
        __threadfence();  // every counted pixel is visible to the pushing lane
        push_tile(s, P, lr0, x0);
    }
}

// First-hit queue entry, 48 bytes (three 128-bit accesses): the refined
// parameter t_star, the ray's end lim and direction (bit-exact: the shade
// stage does not regenerate the ray -- doing that per refill cost more than
// the queue read it saved) and the pixel.  The reciprocal speeds of the
// empty-space skip are recomputed from the direction.  At C3 the queue holds
// ~1.45 M entries: 70 MB (the earlier 96-byte entry: 139 MB, more than L2).
struct __align__(16) HitEntry {
    double t_star, lim;
    double d[3];
    uint32_t pix;  // local row << 16 | column (validate_params: both < 2^16)
    uint32_t pad;
};
static_assert(sizeof(HitEntry) == 48, "hit queue entry layout");
__device__ __forceinline__ uint32_t pack_pix(int lr, int px) { return ((uint32_t)lr << 16) | (uint32_t)px; }

#ifndef VC_STAGE_OVERLAP
#define VC_STAGE_OVERLAP 1
#endif

// Work counters of one launch pair (zeroed together before the frame).
// Zeroed once when the scratch is allocated; afterwards the last kernel-B
// warp of each frame zeroes it for the next one (no memset launch per frame).
struct FrameWork {
    unsigned pixels;   // kernel A: next pixel work item
    unsigned hits;     // kernel A -> B: queue length (tickets taken)
    unsigned shades;   // kernel B: next queue entry
    unsigned fh_done;  // kernel A warps finished (queue length final when all are)
    unsigned sh_done;  // kernel B warps finished (the last one resets the counters)
    unsigned pad[3];
};

// Stage hand-off.  Kernel B is launched with programmatic stream
// serialization and kernel A lets it start at once (griddepcontrol), so B's
// blocks take the SMs A's blocks leave during A's tail.  A hit entry is
// published by a release store of the frame's tag into its last word after
// the payload.  B reads the tag with a strong (L2) load and, once it holds
// this frame's tag, the payload with L1-bypassing loads issued under that
// branch: the release made the payload visible at L2, the point of
// coherence, before the tag.  (An acquire load would order it in the PTX
// model too, but it invalidates the SM's whole L1 -- CCTL.IVALL -- on every
// refill, which cost the gradient-volume and tap gathers 7-9%.)  B's lane
// with queue ticket q is done when every A block has finished and q is past
// the final queue length.  Without the overlap (ncu replay, an event between
// the launches) every tag is already there and nothing waits.
__device__ __forceinline__ unsigned ld_strong_u32(const unsigned* p) {
#ifdef VC_CHECKED
    if (!vc_addr_ok(p, sizeof(unsigned))) return 0u;
#endif
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// a published entry's payload, from L2
__device__ __forceinline__ HitEntry load_hit(const HitEntry* p) {
    HitEntry e;
#ifdef VC_CHECKED
    if (!vc_addr_ok(p, sizeof(HitEntry))) return HitEntry{};
#endif
    const uint4* s = reinterpret_cast<const uint4*>(p);
    uint4* d = reinterpret_cast<uint4*>(&e);
    d[0] = __ldcg(s);
    d[1] = __ldcg(s + 1);
    d[2] = __ldcg(s + 2);
    return e;
}

// kernel B's refill while kernel A may still run: is every A block done
// (warp-uniform; then the final queue length), else is this lane's entry
// published.  st: 0 keep waiting, 1 claim, 2 past the end of the queue.
struct OverlapPoll {
    int st;
    bool fh_all;
    unsigned final_hits;
};
__device__ __noinline__ OverlapPoll overlap_poll(const FrameWork* work, const HitEntry* hits, unsigned nfh,
                                                 unsigned seq, unsigned max_hits, unsigned qt, bool waiting,
                                                 unsigned spin) {
    const unsigned FULL = 0xffffffffu;
    unsigned f = 0u, h = 0u;
    if ((threadIdx.x & 31) == 0) {
        f = ld_strong_u32(&work->fh_done);
        if (f >= nfh) h = ld_strong_u32(&work->hits);
    }
    f = __shfl_sync(FULL, f, 0);
    h = __shfl_sync(FULL, h, 0);
    OverlapPoll r{0, f >= nfh, h};
    if (!waiting) return r;
    if (r.fh_all) r.st = qt < h ? 1 : 2;
    else if (qt < max_hits && ld_strong_u32(&hits[qt].pad) == seq) r.st = 1;
    else if (spin >= (1u << 24)) r.st = 2;  // safety net: never hang the device on a lost entry
    return r;
}

// release: kernel B may read the queue while kernel A runs (overlap on)
__device__ __forceinline__ void publish_hit(HitEntry* hits, unsigned q, HitEntry e, unsigned seq, bool release) {
    HitEntry* d = hits + q;
    if (!vc_st_ok(d, sizeof(HitEntry))) return;
    if (release) {
        e.pad = 0u;
        *d = e;
        st_release_u32(&d->pad, seq);
    } else {
        e.pad = seq;
        *d = e;
    }
}

// end of a kernel-A warp: its hits are published, count it (kernel B
// expects 4 per block)
__device__ __forceinline__ void firsthit_block_done(FrameWork* work) {
    __syncwarp();
    // a release add, not __threadfence + atomicAdd: a full fence invalidates
    // the SM's L1 under the warps still marching (measured 2%)
    if ((threadIdx.x & 31) == 0 && vc_st_ok(&work->fh_done, sizeof(unsigned)))
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&work->fh_done) : "memory");
}

__device__ __forceinline__ void allow_dependent_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ void init_ctx(Ctx<T>& C, const vc_render_params& P, const Vol<T>& vol,
                                         const float4* grad, const RayPos& rp0, const uint8_t* dist, int mx,
                                         int my, int skip_on, const TexArgs& tex) {
    C.v = vol;
    C.tx = tex;
    C.rmu = rcp_for(P.mu_water);
    C.grad = grad;
    C.rp = rp0;
#pragma unroll
    for (int a = 0; a < 3; a++) C.rp.o[a] = P.eye[a];
    C.sk.dist = dist;
    C.sk.mx = mx;
    C.sk.my = my;
    C.sk.on = skip_on != 0;
    C.sk.inv_coarse = 1.0 / P.coarse;
    C.sk.inv_coarse_f = (float)C.sk.inv_coarse;
    C.sk.win = make_winf(P.t_low, P.t_high, vol.amax);
    C.lut = nullptr;
}

__device__ __forceinline__ void commit_counters(unsigned long long* counters, int stage, unsigned nsamp,
                                                unsigned nshade, unsigned nskip, unsigned nhit) {
    if (counters == nullptr) return;
    const unsigned FULL = 0xffffffffu;
    nsamp = __reduce_add_sync(FULL, nsamp);
    nshade = __reduce_add_sync(FULL, nshade);
    nskip = __reduce_add_sync(FULL, nskip);
    nhit = __reduce_add_sync(FULL, nhit);
    if ((threadIdx.x & 31) == 0 && vc_st_ok(counters, VC_NUM_COUNTERS * sizeof(unsigned long long))) {
        if (nsamp) atomicAdd(counters + 0, (unsigned long long)nsamp);
        if (nsamp) atomicAdd(counters + 4 + stage, (unsigned long long)nsamp);
        if (nshade) atomicAdd(counters + 1, (unsigned long long)nshade);
        if (nskip) atomicAdd(counters + 2, (unsigned long long)nskip);
        if (nhit) atomicAdd(counters + 3, (unsigned long long)nhit);
    }
}

// Warp-aggregated ticket: every lane with `want` gets a distinct index from
// *ctr (one atomic per warp).
__device__ __forceinline__ unsigned warp_ticket(unsigned* ctr, bool want) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(FULL, want);
    unsigned base = 0;
    const int leader = __ffs(m) - 1;
    if (m != 0 && lane == leader && vc_st_ok(ctr, sizeof(unsigned))) base = atomicAdd(ctr, (unsigned)__popc(m));
    base = __shfl_sync(FULL, base, leader < 0 ? 0 : leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

// Kernel A -- first hit (wavefront stage 1).  Persistent CTAs; each lane
// pulls pixels from FrameWork::pixels.  Work item w is lane (w % 32) of the
// 8x4 screen tile w / 32 (tiles row-major), so a warp refilled as a whole
// traces a compact tile (L1 locality).  The march runs in lock-step, one
// lattice sample per trip, until every live lane has stopped (hit or ray
// end); then hits are refined (fine scan + bisection) and pushed to the hit
// queue, misses write the background, and finished lanes take new pixels:
// the dynamic ray refill of Aila & Laine keeps warps full although
// neighbouring rays march for very different lengths.
#ifndef VC_FH_MINB
#define VC_FH_MINB 8
#endif

#ifndef VC_SH_MINB
#define VC_SH_MINB 5
#endif
#ifndef VC_SHV_MINB
#define VC_SHV_MINB 7
#endif

template <typename T, int INTERP, bool FXW, bool CNT = true>
__global__ void __launch_bounds__(128, VC_FH_MINB) firsthit_kernel(const __grid_constant__ vc_render_params P, Vol<T> vol,
                                                          RayPos rp0, const uint8_t* __restrict__ dist, int mx,
                                                          int my, int skip_on, PixelSink sink,
                                                          int local_rows, unsigned long long* counters,
                                                          FrameWork* work, HitEntry* __restrict__ hits,
                                                          OctDev oct, TexArgs tex, unsigned seq, int rel) {
    if (rel) allow_dependent_launch();
    const unsigned FULL = 0xffffffffu;
    const int tiles_x = (P.width + 7) >> 3;
    const unsigned total = (unsigned)tiles_x * (unsigned)((local_rows + 3) >> 2) * 32u;
    Ctx<T> C;
    init_ctx(C, P, vol, nullptr, rp0, dist, mx, my, skip_on, tex);
    unsigned nsamp = 0, nshade = 0, nskip = 0, nhit = 0;
    RayState R;
    // FXW: the fixed-point walk (trilinear sampling without the adaptive stride)
    constexpr bool fxw = FXW && INTERP == VC_TRILINEAR;
    __shared__ FxLanes fxs;
    __shared__ double s_rhw[2];  // RN(1/width), RN(1/height)
    __shared__ int s_admit;      // fx_frame_admits
    __shared__ float s_icf;      // (float)(1 / coarse): read at skip events (kept in a register, it was
                                 // re-derived from the float64 value by an XU conversion at each)
    const int me = threadIdx.x;
    if (fxw && me == 0) {
        s_rhw[0] = __drcp_rn((double)P.width);
        s_rhw[1] = __drcp_rn((double)P.height);
        s_admit = fx_frame_admits(P, rp0) ? 1 : 0;
        s_icf = C.sk.inv_coarse_f;
    }
    if (fxw) {
        __syncthreads();
        C.sk.inv_coarse_f = s_icf;
    }
    int kf = 0;         // lattice index of the fixed-point walk
    bool pend = false;  // paused for a float64 sample (fx_exact_step)
    int px = 0, lr = 0;
    bool active = false, done = false;
    for (;;) {
        for (;;) {  // refill idle lanes until each has a live ray or the frame is exhausted
            const bool want = !active && !done;
            if (__ballot_sync(FULL, want) == 0) break;
            const unsigned w = warp_ticket(&work->pixels, want);
            if (want) {
                if (w >= total) {
                    done = true;
                } else {
                    const unsigned tile = w >> 5, r = w & 31u;
                    px = (int)(tile % (unsigned)tiles_x) * 8 + (int)(r & 7u);
                    lr = (int)(tile / (unsigned)tiles_x) * 4 + (int)(r >> 3);
                    if (px < P.width && lr < local_rows) {
                        if (start_ray(C, P, px, image_row(P, lr), R, nullptr, fxw ? s_rhw : nullptr)) {
                            active = true;
                            nhit++;
                            if constexpr (fxw) {
                                fx_setup(C, P, R, fxs, me, s_admit != 0);
                                kf = 0;
                            }
                        } else {
                            put_pixel(sink, P, lr, px, bg_pixel(P));
                        }
                    }
                }
            }
        }
        if (__all_sync(FULL, done)) break;
        if constexpr (fxw) {
            for (;;) {  // march phases: the walk in registers, float64 samples in between
                const FxRay F = fx_load(fxs, me);
                for (;;) {
                    const bool need = active && !R.found && !R.exhausted && !pend;
                    const unsigned mneed = __ballot_sync(FULL, need);
                    if (mneed == 0) break;
                    if (VC_FH_READY < READY_DEN) {  // (at READY_DEN the mneed == 0 exit above is the rule)
                        const unsigned mact = __ballot_sync(FULL, active && !pend);
                        if (__popc(mact & ~mneed) * READY_DEN >= __popc(mact) * VC_FH_READY) break;
                    }
                    if (need) {  // two steps per trip: half the vote / reconvergence overhead
                        pend = !march_step_fx<T>(C, P, R, F, kf, nsamp, nskip);
#if VC_FX_UNROLL2
                        if (!pend && !R.found && !R.exhausted) pend = !march_step_fx<T>(C, P, R, F, kf, nsamp, nskip);
#endif
                    }
                }
                if (__ballot_sync(FULL, pend) == 0) break;
                if (pend) {
                    fx_exact_step<T>(C, P, R, fxs, me, kf, nsamp, nskip);
                    pend = false;
                }
            }
        } else {
            for (;;) {
                const bool need = active && !R.found && !R.exhausted;
                const unsigned mneed = __ballot_sync(FULL, need);
                if (mneed == 0) break;
                if (VC_FH_READY < READY_DEN) {  // (at READY_DEN the mneed == 0 exit above is the rule)
                    const unsigned mact = __ballot_sync(FULL, active);
                    if (__popc(mact & ~mneed) * READY_DEN >= __popc(mact) * VC_FH_READY) break;
                }
                if (need) march_step<T, INTERP, true>(C, P, R, nsamp, nskip, P.use_adaptive ? &oct : nullptr);
            }
        }
        const bool hit = active && R.found;
        double t_star = 0.0;
        if (hit) {
            if constexpr (fxw) t_star = refine_hit_fx<T>(C, P, fxs, me, kf - 1, nsamp);
            else t_star = refine_hit<T, INTERP>(C, P, R, R.t_hit, nsamp);
        }
        const unsigned q = warp_ticket(&work->hits, hit);
        if (hit) {
            HitEntry e;
            e.t_star = t_star;
            if constexpr (fxw) {
                e.lim = fxs.lim[me];
#pragma unroll
                for (int a = 0; a < 3; a++) e.d[a] = fxs.d[a][me];
            } else {
                e.lim = R.lim;
#pragma unroll
                for (int a = 0; a < 3; a++) e.d[a] = C.rp.d[a];
            }
            e.pix = pack_pix(lr, px);
            e.pad = 0u;
            publish_hit(hits, q, e, seq, rel != 0);
        }
        if (active && (R.found || R.exhausted)) {
            if (R.exhausted) put_pixel(sink, P, lr, px, bg_pixel(P));
            active = false;
        }
    }
    if constexpr (CNT) commit_counters(counters, 0, nsamp, nshade, nskip, nhit);  // (CNT false: counters == nullptr)
    firsthit_block_done(work);
}

// use_adaptive with use_octree (raycast.py:494-499, _kernels.py:656): the reference's first
// hit marches only the merged t-segments of the octree leaves whose padded
// range meets the window (collect_segments, _kernels.py:267-342), restarting
// the lattice index at each segment (k = max(k, floor((s0 - t_enter) /
// coarse)), _kernels.py:402-410) and striding adaptively inside.  Since the
// adaptive stride can step over in-window samples, which samples exist
// decides the pixel, so this mode replays the walk exactly: the same
// depth-first near-to-far traversal (children sorted by entry with the same
// insertion sort, so ties pop in the same order) over the level-grid tree,
// consumed lazily -- the next leaf is pulled when the lattice passes the
// current segment end; a leaf that merges (a0 <= s1 + 1e-9) only extends it,
// which is what the eager list would have held.  The reference's segment
// buffer cap (raycast.py:499, 4096: further leaves overwrite the last end)
// is honoured by draining the walk before marching the last segment.
constexpr int SEG_CAP = 4096;
constexpr int SEG_STACK = 1 + 7 * 17;  // depth-first stack bound for <= 17 levels

struct SegWalk {
    unsigned long long stack[SEG_STACK];
    int sp;
    double tray0, tray1;
    double inv[3];  // RN(1.0 / d): the reference's per-node-interval value, once per ray
};

__device__ __forceinline__ unsigned long long seg_node(int L, int bx, int by, int bz) {
    return ((unsigned long long)L << 57) | ((unsigned long long)bz << 38) | ((unsigned long long)by << 19) |
           (unsigned long long)bx;
}

// One node of the walk: 1 = a leaf interval [a0, b0] was emitted, 0 = the
// node was skipped or expanded, -1 = the walk is finished.
constexpr int SEG_LEAF = 1, SEG_MORE = 0, SEG_DONE = -1;
__device__ __noinline__ int seg_step(const OctDev& o, SegWalk& W, const StrideArgs& A, double t_low,
                                     double t_high, double& a0, double& b0) {
    const unsigned M = (1u << 19) - 1u;
    if (W.sp <= 0) return SEG_DONE;
    {
        const unsigned long long node = W.stack[--W.sp];
        const int L = (int)(node >> 57);
        const int b[3] = {(int)(node & M), (int)((node >> 19) & M), (int)((node >> 38) & M)};
        double ta, tb;
        if (!oct_node_interval(o, L, b, A.o, A.d, W.inv, A.s, ta, tb)) return SEG_MORE;
        if (ta < W.tray0) ta = W.tray0;
        if (tb > W.tray1) tb = W.tray1;
        if (tb < ta) return SEG_MORE;
        const long long box = vc_ldg(o.box_off + L) +
                              ((long long)b[2] * vc_ldg(o.dims + 3 * L + 1) + b[1]) * vc_ldg(o.dims + 3 * L + 0) + b[0];
        // a box whose padded range misses the window holds no leaf that
        // does (a child's padded box lies inside its parent's): the whole
        // subtree would emit nothing, so it is pruned without changing the
        // emitted sequence
        const bool meets = vc_ldg(o.srange + 2 * box) <= t_high && vc_ldg(o.srange + 2 * box + 1) >= t_low;
        if (!meets) return SEG_MORE;
        if (vc_ldg(o.state + box) == 2) {  // leaf
            a0 = ta;
            b0 = tb;
            return SEG_LEAF;
        }
        // children: the next level's boxes inside this one, z-major like the
        // reference's construction order (octree.py:97-105)
        const int stride_map = A.nx + A.ny + A.nz;
        const int* m = o.amap + (size_t)(L + 1) * stride_map;
        int c0[3], cn[3];
        const int axoff[3] = {0, A.nx, A.nx + A.ny};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const int* iv = o.ivl + vc_ldg(o.ivl_off + 3 * L + a) + 2 * b[a];
            const int lo = vc_ldg(iv), hi = vc_ldg(iv + 1);
            c0[a] = vc_ldg(m + axoff[a] + lo);
            cn[a] = hi - lo >= 2 ? 2 : 1;
        }
        // oct_node_interval is separable: a child's slab along axis a depends
        // only on its index along a, so the <= 2 slabs per axis are evaluated
        // once (<= 6 instead of 24) and each child takes the max / min of its
        // three -- the same doubles, so the same intervals, bit for bit
        double sa[3][2], sb[3][2];
        bool sok[3][2];
#pragma unroll
        for (int a = 0; a < 3; a++) {
#pragma unroll
            for (int c = 0; c < 2; c++) {
                sa[a][c] = -1e300;
                sb[a][c] = 1e300;
                sok[a][c] = true;
                if (c < cn[a]) {
                    const int* iv = o.ivl + vc_ldg(o.ivl_off + 3 * (L + 1) + a) + 2 * (c0[a] + c);
                    const double lo = dmul(u2d((uint32_t)vc_ldg(iv)), A.s[a]);
                    const double hi = dmul(u2d((uint32_t)vc_ldg(iv + 1)), A.s[a]);
                    const double ov = A.o[a];
                    if (A.d[a] == 0.0) {
                        sok[a][c] = !(ov < lo || ov > hi);
                    } else {
                        double ta = dmul(dsub(lo, ov), W.inv[a]), tb = dmul(dsub(hi, ov), W.inv[a]);
                        if (ta > tb) {
                            const double sw = ta;
                            ta = tb;
                            tb = sw;
                        }
                        sa[a][c] = ta;
                        sb[a][c] = tb;
                    }
                }
            }
        }
        double ct[8];
        unsigned long long ci[8];
        int cnt = 0;
        for (int cz = 0; cz < cn[2]; cz++)
            for (int cy = 0; cy < cn[1]; cy++)
                for (int cx = 0; cx < cn[0]; cx++) {
                    // register selects (no local-memory indexing)
                    const bool ok = (cx ? sok[0][1] : sok[0][0]) && (cy ? sok[1][1] : sok[1][0]) &&
                                    (cz ? sok[2][1] : sok[2][0]);
                    if (!ok) continue;
                    const int cb[3] = {c0[0] + cx, c0[1] + cy, c0[2] + cz};
                    const double ax = cx ? sa[0][1] : sa[0][0], bx = cx ? sb[0][1] : sb[0][0];
                    const double ay = cy ? sa[1][1] : sa[1][0], by = cy ? sb[1][1] : sb[1][0];
                    const double az = cz ? sa[2][1] : sa[2][0], bz = cz ? sb[2][1] : sb[2][0];
                    // the same strict compares in the same axis order as oct_node_interval
                    double ca = -1e300, cbb = 1e300;
                    if (ax > ca) ca = ax;
                    if (bx < cbb) cbb = bx;
                    if (ay > ca) ca = ay;
                    if (by < cbb) cbb = by;
                    if (az > ca) ca = az;
                    if (bz < cbb) cbb = bz;
                    if (ca > cbb || cbb < W.tray0 || ca > W.tray1) continue;
                    ct[cnt] = ca;
                    ci[cnt] = seg_node(L + 1, cb[0], cb[1], cb[2]);
                    cnt++;
                }
        for (int a = 1; a < cnt; a++) {  // farthest entry first: the nearest pops first
            const double tv = ct[a];
            const unsigned long long iv = ci[a];
            int j = a - 1;
            while (j >= 0 && ct[j] < tv) {
                ct[j + 1] = ct[j];
                ci[j + 1] = ci[j];
                j--;
            }
            ct[j + 1] = tv;
            ci[j + 1] = iv;
        }
        for (int a = 0; a < cnt && W.sp < SEG_STACK; a++) W.stack[W.sp++] = ci[a];
    }
    return SEG_MORE;
}

// next emitted leaf interval [a0, b0] of the walk (false: walk finished)
__device__ __forceinline__ bool seg_next_leaf(const OctDev& o, SegWalk& W, const StrideArgs& A, double t_low,
                                              double t_high, double& a0, double& b0) {
    for (;;) {
        const int r = seg_step(o, W, A, t_low, t_high, a0, b0);
        if (r != SEG_MORE) return r == SEG_LEAF;
    }
}

template <typename T>
__device__ __forceinline__ StrideArgs make_stride_args(const Ctx<T>& C, const vc_render_params& P) {
    StrideArgs A;
    A.nx = C.v.nx;
    A.ny = C.v.ny;
    A.nz = C.v.nz;
    A.adapt_jump = P.adapt_jump;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        A.o[a] = C.rp.o[a];
        A.d[a] = C.rp.d[a];
        A.s[a] = C.rp.s[a];
    }
    A.detail_eps = P.detail_eps;
    A.coarse = P.coarse;
    return A;
}

// Per-ray state of the segment walk between work units.
struct SegRay {
    double t_exit, s0, s1;
    int nseg;
    bool walking;  // pulling the next leaf (else marching the current segment)
    bool has_seg;
};

// Start the next segment at leaf [a0, b0] (the reference's segment loop
// head, _kernels.py:402-410), honouring the segment-buffer cap.
template <typename T>
__device__ __forceinline__ void seg_open(const Ctx<T>& C, const vc_render_params& P, const OctDev& o,
                                         SegWalk& W, const StrideArgs& A, SegRay& S, RayState& R, double a0,
                                         double b0) {
    S.s0 = a0;
    S.s1 = b0;
    S.has_seg = true;
    if (++S.nseg == SEG_CAP) {  // the reference's last buffer slot takes every later leaf
        double c0, c1;
        while (seg_next_leaf(o, W, A, P.t_low, P.t_high, c0, c1)) {
            if (c0 <= dadd(S.s1, 1e-9)) {
                if (c1 > S.s1) S.s1 = c1;
            } else {
                S.s1 = c1;
            }
        }
    }
    const double kk = floor(ddiv(dsub(S.s0, R.t_enter), P.coarse));
    if (kk > R.k) R.k = kk;
    S.walking = false;
}

// Kernel A for the segment mode, as a wavefront like Kernel A: persistent
// CTAs, lanes refilled with new rays as theirs finish, and each trip of
// the loop advances every live lane by one unit -- one node of its walk or
// one lattice sample -- so rays with long walks do not hold their warp's
// other lanes idle.  Same work-item tiling, hit queue and counters.
template <typename T, int INTERP>
__global__ void __launch_bounds__(128) firsthit_seg_kernel(const __grid_constant__ vc_render_params P, Vol<T> vol,
                                                           RayPos rp0, PixelSink sink, int local_rows,
                                                           unsigned long long* counters, FrameWork* work,
                                                           HitEntry* __restrict__ hits, OctDev oct, unsigned seq,
                                                           int rel) {
    if (rel) allow_dependent_launch();
    const unsigned FULL = 0xffffffffu;
    const int tiles_x = (P.width + 7) >> 3;
    const unsigned total = (unsigned)tiles_x * (unsigned)((local_rows + 3) >> 2) * 32u;
    Ctx<T> C;
    init_ctx(C, P, vol, nullptr, rp0, nullptr, 0, 0, 0, TexArgs{});
    unsigned nsamp = 0, nhit = 0;
    RayState R;
    SegRay S;
    SegWalk W;
    StrideArgs A;
    int px = 0, lr = 0;
    bool active = false, done = false;
    for (;;) {
        for (;;) {  // refill idle lanes
            const bool want = !active && !done;
            if (__ballot_sync(FULL, want) == 0) break;
            const unsigned w = warp_ticket(&work->pixels, want);
            if (want) {
                if (w >= total) {
                    done = true;
                } else {
                    const unsigned tile = w >> 5, r = w & 31u;
                    px = (int)(tile % (unsigned)tiles_x) * 8 + (int)(r & 7u);
                    lr = (int)(tile / (unsigned)tiles_x) * 4 + (int)(r >> 3);
                    if (px < P.width && lr < local_rows) {
                        if (start_ray(C, P, px, image_row(P, lr), R, &S.t_exit)) {
                            nhit++;
                            A = make_stride_args(C, P);
                            W.sp = 0;
                            W.stack[W.sp++] = seg_node(0, 0, 0, 0);
                            W.tray0 = R.t_enter;
                            W.tray1 = S.t_exit;
#pragma unroll
                            for (int a = 0; a < 3; a++) W.inv[a] = A.d[a] == 0.0 ? 0.0 : __drcp_rn(A.d[a]);
                            S.nseg = 0;
                            S.walking = true;
                            S.has_seg = false;
                            active = true;
                        } else {
                            put_pixel(sink, P, lr, px, bg_pixel(P));
                        }
                    }
                }
            }
        }
        if (__all_sync(FULL, done)) break;
        bool miss = false;
        if (active) {
            if (S.walking) {
                double a0, b0;
                const int st = seg_step(oct, W, A, P.t_low, P.t_high, a0, b0);  // one node per trip (measured best)
                if (st == SEG_DONE) {
                    miss = true;
                } else if (st == SEG_LEAF) {
                    if (S.has_seg && a0 <= dadd(S.s1, 1e-9)) {  // merges into the current segment
                        if (b0 > S.s1) S.s1 = b0;
                        S.walking = false;
                    } else {
                        seg_open(C, P, oct, W, A, S, R, a0, b0);
                    }
                }
            } else {
                const double t = dadd(R.t_enter, dmul(R.k, P.coarse));
                if (t > R.lim) {  // every later segment starts at or after t
                    miss = true;
                } else if (t > dadd(S.s1 > S.t_exit ? S.t_exit : S.s1, 1e-12)) {
                    if (S.nseg == SEG_CAP) miss = true;
                    else S.walking = true;
                } else {
                    double p[3];
                    C.rp.at(t, p);
                    nsamp++;
                    if (window_at<T, INTERP>(C, P, p)) {
                        R.found = true;
                        R.t_hit = t;
                    } else {
                        R.k += P.use_adaptive ? adaptive_stride(oct, A, p[0], p[1], p[2], R.k, R.t_enter) : 1.0;
                    }
                }
            }
        }
        const bool hit = active && R.found;
        double t_star = 0.0;
        if (hit) t_star = refine_hit<T, INTERP>(C, P, R, R.t_hit, nsamp);
        const unsigned q = warp_ticket(&work->hits, hit);
        if (hit) {
            HitEntry e;
            e.t_star = t_star;
            e.lim = R.lim;
            e.d[0] = C.rp.d[0];
            e.d[1] = C.rp.d[1];
            e.d[2] = C.rp.d[2];
            e.pix = pack_pix(lr, px);
            e.pad = 0u;
            publish_hit(hits, q, e, seq, rel != 0);
            active = false;
        }
        if (miss) {
            put_pixel(sink, P, lr, px, bg_pixel(P));
            active = false;
        }
    }
    commit_counters(counters, 0, nsamp, 0, 0, nhit);
    firsthit_block_done(work);
}

// Kernel B -- shade + composite (wavefront stage 2).  Persistent CTAs pull
// first hits from the queue, regenerate the ray, shade at t_star and, in
// composited mode, keep marching t_star + m*coarse and shading in-window
// samples until early ray termination or the ray leaves the box.  Lanes
// refill from the queue as their pixel finishes.
template <typename T, int OP, int INTERP, bool GV, bool CNT = true>
__global__ void __launch_bounds__(128, GV ? VC_SHV_MINB : VC_SH_MINB) shade_kernel(const __grid_constant__ vc_render_params P, Vol<T> vol,
                                                       const float4* __restrict__ grad, RayPos rp0,
                                                       const uint8_t* __restrict__ dist, int mx, int my,
                                                       int skip_on, PixelSink sink,
                                                       unsigned long long* counters, FrameWork* work,
                                                       const HitEntry* __restrict__ hits, TexArgs tex,
                                                       unsigned seq, unsigned nfh, unsigned max_hits) {
    const unsigned FULL = 0xffffffffu;
    // the overlapped stage hand-off: gradient-volume shading (the taps
    // kernel keeps the plain refill; measured slower with it, register bound)
    constexpr bool OV = GV && VC_STAGE_OVERLAP;
    __shared__ SharedLut s_lut;
    load_shared_lut(P, s_lut);
    Ctx<T> C;
    init_ctx(C, P, vol, grad, rp0, dist, mx, my, skip_on, tex);
    C.lut = &s_lut;
    unsigned nsamp = 0, nshade = 0, nskip = 0, nhit = 0;
    RayState R;
    int px = 0, lr = 0;
    bool active = false, done = false;
    unsigned qt = 0;
    bool waiting = false;      // OV: holds queue ticket qt, entry not published yet
    bool fh_all = !OV;         // every kernel-A block has finished (warp-uniform)
    unsigned final_hits = 0u;  // the queue length then
    if constexpr (!OV) final_hits = *(volatile unsigned*)&work->hits;
#ifdef VC_DEBUG_RAYCOST
    unsigned dbg_march = 0, dbg_shade = 0;  // per-ray work, written as the pixel (tools/raycost_probe.py)
#endif
    // a lane takes the entry of its ticket: regenerate the ray at t_star
    auto start = [&](const HitEntry& e) {
        px = (int)(e.pix & 0xffffu);
        lr = (int)(e.pix >> 16);
#pragma unroll
        for (int a = 0; a < 3; a++) C.rp.d[a] = e.d[a];
        R.lim = e.lim;
        R.base = e.t_star;
        R.k = 1.0;
        R.acc_r = R.acc_g = R.acc_b = 0.0;
        R.remain = 1.0;
        R.t_hit = e.t_star;
        R.found = true;
        R.exhausted = false;
        active = true;
#ifdef VC_DEBUG_RAYCOST
        dbg_march = dbg_shade = 0;
#endif
    };
    for (;;) {
        // refill: a fresh lane starts "found" at its t_star, so its first
        // shade joins the other lanes' shades in the single resolve step below
        // (only once VC_SH_REFILL lanes are idle, or none is active: each
        // refill stalls the warp on the queue reads)
        if constexpr (OV) {
            for (unsigned spin = 0;; spin++) {
                const bool want = !active && !done && !waiting;
                const unsigned mw = __ballot_sync(FULL, want);
                if (mw != 0 && (__popc(mw) >= VC_SH_REFILL || __ballot_sync(FULL, active) == 0)) {
                    const unsigned q = warp_ticket(&work->shades, want);
                    if (want) {
                        qt = q;
                        waiting = true;
                    }
                }
                if (__ballot_sync(FULL, waiting) == 0) break;
                bool claim = false;
                if (!fh_all) {  // kernel A may still be running (out of line: keeps the hot code compact)
                    const OverlapPoll r = overlap_poll(work, hits, nfh, seq, max_hits, qt, waiting, spin);
                    fh_all = r.fh_all;
                    final_hits = r.final_hits;
                    claim = r.st == 1;
                    if (r.st == 2) {
                        waiting = false;
                        done = true;
                    }
                } else if (waiting) {  // the queue is complete: every entry below final_hits is published
                    claim = qt < final_hits;
                    if (!claim) {
                        waiting = false;
                        done = true;
                    }
                }
                if (claim) {
                    waiting = false;
                    start(load_hit(hits + qt));
                }
                if (__ballot_sync(FULL, active) != 0 || __all_sync(FULL, done)) break;
                // nothing to shade yet: lanes wait for entries kernel A is still producing
                if (__ballot_sync(FULL, waiting) != 0) __nanosleep(spin < 8 ? 256u : 2048u);
            }
        } else {
            for (;;) {
                const bool want = !active && !done;
                const unsigned mw = __ballot_sync(FULL, want);
                if (mw == 0) break;
                if (__popc(mw) < VC_SH_REFILL && __ballot_sync(FULL, active) != 0) break;
                const unsigned q = warp_ticket(&work->shades, want);
                if (want) {
                    if (q >= final_hits) done = true;
                    else start(vc_ld(hits + q));
                }
            }
        }
        if (__all_sync(FULL, done)) break;
        for (;;) {
            const bool need = active && !R.found && !R.exhausted;
            const unsigned mneed = __ballot_sync(FULL, need);
            if (mneed == 0) break;
            const unsigned mact = __ballot_sync(FULL, active);
            if (__popc(mact & ~mneed) * READY_DEN >= __popc(mact) * (GV ? VC_SHV_READY : VC_SH_READY)) break;
            if (need) march_step<T, INTERP, true>(C, P, R, nsamp, nskip);
#ifdef VC_DEBUG_RAYCOST
            if (need) dbg_march++;
#endif
        }
        if (active && (R.found || R.exhausted)) {
            uchar4 o;
            bool fin;
            if (R.exhausted) {
                o = composite_pixel(P, R);
                fin = true;
            } else {
                R.found = false;
                fin = shade_and_composite<T, OP, INTERP, GV>(C, P, R, R.t_hit, o, nshade);
#ifdef VC_DEBUG_RAYCOST
                dbg_shade++;
#endif
            }
            if (fin) {
#ifdef VC_DEBUG_RAYCOST
                o = make_uchar4(dbg_march & 255u, (dbg_march >> 8) & 255u, dbg_shade & 255u, (dbg_shade >> 8) & 255u);
#endif
                put_pixel(sink, P, lr, px, o);
                active = false;
            }

        }
    }
    if constexpr (CNT) commit_counters(counters, 1, nsamp, nshade, nskip, nhit);  // (CNT false: counters == nullptr)
    // the frame's last kernel-B warp resets the work counters for the next
    // frame on this scratch: every kernel-A warp has finished (B's lanes end
    // only after seeing that) and every other B warp has made its last
    // counter access (its lanes' atomics returned before its count)
    __syncwarp();
    if ((threadIdx.x & 31) == 0 && vc_st_ok(work, sizeof(FrameWork))) {
        const unsigned nw = gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(&work->sh_done, 1u) + 1u == nw) {
            work->pixels = 0u;
            work->hits = 0u;
            work->shades = 0u;
            work->fh_done = 0u;
            work->sh_done = 0u;
        }
    }
}

}  // namespace vc

namespace vc {

static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <typename K>
static unsigned persistent_blocks(K kernel, long long max_useful) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 128, 0);
    if (per_sm < 1) per_sm = 1;
    long long b = (long long)sm_count() * per_sm;
    if (b > max_useful) b = max_useful;
    return (unsigned)(b < 1 ? 1 : b);
}

template <typename T, int OP, int INTERP>
static cudaError_t launch_t(const RenderLaunch& L, cudaStream_t stream) {
    const Vol<T> vol = make_vol(static_cast<const T*>(L.data), L.nx, L.ny, L.nz, L.amax);
    FrameWork* fw = reinterpret_cast<FrameWork*>(L.work);
    HitEntry* hits = reinterpret_cast<HitEntry*>(L.hits);
    cudaError_t e = cudaSuccess;  // fw: zero on entry (see FrameWork)
    const long long tiles = (long long)((L.p->width + 7) / 8) * ((L.local_rows + 3) / 4);
    PixelSink sink{reinterpret_cast<uchar4*>(L.out), reinterpret_cast<uchar4* const*>(L.peers), L.npeers,
                   L.peer_self, L.peer_dest, L.tile_cnt, (L.p->width + 7) / 8, L.local_rows};
    if (L.tile_cnt != nullptr) {
        e = cudaMemsetAsync(L.tile_cnt, 0, sizeof(unsigned) * (size_t)tiles, stream);
        if (e != cudaSuccess) return e;
    }
    TexArgs tex{L.tex_value, L.tex_grad, L.tex_scale, 0.0f, 0.0f};
    // v >= t_low <=> v >= RU(t_low) for a float v (and v <= t_high <=> v <= RD(t_high))
    tex.lo = (float)L.p->t_low;
    if ((double)tex.lo < L.p->t_low) tex.lo = std::nextafter(tex.lo, INFINITY);
    tex.hi = (float)L.p->t_high;
    if ((double)tex.hi > L.p->t_high) tex.hi = std::nextafter(tex.hi, -INFINITY);
    if (L.ev[0]) cudaEventRecord(L.ev[0], stream);
    // use_adaptive + use_octree, or use_octree with 0 in the window: the
    // octree-segment first hit (exact reference walk, capi.cu render_impl)
    const bool seg = INTERP != VC_TEX && L.seg_walk;
    unsigned nfh = 0;  // kernel-A blocks (kernel B's end-of-queue test)
    // the overlapped hand-off: gradient-volume shading, composited frames
    // (a surface frame's shade stage is too short to gain from it)
    const int overlap = (VC_STAGE_OVERLAP && L.overlap_stages && L.grad != nullptr && L.p->mode != VC_SURFACE) ? 1 : 0;
    if (seg) {
        if constexpr (INTERP != VC_TEX) {
            nfh = persistent_blocks(firsthit_seg_kernel<T, INTERP>, (tiles + 3) / 4);
            firsthit_seg_kernel<T, INTERP><<<nfh, 128, 0, stream>>>(
                *L.p, vol, L.rp, sink, L.local_rows, reinterpret_cast<unsigned long long*>(L.counters), fw,
                hits, L.oct, L.seq, overlap);
        }
    } else {
        // the fixed-point walk: trilinear sampling without the adaptive stride
        auto k = firsthit_kernel<T, INTERP, false>;
        if constexpr (INTERP == VC_TRILINEAR) {
            // the fixed-point walk; without work counters the counting compiles out
            if (!L.p->use_adaptive)
                k = L.counters ? firsthit_kernel<T, INTERP, true, true> : firsthit_kernel<T, INTERP, true, false>;
        }
        nfh = persistent_blocks(k, (tiles + 3) / 4);
        k<<<nfh, 128, 0, stream>>>(*L.p, vol, L.rp, L.occ, L.mx, L.my, L.skip_on, sink, L.local_rows,
                                   reinterpret_cast<unsigned long long*>(L.counters), fw, hits, L.oct, tex, L.seq,
                                   overlap);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (L.ev[1]) cudaEventRecord(L.ev[1], stream);
    const float4* grad = static_cast<const float4*>(L.grad);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(L.counters);
    // kernel B may start while kernel A finishes (programmatic stream
    // serialization; see "Stage hand-off")
    auto launch_b = [&](auto kernel) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(persistent_blocks(kernel, (tiles + 3) / 4));
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = overlap;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kernel, *L.p, vol, grad, L.rp, L.occ, L.mx, L.my, L.skip_on, sink, cnt, fw,
                                  hits, tex, L.seq, nfh * 4u, (unsigned)((long long)L.local_rows * L.p->width));
    };
    if (grad != nullptr) {
        if constexpr (INTERP == VC_TRILINEAR) {
            e = cnt ? launch_b(shade_kernel<T, OP, INTERP, true, true>) : launch_b(shade_kernel<T, OP, INTERP, true, false>);
        } else {
            e = launch_b(shade_kernel<T, OP, INTERP, true>);
        }
    } else {
        e = launch_b(shade_kernel<T, OP, INTERP, false>);
    }
    if (e != cudaSuccess) return e;
    if (L.ev[2]) cudaEventRecord(L.ev[2], stream);
    return cudaGetLastError();
}

template <typename T, int OP>
static cudaError_t launch_op(const RenderLaunch& L, cudaStream_t s) {
    if (L.p->sampler == VC_SAMPLER_TEXTURE) return launch_t<T, OP, VC_TEX>(L, s);  // trilinear (validated)
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

#ifdef VC_CHECKED
VC_CHECKED_HOST_API(raycast)
#endif

cudaError_t launch_raycast(const RenderLaunch& L, cudaStream_t s) {
#ifdef VC_CHECKED
    if (L.regions) {
        cudaError_t e = vc_set_regions_raycast(L.regions, L.nregions, s);
        if (e != cudaSuccess) return e;
    }
#endif
    switch (L.dtype) {
        case VC_U8: return launch_dtype<uint8_t>(L, s);
        case VC_U16: return launch_dtype<uint16_t>(L, s);
        default: return launch_dtype<float>(L, s);
    }
}

size_t hit_entry_bytes() { return sizeof(HitEntry); }
size_t frame_work_bytes() { return sizeof(FrameWork); }

}  // namespace vc
