// vc_device.cuh -- device-side restatement of the reference arithmetic.
//
// Every function mirrors one of /root/reference/pkg/src/voxelcast/_kernels.py
// operation for operation in float64.  The translation units that include
// this header are built with -fmad=false and the helpers below use the
// explicit round-to-nearest intrinsics, so no multiply-add is ever
// contracted (numba emits none either): the FP64
// path is meant to be bit-identical to the reference.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voxelcast_b200.h"

namespace vc {

// _kernels.py:25-30
constexpr double GRAD_EPS = 1e-8;
constexpr double OPAQUE_ALPHA = 1.0 - 1e-6;
constexpr double MIN_REMAINING = 0.01;
__host__ __device__ constexpr int grad_samples(int op) { return op == VC_OP_CENTRAL ? 6 : 26; }

// 1/sqrt(2), 1/sqrt(3) exactly as the reference rounds them:
// 1.0 / math.sqrt(2.0) and 1.0 / math.sqrt(3.0) (_kernels.py:173)
constexpr double INV_SQRT2 = 0x1.6a09e667f3bccp-1;  // 0.7071067811865475
constexpr double INV_SQRT3 = 0x1.279a74590331dp-1;  // 0.5773502691896258

// ---- bounds-checked build (VC_CHECKED) ------------------------------------
// compute-sanitizer is not available on this pool, so the library has a
// checked variant of its own (paper_1609_01317_b200/_lib/checked, built by
// build()): every global load and store of the raycast and point kernels
// goes through vc_ldg / vc_st_ok, which test the address against the
// buffers the launch was given (vc_set_regions, one table per translation
// unit) and count -- and skip -- anything outside them.  The production
// build compiles both to plain accesses.
#ifdef VC_CHECKED
struct VcRegion {
    unsigned long long lo, hi;  // [lo, hi) byte addresses
};
constexpr int VC_MAX_REGIONS = 96;
static __constant__ VcRegion vc_regions[VC_MAX_REGIONS];
static __constant__ int vc_nregions;
static __device__ unsigned long long vc_viol_count;
static __device__ unsigned long long vc_viol_first;
static __device__ __noinline__ bool vc_addr_ok(const void* p, unsigned n) {
    const unsigned long long a = reinterpret_cast<unsigned long long>(p);
    for (int r = 0; r < vc_nregions; r++)
        if (a >= vc_regions[r].lo && a + n <= vc_regions[r].hi) return true;
    if (atomicAdd(&vc_viol_count, 1ull) == 0ull) vc_viol_first = a;
    return false;
}
template <typename T>
__device__ __forceinline__ T vc_ldg(const T* p) {
    return vc_addr_ok(p, sizeof(T)) ? __ldg(p) : T{};
}
template <typename T>
__device__ __forceinline__ T vc_ld(const T* p) {
    return vc_addr_ok(p, sizeof(T)) ? *p : T{};
}
__device__ __forceinline__ bool vc_st_ok(const void* p, unsigned n) { return vc_addr_ok(p, n); }
// host side, one copy per translation unit (static device symbols)
#define VC_CHECKED_HOST_API(tu)                                                                          \
    cudaError_t vc_set_regions_##tu(const unsigned long long* lohi, int n, cudaStream_t s) {           \
        if (n > VC_MAX_REGIONS) n = VC_MAX_REGIONS;                                                       \
        cudaError_t e = cudaMemcpyToSymbolAsync(vc_regions, lohi, sizeof(VcRegion) * n, 0,              \
                                                cudaMemcpyHostToDevice, s);                              \
        if (e == cudaSuccess)                                                                            \
            e = cudaMemcpyToSymbolAsync(vc_nregions, &n, sizeof(int), 0, cudaMemcpyHostToDevice, s);     \
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);                                              \
        return e;                                                                                        \
    }                                                                                                    \
    unsigned long long vc_take_violations_##tu(unsigned long long* first) {                            \
        unsigned long long c = 0, f = 0, z = 0;                                                          \
        cudaDeviceSynchronize();                                                                         \
        cudaMemcpyFromSymbol(&c, vc_viol_count, sizeof(c));                                              \
        cudaMemcpyFromSymbol(&f, vc_viol_first, sizeof(f));                                              \
        cudaMemcpyToSymbol(vc_viol_count, &z, sizeof(z));                                                \
        if (first) *first = f;                                                                           \
        return c;                                                                                        \
    }
#else
template <typename T>
__device__ __forceinline__ T vc_ldg(const T* p) {
    return __ldg(p);
}
template <typename T>
__device__ __forceinline__ T vc_ld(const T* p) {
    return *p;
}
__device__ __forceinline__ constexpr bool vc_st_ok(const void*, unsigned) { return true; }
#endif

// ---- strict float64 helpers -----------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
// IEEE division.  A zero numerator (frequent: hu = (v - mu)/mu on voxels
// equal to mu_water) takes the slow, divergent branch of __ddiv_rn; 0 / b
// is +-0 with the xor of the signs for every finite non-zero b, which
// 0 * copysign(1, b) reproduces exactly.
__device__ __forceinline__ double ddiv(double a, double b) {
#ifndef VC_DDIV_PLAIN
    if (a == 0.0 && b != 0.0 && fabs(b) < 1.0 / 0.0) return __dmul_rn(a, copysign(1.0, b));
#endif
    return __ddiv_rn(a, b);
}

// a / b, correctly rounded, from y = RN(1/b) (Markstein: q = RN(a y) is
// within 1 ulp of a/b; the fma residual and one fma correction give
// RN(a/b)).  Three FP64 instructions instead of the ~40 of __ddiv_rn.
// Used for b = voxel spacing (per-volume constant y = 1.0 / s from the
// host); spacings with an all-ones significand, which the classic statement
// of the theorem excludes, take ddiv_cold instead (RayPos::rcp).
__device__ __forceinline__ double ddiv_rcp(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    return __fma_rn(r, y, q);
}
static __device__ __noinline__ double ddiv_cold(double a, double b) { return ddiv(a, b); }
// y = rcp_for(b): RN(1/b), or 0 when b is not a positive finite value with
// a usable significand; div_rcp(a, b, y) = RN(a / b) either way
__device__ __forceinline__ double rcp_for(double b) {
    const bool ok = b > 0.0 && b < 1e300 &&
                    (__double_as_longlong(b) & 0xFFFFFFFFFFFFFLL) != 0xFFFFFFFFFFFFFLL;
    return ok ? __drcp_rn(b) : 0.0;
}
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
    return y != 0.0 ? ddiv_rcp(a, b, y) : ddiv_cold(a, b);
}

// _kernels.py:35-37
__device__ __forceinline__ double lerp(double f0, double f1, double t) {
    return dadd(f0, dmul(dsub(f1, f0), t));
}

// integer voxels are carried in 32-bit registers once loaded (zero
// extended), float voxels as themselves
template <typename T>
struct Wide {
    using type = uint32_t;
};
template <>
struct Wide<float> {
    using type = float;
};
template <typename T>
using wide_t = typename Wide<T>::type;

template <typename T>
struct Vol {
    const T* __restrict__ data;
    int nx, ny, nz;
    // n-1 and max(n-2, 0) as doubles: range checks and cell clamps without
    // an I2F.F64 per sample (make_vol fills them)
    double mx, my, mz, cx, cy, cz;
    // max |voxel value| (bounds the float32 pre-test error); <= 0: unknown
    double amax;
    // max(n-2, 0): the clamped lower cell corner; element offsets of the
    // +1 corner along x / y / z (0 on a one-voxel axis, _kernels.py:53-64)
    int kx, ky, kz;
    uint32_t sx1, sy1, sz1;
    uint32_t syb, szb;  // sy1 / sz1 in bytes
};

template <typename T>
__host__ __device__ inline Vol<T> make_vol(const T* data, int nx, int ny, int nz, double amax = -1.0) {
    Vol<T> v;
    v.amax = amax;
    v.data = data;
    v.nx = nx;
    v.ny = ny;
    v.nz = nz;
    v.mx = (double)(nx - 1);
    v.my = (double)(ny - 1);
    v.mz = (double)(nz - 1);
    v.cx = (double)(nx - 2 < 0 ? 0 : nx - 2);
    v.cy = (double)(ny - 2 < 0 ? 0 : ny - 2);
    v.cz = (double)(nz - 2 < 0 ? 0 : nz - 2);
    v.kx = nx - 2 < 0 ? 0 : nx - 2;
    v.ky = ny - 2 < 0 ? 0 : ny - 2;
    v.kz = nz - 2 < 0 ? 0 : nz - 2;
    v.sx1 = nx > 1 ? 1u : 0u;
    v.sy1 = ny > 1 ? (uint32_t)nx : 0u;
    v.sz1 = nz > 1 ? (uint32_t)nx * (uint32_t)ny : 0u;
    v.syb = v.sy1 * (uint32_t)sizeof(T);
    v.szb = v.sz1 * (uint32_t)sizeof(T);
    return v;
}

// The 8 corners of the (clamped) cell with lower corner (i, j, k): one
// 64-bit base address and two row offsets, the x neighbours at an
// immediate +1 element (x-degenerate grids, nx == 1, read the same voxel
// twice on a uniform branch).  Corner order c000 c100 c010 c110 c001 c101
// c011 c111.
// The +1 reads of an x-degenerate grid land on the next row or on the
// allocation's zeroed tail padding (VC_VOLUME_PAD) and are replaced.
constexpr size_t VC_VOLUME_PAD = 64;
template <typename T>
__device__ __forceinline__ void gather8(const Vol<T>& v, int i, int j, int k, wide_t<T> c[8]) {
    const uint32_t idx = ((uint32_t)k * (uint32_t)v.ny + (uint32_t)j) * (uint32_t)v.nx + (uint32_t)i;
    const T* p0 = v.data + idx;
    const T* p1 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p0) + v.syb);
    const T* p2 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p0) + v.szb);
    const T* p3 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p2) + v.syb);
    c[0] = vc_ldg(p0);
    c[1] = vc_ldg(p0 + 1);
    c[2] = vc_ldg(p1);
    c[3] = vc_ldg(p1 + 1);
    c[4] = vc_ldg(p2);
    c[5] = vc_ldg(p2 + 1);
    c[6] = vc_ldg(p3);
    c[7] = vc_ldg(p3 + 1);
    if (v.sx1 == 0u) {
        c[1] = c[0];
        c[3] = c[2];
        c[5] = c[4];
        c[7] = c[6];
    }
}

template <typename T>
__device__ __forceinline__ T ldv(const T* p) { return vc_ldg(p); }

// _kernels.py:40-42
template <typename T>
__device__ __forceinline__ double fetch(const Vol<T>& v, int i, int j, int k) {
    uint32_t idx = ((uint32_t)k * (uint32_t)v.ny + (uint32_t)j) * (uint32_t)v.nx + (uint32_t)i;
    return (double)ldv(v.data + idx);
}

// _kernels.py:45-49
__device__ __forceinline__ double round_half_away(double x) {
    if (x >= 0.0) return floor(dadd(x, 0.5));
    return ceil(dsub(x, 0.5));
}

// ---- conversion-free integer <-> float64 helpers ---------------------------
// On sm_100 the float64 conversions (I2F.F64, F2I.F64.FLOOR, F2F.F64.F32)
// issue on the narrow XU pipe, which the first profile showed saturated
// (profiles/r01_*).  These replacements run on the FP64 / integer pipes and
// are exact: 2^52 + v is representable for every 0 <= v < 2^32.
constexpr double TWO52 = 0x1p52;
constexpr double TWO52_31 = 0x1.000008p52;  // 2^52 + 2^31

// exact double of an unsigned 32-bit integer
__device__ __forceinline__ double u2d(uint32_t v) { return __dsub_rn(__hiloint2double(0x43300000, (int)v), TWO52); }
// exact double of a signed integer d, given biased = d + 2^31 (mod 2^32)
__device__ __forceinline__ double biased2d(uint32_t biased) {
    return __dsub_rn(__hiloint2double(0x43300000, (int)biased), TWO52_31);
}

// floor(x) for |x| < 2^31: returns the integer, r = (double)floor(x).
// (VC_FLOOR_MAGIC variant: x + 1.5*2^52 lies in [2^52, 2^53) where the ulp
// is 1, so the sum is x rounded to the nearest integer and its low word is
// that integer.)
constexpr double MAGIC_RND = 0x1.8p52;
__device__ __forceinline__ int floor_pos(double x, double& r) {
#ifndef VC_FLOOR_MAGIC
    // one XU op + one DADD beat the 5-op magic-number floor here (measured
    // +4% frame rate); XU stays far from saturation since voxel and index
    // conversions no longer use it
    const int i = __double2int_rd(x);                    // F2I.F64.FLOOR
    r = biased2d((uint32_t)i + 0x80000000u);             // exact (double)i on the FP64 pipe
    return i;
#else
    const double t = __dadd_rn(x, MAGIC_RND);
    int i = __double2loint(t);
    r = __dsub_rn(t, MAGIC_RND);
    if (r > x) {
        r = __dsub_rn(r, 1.0);
        i -= 1;
    }
    return i;
#endif
}

// _kernels.py:52-64 for an in-range coordinate 0 <= v <= n-1: lower cell
// corner clamped to n-2 (and to 0 when n == 1), fraction f = v - i0.
// nm2 = (double)max(n-2, 0).
__device__ __forceinline__ int cell(double v, int n, double nm2, double& f) {
    double r;
    int i0 = floor_pos(v, r);
    if (i0 > n - 2) {
        i0 = n - 2 < 0 ? 0 : n - 2;
        r = nm2;
    }
    f = dsub(v, r);
    return i0;
}
__device__ __forceinline__ int cell_hi(int i0, int n) {
    int i1 = i0 + 1;
    return i1 > n - 1 ? n - 1 : i1;
}

template <typename T>
struct VoxelBits;  // raw voxel -> exact double, and lerp over a voxel pair
template <>
struct VoxelBits<uint8_t> {
    static constexpr bool integral = true;
};
template <>
struct VoxelBits<uint16_t> {
    static constexpr bool integral = true;
};
template <>
struct VoxelBits<float> {
    static constexpr bool integral = false;
};

// lerp(c0, c1, t) = c0 + (c1 - c0) * t over two voxel values, bit-identical
// to the reference's float64 expression (c1 - c0 is exact for integer data).
template <typename T>
__device__ __forceinline__ double lerp_vox(wide_t<T> c0, wide_t<T> c1, double t) {
    if constexpr (VoxelBits<T>::integral) {
        const double f0 = u2d((uint32_t)c0);
        const double d = biased2d((uint32_t)c1 - (uint32_t)c0 + 0x80000000u);
        return dadd(f0, dmul(d, t));
    } else {
        return lerp((double)c0, (double)c1, t);
    }
}

// _kernels.py:104-115 for an in-range position (sample_any checked it).
// All eight gathers are issued before any arithmetic (memory-level
// parallelism); offsets are 32-bit from the cell's base corner.
template <typename T>
__device__ __forceinline__ double sample_trilinear(const Vol<T>& v, double x, double y, double z) {
    double fx, fy, fz;
    const int i0 = cell(x, v.nx, v.cx, fx), i1 = cell_hi(i0, v.nx);
    const int j0 = cell(y, v.ny, v.cy, fy), j1 = cell_hi(j0, v.ny);
    const int k0 = cell(z, v.nz, v.cz, fz), k1 = cell_hi(k0, v.nz);
    const uint32_t sx = (uint32_t)(i1 - i0);
    const uint32_t sy = (uint32_t)(j1 - j0) * (uint32_t)v.nx;
    const uint32_t sz = (uint32_t)(k1 - k0) * (uint32_t)v.nx * (uint32_t)v.ny;
    const T* b = v.data + (((uint32_t)k0 * (uint32_t)v.ny + (uint32_t)j0) * (uint32_t)v.nx + (uint32_t)i0);
    const T c000 = ldv(b), c100 = ldv(b + sx), c010 = ldv(b + sy), c110 = ldv(b + sy + sx);
    const T c001 = ldv(b + sz), c101 = ldv(b + sz + sx), c011 = ldv(b + sz + sy),
            c111 = ldv(b + sz + sy + sx);
    const double x00 = lerp_vox<T>(c000, c100, fx);
    const double x10 = lerp_vox<T>(c010, c110, fx);
    const double x01 = lerp_vox<T>(c001, c101, fx);
    const double x11 = lerp_vox<T>(c011, c111, fx);
    const double y0 = lerp(x00, x10, fy);
    const double y1 = lerp(x01, x11, fy);
    return lerp(y0, y1, fz);
}

// Cell location of a position, computed once and shared by the range
// check, the macrocell lookup and the trilinear gather.  Valid for
// |coordinate| < 2^31 (ray positions stay within the volume box).
struct Loc {
    int i, j, k;        // lower cell corner, clamped like _kernels.py:52-64
    double fx, fy, fz;  // fractions v - i0
};

// n1 = n-1, kmax = max(n-2, 0), nm1 = (double)(n-1).  L (i0, f) is only
// meaningful when the result is true.
__device__ __forceinline__ bool locate_axis(double x, int n1, int kmax, double nm1, int& i0, double& f) {
    int i = __double2int_rd(x);  // F2I.F64.FLOOR, exact for negative x too
    // in range  <=>  0 <= x <= n-1  <=>  0 <= i < n-1, or x == n-1
    const bool inr = (uint32_t)i < (uint32_t)n1 || x == nm1;
    i = min(i, kmax);            // the clamp of _kernels.py:53-64 (x == n-1)
    i0 = i;
    f = dsub(x, biased2d((uint32_t)i + 0x80000000u));
    return inr;
}

template <typename T>
__device__ __forceinline__ bool locate(const Vol<T>& v, const double p[3], Loc& L) {
    const bool a = locate_axis(p[0], v.nx - 1, v.kx, v.mx, L.i, L.fx);
    const bool b = locate_axis(p[1], v.ny - 1, v.ky, v.my, L.j, L.fy);
    const bool c = locate_axis(p[2], v.nz - 1, v.kz, v.mz, L.k, L.fz);
    return a && b && c;
}

// sample_trilinear (_kernels.py:104-115) from a precomputed in-range Loc
template <typename T>
__device__ __forceinline__ double trilinear_at(const Vol<T>& v, const Loc& L) {
    wide_t<T> c[8];  // L is clamped: i+1 < n unless n == 1
    gather8(v, L.i, L.j, L.k, c);
    const wide_t<T> c000 = c[0], c100 = c[1], c010 = c[2], c110 = c[3], c001 = c[4], c101 = c[5], c011 = c[6],
                    c111 = c[7];
    const double x00 = lerp_vox<T>(c000, c100, L.fx);
    const double x10 = lerp_vox<T>(c010, c110, L.fx);
    const double x01 = lerp_vox<T>(c001, c101, L.fx);
    const double x11 = lerp_vox<T>(c011, c111, L.fx);
    const double y0 = lerp(x00, x10, L.fy);
    const double y1 = lerp(x01, x11, L.fy);
    return lerp(y0, y1, L.fz);
}

// ---- in-window test with a float32 pre-test -------------------------------
// March, fine-scan, bisection and composite-march samples are only ever
// compared with the threshold window.  The trilinear value is first formed
// in float32 from the same eight voxels and the float64 fractions; its
// error is below E = amax * 2^-16 (corners exact in float32, each of the
// three lerp levels adds at most a few ulp of amax -- about 34 * 2^-24 *
// amax in total, so E has a 4x margin).  Only a value within E of a
// threshold is re-evaluated with the reference's float64 cascade, so every
// decision equals the reference's.
struct WinF {
    float lo_out, lo_in, hi_in, hi_out;  // v < lo_out or > hi_out: out; lo_in <= v <= hi_in: in
};

__host__ __device__ inline double prefilter_error(double amax) { return amax > 0.0 ? amax * 0x1p-16 + 1e-30 : 1e300; }

__device__ __forceinline__ WinF make_winf(double t_low, double t_high, double amax) {
    const double e = prefilter_error(amax);
    WinF w;
    if (e > 1e200) {  // unknown range: always take the exact path
        w.lo_out = -INFINITY;
        w.hi_out = INFINITY;
        w.lo_in = INFINITY;
        w.hi_in = -INFINITY;
        return w;
    }
    w.lo_out = __double2float_rd(t_low - e);
    w.lo_in = __double2float_ru(t_low + e);
    w.hi_in = __double2float_rd(t_high - e);
    w.hi_out = __double2float_ru(t_high + e);
    return w;
}

template <typename T>
__device__ __forceinline__ float vox_f32(wide_t<T> c) {
    if constexpr (VoxelBits<T>::integral) return __int_as_float(0x4B000000 | (int)c) - 8388608.0f;
    else return (float)c;
}

template <typename T>
__device__ __forceinline__ bool in_window_corners(const wide_t<T> c[8], const Loc& L, double t_low, double t_high,
                                                  const WinF& w) {
    const wide_t<T> c000 = c[0], c100 = c[1], c010 = c[2], c110 = c[3], c001 = c[4], c101 = c[5], c011 = c[6],
                    c111 = c[7];
    const float fx = __double2float_rn(L.fx), fy = __double2float_rn(L.fy), fz = __double2float_rn(L.fz);
    auto l32 = [](float a, float bb, float t) { return __fmaf_rn(bb - a, t, a); };
    const float y0 = l32(l32(vox_f32<T>(c000), vox_f32<T>(c100), fx), l32(vox_f32<T>(c010), vox_f32<T>(c110), fx), fy);
    const float y1 = l32(l32(vox_f32<T>(c001), vox_f32<T>(c101), fx), l32(vox_f32<T>(c011), vox_f32<T>(c111), fx), fy);
    const float v32 = l32(y0, y1, fz);
    if (v32 < w.lo_out || v32 > w.hi_out) return false;
    if (v32 >= w.lo_in && v32 <= w.hi_in) return true;
    // ambiguous: the reference's float64 cascade on the same corners
    const double x00 = lerp_vox<T>(c000, c100, L.fx);
    const double x10 = lerp_vox<T>(c010, c110, L.fx);
    const double x01 = lerp_vox<T>(c001, c101, L.fx);
    const double x11 = lerp_vox<T>(c011, c111, L.fx);
    const double val = lerp(lerp(x00, x10, L.fy), lerp(x01, x11, L.fy), L.fz);
    return t_low <= val && val <= t_high;
}

// the float32 pre-test alone, from float32 fractions: 0 out, 1 in, -1
// ambiguous (the caller re-evaluates with the reference's float64 cascade)
template <typename T>
__device__ __forceinline__ int window_corners_f(const wide_t<T> c[8], float fx, float fy, float fz, const WinF& w) {
    auto l32 = [](float a, float bb, float t) { return __fmaf_rn(bb - a, t, a); };
    const float y0 = l32(l32(vox_f32<T>(c[0]), vox_f32<T>(c[1]), fx), l32(vox_f32<T>(c[2]), vox_f32<T>(c[3]), fx), fy);
    const float y1 = l32(l32(vox_f32<T>(c[4]), vox_f32<T>(c[5]), fx), l32(vox_f32<T>(c[6]), vox_f32<T>(c[7]), fx), fy);
    const float v32 = l32(y0, y1, fz);
    if (v32 < w.lo_out || v32 > w.hi_out) return 0;
    if (v32 >= w.lo_in && v32 <= w.hi_in) return 1;
    return -1;
}

// window_corners_f of interior cell (i, j, k): i < nx-1, j < ny-1, k < nz-1
// (no one-voxel-axis case).  Integer voxels: the x-lerp's left value and
// the pair difference each come from one integer op + one FADD (magic
// 2^23 / 1.5 * 2^23 biases, exact for |value| < 2^22).
template <typename T>
__device__ __forceinline__ int window_cell_f(const Vol<T>& v, int i, int j, int k, float fx, float fy, float fz,
                                             const WinF& w) {
    const uint32_t idx = ((uint32_t)k * (uint32_t)v.ny + (uint32_t)j) * (uint32_t)v.nx + (uint32_t)i;
    const T* p0 = v.data + idx;
    const T* p1 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p0) + v.syb);
    const T* p2 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p0) + v.szb);
    const T* p3 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p2) + v.syb);
    const wide_t<T> c0 = vc_ldg(p0), c1 = vc_ldg(p0 + 1), c2 = vc_ldg(p1), c3 = vc_ldg(p1 + 1);
    const wide_t<T> c4 = vc_ldg(p2), c5 = vc_ldg(p2 + 1), c6 = vc_ldg(p3), c7 = vc_ldg(p3 + 1);
    float x0, x1, x2, x3;
    if constexpr (VoxelBits<T>::integral) {
        auto left = [](wide_t<T> a) { return __fsub_rn(__int_as_float(0x4B000000 + (int)a), 8388608.0f); };
        auto diff = [](wide_t<T> a, wide_t<T> b) {
            return __fsub_rn(__int_as_float((int)b - (int)a + 0x4B400000), 12582912.0f);
        };
        x0 = __fmaf_rn(diff(c0, c1), fx, left(c0));
        x1 = __fmaf_rn(diff(c2, c3), fx, left(c2));
        x2 = __fmaf_rn(diff(c4, c5), fx, left(c4));
        x3 = __fmaf_rn(diff(c6, c7), fx, left(c6));
    } else {
        auto l32 = [](float a, float bb, float t) { return __fmaf_rn(bb - a, t, a); };
        x0 = l32(c0, c1, fx);
        x1 = l32(c2, c3, fx);
        x2 = l32(c4, c5, fx);
        x3 = l32(c6, c7, fx);
    }
    const float y0 = __fmaf_rn(x1 - x0, fy, x0);
    const float y1 = __fmaf_rn(x3 - x2, fy, x2);
    const float v32 = __fmaf_rn(y1 - y0, fz, y0);
    if (v32 < w.lo_out || v32 > w.hi_out) return 0;
    if (v32 >= w.lo_in && v32 <= w.hi_in) return 1;
    return -1;
}

// window_cell_f with the cell's x-lerp operands cached across calls
// (bisection: successive positions almost always share the cell)
struct CellCache {
    int i, j, k;
    float l[4], d[4];  // x-lerp left value and pair difference, four x-edges
};

template <typename T>
__device__ __forceinline__ int window_cell_cached(const Vol<T>& v, int i, int j, int k, float fx, float fy, float fz,
                                                  const WinF& w, CellCache& cc) {
    if (i != cc.i || j != cc.j || k != cc.k) {
        const uint32_t idx = ((uint32_t)k * (uint32_t)v.ny + (uint32_t)j) * (uint32_t)v.nx + (uint32_t)i;
        const T* p0 = v.data + idx;
        const T* p1 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p0) + v.syb);
        const T* p2 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p0) + v.szb);
        const T* p3 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(p2) + v.syb);
        const T* row[4] = {p0, p1, p2, p3};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const wide_t<T> a = vc_ldg(row[e]), b = vc_ldg(row[e] + 1);
            if constexpr (VoxelBits<T>::integral) {
                cc.l[e] = __fsub_rn(__int_as_float(0x4B000000 + (int)a), 8388608.0f);
                cc.d[e] = __fsub_rn(__int_as_float((int)b - (int)a + 0x4B400000), 12582912.0f);
            } else {
                cc.l[e] = a;
                cc.d[e] = b - a;
            }
        }
        cc.i = i;
        cc.j = j;
        cc.k = k;
    }
    const float x0 = __fmaf_rn(cc.d[0], fx, cc.l[0]), x1 = __fmaf_rn(cc.d[1], fx, cc.l[1]);
    const float x2 = __fmaf_rn(cc.d[2], fx, cc.l[2]), x3 = __fmaf_rn(cc.d[3], fx, cc.l[3]);
    const float y0 = __fmaf_rn(x1 - x0, fy, x0);
    const float y1 = __fmaf_rn(x3 - x2, fy, x2);
    const float v32 = __fmaf_rn(y1 - y0, fz, y0);
    if (v32 < w.lo_out || v32 > w.hi_out) return 0;
    if (v32 >= w.lo_in && v32 <= w.hi_in) return 1;
    return -1;
}

template <typename T>
__device__ __forceinline__ bool in_window_trilinear(const Vol<T>& v, const Loc& L, double t_low, double t_high,
                                                    const WinF& w) {
    wide_t<T> c[8];  // L is clamped: i+1 < n unless n == 1
    gather8(v, L.i, L.j, L.k, c);
    return in_window_corners<T>(c, L, t_low, t_high, w);
}

// _kernels.py:67-72
template <typename T>
__device__ __forceinline__ double sample_nearest(const Vol<T>& v, double x, double y, double z) {
    return fetch(v, (int)round_half_away(x), (int)round_half_away(y), (int)round_half_away(z));
}

// _kernels.py:75-101
template <typename T>
__device__ double sample_linear(const Vol<T>& v, double x, double y, double z) {
    const double fx = fabs(dsub(x, round_half_away(x)));
    const double fy = fabs(dsub(y, round_half_away(y)));
    const double fz = fabs(dsub(z, round_half_away(z)));
    int axis;
    if (fy > fx && fy >= fz) axis = 1;
    else if (fz > fx && fz > fy) axis = 2;
    else axis = 0;
    double f;
    if (axis == 0) {
        const int j = (int)round_half_away(y), k = (int)round_half_away(z);
        const int a0 = cell(x, v.nx, v.cx, f), a1 = cell_hi(a0, v.nx);
        return lerp(fetch(v, a0, j, k), fetch(v, a1, j, k), f);
    }
    if (axis == 1) {
        const int i = (int)round_half_away(x), k = (int)round_half_away(z);
        const int a0 = cell(y, v.ny, v.cy, f), a1 = cell_hi(a0, v.ny);
        return lerp(fetch(v, i, a0, k), fetch(v, i, a1, k), f);
    }
    const int i = (int)round_half_away(x), j = (int)round_half_away(y);
    const int a0 = cell(z, v.nz, v.cz, f), a1 = cell_hi(a0, v.nz);
    return lerp(fetch(v, i, j, a0), fetch(v, i, j, a1), f);
}

template <typename T>
__device__ __forceinline__ bool in_range(const Vol<T>& v, double x, double y, double z) {
    return !(x < 0.0 || x > v.mx || y < 0.0 || y > v.my || z < 0.0 || z > v.mz);
}

// _kernels.py:118-127
template <typename T, int INTERP>
__device__ __forceinline__ double sample_any(const Vol<T>& v, double x, double y, double z) {
    if (!in_range(v, x, y, z)) return 0.0;
    if (INTERP == VC_TRILINEAR) return sample_trilinear(v, x, y, z);
    if (INTERP == VC_LINEAR) return sample_linear(v, x, y, z);
    return sample_nearest(v, x, y, z);
}

template <typename T>
__device__ __forceinline__ double tap(const Vol<T>& v, double x, double y, double z) {
    return sample_any<T, VC_TRILINEAR>(v, x, y, z);
}

// _kernels.py:130-137
__host__ __device__ constexpr double smooth_weight(int u, int w) {
    return (u == 0 && w == 0) ? 6.0 : ((u == 0 || w == 0) ? 3.0 : 1.0);
}
__host__ __device__ constexpr double zh_inv(int i, int j, int k) {
    return (i * i + j * j + k * k) == 1 ? 1.0 : ((i * i + j * j + k * k) == 2 ? INV_SQRT2 : INV_SQRT3);
}

// _kernels.py:140-177 -- taps always trilinear, i->j->k accumulation order.
// Terms whose weight is 0 add +0.0 to a sum that can never be -0.0 (it
// starts at +0.0 and round-to-nearest never produces -0.0 from a sum
// of non-(-0.0) operands), so they are dropped without changing a bit.
// ROLL: the 26-tap loop is not unrolled.  This general path serves the
// shading samples of the boundary band, where the shared footprint does not
// apply; unrolled, its 26 inlined trilinear taps are ~4k instructions, and
// where the band is frequent (noise / Marschner-Lobb faces, C4) they evicted
// the march and shade loop from the instruction cache (50% of the C4 shade
// stage's stalls "no instruction"; rolled: 4.48 -> 3.26 ms).  Where the band
// is rare and the kernel tight on registers (C3's gradient-volume kernel)
// the unrolled form keeps fewer spills.
template <typename T, int OP>
__device__ __forceinline__ void grad_tap_term(const Vol<T>& v, double x, double y, double z, int i, int j, int k,
                                              double& gx, double& gy, double& gz) {
    const double s = tap(v, dadd(x, (double)i), dadd(y, (double)j), dadd(z, (double)k));
    double wx, wy, wz;
    if (OP == VC_OP_SOBEL3D) {
        wx = (double)i * smooth_weight(j, k);
        wy = (double)j * smooth_weight(i, k);
        wz = (double)k * smooth_weight(i, j);
    } else {
        const double inv = zh_inv(i, j, k);
        wx = (double)i * inv;
        wy = (double)j * inv;
        wz = (double)k * inv;
    }
    if (i != 0) gx = dadd(gx, dmul(wx, s));
    if (j != 0) gy = dadd(gy, dmul(wy, s));
    if (k != 0) gz = dadd(gz, dmul(wz, s));
}

template <typename T, int OP, bool ROLL = false>
__device__ __forceinline__ void grad_raw(const Vol<T>& v, double x, double y, double z, double g[3]) {
    if (OP == VC_OP_CENTRAL) {
        g[0] = dsub(tap(v, dadd(x, 1.0), y, z), tap(v, dsub(x, 1.0), y, z));
        g[1] = dsub(tap(v, x, dadd(y, 1.0), z), tap(v, x, dsub(y, 1.0), z));
        g[2] = dsub(tap(v, x, y, dadd(z, 1.0)), tap(v, x, y, dsub(z, 1.0)));
        return;
    }
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if constexpr (ROLL) {
#pragma unroll 1
        for (int i = -1; i < 2; i++)
#pragma unroll 1
            for (int j = -1; j < 2; j++)
#pragma unroll 1
                for (int k = -1; k < 2; k++)
                    if (!(i == 0 && j == 0 && k == 0)) grad_tap_term<T, OP>(v, x, y, z, i, j, k, gx, gy, gz);
    } else {
#pragma unroll
        for (int i = -1; i < 2; i++)
#pragma unroll
            for (int j = -1; j < 2; j++)
#pragma unroll
                for (int k = -1; k < 2; k++)
                    if (!(i == 0 && j == 0 && k == 0)) grad_tap_term<T, OP>(v, x, y, z, i, j, k, gx, gy, gz);
    }
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
}

// grad_raw for the common interior case, sharing one 4x4x4 voxel footprint
// between the 26 (6) taps.  When every tap coordinate x+i is exact -- x >= 1,
// x+1 < n-1 and x+1 does not cross a binade with rounding -- all taps have
// the fractions of x and cells shifted by i, none is clamped and all are in
// range, so each tap's x-lerps are the shared X[j][k] below, its y-lerps the
// shared Y, its z-lerp Z: the same float64 operations on the same operands
// as grad_raw / sample_trilinear, accumulated in the same i->j->k order, so
// the result is bit-identical (3.5x fewer loads and FP64 ops).  `center`
// receives sample_trilinear(x, y, z).  Returns false when the fast path does
// not apply (the caller then uses grad_raw).
template <typename T, int OP>
__device__ __forceinline__ bool grad_raw_shared(const Vol<T>& v, double x, double y, double z, double g[3],
                                                double& center) {
    const double xp = dadd(x, 1.0), yp = dadd(y, 1.0), zp = dadd(z, 1.0);
    if (!(x >= 1.0 && xp < v.mx && dsub(xp, x) == 1.0 && y >= 1.0 && yp < v.my && dsub(yp, y) == 1.0 &&
          z >= 1.0 && zp < v.mz && dsub(zp, z) == 1.0))
        return false;
    double r;
    const int i0 = floor_pos(x, r);
    const double fx = dsub(x, r);
    const int j0 = floor_pos(y, r);
    const double fy = dsub(y, r);
    const int k0 = floor_pos(z, r);
    const double fz = dsub(z, r);
    const uint32_t sy = (uint32_t)v.nx, sz = (uint32_t)v.nx * (uint32_t)v.ny;
    // corner (i0-1, j0-1, k0-1) of the footprint
    const T* b = v.data + (((uint32_t)(k0 - 1) * (uint32_t)v.ny + (uint32_t)(j0 - 1)) * (uint32_t)v.nx +
                           (uint32_t)(i0 - 1));
    if (OP == VC_OP_CENTRAL) {
        // tap at cell offset (di, dj, dk): trilinear over footprint cell (1+di, 1+dj, 1+dk)
        auto tri = [&](int di, int dj, int dk) {
            const T* c = b + (uint32_t)(1 + dk) * sz + (uint32_t)(1 + dj) * sy + (uint32_t)(1 + di);
            const double x00 = lerp_vox<T>(ldv(c), ldv(c + 1), fx);
            const double x10 = lerp_vox<T>(ldv(c + sy), ldv(c + sy + 1), fx);
            const double x01 = lerp_vox<T>(ldv(c + sz), ldv(c + sz + 1), fx);
            const double x11 = lerp_vox<T>(ldv(c + sz + sy), ldv(c + sz + sy + 1), fx);
            return lerp(lerp(x00, x10, fy), lerp(x01, x11, fy), fz);
        };
        g[0] = dsub(tri(1, 0, 0), tri(-1, 0, 0));
        g[1] = dsub(tri(0, 1, 0), tri(0, -1, 0));
        g[2] = dsub(tri(0, 0, 1), tri(0, 0, -1));
        center = tri(0, 0, 0);
        return true;
    }
    double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
    for (int i = -1; i < 2; i++) {
        double X[4][4];  // [row j0-1+jj][slice k0-1+kk], x-lerp over cells i0+i, i0+i+1
#pragma unroll
        for (int kk = 0; kk < 4; kk++)
#pragma unroll
            for (int jj = 0; jj < 4; jj++) {
                const T* c = b + (uint32_t)kk * sz + (uint32_t)jj * sy + (uint32_t)(i + 1);
                X[jj][kk] = lerp_vox<T>(ldv(c), ldv(c + 1), fx);
            }
        double Y[3][4];  // tap row j: lerp(X[j+1], X[j+2], fy)
#pragma unroll
        for (int j = 0; j < 3; j++)
#pragma unroll
            for (int kk = 0; kk < 4; kk++) Y[j][kk] = lerp(X[j][kk], X[j + 1][kk], fy);
#pragma unroll
        for (int j = -1; j < 2; j++) {
#pragma unroll
            for (int k = -1; k < 2; k++) {
                const double s = lerp(Y[j + 1][k + 1], Y[j + 1][k + 2], fz);
                if (i == 0 && j == 0 && k == 0) {
                    center = s;
                    continue;
                }
                double wx, wy, wz;
                if (OP == VC_OP_SOBEL3D) {
                    wx = (double)i * smooth_weight(j, k);
                    wy = (double)j * smooth_weight(i, k);
                    wz = (double)k * smooth_weight(i, j);
                } else {
                    const double inv = zh_inv(i, j, k);
                    wx = (double)i * inv;
                    wy = (double)j * inv;
                    wz = (double)k * inv;
                }
                if (i != 0) gx = dadd(gx, dmul(wx, s));
                if (j != 0) gy = dadd(gy, dmul(wy, s));
                if (k != 0) gz = dadd(gz, dmul(wz, s));
            }
        }
    }
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
    return true;
}

// _kernels.py:180-185
__device__ __forceinline__ void normalize3(const double g[3], double u[3]) {
    const double s = dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2]));
    // zero gradients (flat regions, frequent) would take the slow sqrt path;
    // sqrt(0) = 0 <= eps gives the zero vector either way
    const double n = s == 0.0 ? 0.0 : __dsqrt_rn(s);
    if (n <= GRAD_EPS) {
        u[0] = u[1] = u[2] = 0.0;
        return;
    }
    const double y = rcp_for(n);
    u[0] = div_rcp(g[0], n, y);
    u[1] = div_rcp(g[1], n, y);
    u[2] = div_rcp(g[2], n, y);
}

// _kernels.py:188-224 (slab_interval + box_interval)
// inv_out (optional): RN(1 / d) per axis, 0 for d == 0 (valid when true is returned)
__device__ __forceinline__ bool box_interval(const double o[3], const double d[3], const double lo[3],
                                             const double hi[3], double& t0, double& t1,
                                             double* inv_out = nullptr) {
    double tmin = -1e300, tmax = 1e300;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (inv_out) inv_out[a] = 0.0;
        if (d[a] == 0.0) {
            if (o[a] < lo[a] || o[a] > hi[a]) return false;
        } else {
            const double inv = __drcp_rn(d[a]);  // = RN(1.0 / d), the reference's value
            if (inv_out) inv_out[a] = inv;
            double ta = dmul(dsub(lo[a], o[a]), inv);
            double tb = dmul(dsub(hi[a], o[a]), inv);
            if (ta > tb) {
                const double s = ta;
                ta = tb;
                tb = s;
            }
            if (ta > tmin) tmin = ta;
            if (tb < tmax) tmax = tb;
        }
    }
    if (tmin > tmax) return false;
    if (tmax < 0.0) return false;
    t0 = tmin < 0.0 ? 0.0 : tmin;
    t1 = tmax;
    return true;
}

// Ray-to-voxel-space position, _kernels.py:414-416: (o + t*d)/s - 0.5.
// When every spacing is a power of two the division is exact as a
// multiply by the (exact) reciprocal, so UNIT/POW2 spacing takes the fast
// form without changing a bit.
// Other spacings divide through the correctly rounded reciprocal rs
// (ddiv_rcp, exact).
struct RayPos {
    double o[3], d[3], s[3], rs[3];
    bool pow2;
    bool rcp;  // every rs[a] usable by ddiv_rcp (host: make_raypos)
    __device__ __forceinline__ double vox(double w, int a) const {
        return pow2 ? dmul(w, rs[a]) : (rcp ? ddiv_rcp(w, s[a], rs[a]) : ddiv_cold(w, s[a]));
    }
    __device__ __forceinline__ void at(double t, double p[3]) const {
#pragma unroll
        for (int a = 0; a < 3; a++) p[a] = dsub(vox(dadd(o[a], dmul(t, d[a])), a), 0.5);
    }
};

// _kernels.py:514-525
__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
__device__ __forceinline__ uint8_t quant(double v) {
    return (uint8_t)(int)dadd(dmul(clamp01(v), 255.0), 0.5);
}

// _kernels.py:490-511; breakpoints read from the kernel-parameter bank
__device__ __forceinline__ void lut_eval(const vc_render_params& P, double hu, double out[4]) {
    const int n = P.lut_n;
    if (hu <= P.lut_hu[0]) {
#pragma unroll
        for (int c = 0; c < 4; c++) out[c] = P.lut_rgba[0][c];
        return;
    }
    if (hu >= P.lut_hu[n - 1]) {
#pragma unroll
        for (int c = 0; c < 4; c++) out[c] = P.lut_rgba[n - 1][c];
        return;
    }
    int i = 0;
    while (i + 1 < n - 1 && P.lut_hu[i + 1] <= hu) i++;
    const double t = ddiv(dsub(hu, P.lut_hu[i]), dsub(P.lut_hu[i + 1], P.lut_hu[i]));
#pragma unroll
    for (int c = 0; c < 4; c++) out[c] = lerp(P.lut_rgba[i][c], P.lut_rgba[i + 1][c], t);
}

// The same evaluation over a shared-memory copy of the breakpoints: lanes
// of a warp sit in different LUT segments, and divergent indices into the
// constant bank serialise, shared memory does not.
struct SharedLut {
    double hu[VC_MAX_LUT];
    double rgba[VC_MAX_LUT][4];
    double rw[VC_MAX_LUT];  // rcp_for(hu[i+1] - hu[i]) for the segment division
    int n;
};

__device__ __forceinline__ void lut_eval(const SharedLut& L, double hu, double out[4]) {
    const int n = L.n;
    int i;
    if (hu <= L.hu[0]) {
        i = 0;
    } else if (hu >= L.hu[n - 1]) {
        i = n - 1;
    } else {
        i = -1;
    }
    if (i >= 0) {
#pragma unroll
        for (int c = 0; c < 4; c++) out[c] = L.rgba[i][c];
        return;
    }
    i = 0;
    while (i + 1 < n - 1 && L.hu[i + 1] <= hu) i++;
    const double t = div_rcp(dsub(hu, L.hu[i]), dsub(L.hu[i + 1], L.hu[i]), L.rw[i]);
#pragma unroll
    for (int c = 0; c < 4; c++) out[c] = lerp(L.rgba[i][c], L.rgba[i + 1][c], t);
}

__device__ __forceinline__ void load_shared_lut(const vc_render_params& P, SharedLut& L) {
    for (int k = threadIdx.x; k < P.lut_n; k += blockDim.x) {
        L.hu[k] = P.lut_hu[k];
#pragma unroll
        for (int c = 0; c < 4; c++) L.rgba[k][c] = P.lut_rgba[k][c];
        L.rw[k] = k + 1 < P.lut_n ? rcp_for(dsub(P.lut_hu[k + 1], P.lut_hu[k])) : 0.0;
    }
    if (threadIdx.x == 0) L.n = P.lut_n;
    __syncthreads();
}

}  // namespace vc
