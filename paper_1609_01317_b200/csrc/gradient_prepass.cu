// gradient_prepass.cu -- Kernel 1: lattice gradient volume, packed float4.
//
// Output voxel (i,j,k) = (gx, gy, gz, value) where g is the reference's
// raw gradient grad_raw evaluated at the integer point (i,j,k)
// (/root/reference/pkg/src/voxelcast/_kernels.py:140-177).  At lattice
// points every trilinear tap returns a voxel value exactly and
// out-of-range taps read 0 (_kernels.py:52-64, :118-127), so the operator
// is a zero-padded 3x3x3 stencil:
//   CentralDifference  gx = v(x+1) - v(x-1)                       (:146-155)
//   Sobel3D            gx = sum_i,j,k  i * w(j,k) * v,  w = [[1,3,1],[3,6,3],[1,3,1]]  (:156-165)
//   Zucker-Hummel      gx = sum_i,j,k  i / |(i,j,k)| * v                                (:166-176)
//
// HBM-bound stencil: 2 B in (u16) + 16 B out per voxel.  Each CTA owns a
// 32x8 (x,y) column tile and a 16-plane z-chunk.  The chunk plus a 1-voxel
// halo is staged in shared memory in one go: by one TMA 3-D tile load
// (cp.async.bulk.tensor, the tensor map's out-of-bounds zero fill is the
// reference's zero padding at the faces, no address arithmetic in the
// threads) when the row pitch is a multiple of 16 bytes, else by coalesced
// per-thread loads; each thread then
// sweeps its column, reducing every plane to seven partial sums, and
// combines three planes in registers -- every input voxel is read from HBM
// once (plus the halo), every output float4 is written once with a
// streaming 16-byte store, a warp storing 512 contiguous bytes.
//
// Integer grids (u8/u16) accumulate in int32: CD and Sobel3D results are
// exact integers (|g| <= 44 * 65535 < 2^24), bit-identical to the
// reference.  Zucker-Hummel groups the integer taps by weight class
// (1, 1/sqrt2, 1/sqrt3) and combines the three class sums in float64;
// float32 grids accumulate in float64.  Both round to float32 on store
// (relative error <= 2^-24 vs the reference's float64 sum).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "vc_internal.h"

namespace vc {

constexpr int GX = 32, GY = 8, GZC = 16;

// Exact int -> float / double without the XU conversion pipe (profiled at
// 34% XU on the first version): |v| < 2^22 added into the mantissa of
// 1.5*2^23, and v + 2^31 into 2^52 (see vc_device.cuh).
__device__ __forceinline__ float i2f_exact(int v) { return __int_as_float(0x4B400000 + v) - 12582912.0f; }
template <typename A>
__device__ __forceinline__ float tof(A v) {
    if constexpr (sizeof(A) == 4) return i2f_exact(v);
    else return (float)v;
}
template <typename A>
__device__ __forceinline__ double tod(A v) {
    if constexpr (sizeof(A) == 4) return biased2d((uint32_t)v + 0x80000000u);
    else return v;
}

template <typename A>
struct Planar {  // per-plane partial sums at one (x, y)
    A d0x, d1x, d0y, d1y, e0, e1, e2;
};

// Tile layout.  Column lx of the staged tile holds x = x0 - tile_x0() + lx.
// The TMA box must start on a 16-byte boundary in x (an unaligned start
// faults on sm_100a -- tools/probe/tma_probe.cu), so the TMA tile starts 16
// bytes left of the CTA's first column and is 16-byte multiple wide; the
// per-thread staging keeps the plain one-voxel halo.
template <typename T, bool TMA>
constexpr int tile_x0() { return TMA ? (int)(16 / sizeof(T)) : 1; }
template <typename T, bool TMA>
constexpr int tile_w() {
    return TMA ? (tile_x0<T, TMA>() + GX + 1 + tile_x0<T, TMA>() - 1) / tile_x0<T, TMA>() * tile_x0<T, TMA>()
               : GX + 2;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <typename T, typename A, int OP, bool TMA>
__global__ void __launch_bounds__(GX* GY) gradient_prepass_kernel(const T* __restrict__ vol, int nx, int ny,
                                                                  int nz, float4* __restrict__ out,
                                                                  const __grid_constant__ CUtensorMap tmap) {
    // the whole (GZC+2) x (GY+2) x (GX+2) halo'd chunk is staged once
    constexpr int TW = tile_w<T, TMA>(), XO = tile_x0<T, TMA>(), TH = GY + 2, TD = GZC + 2;
    __shared__ __align__(128) T tile[TD][TH][TW];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * GX + tx;
    const int x0 = blockIdx.x * GX, y0 = blockIdx.y * GY;
    const int z0 = blockIdx.z * GZC, z1 = min(z0 + GZC, nz);
    const int x = x0 + tx, y = y0 + ty;
    const size_t plane = (size_t)nx * ny;

    if constexpr (TMA) {
        // one elected thread: tensor-map tile load at (x0-XO, y0-1, z0-1);
        // elements outside the volume arrive as zeros (out-of-bounds fill)
        __shared__ __align__(8) uint64_t bar;
        const uint32_t b = smem_u32(&bar);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                         "r"((uint32_t)sizeof(tile))
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];" ::"r"(smem_u32(&tile[0][0][0])),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0 - XO), "r"(y0 - 1), "r"(z0 - 1), "r"(b)
                : "memory");
        }
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(b)
            : "memory");
    } else {
        // every thread issues all of its global loads before the single
        // barrier, so the loads overlap instead of one plane's latency per step
        constexpr int TN = TW * TH * TD;
        constexpr int PER = (TN + GX * GY - 1) / (GX * GY);
        T vals[PER];
#pragma unroll
        for (int r = 0; r < PER; r++) {
            const int e = tid + r * GX * GY;
            T v = T(0);
            if (e < TN) {
                const int lz = e / (TW * TH), rem = e - lz * (TW * TH);
                const int ly = rem / TW, lx = rem - ly * TW;
                const int gx = x0 + lx - 1, gy = y0 + ly - 1, gz = z0 + lz - 1;
                if (gz >= 0 && gz < nz && gx >= 0 && gx < nx && gy >= 0 && gy < ny)
                    v = __ldg(vol + (size_t)gz * plane + (size_t)gy * nx + gx);
            }
            vals[r] = v;
        }
#pragma unroll
        for (int r = 0; r < PER; r++) {
            const int e = tid + r * GX * GY;
            if (e < TN) (&tile[0][0][0])[e] = vals[r];
        }
        __syncthreads();
    }
    if (x >= nx || y >= ny) return;

    Planar<A> pp{}, pc{}, pn{};
    const int cx = tx + XO, cy = ty + 1;
    auto plane_step = [&](int lz) {
        const T(*s)[TW] = tile[lz];
        const A vmm = (A)s[cy - 1][cx - 1], v0m = (A)s[cy - 1][cx], vpm = (A)s[cy - 1][cx + 1];
        const A vm0 = (A)s[cy][cx - 1], v00 = (A)s[cy][cx], vp0 = (A)s[cy][cx + 1];
        const A vmp = (A)s[cy + 1][cx - 1], v0p = (A)s[cy + 1][cx], vpp = (A)s[cy + 1][cx + 1];
        pn.d0x = vp0 - vm0;
        pn.d1x = (vpm - vmm) + (vpp - vmp);
        pn.d0y = v0p - v0m;
        pn.d1y = (vmp - vmm) + (vpp - vpm);
        pn.e0 = v00;
        pn.e1 = (vm0 + vp0) + (v0m + v0p);
        pn.e2 = (vmm + vpm) + (vmp + vpp);
        if (lz >= 2) {
            float4 o;
            if (OP == VC_OP_CENTRAL) {
                o.x = tof(pc.d0x);
                o.y = tof(pc.d0y);
                o.z = tof(pn.e0 - pp.e0);
            } else if (OP == VC_OP_SOBEL3D) {
                const A side_x = (A)3 * pp.d0x + pp.d1x + ((A)3 * pn.d0x + pn.d1x);
                const A side_y = (A)3 * pp.d0y + pp.d1y + ((A)3 * pn.d0y + pn.d1y);
                o.x = tof(side_x + ((A)6 * pc.d0x + (A)3 * pc.d1x));
                o.y = tof(side_y + ((A)6 * pc.d0y + (A)3 * pc.d1y));
                o.z = tof(((A)6 * pn.e0 + (A)3 * pn.e1 + pn.e2) - ((A)6 * pp.e0 + (A)3 * pp.e1 + pp.e2));
            } else {
                const A a1x = pc.d0x, a2x = pc.d1x + (pp.d0x + pn.d0x), a3x = pp.d1x + pn.d1x;
                const A a1y = pc.d0y, a2y = pc.d1y + (pp.d0y + pn.d0y), a3y = pp.d1y + pn.d1y;
                const A a1z = pn.e0 - pp.e0, a2z = pn.e1 - pp.e1, a3z = pn.e2 - pp.e2;
                o.x = (float)dadd(dadd(tod(a1x), dmul(tod(a2x), INV_SQRT2)), dmul(tod(a3x), INV_SQRT3));
                o.y = (float)dadd(dadd(tod(a1y), dmul(tod(a2y), INV_SQRT2)), dmul(tod(a3y), INV_SQRT3));
                o.z = (float)dadd(dadd(tod(a1z), dmul(tod(a2z), INV_SQRT2)), dmul(tod(a3z), INV_SQRT3));
            }
            o.w = tof(pc.e0);
            __stcs(out + (size_t)(z0 + lz - 2) * plane + (size_t)y * nx + x, o);
        }
        pp = pc;
        pc = pn;
    };
    if (z1 - z0 == GZC) {  // full chunk: unrolled sweep (independent planes overlap)
#pragma unroll
        for (int lz = 0; lz < GZC + 2; lz++) plane_step(lz);
    } else {
        for (int lz = 0; lz < z1 - z0 + 2; lz++) plane_step(lz);
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link); nullptr when unavailable
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <typename T>
static bool make_tile_map(const void* data, int nx, int ny, int nz, CUtensorMap* m) {
    auto enc = tensor_map_encoder();
    const size_t es = sizeof(T);
    if (!enc || ((size_t)nx * es) % 16 != 0 || (reinterpret_cast<uintptr_t>(data) & 15) != 0) return false;
    const CUtensorMapDataType dt = sizeof(T) == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[2] = {(cuuint64_t)nx * es, (cuuint64_t)nx * ny * es};
    const cuuint32_t box[3] = {(cuuint32_t)tile_w<T, true>(), (cuuint32_t)(GY + 2), (cuuint32_t)(GZC + 2)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, dt, 3, const_cast<void*>(data), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, typename A, int OP>
static void launch_op_pre(const T* v, int nx, int ny, int nz, float4* out, bool tma, const CUtensorMap& m,
                          dim3 grid, dim3 block, cudaStream_t s) {
    if (tma)
        gradient_prepass_kernel<T, A, OP, true><<<grid, block, 0, s>>>(v, nx, ny, nz, out, m);
    else
        gradient_prepass_kernel<T, A, OP, false><<<grid, block, 0, s>>>(v, nx, ny, nz, out, m);
}

template <typename T, typename A>
static cudaError_t launch_pre(const void* data, int nx, int ny, int nz, int op, float4* out,
                              cudaStream_t s) {
    const dim3 block(GX, GY);
    const dim3 grid((nx + GX - 1) / GX, (ny + GY - 1) / GY, (nz + GZC - 1) / GZC);
    const T* v = static_cast<const T*>(data);
    CUtensorMap m{};
    bool tma = make_tile_map<T>(data, nx, ny, nz, &m);
#ifdef VC_NO_TMA
    tma = false;
#endif
    switch (op) {
        case VC_OP_CENTRAL: launch_op_pre<T, A, VC_OP_CENTRAL>(v, nx, ny, nz, out, tma, m, grid, block, s); break;
        case VC_OP_SOBEL3D: launch_op_pre<T, A, VC_OP_SOBEL3D>(v, nx, ny, nz, out, tma, m, grid, block, s); break;
        default: launch_op_pre<T, A, VC_OP_ZUCKER_HUMMEL>(v, nx, ny, nz, out, tma, m, grid, block, s);
    }
    return cudaGetLastError();
}

cudaError_t launch_gradient_prepass(int dtype, const void* data, int nx, int ny, int nz, int op,
                                    float4* out, cudaStream_t s) {
    switch (dtype) {
        case VC_U8: return launch_pre<uint8_t, int>(data, nx, ny, nz, op, out, s);
        case VC_U16: return launch_pre<uint16_t, int>(data, nx, ny, nz, op, out, s);
        default: return launch_pre<float, double>(data, nx, ny, nz, op, out, s);
    }
}

}  // namespace vc
