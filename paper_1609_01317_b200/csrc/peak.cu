// peak.cu -- measured ceiling of the raycaster's unit of work.
//
// The march kernels are bound by L1-resident gathers and FP64/ALU issue,
// not by HBM.  This microbenchmark runs the exact per-sample code of the
// march (ray position in float64, cell location, 8-corner gather, float32
// pre-test with float64 fallback) on a 16^3 volume that stays in L1, with
// every lane busy and no divergence, and reports samples/s.  bench.py uses
// it as the "sample roofline" next to the HBM one.
#include "vc_internal.h"

namespace vc {

template <typename T>
__global__ void __launch_bounds__(128) sample_peak_kernel(Vol<T> v, RayPos rp, double t_low, double t_high,
                                                          int iters, unsigned long long* out) {
    const WinF w = make_winf(t_low, t_high, v.amax);
    // a per-thread ray through the small volume; samples wrap around its box
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
    const double fx = 0.37 + 0.001 * (double)(tid & 255), fy = 0.29 + 0.0013 * (double)((tid >> 8) & 127);
    rp.o[0] = 0.5 + 7.0 * fx;
    rp.o[1] = 0.5 + 7.0 * fy;
    rp.o[2] = 0.5;
    const double n = __dsqrt_rn(fx * fx + fy * fy + 1.0);
    rp.d[0] = fx / n;
    rp.d[1] = fy / n;
    rp.d[2] = 1.0 / n;
    unsigned hits = 0;
    double t = 0.0;
    for (int k = 0; k < iters; k++) {
        double p[3];
        rp.at(t, p);
        Loc L;
        if (locate(v, p, L) && in_window_trilinear(v, L, t_low, t_high, w)) hits++;
        t = dadd(t, 0.61);
        if (t > 12.0) t = dsub(t, 12.0);
    }
    hits = __reduce_add_sync(0xffffffffu, hits);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)hits);
}

// the same march through the texture unit (VC_SAMPLER_TEXTURE's sample)
__global__ void __launch_bounds__(128) sample_peak_tex_kernel(cudaTextureObject_t tex, float scale, float lo,
                                                              float hi, int iters, unsigned long long* out) {
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
    const double fx = 0.37 + 0.001 * (double)(tid & 255), fy = 0.29 + 0.0013 * (double)((tid >> 8) & 127);
    double o[3] = {0.5 + 7.0 * fx, 0.5 + 7.0 * fy, 0.5}, d[3];
    const double n = __dsqrt_rn(fx * fx + fy * fy + 1.0);
    d[0] = fx / n;
    d[1] = fy / n;
    d[2] = 1.0 / n;
    unsigned hits = 0;
    double t = 0.0;
    for (int k = 0; k < iters; k++) {
        double p[3];
#pragma unroll
        for (int a = 0; a < 3; a++) p[a] = dsub(dadd(o[a], dmul(t, d[a])), 0.5);
        const bool inr = p[0] >= 0.0 && p[0] <= 15.0 && p[1] >= 0.0 && p[1] <= 15.0 && p[2] >= 0.0 && p[2] <= 15.0;
        if (inr) {
            const float v = tex3D<float>(tex, __double2float_rn(p[0]) + 0.5f, __double2float_rn(p[1]) + 0.5f,
                                         __double2float_rn(p[2]) + 0.5f) * scale;
            if (v >= lo && v <= hi) hits++;
        }
        t = dadd(t, 0.61);
        if (t > 12.0) t = dsub(t, 12.0);
    }
    hits = __reduce_add_sync(0xffffffffu, hits);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)hits);
}

}  // namespace vc

extern "C" VC_API int vc_sample_peak_texture(int device, double* gsamples_per_s) {
    using namespace vc;
    if (!gsamples_per_s) return VC_ERR_INVALID;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const int n = 16;
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    unsigned long long* cnt = nullptr;
    int rc = VC_OK;
    cudaChannelFormatDesc desc = cudaCreateChannelDesc<unsigned short>();
    if (cudaMalloc3DArray(&arr, &desc, make_cudaExtent(n, n, n), 0) != cudaSuccess ||
        cudaMalloc(&cnt, sizeof(unsigned long long)) != cudaSuccess)
        rc = VC_ERR_CUDA;
    if (rc == VC_OK) {
        uint16_t h[16 * 16 * 16];
        for (int i = 0; i < n * n * n; i++) h[i] = (uint16_t)((i * 2654435761u >> 20) & 4095);
        cudaMemcpy3DParms cp{};
        cp.srcPtr = make_cudaPitchedPtr(h, n * sizeof(uint16_t), n, n);
        cp.dstArray = arr;
        cp.extent = make_cudaExtent(n, n, n);
        cp.kind = cudaMemcpyHostToDevice;
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = arr;
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModeLinear;
        td.readMode = cudaReadModeNormalizedFloat;
        if (cudaMemcpy3D(&cp) != cudaSuccess || cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess)
            rc = VC_ERR_CUDA;
    }
    if (rc == VC_OK) {
        cudaMemset(cnt, 0, sizeof(unsigned long long));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sample_peak_tex_kernel, 128, 0);
        const int blocks = sms * per_sm, iters = 4096;
        sample_peak_tex_kernel<<<blocks, 128>>>(tex, 65535.0f, 500.0f, 3000.0f, 256, cnt);  // warm-up
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        sample_peak_tex_kernel<<<blocks, 128>>>(tex, 65535.0f, 500.0f, 3000.0f, iters, cnt);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) rc = VC_ERR_CUDA;
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        *gsamples_per_s = (double)blocks * 128.0 * iters / (ms * 1e-3) / 1e9;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    if (tex) cudaDestroyTextureObject(tex);
    if (arr) cudaFreeArray(arr);
    cudaFree(cnt);
    cudaSetDevice(prev);
    return rc;
}

extern "C" VC_API int vc_sample_peak(int device, double* gsamples_per_s) {
    using namespace vc;
    if (!gsamples_per_s) return VC_ERR_INVALID;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const int n = 16;
    uint16_t* d = nullptr;
    unsigned long long* cnt = nullptr;
    int rc = VC_OK;
    if (cudaMalloc(&d, n * n * n * sizeof(uint16_t)) != cudaSuccess ||
        cudaMalloc(&cnt, sizeof(unsigned long long)) != cudaSuccess)
        rc = VC_ERR_CUDA;
    if (rc == VC_OK) {
        uint16_t h[16 * 16 * 16];
        for (int i = 0; i < n * n * n; i++) h[i] = (uint16_t)((i * 2654435761u >> 20) & 4095);
        cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
        cudaMemset(cnt, 0, sizeof(unsigned long long));
        Vol<uint16_t> v = make_vol<uint16_t>(d, n, n, n, 4095.0);
        RayPos rp{};
        for (int a = 0; a < 3; a++) {
            rp.s[a] = 1.0;
            rp.rs[a] = 1.0;
        }
        rp.pow2 = true;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sample_peak_kernel<uint16_t>, 128, 0);
        const int blocks = sms * per_sm, iters = 4096;
        sample_peak_kernel<uint16_t><<<blocks, 128>>>(v, rp, 500.0, 3000.0, 256, cnt);  // warm-up
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        sample_peak_kernel<uint16_t><<<blocks, 128>>>(v, rp, 500.0, 3000.0, iters, cnt);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) rc = VC_ERR_CUDA;
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        *gsamples_per_s = (double)blocks * 128.0 * iters / (ms * 1e-3) / 1e9;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    cudaFree(d);
    cudaFree(cnt);
    cudaSetDevice(prev);
    return rc;
}
