// Standalone TMA 3-D tile load probe (development).  ./tma_probe V
//   V=0 baseline box 40x10x18 at (-1,-1,-1), map as __grid_constant__ param
//   V=1 same at (0,0,0);  V=2 box 32x8x16;  V=3 map in global memory
//   V=4 barrier only (arrive with no TMA, plain arrive)
//   V=5 start (31,1,1) inside (x start not 16-byte aligned)
//   V=6 start (32,56,50): box crosses the high faces
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int MAXE = 40 * 10 * 18;

__global__ void probe(uint16_t* out, const __grid_constant__ CUtensorMap tmap, const CUtensorMap* gmap, int v,
                      int cx, int cy, int cz, int nbytes) {
    __shared__ __align__(1024) uint16_t tile[MAXE];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t t = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (v == 4) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
        } else {
            const uint64_t desc = v == 3 ? reinterpret_cast<uint64_t>(gmap) : reinterpret_cast<uint64_t>(&tmap);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbytes) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(t), "l"(desc), "r"(cx), "r"(cy), "r"(cz), "r"(b) : "memory");
        }
    }
    uint32_t phase = 0;
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(b), "r"(phase) : "memory");
    for (int i = threadIdx.x; i < nbytes / 2; i += blockDim.x) out[i] = tile[i];
}

int main(int argc, char** argv) {
    const int v = argc > 1 ? atoi(argv[1]) : 0;
    const int n = 64;
    std::vector<uint16_t> h(n * n * n);
    for (size_t i = 0; i < h.size(); i++) h[i] = (uint16_t)(i % 4093 + 1);
    uint16_t *d, *o;
    CUtensorMap* gm;
    cudaMalloc(&d, h.size() * 2);
    cudaMalloc(&o, MAXE * 2);
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    alignas(64) CUtensorMap m;
    const cuuint32_t bw = v == 2 ? 32 : 40, bh = v == 2 ? 8 : 10, bd = v == 2 ? 16 : 18;
    cuuint64_t dims[3] = {n, n, n};
    cuuint64_t str[2] = {n * 2, (cuuint64_t)n * n * 2};
    cuuint32_t box[3] = {bw, bh, bd};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    int cx = v == 1 ? 0 : -1, cy = cx, cz = cx;
    if (v == 5) { cx = 31; cy = 1; cz = 1; }
    if (v == 6) { cx = 32; cy = 56; cz = 50; }
    if (v == 7) { cx = -8; cy = -1; cz = -1; }
    if (v == 8) { cx = 0; cy = -1; cz = -1; }
    if (v == 9) { cx = -8; cy = 0; cz = 0; }
    if (v == 10) { cx = 24; cy = 7; cz = 15; }
    const int nbytes = (int)(bw * bh * bd * 2);
    probe<<<1, 128>>>(o, m, gm, v, cx, cy, cz, nbytes);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d encode %d launch: %s\n", v, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess || v == 4) return 0;
    std::vector<uint16_t> g(nbytes / 2);
    cudaMemcpy(g.data(), o, nbytes, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int z = 0; z < (int)bd; z++)
        for (int y = 0; y < (int)bh; y++)
            for (int x = 0; x < (int)bw; x++) {
                int gx = x + cx, gy = y + cy, gz = z + cz;
                uint16_t want = (gx < 0 || gy < 0 || gz < 0 || gx >= n || gy >= n || gz >= n)
                                    ? 0 : h[(size_t)gz * n * n + gy * n + gx];
                if (g[(z * bh + y) * bw + x] != want) bad++;
            }
    printf("variant %d mismatches: %d\n", v, bad);
    return 0;
}
