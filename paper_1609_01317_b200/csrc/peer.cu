// peer.cu -- device-side completion flags of the multi-GPU image-tile gather.
//
// Each rank's IPC allocation holds its frame buffer and two flag blocks of
// VC_MAX_PEERS uint32 slots: "done" (slot r = the last frame sequence number
// rank r finished storing into this buffer) and "free" (slot c = the last
// frame consumer c finished reading from the writer's target buffer, in the
// writer's block).  A producer signals after its kernels with a system-scope
// release; a consumer's stream waits on an acquire spin in one thread -- no
// host synchronisation and no host barrier in the per-frame path.  The spin
// is bounded (timeout_us) and reports a timeout through *status instead of
// hanging the GPU.
#include "vc_internal.h"

namespace vc {

__global__ void signal_flags_kernel(uint32_t* const* blocks, int n, int dest, int slot, uint32_t seq) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // everything this stream wrote before (the raycast kernels' local and
    // NVLink stores, or a finished read) is ordered before the flags
    __threadfence_system();
    for (int r = 0; r < n; r++) {
        if (dest >= 0 && r != dest) continue;
        uint32_t* f = blocks[r] + slot;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(seq) : "memory");
    }
}

__global__ void wait_flags_kernel(const uint32_t* block, int first, int count, uint32_t seq, uint64_t timeout_ns,
                                  int32_t* status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = first; i < first + count; i++) {
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(block + i) : "memory");
            if ((int32_t)(v - seq) >= 0) break;  // sequence numbers wrap
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                if (status) *status = 1;
                return;
            }
            __nanosleep(256);
        }
    }
    if (status) *status = 0;
}

cudaError_t launch_signal_flags(uint32_t* const* blocks, int n, int dest, int slot, uint32_t seq, cudaStream_t s) {
    signal_flags_kernel<<<1, 32, 0, s>>>(blocks, n, dest, slot, seq);
    return cudaGetLastError();
}

cudaError_t launch_wait_flags(const uint32_t* block, int first, int count, uint32_t seq, uint32_t timeout_us,
                              int32_t* status, cudaStream_t s) {
    wait_flags_kernel<<<1, 32, 0, s>>>(block, first, count, seq, (uint64_t)timeout_us * 1000ull, status);
    return cudaGetLastError();
}

}  // namespace vc
