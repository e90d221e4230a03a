// capi.cu -- the C ABI (include/voxelcast_b200.h): device-resident volume
// objects, their caches, and the launch wrappers.
//
// A vc_volume owns, on one device:
//   * the voxel grid (immutable after create; the reference Volume is frozen,
//     volume.py:47, :71-72)
//   * the 4^3 macrocell min/max grid (built once) and the Chebyshev
//     distance fields of the last 8 threshold windows (LRU)
//   * one packed float4 gradient volume per operator (Kernel 1, lazily)
//   * scratch for the host-facing render path.
// The reference API is stateless per call (raycast.py:431-438); keeping the
// upload and the derived grids on the volume object is what lets a frame be
// a single kernel launch.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "vc_internal.h"

struct vc_volume {
    int device = 0;
    int dtype = VC_U16;
    int nx = 0, ny = 0, nz = 0;
    double spacing[3] = {1.0, 1.0, 1.0};
    void* d_data = nullptr;
    size_t bytes = 0;
    float2* d_mm = nullptr;
    // macrocell distance fields, one per threshold window seen (LRU, at most
    // MAX_FIELDS); `ready` orders the build before renders on other streams
    struct WindowField {
        double lo = 0.0, hi = 0.0;
        uint8_t* dist = nullptr;
        uint8_t* tmp = nullptr;
        cudaEvent_t ready = nullptr;
        uint64_t stamp = 0;
    };
    std::vector<WindowField> fields;
    uint64_t clock = 0;
    int mx = 0, my = 0, mz = 0;
    double vmin = 0.0, vmax = 0.0;  // value range (from the macrocell grid)
    float4* d_grad[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t grad_ready[3] = {nullptr, nullptr, nullptr};
    // VC_SAMPLER_TEXTURE: cudaArray copies + texture objects, built lazily
    cudaArray_t val_arr = nullptr, grad_arr[3] = {nullptr, nullptr, nullptr};
    cudaTextureObject_t val_tex = 0, grad_tex[3] = {0, 0, 0};
    vc::OctDev oct{};  // device octree for adaptive stepping (owned buffers)
    long long oct_n_ivl = 0, oct_n_boxes = 0;  // its array sizes (checked builds' regions)
    uint8_t* d_scratch = nullptr;
    size_t scratch_bytes = 0;
    uint64_t* d_counters = nullptr;
    // per-stream scratch of the two-stage raycast: frame work counters and the
    // first-hit queue (renders on different streams never share them)
    struct StreamScratch {
        void* work = nullptr;
        void* hits = nullptr;
        size_t hit_cap = 0;
        unsigned* tiles = nullptr;  // 8x4 tile counters of the peer tile pushes
        size_t tile_cap = 0;
        cudaEvent_t done = nullptr;  // recorded after each render that used it
        uint64_t stamp = 0;
        unsigned seq = 0;            // hit-entry tag of the last render (0: none yet)
        bool work_dirty = true;      // the work counters need zeroing before the next render
    };
    std::unordered_map<cudaStream_t, StreamScratch> scratch;
    uint64_t scratch_clock = 0;
    cudaStream_t host_stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::mutex mu;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(VC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define VC_CUDA(call)                                   \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

size_t dtype_size(int dtype) { return dtype == VC_U8 ? 1 : (dtype == VC_U16 ? 2 : 4); }

bool is_pow2(double s) {
    int e = 0;
    return std::frexp(s, &e) == 0.5;
}

vc::RayPos make_raypos(const vc_volume* v) {
    vc::RayPos rp{};
    bool pow2 = true;
    for (int a = 0; a < 3; a++) {
        rp.s[a] = v->spacing[a];
        rp.rs[a] = 1.0 / v->spacing[a];
        pow2 = pow2 && is_pow2(v->spacing[a]);
    }
    rp.pow2 = pow2;
    // ddiv_rcp needs rs = RN(1/s) (1.0 / s above) and no all-ones significand
    rp.rcp = true;
    for (int a = 0; a < 3; a++) {
        uint64_t bits;
        memcpy(&bits, &v->spacing[a], sizeof(bits));
        if ((bits & 0xFFFFFFFFFFFFFull) == 0xFFFFFFFFFFFFFull) rp.rcp = false;
    }
    return rp;
}

class DeviceGuard {
   public:
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev_);
        if (prev_ != dev) cudaSetDevice(dev);
        dev_ = dev;
    }
    ~DeviceGuard() {
        if (prev_ != dev_) cudaSetDevice(prev_);
    }

   private:
    int prev_ = 0, dev_ = 0;
};

int validate_dims(int dtype, int nx, int ny, int nz, const double* spacing) {
    if (dtype < VC_U8 || dtype > VC_F32) return fail(VC_ERR_INVALID, "dtype must be VC_U8, VC_U16 or VC_F32");
    if (nx <= 0 || ny <= 0 || nz <= 0) return fail(VC_ERR_INVALID, "volume must contain at least one voxel");
    if ((double)nx * ny * nz > 4294967295.0)
        return fail(VC_ERR_UNSUPPORTED, "volumes above 2^32 - 1 voxels are not supported");
    if (spacing == nullptr) return fail(VC_ERR_INVALID, "spacing is required");
    for (int a = 0; a < 3; a++)
        if (!(spacing[a] > 0.0) || !std::isfinite(spacing[a]))
            return fail(VC_ERR_INVALID, "spacing must be positive");
    return VC_OK;
}

// Runs on v->host_stream after the voxel upload was queued there: the
// min/max kernel is stream-ordered after the copy, and the final
// synchronize completes both before any render (on any stream) can start.
int finish_create(vc_volume* v) {
    // macrocells over interpolation cells [0, max(n-2,0)] per axis
    v->mx = std::max(v->nx - 2, 0) / vc::MC_EDGE + 1;
    v->my = std::max(v->ny - 2, 0) / vc::MC_EDGE + 1;
    v->mz = std::max(v->nz - 2, 0) / vc::MC_EDGE + 1;
    const size_t mc = (size_t)v->mx * v->my * v->mz;
    VC_CUDA(cudaMalloc(&v->d_mm, mc * sizeof(float2)));
    VC_CUDA(cudaMalloc(&v->d_counters, VC_NUM_COUNTERS * sizeof(uint64_t)));
    VC_CUDA(cudaEventCreate(&v->ev0));
    VC_CUDA(cudaEventCreate(&v->ev1));
    VC_CUDA(vc::launch_macrocell_minmax(v->dtype, v->d_data, v->nx, v->ny, v->nz, v->d_mm, v->mx, v->my,
                                        v->mz, v->host_stream));
    std::vector<float2> mm(mc);
    VC_CUDA(cudaMemcpyAsync(mm.data(), v->d_mm, mc * sizeof(float2), cudaMemcpyDeviceToHost, v->host_stream));
    VC_CUDA(cudaStreamSynchronize(v->host_stream));
    double lo = mm[0].x, hi = mm[0].y;
    for (const auto& r : mm) {
        lo = std::min(lo, (double)r.x);
        hi = std::max(hi, (double)r.y);
    }
    v->vmin = lo;
    v->vmax = hi;
    return VC_OK;
}

void free_octree(vc_volume* v) {
    cudaFree((void*)v->oct.dims);
    cudaFree((void*)v->oct.amap);
    cudaFree((void*)v->oct.ivl_off);
    cudaFree((void*)v->oct.ivl);
    cudaFree((void*)v->oct.box_off);
    cudaFree((void*)v->oct.state);
    cudaFree((void*)v->oct.srange);
    v->oct = vc::OctDev{};
}

void release(vc_volume* v) {
    if (!v) return;
    DeviceGuard g(v->device);
    cudaFree(v->d_data);
    cudaFree(v->d_mm);
    for (auto& f : v->fields) {
        cudaFree(f.dist);
        cudaFree(f.tmp);
        if (f.ready) cudaEventDestroy(f.ready);
    }
    for (auto& e : v->grad_ready)
        if (e) cudaEventDestroy(e);
    free_octree(v);
    for (auto& p : v->d_grad) cudaFree(p);
    if (v->val_tex) cudaDestroyTextureObject(v->val_tex);
    if (v->val_arr) cudaFreeArray(v->val_arr);
    for (int i = 0; i < 3; i++) {
        if (v->grad_tex[i]) cudaDestroyTextureObject(v->grad_tex[i]);
        if (v->grad_arr[i]) cudaFreeArray(v->grad_arr[i]);
    }
    cudaFree(v->d_scratch);
    cudaFree(v->d_counters);
    for (auto& kv : v->scratch) {
        cudaFree(kv.second.work);
        cudaFree(kv.second.hits);
        cudaFree(kv.second.tiles);
        if (kv.second.done) cudaEventDestroy(kv.second.done);
    }
    if (v->host_stream) cudaStreamDestroy(v->host_stream);
    if (v->ev0) cudaEventDestroy(v->ev0);
    if (v->ev1) cudaEventDestroy(v->ev1);
    delete v;
}

int create_common(int device, const void* src, cudaMemcpyKind kind, int dtype, int nx, int ny, int nz,
                  const double spacing[3], vc_volume** out) {
    if (out == nullptr) return fail(VC_ERR_INVALID, "out is null");
    *out = nullptr;
    if (src == nullptr) return fail(VC_ERR_INVALID, "volume data is null");
    int rc = validate_dims(dtype, nx, ny, nz, spacing);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(VC_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(VC_ERR_INVALID, "device ordinal out of range");
    DeviceGuard g(device);
    vc_volume* v = new vc_volume();
    v->device = device;
    v->dtype = dtype;
    v->nx = nx;
    v->ny = ny;
    v->nz = nz;
    for (int a = 0; a < 3; a++) v->spacing[a] = spacing[a];
    v->bytes = (size_t)nx * ny * nz * dtype_size(dtype);
    // zeroed tail padding: gather8 reads one element past an x-degenerate row
    cudaError_t e = cudaMalloc(&v->d_data, v->bytes + vc::VC_VOLUME_PAD);
    if (e == cudaSuccess) e = cudaMemset(static_cast<char*>(v->d_data) + v->bytes, 0, vc::VC_VOLUME_PAD);
    if (e != cudaSuccess) {
        release(v);
        return fail(VC_ERR_NOMEM, std::string("cudaMalloc(volume): ") + cudaGetErrorString(e));
    }
    // The upload goes on the volume's own (non-blocking) stream so that the
    // macrocell min/max kernel queued behind it in finish_create reads the
    // finished copy.  A device source may still be being written by a
    // producer on any stream (e.g. the ingest path's torch stream): drain the
    // device first -- once per volume, so the cost does not matter.
    e = cudaStreamCreateWithFlags(&v->host_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && kind == cudaMemcpyDeviceToDevice) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpyAsync(v->d_data, src, v->bytes, kind, v->host_stream);
    if (e != cudaSuccess) {
        release(v);
        return cuda_fail(e, "cudaMemcpyAsync(volume)");
    }
    rc = finish_create(v);
    if (rc) {
        release(v);
        return rc;
    }
    *out = v;
    return VC_OK;
}

int ensure_grad(vc_volume* v, int op, cudaStream_t s) {
    if (v->d_grad[op]) {
        VC_CUDA(cudaStreamWaitEvent(s, v->grad_ready[op], 0));  // built on another stream
        return VC_OK;
    }
    float4* g = nullptr;
    cudaError_t e = cudaMalloc(&g, (size_t)v->nx * v->ny * v->nz * sizeof(float4));
    if (e != cudaSuccess) return fail(VC_ERR_NOMEM, std::string("cudaMalloc(gradient volume): ") + cudaGetErrorString(e));
    e = vc::launch_gradient_prepass(v->dtype, v->d_data, v->nx, v->ny, v->nz, op, g, s);
    if (e != cudaSuccess) {
        cudaFree(g);
        return cuda_fail(e, "gradient pre-pass launch");
    }
    v->d_grad[op] = g;
    if (!v->grad_ready[op]) VC_CUDA(cudaEventCreateWithFlags(&v->grad_ready[op], cudaEventDisableTiming));
    VC_CUDA(cudaEventRecord(v->grad_ready[op], s));
    return VC_OK;
}

// 3-D texture over a cudaArray copy of `src` (x fastest, elem bytes per
// texel), hardware trilinear filtering, unnormalized coordinates (texel
// centres at i + 0.5), clamp addressing (callers test the reference's
// [0, n-1] range first).
int make_texture(const vc_volume* v, const void* src, const cudaChannelFormatDesc& desc, size_t elem,
                 bool normalized_read, cudaStream_t s, cudaArray_t* arr, cudaTextureObject_t* tex) {
    const cudaExtent ext = make_cudaExtent(v->nx, v->ny, v->nz);
    cudaError_t e = cudaMalloc3DArray(arr, &desc, ext, 0);
    if (e != cudaSuccess) return fail(VC_ERR_NOMEM, std::string("cudaMalloc3DArray: ") + cudaGetErrorString(e));
    cudaMemcpy3DParms cp{};
    cp.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), (size_t)v->nx * elem, v->nx, v->ny);
    cp.dstArray = *arr;
    cp.extent = ext;
    cp.kind = cudaMemcpyDeviceToDevice;
    VC_CUDA(cudaMemcpy3DAsync(&cp, s));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = *arr;
    cudaTextureDesc td{};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModeLinear;
    td.readMode = normalized_read ? cudaReadModeNormalizedFloat : cudaReadModeElementType;
    td.normalizedCoords = 0;
    VC_CUDA(cudaCreateTextureObject(tex, &rd, &td, nullptr));
    return VC_OK;
}

int ensure_textures(vc_volume* v, int op, bool want_grad, cudaStream_t s) {
    if (!v->val_tex) {
        cudaChannelFormatDesc d = v->dtype == VC_U8    ? cudaCreateChannelDesc<unsigned char>()
                                  : v->dtype == VC_U16 ? cudaCreateChannelDesc<unsigned short>()
                                                       : cudaCreateChannelDesc<float>();
        int rc = make_texture(v, v->d_data, d, dtype_size(v->dtype), v->dtype != VC_F32, s, &v->val_arr,
                              &v->val_tex);
        if (rc) return rc;
    }
    if (want_grad && !v->grad_tex[op]) {
        int rc = make_texture(v, v->d_grad[op], cudaCreateChannelDesc<float4>(), sizeof(float4), false, s,
                              &v->grad_arr[op], &v->grad_tex[op]);
        if (rc) return rc;
    }
    // one-time copies: finish them before any stream samples the arrays
    VC_CUDA(cudaStreamSynchronize(s));
    return VC_OK;
}

constexpr size_t MAX_FIELDS = 8;

// distance field of window [lo, hi], built on stream s if not cached
int window_field(vc_volume* v, double lo, double hi, cudaStream_t s, vc_volume::WindowField** out) {
    v->clock++;
    for (auto& f : v->fields)
        if (f.lo == lo && f.hi == hi) {
            f.stamp = v->clock;
            VC_CUDA(cudaStreamWaitEvent(s, f.ready, 0));
            *out = &f;
            return VC_OK;
        }
    vc_volume::WindowField* f = nullptr;
    if (v->fields.size() < MAX_FIELDS) {
        v->fields.emplace_back();
        f = &v->fields.back();
        const size_t mc = (size_t)v->mx * v->my * v->mz;
        VC_CUDA(cudaMalloc(&f->dist, mc));
        VC_CUDA(cudaMalloc(&f->tmp, mc));
        VC_CUDA(cudaEventCreateWithFlags(&f->ready, cudaEventDisableTiming));
    } else {
        f = &v->fields[0];
        for (auto& g : v->fields)
            if (g.stamp < f->stamp) f = &g;
        // Renders still reading the evicted field may run on any stream:
        // eviction is rare (a ninth threshold window), so wait for the whole
        // device rather than track every reader.
        VC_CUDA(cudaDeviceSynchronize());
    }
    f->lo = lo;
    f->hi = hi;
    f->stamp = v->clock;
    VC_CUDA(vc::launch_occupancy(v->d_mm, v->mx, v->my, v->mz, lo, hi, f->dist, f->tmp, s));
    VC_CUDA(cudaEventRecord(f->ready, s));
    *out = f;
    return VC_OK;
}

int validate_params(const vc_render_params* p, int* local_rows) {
    if (p == nullptr) return fail(VC_ERR_INVALID, "params is null");
    if (p->width <= 0 || p->height <= 0) return fail(VC_ERR_INVALID, "image size must be positive");
    if (p->width > 65535 || p->height > 65535)  // hit-queue entries pack (row, column) in 16 bits each
        return fail(VC_ERR_UNSUPPORTED, "frames wider or taller than 65535 pixels are not supported");
    if (p->band_rows < 1 || p->band_step < 1 || p->band_first < 0)
        return fail(VC_ERR_INVALID, "band_rows/band_step must be >= 1 and band_first >= 0");
    if (p->lut_n < 1 || p->lut_n > VC_MAX_LUT) return fail(VC_ERR_INVALID, "lut_n must be in [1, VC_MAX_LUT]");
    for (int i = 0; i + 1 < p->lut_n; i++)
        if (!(p->lut_hu[i + 1] > p->lut_hu[i])) return fail(VC_ERR_INVALID, "transfer breakpoints must strictly increase");
    if (p->op < 0 || p->op > 2) return fail(VC_ERR_INVALID, "op must be 0, 1 or 2");
    if (p->interp < 0 || p->interp > 2) return fail(VC_ERR_INVALID, "interp must be 0, 1 or 2");
    if (p->mode < 0 || p->mode > 1) return fail(VC_ERR_INVALID, "mode must be 0 or 1");
    if (!(p->coarse > 0.0) || !(p->fine > 0.0)) return fail(VC_ERR_INVALID, "steps must be positive");
    if (p->refine_iters < 0) return fail(VC_ERR_INVALID, "refine_iters must be >= 0");
    if (!(p->mu_water > 0.0)) return fail(VC_ERR_INVALID, "mu_water must be positive");
    if (p->use_adaptive && p->adapt_jump < 1) return fail(VC_ERR_INVALID, "adaptive_factor must be >= 1");
    if (p->grad_source != VC_GRAD_TAPS && p->grad_source != VC_GRAD_VOLUME)
        return fail(VC_ERR_INVALID, "grad_source must be VC_GRAD_TAPS or VC_GRAD_VOLUME");
    if (p->sampler != VC_SAMPLER_SOFTWARE && p->sampler != VC_SAMPLER_TEXTURE)
        return fail(VC_ERR_INVALID, "sampler must be VC_SAMPLER_SOFTWARE or VC_SAMPLER_TEXTURE");
    if (p->sampler == VC_SAMPLER_TEXTURE && p->interp != VC_TRILINEAR)
        return fail(VC_ERR_INVALID, "the texture sampler is trilinear only");
    if (p->sampler == VC_SAMPLER_TEXTURE && p->use_adaptive)
        return fail(VC_ERR_UNSUPPORTED, "adaptive stepping runs on the software sampler only");
    if (p->row_end < 0) return fail(VC_ERR_INVALID, "row_end must be >= 0");
    // bands ascend, so the first local_rows rows of the band set are exactly
    // those below row_end: the kernels need no extra test
    const long long h = p->row_end > 0 ? std::min(p->height, p->row_end) : p->height;
    const long long nb = (h + p->band_rows - 1) / p->band_rows;
    long long rows = 0;
    for (long long b = p->band_first; b < nb; b += p->band_step)
        rows += std::min<long long>(p->band_rows, h - b * p->band_rows);
    if (rows > (1LL << 30)) return fail(VC_ERR_INVALID, "too many rows");
    *local_rows = (int)rows;
    return VC_OK;
}

// The byte ranges a launch may touch (VC_CHECKED builds upload them; the
// kernels count and skip any access outside).  Peer frames are read back
// from the device table.
struct Regions {
    std::vector<unsigned long long> lohi;
    void add(const void* p, size_t bytes) {
        if (!p || !bytes) return;
        lohi.push_back((unsigned long long)p);
        lohi.push_back((unsigned long long)p + bytes);
    }
};

int render_impl(vc_volume* v, const vc_render_params* p, uint8_t* d_rgba, uint64_t* d_counters,
                cudaStream_t s, int local_rows, cudaEvent_t* stage_events = nullptr,
                const vc_peer_frames* pf = nullptr) {
    vc::RenderLaunch L{};
    void* const* d_peers = pf ? pf->d_frames : nullptr;
    const int npeers = pf ? pf->n : 0;
    const size_t peer_bytes = pf ? (size_t)pf->frame_bytes : 0;
    L.peers = d_peers;
    L.npeers = npeers;
    L.peer_self = pf ? pf->self : 0;
    L.peer_dest = pf ? pf->dest : -1;
    L.tile_cnt = nullptr;
    if (stage_events)
        for (int i = 0; i < 3; i++) L.ev[i] = stage_events[i];
    L.p = p;
    L.dtype = v->dtype;
    L.data = v->d_data;
    L.nx = v->nx;
    L.ny = v->ny;
    L.nz = v->nz;
    L.amax = std::max(std::fabs(v->vmin), std::fabs(v->vmax));
    if (!std::isfinite(L.amax)) L.amax = -1.0;  // no float32 pre-test
    L.rp = make_raypos(v);
    L.oct = v->oct;
    L.out = d_rgba;
    L.local_rows = local_rows;
    L.counters = d_counters;
    vc_volume::StreamScratch* scp = nullptr;
    {
        // per-stream scratch, at most MAX_STREAM_SCRATCH streams: the least
        // recently used one is released once its last render has finished
        constexpr size_t MAX_STREAM_SCRATCH = 8;
        if (v->scratch.find(s) == v->scratch.end() && v->scratch.size() >= MAX_STREAM_SCRATCH) {
            auto old = v->scratch.begin();
            for (auto it = v->scratch.begin(); it != v->scratch.end(); ++it)
                if (it->second.stamp < old->second.stamp) old = it;
            if (old->second.done) VC_CUDA(cudaEventSynchronize(old->second.done));
            cudaFree(old->second.work);
            cudaFree(old->second.hits);
            cudaFree(old->second.tiles);
            if (old->second.done) cudaEventDestroy(old->second.done);
            v->scratch.erase(old);
        }
        auto& sc = v->scratch[s];
        sc.stamp = ++v->scratch_clock;
        if (!sc.done) VC_CUDA(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming));
        scp = &sc;
        const size_t need = (size_t)local_rows * p->width;
        if (sc.work == nullptr) {
            VC_CUDA(cudaMalloc(&sc.work, vc::frame_work_bytes()));
            sc.work_dirty = true;
        }
        // the frame's work counters are reset by its own last kernel; after a
        // failed render (or on a fresh scratch) they are zeroed here
        if (sc.work_dirty) {
            VC_CUDA(cudaMemsetAsync(sc.work, 0, vc::frame_work_bytes(), s));
            sc.work_dirty = false;
        }
        if (sc.hit_cap < need) {
            cudaFree(sc.hits);
            sc.hits = nullptr;
            sc.hit_cap = 0;
            cudaError_t e = cudaMalloc(&sc.hits, need * vc::hit_entry_bytes());
            if (e != cudaSuccess) return fail(VC_ERR_NOMEM, std::string("cudaMalloc(hit queue): ") + cudaGetErrorString(e));
            sc.hit_cap = need;
            sc.seq = 0;
        }
        // hit entries carry the render's tag (kernel B reads an entry once it
        // holds this render's tag): a fresh queue, or a tag counter about to
        // wrap, starts from zeroed entries
        if (sc.seq == 0 || sc.seq == 0xffffffffu) {
            VC_CUDA(cudaMemsetAsync(sc.hits, 0, sc.hit_cap * vc::hit_entry_bytes(), s));
            sc.seq = 0;
        }
        L.seq = ++sc.seq;
        // overlap the two stages (kernel B starting in kernel A's tail) only
        // when this render is alone on the device: with renders of other
        // streams in flight (render_sequence) the tail is filled anyway and
        // kernel B's early blocks would only poll
        static const bool no_overlap = getenv("VC_NO_STAGE_OVERLAP") != nullptr;
        bool alone = true;
        for (auto& kv : v->scratch)
            if (kv.first != s && kv.second.done && cudaEventQuery(kv.second.done) == cudaErrorNotReady) alone = false;
        if (!alone) (void)cudaGetLastError();  // a not-ready status is not this render's error
        L.overlap_stages = (!no_overlap && alone) ? 1 : 0;
        L.work = sc.work;
        L.hits = sc.hits;
        // tile pushes need whole 8x4 tiles inside one band (band_rows % 4 == 0)
        if (npeers > 0 && p->band_rows % 4 == 0) {
            const size_t tiles = (size_t)((p->width + 7) / 8) * (size_t)((local_rows + 3) / 4);
            if (sc.tile_cap < tiles) {
                cudaFree(sc.tiles);
                sc.tiles = nullptr;
                sc.tile_cap = 0;
                VC_CUDA(cudaMalloc(&sc.tiles, tiles * sizeof(unsigned)));
                sc.tile_cap = tiles;
            }
            L.tile_cnt = sc.tiles;
        }
    }
    L.mx = v->mx;
    L.my = v->my;
    L.occ = nullptr;
    const bool zero_in_window = p->t_low <= 0.0 && 0.0 <= p->t_high;
    // adaptive strides depend on the exact lattice sequence: no skipping
    L.skip_on = (p->skip_empty && !zero_in_window && !p->use_adaptive) ? 1 : 0;
    // With use_octree the reference's first hit marches only the merged
    // segments of the octree leaves whose padded range meets the window
    // (collect_segments, _kernels.py:290-364, 656-669).  Away from the grid
    // that drops only out-of-window samples, so the macrocell skip above gives
    // the same pixels.  But a sample in the half-voxel border band reads 0
    // (_kernels.py:121-122): with 0 in the window it is in-window, and the
    // reference still skips it whenever its border leaf's padded range misses
    // the window.  That case (and use_adaptive, whose stride depends on the
    // lattice sequence) replays the reference's segment walk on the device.
    L.seg_walk = (p->skip_empty && p->sampler != VC_SAMPLER_TEXTURE && (p->use_adaptive || zero_in_window)) ? 1 : 0;
    if ((p->use_adaptive || L.seg_walk) && v->oct.levels == 0)
        return fail(VC_ERR_INVALID, "use_adaptive, or use_octree with 0 inside the threshold window, needs an "
                                    "octree (vc_volume_set_octree)");
    vc_volume::WindowField* field = nullptr;
    if (L.skip_on) {
        int rc = window_field(v, p->t_low, p->t_high, s, &field);
        if (rc) return rc;
        L.occ = field->dist;
    }
    L.grad = nullptr;
    if (p->grad_source == VC_GRAD_VOLUME) {
        int rc = ensure_grad(v, p->op, s);
        if (rc) return rc;
        L.grad = v->d_grad[p->op];
    }
    L.tex_value = 0;
    L.tex_grad = 0;
    L.tex_scale = v->dtype == VC_U8 ? 255.0f : (v->dtype == VC_U16 ? 65535.0f : 1.0f);
    if (p->sampler == VC_SAMPLER_TEXTURE) {
        int rc = ensure_textures(v, p->op, L.grad != nullptr, s);
        if (rc) return rc;
        L.tex_value = v->val_tex;
        L.tex_grad = L.grad ? v->grad_tex[p->op] : 0;
    }
    if (d_counters) VC_CUDA(cudaMemsetAsync(d_counters, 0, VC_NUM_COUNTERS * sizeof(uint64_t), s));
    if (local_rows == 0) return VC_OK;
#ifdef VC_CHECKED
    Regions R;
    R.add(v->d_data, v->bytes + vc::VC_VOLUME_PAD);
    if (L.grad) R.add(L.grad, (size_t)v->nx * v->ny * v->nz * sizeof(float4));
    if (L.occ) R.add(L.occ, (size_t)v->mx * v->my * v->mz);
    R.add(L.work, vc::frame_work_bytes());
    // negative control of the checker itself (tests/test_checked_gpu.py):
    // leave the hit queue out and every queue access must be reported
    if (!getenv("VC_CHECKED_DROP_QUEUE")) R.add(L.hits, scp->hit_cap * vc::hit_entry_bytes());
    R.add(d_counters, VC_NUM_COUNTERS * sizeof(uint64_t));
    if (d_rgba) R.add(d_rgba, (size_t)local_rows * p->width * 4);
    if (npeers > 0) {
        R.add(d_peers, (size_t)npeers * sizeof(void*));
        std::vector<void*> hp(npeers);
        VC_CUDA(cudaMemcpy(hp.data(), d_peers, npeers * sizeof(void*), cudaMemcpyDeviceToHost));
        for (void* q : hp) R.add(q, peer_bytes);
        if (L.tile_cnt) R.add(L.tile_cnt, scp->tile_cap * sizeof(unsigned));
    }
    if (v->oct.levels > 0) {
        const size_t lv = (size_t)v->oct.levels;
        R.add(v->oct.dims, lv * 3 * sizeof(int32_t));
        R.add(v->oct.amap, lv * (size_t)(v->nx + v->ny + v->nz) * sizeof(int32_t));
        R.add(v->oct.ivl_off, lv * 3 * sizeof(int32_t));
        R.add(v->oct.ivl, (size_t)v->oct_n_ivl * sizeof(int32_t));
        R.add(v->oct.box_off, lv * sizeof(int64_t));
        R.add(v->oct.state, (size_t)v->oct_n_boxes);
        R.add(v->oct.srange, (size_t)v->oct_n_boxes * 2 * sizeof(double));
    }
    L.regions = R.lohi.data();
    L.nregions = (int)(R.lohi.size() / 2);
#endif
    {
        const cudaError_t le = vc::launch_raycast(L, s);
        if (le != cudaSuccess) {
            scp->work_dirty = true;  // the kernels may not have reset the counters
            VC_CUDA(le);
        }
    }
    if (pf && pf->d_done)  // this rank's bands are in every receiver's frame
        VC_CUDA(vc::launch_signal_flags(pf->d_done, pf->n, pf->dest, pf->self, pf->seq, s));
    VC_CUDA(cudaEventRecord(scp->done, s));
    return VC_OK;
}

}  // namespace

extern "C" {

int vc_abi_version(void) { return VC_ABI_VERSION; }

#ifdef VC_CHECKED
// checked builds only (not in the public header): accesses outside the
// launches' regions since the last call, and the first offending address
VC_API unsigned long long vc_checked_violations(unsigned long long* first) {
    unsigned long long f1 = 0, f2 = 0;
    const unsigned long long a = vc::vc_take_violations_raycast(&f1), b = vc::vc_take_violations_points(&f2);
    if (first) *first = a ? f1 : f2;
    return a + b;
}
#endif
int vc_render_params_size(void) { return (int)sizeof(vc_render_params); }
const char* vc_last_error(void) { return g_err.c_str(); }

int vc_device_count(int* out) {
    if (!out) return fail(VC_ERR_INVALID, "out is null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *out = n;
    return VC_OK;
}

int vc_volume_create(int device, const void* h_data, int dtype, int nx, int ny, int nz,
                     const double spacing[3], vc_volume** out) {
    return create_common(device, h_data, cudaMemcpyHostToDevice, dtype, nx, ny, nz, spacing, out);
}

int vc_volume_create_device(int device, const void* d_data, int dtype, int nx, int ny, int nz,
                            const double spacing[3], vc_volume** out) {
    return create_common(device, d_data, cudaMemcpyDeviceToDevice, dtype, nx, ny, nz, spacing, out);
}

int vc_volume_destroy(vc_volume* vol) {
    release(vol);
    return VC_OK;
}

int vc_volume_set_octree(vc_volume* vol, const vc_octree_desc* d) {
    if (!vol || !d) return fail(VC_ERR_INVALID, "null argument");
    if (d->levels < 1 || d->levels > 17) return fail(VC_ERR_INVALID, "octree levels must be in [1, 17]");
    if (!d->dims || !d->axis_map || !d->ivl_off || !d->ivl || !d->box_off || !d->state || !d->srange ||
        d->n_ivl <= 0 || d->n_boxes <= 0)
        return fail(VC_ERR_INVALID, "incomplete octree description");
    DeviceGuard g(vol->device);
    std::lock_guard<std::mutex> lk(vol->mu);
    VC_CUDA(cudaDeviceSynchronize());  // renders in flight may read the old tree
    free_octree(vol);
    const size_t L = (size_t)d->levels, nmap = L * (size_t)(vol->nx + vol->ny + vol->nz);
    auto up = [](const void* src, size_t bytes, const void** dst) -> cudaError_t {
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) return e;
        *dst = p;
        return cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
    };
    vc::OctDev o{};
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = up(d->dims, L * 3 * sizeof(int32_t), (const void**)&o.dims);
    if (e == cudaSuccess) e = up(d->axis_map, nmap * sizeof(int32_t), (const void**)&o.amap);
    if (e == cudaSuccess) e = up(d->ivl_off, L * 3 * sizeof(int32_t), (const void**)&o.ivl_off);
    if (e == cudaSuccess) e = up(d->ivl, (size_t)d->n_ivl * sizeof(int32_t), (const void**)&o.ivl);
    if (e == cudaSuccess) e = up(d->box_off, L * sizeof(int64_t), (const void**)&o.box_off);
    if (e == cudaSuccess) e = up(d->state, (size_t)d->n_boxes, (const void**)&o.state);
    if (e == cudaSuccess) e = up(d->srange, (size_t)d->n_boxes * 2 * sizeof(double), (const void**)&o.srange);
    vol->oct = o;
    if (e != cudaSuccess) {
        free_octree(vol);
        return cuda_fail(e, "octree upload");
    }
    vol->oct.levels = d->levels;
    vol->oct_n_ivl = d->n_ivl;
    vol->oct_n_boxes = d->n_boxes;
    return VC_OK;
}

int vc_volume_data(const vc_volume* vol, const void** d_data) {
    if (!vol || !d_data) return fail(VC_ERR_INVALID, "null argument");
    *d_data = vol->d_data;
    return VC_OK;
}

int vc_gradient_prepass(vc_volume* vol, int op, void* stream) {
    if (!vol) return fail(VC_ERR_INVALID, "volume is null");
    if (op < 0 || op > 2) return fail(VC_ERR_INVALID, "op must be 0, 1 or 2");
    DeviceGuard g(vol->device);
    std::lock_guard<std::mutex> lk(vol->mu);
    return ensure_grad(vol, op, static_cast<cudaStream_t>(stream));
}

int vc_gradient_volume(const vc_volume* vol, int op, const void** d_grad) {
    if (!vol || !d_grad) return fail(VC_ERR_INVALID, "null argument");
    if (op < 0 || op > 2) return fail(VC_ERR_INVALID, "op must be 0, 1 or 2");
    *d_grad = vol->d_grad[op];
    return VC_OK;
}

int vc_gradient_prepass_into(const vc_volume* vol, int op, void* d_out, void* stream) {
    if (!vol || !d_out) return fail(VC_ERR_INVALID, "null argument");
    if (op < 0 || op > 2) return fail(VC_ERR_INVALID, "op must be 0, 1 or 2");
    DeviceGuard g(vol->device);
    VC_CUDA(vc::launch_gradient_prepass(vol->dtype, vol->d_data, vol->nx, vol->ny, vol->nz, op,
                                        static_cast<float4*>(d_out), static_cast<cudaStream_t>(stream)));
    return VC_OK;
}

int vc_render(vc_volume* vol, const vc_render_params* p, uint8_t* d_rgba, uint64_t* d_counters,
              void* stream) {
    if (!vol) return fail(VC_ERR_INVALID, "volume is null");
    int local_rows = 0;
    int rc = validate_params(p, &local_rows);
    if (rc) return rc;
    if (!d_rgba && local_rows > 0) return fail(VC_ERR_INVALID, "output buffer is null");
    DeviceGuard g(vol->device);
    std::lock_guard<std::mutex> lk(vol->mu);
    return render_impl(vol, p, d_rgba, d_counters, static_cast<cudaStream_t>(stream), local_rows);
}

int vc_render_to_peers(vc_volume* vol, const vc_render_params* p, const vc_peer_frames* pf, uint64_t* d_counters,
                       void* stream) {
    if (!vol || !pf || !pf->d_frames) return fail(VC_ERR_INVALID, "null argument");
    if (pf->n < 1 || pf->n > VC_MAX_PEERS) return fail(VC_ERR_INVALID, "need 1..VC_MAX_PEERS frame buffers");
    if (pf->self < 0 || pf->self >= pf->n || pf->dest < -1 || pf->dest >= pf->n)
        return fail(VC_ERR_INVALID, "self / dest out of range");
    int local_rows = 0;
    int rc = validate_params(p, &local_rows);
    if (rc) return rc;
    // every receiver's frame is stored at image_row * width + px: each buffer
    // must hold the whole (height, width, 4) frame
    if (pf->frame_bytes < (uint64_t)p->height * p->width * 4)
        return fail(VC_ERR_INVALID, "peer frame buffers are smaller than height * width * 4 bytes");
    DeviceGuard g(vol->device);
    std::lock_guard<std::mutex> lk(vol->mu);
    return render_impl(vol, p, nullptr, d_counters, static_cast<cudaStream_t>(stream), local_rows, nullptr, pf);
}

int vc_signal_flags(uint32_t* const* d_blocks, int n, int dest, int slot, uint32_t seq, void* stream) {
    if (!d_blocks || n < 1 || n > VC_MAX_PEERS || slot < 0 || slot >= VC_MAX_PEERS || dest < -1 || dest >= n)
        return fail(VC_ERR_INVALID, "bad flag-block arguments");
    VC_CUDA(vc::launch_signal_flags(d_blocks, n, dest, slot, seq, static_cast<cudaStream_t>(stream)));
    return VC_OK;
}

int vc_wait_flags(const uint32_t* d_block, int first, int count, uint32_t seq, uint32_t timeout_us, int32_t* d_status,
                  void* stream) {
    if (!d_block || first < 0 || count < 0 || first + count > VC_MAX_PEERS)
        return fail(VC_ERR_INVALID, "bad flag-block arguments");
    VC_CUDA(vc::launch_wait_flags(d_block, first, count, seq, timeout_us, d_status, static_cast<cudaStream_t>(stream)));
    return VC_OK;
}

int vc_device_alloc(int device, size_t bytes, void** d_ptr) {
    if (!d_ptr || bytes == 0) return fail(VC_ERR_INVALID, "bad allocation request");
    DeviceGuard g(device);
    cudaError_t e = cudaMalloc(d_ptr, bytes);
    if (e != cudaSuccess) return fail(VC_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return VC_OK;
}

int vc_device_free(void* d_ptr) {
    cudaFree(d_ptr);
    return VC_OK;
}

int vc_memcpy_to_host(void* h_dst, const void* d_src, size_t bytes, void* stream) {
    if (!h_dst || !d_src) return fail(VC_ERR_INVALID, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    VC_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, s));
    VC_CUDA(cudaStreamSynchronize(s));
    return VC_OK;
}

int vc_ipc_handle(const void* d_ptr, void* handle_out) {
    if (!d_ptr || !handle_out) return fail(VC_ERR_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    VC_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    memcpy(handle_out, &h, sizeof(h));
    return VC_OK;
}

int vc_ipc_open(int device, const void* handle, void** d_ptr) {
    if (!handle || !d_ptr) return fail(VC_ERR_INVALID, "null argument");
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    VC_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return VC_OK;
}

int vc_ipc_close(void* d_ptr) {
    if (!d_ptr) return fail(VC_ERR_INVALID, "null argument");
    VC_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return VC_OK;
}

int vc_render_profiled(vc_volume* vol, const vc_render_params* p, uint8_t* d_rgba, uint64_t* d_counters,
                       void* stream, float* stage_ms) {
    if (!vol || !stage_ms) return fail(VC_ERR_INVALID, "null argument");
    int local_rows = 0;
    int rc = validate_params(p, &local_rows);
    if (rc) return rc;
    if (!d_rgba && local_rows > 0) return fail(VC_ERR_INVALID, "output buffer is null");
    DeviceGuard g(vol->device);
    std::lock_guard<std::mutex> lk(vol->mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    for (auto& e : ev) VC_CUDA(cudaEventCreate(&e));
    rc = render_impl(vol, p, d_rgba, d_counters, s, local_rows, ev);
    if (rc == VC_OK) {
        cudaError_t e = cudaEventSynchronize(ev[2]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&stage_ms[0], ev[0], ev[1]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&stage_ms[1], ev[1], ev[2]);
        if (e != cudaSuccess) rc = cuda_fail(e, "stage timing");
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return rc;
}

int vc_render_host(vc_volume* vol, const vc_render_params* p, uint8_t* h_rgba, uint64_t* h_counters,
                   float* ms) {
    if (!vol) return fail(VC_ERR_INVALID, "volume is null");
    int local_rows = 0;
    int rc = validate_params(p, &local_rows);
    if (rc) return rc;
    if (!h_rgba && local_rows > 0) return fail(VC_ERR_INVALID, "output buffer is null");
    DeviceGuard g(vol->device);
    std::lock_guard<std::mutex> lk(vol->mu);
    const size_t bytes = (size_t)local_rows * p->width * 4;
    if (bytes > vol->scratch_bytes) {
        cudaFree(vol->d_scratch);
        vol->d_scratch = nullptr;
        vol->scratch_bytes = 0;
        cudaError_t e = cudaMalloc(&vol->d_scratch, bytes);
        if (e != cudaSuccess) return fail(VC_ERR_NOMEM, std::string("cudaMalloc(frame): ") + cudaGetErrorString(e));
        vol->scratch_bytes = bytes;
    }
    cudaStream_t s = vol->host_stream;
    VC_CUDA(cudaEventRecord(vol->ev0, s));
    rc = render_impl(vol, p, vol->d_scratch, vol->d_counters, s, local_rows);
    if (rc) return rc;
    if (bytes) VC_CUDA(cudaMemcpyAsync(h_rgba, vol->d_scratch, bytes, cudaMemcpyDeviceToHost, s));
    if (h_counters)
        VC_CUDA(cudaMemcpyAsync(h_counters, vol->d_counters, VC_NUM_COUNTERS * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, s));
    VC_CUDA(cudaEventRecord(vol->ev1, s));
    VC_CUDA(cudaStreamSynchronize(s));
    if (ms) VC_CUDA(cudaEventElapsedTime(ms, vol->ev0, vol->ev1));
    return VC_OK;
}

// ---- point queries ------------------------------------------------------

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

}  // namespace

#ifdef VC_CHECKED
// point kernels: the volume (their vc_device.cuh reads) is the checked region
int point_regions(const vc_volume* vol) {
    Regions R;
    R.add(vol->d_data, vol->bytes + vc::VC_VOLUME_PAD);
    VC_CUDA(vc::vc_set_regions_points(R.lohi.data(), (int)(R.lohi.size() / 2), 0));
    return VC_OK;
}
#define VC_POINT_REGIONS(vol)           \
    do {                                \
        int _rc = point_regions(vol);   \
        if (_rc) return _rc;            \
    } while (0)
#else
#define VC_POINT_REGIONS(vol) \
    do {                      \
    } while (0)
#endif

int vc_sample_points(const vc_volume* vol, int interp, const double* h_pts, int64_t n, double* h_out) {
    if (!vol || (n > 0 && (!h_pts || !h_out))) return fail(VC_ERR_INVALID, "null argument");
    if (interp < 0 || interp > 2) return fail(VC_ERR_INVALID, "interp must be 0, 1 or 2");
    if (n <= 0) return VC_OK;
    DeviceGuard g(vol->device);
    DevBuf dp, dout;
    VC_CUDA(cudaMalloc(&dp.p, n * 3 * sizeof(double)));
    VC_CUDA(cudaMalloc(&dout.p, n * sizeof(double)));
    VC_CUDA(cudaMemcpy(dp.p, h_pts, n * 3 * sizeof(double), cudaMemcpyHostToDevice));
    VC_POINT_REGIONS(vol);
    VC_CUDA(vc::launch_sample_points(vol->dtype, vol->d_data, vol->nx, vol->ny, vol->nz, interp,
                                     (const double*)dp.p, n, (double*)dout.p, 0));
    VC_CUDA(cudaMemcpy(h_out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    return VC_OK;
}

int vc_gradient_points(const vc_volume* vol, int op, const double* h_pts, int64_t n, double* h_out) {
    if (!vol || (n > 0 && (!h_pts || !h_out))) return fail(VC_ERR_INVALID, "null argument");
    if (op < 0 || op > 2) return fail(VC_ERR_INVALID, "op must be 0, 1 or 2");
    if (n <= 0) return VC_OK;
    DeviceGuard g(vol->device);
    DevBuf dp, dout;
    VC_CUDA(cudaMalloc(&dp.p, n * 3 * sizeof(double)));
    VC_CUDA(cudaMalloc(&dout.p, n * 3 * sizeof(double)));
    VC_CUDA(cudaMemcpy(dp.p, h_pts, n * 3 * sizeof(double), cudaMemcpyHostToDevice));
    VC_POINT_REGIONS(vol);
    VC_CUDA(vc::launch_gradient_points(vol->dtype, vol->d_data, vol->nx, vol->ny, vol->nz, op,
                                       (const double*)dp.p, n, (double*)dout.p, 0));
    VC_CUDA(cudaMemcpy(h_out, dout.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost));
    return VC_OK;
}

int vc_box_interval_rays(const double* h_rays, int64_t n, const double lo[3], const double hi[3],
                         double* h_out) {
    if (n > 0 && (!h_rays || !h_out || !lo || !hi)) return fail(VC_ERR_INVALID, "null argument");
    if (n <= 0) return VC_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(VC_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    DevBuf dr, dbox, dout;
    double lohi[6] = {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]};
    VC_CUDA(cudaMalloc(&dr.p, n * 6 * sizeof(double)));
    VC_CUDA(cudaMalloc(&dbox.p, sizeof(lohi)));
    VC_CUDA(cudaMalloc(&dout.p, n * 3 * sizeof(double)));
    VC_CUDA(cudaMemcpy(dr.p, h_rays, n * 6 * sizeof(double), cudaMemcpyHostToDevice));
    VC_CUDA(cudaMemcpy(dbox.p, lohi, sizeof(lohi), cudaMemcpyHostToDevice));
    VC_CUDA(vc::launch_box_rays((const double*)dr.p, n, (const double*)dbox.p, (double*)dout.p, 0));
    VC_CUDA(cudaMemcpy(h_out, dout.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost));
    return VC_OK;
}

int vc_first_hit_rays(const vc_volume* vol, const double* h_rays, int64_t n, double coarse, double fine,
                      double t_low, double t_high, int interp, double* h_out, uint64_t* h_samples) {
    if (!vol || (n > 0 && (!h_rays || !h_out))) return fail(VC_ERR_INVALID, "null argument");
    if (!(coarse > 0.0) || !(fine > 0.0) || fine > coarse)
        return fail(VC_ERR_INVALID, "need 0 < fine_step <= coarse_step");
    if (interp < 0 || interp > 2) return fail(VC_ERR_INVALID, "interp must be 0, 1 or 2");
    if (n <= 0) return VC_OK;
    DeviceGuard g(vol->device);
    DevBuf dr, dout, dc;
    VC_CUDA(cudaMalloc(&dr.p, n * 8 * sizeof(double)));
    VC_CUDA(cudaMalloc(&dout.p, n * 4 * sizeof(double)));
    VC_CUDA(cudaMalloc(&dc.p, sizeof(unsigned long long)));
    VC_CUDA(cudaMemset(dc.p, 0, sizeof(unsigned long long)));
    VC_CUDA(cudaMemcpy(dr.p, h_rays, n * 8 * sizeof(double), cudaMemcpyHostToDevice));
    VC_POINT_REGIONS(vol);
    VC_CUDA(vc::launch_first_hit_rays(vol->dtype, vol->d_data, vol->nx, vol->ny, vol->nz, make_raypos(vol),
                                      (const double*)dr.p, n, coarse, fine, t_low, t_high, interp,
                                      (double*)dout.p, (unsigned long long*)dc.p, 0));
    VC_CUDA(cudaMemcpy(h_out, dout.p, n * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    if (h_samples) VC_CUDA(cudaMemcpy(h_samples, dc.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return VC_OK;
}

int vc_bisect_rays(const vc_volume* vol, const double* h_rays, int64_t n, double t_low, double t_high,
                   int iters, int interp, double* h_out, uint64_t* h_samples) {
    if (!vol || (n > 0 && (!h_rays || !h_out))) return fail(VC_ERR_INVALID, "null argument");
    if (iters < 0) return fail(VC_ERR_INVALID, "iters must be >= 0");
    if (interp < 0 || interp > 2) return fail(VC_ERR_INVALID, "interp must be 0, 1 or 2");
    if (n <= 0) return VC_OK;
    DeviceGuard g(vol->device);
    DevBuf dr, dout, dc;
    VC_CUDA(cudaMalloc(&dr.p, n * 8 * sizeof(double)));
    VC_CUDA(cudaMalloc(&dout.p, n * sizeof(double)));
    VC_CUDA(cudaMalloc(&dc.p, sizeof(unsigned long long)));
    VC_CUDA(cudaMemset(dc.p, 0, sizeof(unsigned long long)));
    VC_CUDA(cudaMemcpy(dr.p, h_rays, n * 8 * sizeof(double), cudaMemcpyHostToDevice));
    VC_POINT_REGIONS(vol);
    VC_CUDA(vc::launch_bisect_rays(vol->dtype, vol->d_data, vol->nx, vol->ny, vol->nz, make_raypos(vol),
                                   (const double*)dr.p, n, t_low, t_high, iters, interp, (double*)dout.p,
                                   (unsigned long long*)dc.p, 0));
    VC_CUDA(cudaMemcpy(h_out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (h_samples) VC_CUDA(cudaMemcpy(h_samples, dc.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return VC_OK;
}

}  // extern "C"
