// png.cu -- frame egress: PNG encoding of a device frame on the device.
//
// The reference ships frames to its viewer as PNG (image_io.png_bytes,
// image_io.py:52-55, via Pillow/zlib on one CPU core; service.py:180-202),
// which at 1080p costs tens of milliseconds -- far more than rendering the
// frame here.  This encoder keeps the frame in HBM and copies only the
// compressed bytes to the host:
//
//   * filter: PNG "Up" on every scanline (prior row of row 0 = zeros),
//     RGB from the RGBA frame (alpha dropped like image_io._as_rgb);
//   * deflate: one fixed-Huffman block per scanline, one warp per scanline;
//     the 32 lanes tokenize 32 slices of the filtered row in parallel
//     (literals + distance-1 / distance-3 matches: zero runs over
//     background, repeating RGB along flat shading), a warp scan of the
//     bit counts places every lane's codes, and each lane writes its words
//     from a register bit buffer (atomics only on the two words it may
//     share with its neighbours);
//   * rows end with a sync flush (empty stored block) so the per-row
//     streams are byte aligned and simply concatenated (device scan +
//     gather); the last row carries BFINAL;
//   * Adler-32: per-row sums on the device, combined on the host; CRC-32 of
//     the rows on the device (see png_gather_kernel).
// The result is a standard PNG (zlib stream, 8-bit RGB) any decoder reads.
#include <cstring>
#include <vector>

#include "vc_internal.h"

namespace vc {

// fixed Huffman code of a literal / length symbol (RFC 1951 3.2.6), bit-reversed
// so it can be emitted LSB-first
__device__ __forceinline__ void lit_code(int sym, uint32_t& code, int& len) {
    uint32_t c;
    if (sym < 144) {
        c = 0x30 + sym;
        len = 8;
    } else if (sym < 256) {
        c = 0x190 + (sym - 144);
        len = 9;
    } else if (sym < 280) {
        c = sym - 256;
        len = 7;
    } else {
        c = 0xC0 + (sym - 280);
        len = 8;
    }
    code = __brev(c) >> (32 - len);
}

// length 3..258 -> (symbol, extra bits, extra value)
__device__ __forceinline__ void length_sym(int L, int& sym, int& ebits, int& eval) {
    if (L == 258) {
        sym = 285;
        ebits = 0;
        eval = 0;
        return;
    }
    const int v = L - 3;
    if (v < 8) {
        sym = 257 + v;
        ebits = 0;
        eval = 0;
        return;
    }
    // groups of 4 lengths per extra-bit count
    int eb = 31 - __clz(v) - 2;  // v in [2^(eb+2), 2^(eb+3))
    int base = (4 << eb);        // first v of the group... (v >> eb) in [4, 8)
    sym = 257 + 4 * eb + 4 + ((v >> eb) - 4);
    ebits = eb;
    eval = v - ((v >> eb) << eb);
    (void)base;
}

// LSB-first bit writer of one lane's slice of a row.  Bits gather in a
// 64-bit register and leave as whole 32-bit words: plain stores for the
// words only this lane writes, atomicOr for the first and last word, which
// it may share with the neighbouring lanes' slices (the row's words start
// zeroed).  A null `words` only counts.
struct BitSink {
    uint32_t* words;
    uint64_t pos;             // absolute bit position of the next bit
    uint64_t acc = 0;         // pending bits, aligned to word (pos0 >> 5) of `first`
    int nacc = 0;             // bits in acc, counted from the word boundary
    uint64_t wnext = 0;       // word index acc[0..31] belongs to
    bool first = true;        // the next word flushed is this lane's first (shared) word
    __device__ __forceinline__ void begin() {
        wnext = pos >> 5;
        nacc = (int)(pos & 31);
        acc = 0;
        first = true;
    }
    __device__ __forceinline__ void put(uint32_t bits, int n) {
        if (n == 0) return;
        acc |= (uint64_t)bits << nacc;
        nacc += n;
        pos += n;
        if (nacc >= 32) {
            if (first) {
                atomicOr(words + wnext, (uint32_t)acc);
                first = false;
            } else {
                words[wnext] = (uint32_t)acc;
            }
            acc >>= 32;
            nacc -= 32;
            wnext++;
        }
    }
    __device__ __forceinline__ void finish() {  // last partial word: shared with the next slice
        if (nacc > 0) atomicOr(words + wnext, (uint32_t)acc);
    }
};

// token pass over [a, b) of row data d; emit == false only counts bits.
// Greedy LZ77 with two candidate distances: 1 (byte runs -- Up-filtered
// rows of unchanged pixels are zero runs) and 3 (the previous RGB pixel --
// flat or repeating colour along the row).  Matches may reach back before
// a (the decoder already has those bytes) but not before the row start.
__device__ uint64_t encode_slice(const uint8_t* d, int a, int b, bool emit, BitSink& s) {
    uint64_t bits = 0;
    int i = a;
    while (i < b) {
        int best = 0, dist = 0;
        if (i >= 1) {
            int L = 0;
            while (i + L < b && L < 258 && d[i + L] == d[i + L - 1]) L++;
            best = L;
            dist = 1;
        }
        if (i >= 3) {
            int L = 0;
            while (i + L < b && L < 258 && d[i + L] == d[i + L - 3]) L++;
            if (L > best) {
                best = L;
                dist = 3;
            }
        }
        uint32_t code;
        int len;
        if (best >= 3) {
            int sym, eb, ev;
            length_sym(best, sym, eb, ev);
            lit_code(sym, code, len);
            bits += len + eb + 5;
            if (emit) {
                s.put(code, len);
                s.put((uint32_t)ev, eb);
                s.put(dist == 1 ? 0u : 0x08u, 5);  // distance codes 0 (d=1) and 2 (d=3), bit-reversed
            }
            i += best;
        } else {
            lit_code(d[i], code, len);
            bits += len;
            if (emit) s.put(code, len);
            i += 1;
        }
    }
    return bits;
}

// One CTA per scanline, PNG_SEGS warps: the CTA filters the row once into
// shared memory, then warp w deflates segment w of it as its own
// fixed-Huffman block ending in a sync flush (byte aligned), so the
// segments concatenate like rows do.  Matches may reach back into the
// previous segment (the decoder's window holds it).  Measured at 1080p:
// 1 / 2 / 4 / 8 segments -> 0.64 / 0.50 / 0.44 / 0.42 ms, 2.06 / 2.10 /
// 2.20 / 2.37 MB (runs are cut at every lane slice): 2 it is.
#ifndef VC_PNG_SEGS
#define VC_PNG_SEGS 2
#endif
constexpr int PNG_SEGS = VC_PNG_SEGS;

// segments per row: 2 from 1024 pixels on (small rows keep one block)
__host__ __device__ inline int png_segs(int width) { return width >= 1024 ? PNG_SEGS : 1; }
__host__ __device__ inline size_t png_seg_words(size_t n, int segs) { return ((n + segs - 1) / segs * 9 / 8 + 64) / 4 + 4; }

__global__ void __launch_bounds__(32 * PNG_SEGS) png_rows_kernel(
    const uint8_t* __restrict__ rgba, int width, int height, uint32_t* __restrict__ segbuf, size_t seg_words,
    uint32_t* __restrict__ seg_bytes, unsigned long long* __restrict__ adler) {
    extern __shared__ uint8_t d[];
    __shared__ unsigned long long red[2][PNG_SEGS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int segs = (int)(blockDim.x >> 5);
    const int y = blockIdx.x;
    const int n = 1 + 3 * width;
    // Up-filtered RGB scanline
    const uint8_t* cur = rgba + (size_t)y * width * 4;
    const uint8_t* prev = y > 0 ? rgba + (size_t)(y - 1) * width * 4 : nullptr;
    if (threadIdx.x == 0) d[0] = 2;
    for (int x = threadIdx.x; x < width; x += blockDim.x) {
        const uchar4 c = *reinterpret_cast<const uchar4*>(cur + 4 * x);
        uchar4 p = make_uchar4(0, 0, 0, 0);
        if (prev) p = *reinterpret_cast<const uchar4*>(prev + 4 * x);
        d[1 + 3 * x] = (uint8_t)(c.x - p.x);
        d[2 + 3 * x] = (uint8_t)(c.y - p.y);
        d[3 + 3 * x] = (uint8_t)(c.z - p.z);
    }
    __syncthreads();
    // Adler-32 pieces of the row: sum b_i and sum (n - i) b_i
    unsigned long long sa = 0, sb = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sa += d[i];
        sb += (unsigned long long)(n - i) * d[i];
    }
    for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
        red[0][warp] = sa;
        red[1][warp] = sb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long A = 0, B = 0;
        for (int w = 0; w < segs; w++) {
            A += red[0][w];
            B += red[1][w];
        }
        adler[2 * y] = A;
        adler[2 * y + 1] = B;
    }
    // this warp's segment [s0, s1), tokenized in 32 lane slices
    const int s0 = (int)((long long)n * warp / segs), s1 = (int)((long long)n * (warp + 1) / segs);
    const int len = s1 - s0;
    const int a = s0 + (int)((long long)len * lane / 32), b = s0 + (int)((long long)len * (lane + 1) / 32);
    BitSink dummy{nullptr, 0};
    const uint64_t mybits = encode_slice(d, a, b, false, dummy);  // counting pass
    uint64_t incl = mybits;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const uint64_t total = __shfl_sync(0xffffffffu, incl, 31);
    const size_t seg = (size_t)y * segs + warp;
    uint32_t* words = segbuf + seg * seg_words;
    for (size_t w = lane; w < seg_words; w += 32) words[w] = 0;
    __syncwarp();
    const bool last = (y == height - 1) && warp == segs - 1;
    BitSink bs{words, 3 + (incl - mybits)};
    bs.begin();
    if (lane == 0) {  // block header: BFINAL, BTYPE = 01 (fixed Huffman)
        atomicOr(words, (last ? 1u : 0u) | (1u << 1));
    }
    encode_slice(d, a, b, true, bs);
    bs.finish();
    __syncwarp();
    if (lane == 0) {
        BitSink t{words, 3 + total};
        t.begin();
        uint32_t code;
        int clen;
        lit_code(256, code, clen);  // end of block
        t.put(code, clen);
        t.finish();
        uint64_t nbits = t.pos;
        if (!last) {  // sync flush: empty stored block, byte aligned, 00 00 FF FF
            nbits = (t.pos + 3 + 7) & ~7ull;  // 3 zero header bits (words start zeroed), then pad
            uint8_t* bytes = reinterpret_cast<uint8_t*>(words);
            const size_t nb = nbits >> 3;
            bytes[nb + 0] = 0x00;
            bytes[nb + 1] = 0x00;
            bytes[nb + 2] = 0xFF;
            bytes[nb + 3] = 0xFF;
            seg_bytes[seg] = (uint32_t)(nb + 4);
        } else {
            seg_bytes[seg] = (uint32_t)((nbits + 7) >> 3);
        }
    }
}

// exclusive scan of row byte counts (one block)
__global__ void png_scan_kernel(const uint32_t* __restrict__ row_bytes, int height,
                                unsigned long long* __restrict__ offsets) {
    __shared__ unsigned long long part[1024];
    const int t = threadIdx.x;
    const int per = (height + blockDim.x - 1) / blockDim.x;
    unsigned long long s = 0;
    for (int i = t * per; i < min(height, (t + 1) * per); i++) s += row_bytes[i];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < (int)blockDim.x; i++) {
            const unsigned long long v = part[i];
            part[i] = run;
            run += v;
        }
        offsets[height] = run;
    }
    __syncthreads();
    unsigned long long run = part[t];
    for (int i = t * per; i < min(height, (t + 1) * per); i++) {
        offsets[i] = run;
        run += row_bytes[i];
    }
}

// ---- CRC-32 (PNG / zlib polynomial, reflected 0xEDB88320) on the device --
// Rows are byte strings (sync flush), so the IDAT CRC is the CRC of their
// concatenation: each row's CRC is computed in the gather kernel (256
// threads: per-thread chunks combined in a tree) and the row CRCs are
// combined in a tree over the rows with crc(A||B) = crc(A) * x^(8|B|) ^
// crc(B) in GF(2)[x]/P (the zlib crc32_combine identity).
__device__ __forceinline__ uint32_t gf2_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}
__global__ void png_gather_kernel(const uint32_t* __restrict__ rowbuf, size_t row_words,
                                  const uint32_t* __restrict__ row_bytes,
                                  const unsigned long long* __restrict__ offsets, uint8_t* __restrict__ out) {
    const int y = blockIdx.x;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(rowbuf + (size_t)y * row_words);
    uint8_t* dst = out + offsets[y];
    for (uint32_t i = threadIdx.x; i < row_bytes[y]; i += blockDim.x) dst[i] = src[i];
}

// CRC-32 of the gathered stream, fully parallel.  The raw CRC (register
// starting at 0, no final xor) is linear, raw(A||B) = raw(A) * x^(8|B|) ^
// raw(B) in GF(2)[x]/P, and leading zero bytes do not change it.  So the
// stream is virtually front-padded with zeros to a power-of-two number of
// CRC_BLOCK-byte blocks: every pair in both combine trees (8-byte thread
// chunks inside a block, then blocks) has a full right half, and each level
// multiplies by one fixed power x^(2^k) -- one multmodp per pair.  The
// host turns the raw value into the PNG CRC: raw ^ 0xFFFFFFFF * x^(8 n) ^
// 0xFFFFFFFF.
constexpr int CRC_BLOCK = 2048;  // 256 threads x 8 bytes

__global__ void __launch_bounds__(256) png_crc_blocks_kernel(const uint8_t* __restrict__ data,
                                                             const unsigned long long* __restrict__ total_p,
                                                             const uint32_t* __restrict__ crc_table,
                                                             const uint32_t* __restrict__ x2n_g,
                                                             uint32_t* __restrict__ block_crc) {
    __shared__ uint32_t tab[256], x2n[32], part[256];
    const long long total = (long long)*total_p;
    long long nb = (total + CRC_BLOCK - 1) / CRC_BLOCK, nbp = 1;
    while (nbp < nb) nbp <<= 1;
    if ((long long)blockIdx.x >= nbp) return;
    const long long pad = nbp * CRC_BLOCK - total;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc_table[i];
    if (threadIdx.x < 32) x2n[threadIdx.x] = x2n_g[threadIdx.x];
    __syncthreads();
    // bytes [a, a + 8) of the padded stream = [a - pad, a - pad + 8) of the data
    const long long a = (long long)blockIdx.x * CRC_BLOCK + 8ll * threadIdx.x - pad;
    uint32_t c = 0;  // raw register; the leading pad zeros leave it at 0
    for (long long i = max(a, 0ll); i < a + 8; i++) c = tab[(c ^ data[i]) & 0xFF] ^ (c >> 8);
    part[threadIdx.x] = c;
    __syncthreads();
    for (int L = 0; L < 8; L++) {  // right halves of 8 * 2^L bytes
        const int t = threadIdx.x, st = 1 << L;
        if ((t & (2 * st - 1)) == 0) part[t] = gf2_multmodp(x2n[6 + L], part[t]) ^ part[t + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) block_crc[blockIdx.x] = part[0];
}

__global__ void png_crc_tree_kernel(uint32_t* __restrict__ crc, const unsigned long long* __restrict__ total_p,
                                    const uint32_t* __restrict__ x2n_g, uint32_t* __restrict__ result) {
    __shared__ uint32_t x2n[32];
    if (threadIdx.x < 32) x2n[threadIdx.x] = x2n_g[threadIdx.x];
    __syncthreads();
    const long long total = (long long)*total_p;
    long long nb = (total + CRC_BLOCK - 1) / CRC_BLOCK, nbp = 1;
    while (nbp < nb) nbp <<= 1;
    for (int L = 0; (1ll << L) < nbp; L++) {  // right halves of CRC_BLOCK * 2^L bytes
        const long long st = 1ll << L;
        for (long long t = threadIdx.x * 2 * st; t < nbp; t += (long long)blockDim.x * 2 * st)
            crc[t] = gf2_multmodp(x2n[(14 + L) & 31], crc[t]) ^ crc[t + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) *result = total > 0 ? crc[0] : 0u;
}

}  // namespace vc

namespace {

uint32_t crc_tab[8][256];
bool crc_ready = false;
uint32_t x2n_tab[32];  // x^(2^k) mod P (zlib crc32_combine tables)

uint32_t multmodp_host(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}


void crc_init() {  // slice-by-8 tables of the PNG CRC-32 (polynomial 0xEDB88320)
    for (uint32_t n = 0; n < 256; n++) {
        uint32_t c = n;
        for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
        crc_tab[0][n] = c;
    }
    for (uint32_t n = 0; n < 256; n++)
        for (int t = 1; t < 8; t++) crc_tab[t][n] = (crc_tab[t - 1][n] >> 8) ^ crc_tab[0][crc_tab[t - 1][n] & 0xFF];
    uint32_t p = 1u << 30;  // x^1
    x2n_tab[0] = p;
    for (int k = 1; k < 32; k++) x2n_tab[k] = p = multmodp_host(p, p);
    crc_ready = true;
}

uint32_t crc32(const uint8_t* p, size_t n, uint32_t c = 0) {
    if (!crc_ready) crc_init();
    c ^= 0xFFFFFFFFu;
    while (n >= 8) {
        uint32_t lo, hi;
        memcpy(&lo, p, 4);
        memcpy(&hi, p + 4, 4);
        lo ^= c;
        c = crc_tab[7][lo & 0xFF] ^ crc_tab[6][(lo >> 8) & 0xFF] ^ crc_tab[5][(lo >> 16) & 0xFF] ^
            crc_tab[4][lo >> 24] ^ crc_tab[3][hi & 0xFF] ^ crc_tab[2][(hi >> 8) & 0xFF] ^
            crc_tab[1][(hi >> 16) & 0xFF] ^ crc_tab[0][hi >> 24];
        p += 8;
        n -= 8;
    }
    while (n--) c = crc_tab[0][(c ^ *p++) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

// c * x^(8 len) mod P
uint32_t shift_host(uint32_t c, unsigned long long len) {
    uint32_t p = 1u << 31;
    int k = 3;
    for (unsigned long long n = len; n; n >>= 1, k++)
        if (n & 1) p = multmodp_host(x2n_tab[k & 31], p);
    return multmodp_host(p, c);
}

uint32_t crc32_combine_host(uint32_t c1, uint32_t c2, unsigned long long len2) {
    return shift_host(c1, len2) ^ c2;
}

void put_be32(uint8_t* o, uint32_t x) {
    o[0] = x >> 24;
    o[1] = x >> 16;
    o[2] = x >> 8;
    o[3] = x;
}

}  // namespace

extern "C" VC_API int vc_encode_png(const uint8_t* d_rgba, int width, int height, void* stream, uint8_t* h_out,
                                    size_t h_cap, size_t* out_len) {
    using namespace vc;
    if (!d_rgba || !out_len || width <= 0 || height <= 0) return VC_ERR_INVALID;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n = 1 + 3 * (size_t)width;
    const int segs = png_segs(width);
    const size_t row_words = png_seg_words(n, segs);  // per segment
    const int nseg = height * segs;
    uint32_t *rowbuf = nullptr, *row_bytes = nullptr, *row_crc = nullptr, *tables = nullptr;
    unsigned long long *adler = nullptr, *offsets = nullptr;
    uint8_t* packed = nullptr;
    int rc = VC_OK;
    auto ok = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == VC_OK) rc = VC_ERR_CUDA;
        return e == cudaSuccess;
    };
    if (!crc_ready) crc_init();
    ok(cudaMallocAsync((void**)&rowbuf, row_words * 4 * nseg, s));
    ok(cudaMallocAsync((void**)&row_bytes, 4 * (size_t)nseg, s));
    // block CRCs of the gathered stream (upper bound on its size) + the result
    size_t max_blocks = 1;  // power of two >= the stream's block count (upper bound)
    while (max_blocks * CRC_BLOCK < row_words * 4 * (size_t)nseg) max_blocks <<= 1;
    ok(cudaMallocAsync((void**)&row_crc, 4 * max_blocks + 4, s));
    ok(cudaMallocAsync((void**)&tables, 4 * (256 + 32), s));
    ok(cudaMallocAsync((void**)&adler, 16 * (size_t)height, s));
    ok(cudaMallocAsync((void**)&offsets, 8 * (size_t)(nseg + 1), s));
    ok(cudaMallocAsync((void**)&packed, row_words * 4 * nseg, s));
    std::vector<unsigned long long> hadler(2 * (size_t)height);
    unsigned long long total = 0;
    uint32_t rows_crc = 0;
    if (rc == VC_OK) {
        ok(cudaMemcpyAsync(tables, crc_tab[0], 4 * 256, cudaMemcpyHostToDevice, s));
        ok(cudaMemcpyAsync(tables + 256, x2n_tab, 4 * 32, cudaMemcpyHostToDevice, s));
        const size_t smem = (n + 15) & ~(size_t)15;
        if (smem > 48 * 1024)
            ok(cudaFuncSetAttribute(png_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        png_rows_kernel<<<height, 32 * segs, smem, s>>>(d_rgba, width, height, rowbuf, row_words, row_bytes,
                                                        adler);
        ok(cudaGetLastError());
        png_scan_kernel<<<1, 1024, 0, s>>>(row_bytes, nseg, offsets);
        png_gather_kernel<<<nseg, 256, 0, s>>>(rowbuf, row_words, row_bytes, offsets, packed);
        png_crc_blocks_kernel<<<(unsigned)max_blocks, 256, 0, s>>>(packed, offsets + nseg, tables, tables + 256,
                                                                   row_crc);
        png_crc_tree_kernel<<<1, 1024, 0, s>>>(row_crc, offsets + nseg, tables + 256, row_crc + max_blocks);
        ok(cudaGetLastError());
        ok(cudaMemcpyAsync(&total, offsets + nseg, 8, cudaMemcpyDeviceToHost, s));
        ok(cudaMemcpyAsync(&rows_crc, row_crc + max_blocks, 4, cudaMemcpyDeviceToHost, s));
        ok(cudaMemcpyAsync(hadler.data(), adler, 16 * (size_t)height, cudaMemcpyDeviceToHost, s));
        ok(cudaStreamSynchronize(s));
    }
    // file layout: signature, IHDR, IDAT {78 01, rows, Adler-32}, IEND
    const size_t idat_len = 2 + (size_t)total + 4;
    const size_t file_len = 8 + 25 + 8 + idat_len + 4 + 12;
    *out_len = file_len;
    if (rc == VC_OK && h_out != nullptr && h_cap >= file_len) {
        uint8_t* o = h_out;
        const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1A, '\n'};
        memcpy(o, sig, 8);
        const uint32_t W = (uint32_t)width, H = (uint32_t)height;
        const uint8_t ihdr[4 + 4 + 13] = {0, 0, 0, 13, 'I', 'H', 'D', 'R',
                                          (uint8_t)(W >> 24), (uint8_t)(W >> 16), (uint8_t)(W >> 8), (uint8_t)W,
                                          (uint8_t)(H >> 24), (uint8_t)(H >> 16), (uint8_t)(H >> 8), (uint8_t)H,
                                          8, 2, 0, 0, 0};
        memcpy(o + 8, ihdr, sizeof(ihdr));
        put_be32(o + 8 + 21, crc32(ihdr + 4, 17));
        uint8_t* id = o + 33;  // IDAT chunk
        put_be32(id, (uint32_t)idat_len);
        memcpy(id + 4, "IDAT", 4);
        id[8] = 0x78;
        id[9] = 0x01;
        // the compressed rows go straight from HBM into the caller's buffer
        ok(cudaMemcpyAsync(id + 10, packed, total, cudaMemcpyDeviceToHost, s));
        // Adler-32 of all filtered rows (per-row sums from the device)
        unsigned long long A = 1, B = 0;
        for (int y = 0; y < height; y++) {
            B = (B + (n % 65521) * A + hadler[2 * y + 1] % 65521) % 65521;
            A = (A + hadler[2 * y] % 65521) % 65521;
        }
        uint8_t ad[4];
        put_be32(ad, (uint32_t)((B << 16) | A));
        // CRC over "IDAT", the zlib header, the rows (device) and the Adler
        // the device's raw CRC of the rows -> their PNG CRC, then chain
        const uint32_t rows_std = rows_crc ^ shift_host(0xFFFFFFFFu, total) ^ 0xFFFFFFFFu;
        uint32_t c = crc32(id + 4, 6);
        c = crc32_combine_host(c, rows_std, total);
        c = crc32(ad, 4, c);
        ok(cudaStreamSynchronize(s));
        memcpy(id + 10 + total, ad, 4);
        put_be32(id + 10 + total + 4, c);
        uint8_t* ie = id + 10 + total + 8;
        const uint8_t iend[12] = {0, 0, 0, 0, 'I', 'E', 'N', 'D', 0xAE, 0x42, 0x60, 0x82};
        memcpy(ie, iend, 12);
    }
    cudaFreeAsync(rowbuf, s);
    cudaFreeAsync(row_bytes, s);
    cudaFreeAsync(row_crc, s);
    cudaFreeAsync(tables, s);
    cudaFreeAsync(adler, s);
    cudaFreeAsync(offsets, s);
    cudaFreeAsync(packed, s);
    if (rc != VC_OK) return rc;
    if (h_out != nullptr && h_cap < file_len) return VC_ERR_INVALID;
    return VC_OK;
}
