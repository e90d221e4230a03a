// png.cu -- frame egress: PNG encoding of a device frame on the device.
//
// The reference ships frames to its viewer as PNG (image_io.png_bytes,
// image_io.py:52-55, via Pillow/zlib on one CPU core; service.py:180-202),
// which at 1080p costs hundreds of milliseconds -- far more than rendering
// the frame here.  This encoder keeps the frame in HBM and copies only the
// compressed bytes to the host:
//
//   * filter: PNG "Up" on every scanline (prior row of row 0 = zeros), RGB
//     from the RGBA frame (alpha dropped like image_io._as_rgb);
//   * tokens: one CTA per scanline, each of its TOK_LANES threads tokenizes
//     a slice of the filtered row (literals + distance-1 / distance-3
//     matches: zero runs over background, repeating RGB along flat shading)
//     into a token buffer and a shared symbol histogram;
//   * code: the frame is ONE dynamic-Huffman deflate block.  The host turns
//     the histogram into length-limited canonical codes (package-merge) and
//     the block header; every thread then knows its bit count, a scan gives
//     its bit offset, and all threads write their codes in parallel at those
//     offsets (whole words from a register bit buffer, atomics only on the
//     two words a slice may share with its neighbours);
//   * Adler-32: per-row sums on the device, combined on the host; CRC-32 of
//     the stream on the device (block tree, see png_crc_blocks_kernel).
// The result is a standard PNG (zlib stream, 8-bit RGB) any decoder reads;
// one shared table makes it about as small as zlib level 6.
#include <algorithm>
#include <cstring>
#include <iterator>
#include <vector>

#include "vc_internal.h"

namespace vc {

constexpr int TOK_LANES = 64;  // tokenizing threads per scanline
constexpr int NLIT = 286, NDIST = 30;

// length 3..258 -> (symbol, extra bits, extra value), RFC 1951 3.2.5
__host__ __device__ inline void length_sym(int L, int& sym, int& ebits, int& eval) {
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
    int eb = 0;  // v in [2^(eb+2), 2^(eb+3))
    while ((v >> (eb + 3)) != 0) eb++;
    sym = 257 + 4 * eb + 4 + ((v >> eb) - 4);
    ebits = eb;
    eval = v - ((v >> eb) << eb);
}

// token: symbol (9 bits) | extra-bit count (3) | extra value (5) | distance (2: 0 none, 1 -> d=1, 2 -> d=3)
__device__ __forceinline__ uint32_t make_token(int sym, int eb, int ev, int dist) {
    return (uint32_t)sym | ((uint32_t)eb << 9) | ((uint32_t)ev << 12) | ((uint32_t)dist << 17);
}

// LSB-first bit writer of one thread's slice of the stream.  Bits gather in a
// 64-bit register and leave as whole 32-bit words: plain stores for words
// only this thread writes, atomicOr for its first and last word, which it
// may share with its neighbours (the buffer starts zeroed).
struct BitSink {
    uint32_t* words;
    uint64_t pos;
    uint64_t acc = 0;
    int nacc = 0;
    uint64_t wnext = 0;
    bool first = true;
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
    __device__ __forceinline__ void finish() {
        if (nacc > 0) atomicOr(words + wnext, (uint32_t)acc);
    }
};

__host__ __device__ inline int tok_slice_max(int n) { return (n + TOK_LANES - 1) / TOK_LANES + 1; }

// Filter + tokenize one scanline per CTA.  Greedy LZ77 with two candidate
// distances, 1 (byte runs -- Up-filtered rows of unchanged pixels are zero
// runs) and 3 (the previous RGB pixel); a match may reach back before the
// slice (the decoder has those bytes) but not before the row start.
__global__ void __launch_bounds__(TOK_LANES) png_tokenize_kernel(
    const uint8_t* __restrict__ rgba, int width, int height, uint32_t* __restrict__ tokens,
    uint32_t* __restrict__ ntok, unsigned int* __restrict__ hist, unsigned long long* __restrict__ adler) {
    extern __shared__ uint8_t d[];
    __shared__ unsigned int h[NLIT + NDIST];
    __shared__ unsigned long long red[2][TOK_LANES / 32];
    const int y = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = 1 + 3 * width;
    for (int i = t; i < NLIT + NDIST; i += blockDim.x) h[i] = 0;
    const uint8_t* cur = rgba + (size_t)y * width * 4;
    const uint8_t* prev = y > 0 ? rgba + (size_t)(y - 1) * width * 4 : nullptr;
    if (t == 0) d[0] = 2;  // filter type Up
    for (int x = t; x < width; x += blockDim.x) {
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
    for (int i = t; i < n; i += blockDim.x) {
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
    // this thread's slice
    const int a = (int)((long long)n * t / TOK_LANES), b = (int)((long long)n * (t + 1) / TOK_LANES);
    uint32_t* out = tokens + ((size_t)y * TOK_LANES + t) * tok_slice_max(n);
    int k = 0, i = a;
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
        if (best >= 3) {
            int sym, eb, ev;
            length_sym(best, sym, eb, ev);
            out[k++] = make_token(sym, eb, ev, dist == 1 ? 1 : 2);
            atomicAdd(&h[sym], 1u);
            atomicAdd(&h[NLIT + (dist == 1 ? 0 : 2)], 1u);  // distance codes 0 (d=1), 2 (d=3)
            i += best;
        } else {
            out[k++] = make_token(d[i], 0, 0, 0);
            atomicAdd(&h[d[i]], 1u);
            i += 1;
        }
    }
    ntok[(size_t)y * TOK_LANES + t] = (uint32_t)k;
    __syncthreads();
    if (t == 0) {
        unsigned long long A = 0, B = 0;
        for (int w = 0; w < TOK_LANES / 32; w++) {
            A += red[0][w];
            B += red[1][w];
        }
        adler[2 * y] = A;
        adler[2 * y + 1] = B;
    }
    for (int s = t; s < NLIT + NDIST; s += blockDim.x)
        if (h[s]) atomicAdd(&hist[s], h[s]);
}

// Huffman code tables from the host: code (bit-reversed for LSB-first
// output) in the low 16 bits, length in the high 16
struct CodeTables {
    uint32_t lit[NLIT];
    uint32_t dist[NDIST];
};

__device__ __forceinline__ uint32_t token_bits(const CodeTables& c, uint32_t tk) {
    const int sym = tk & 511, eb = (tk >> 9) & 7, dist = (tk >> 17) & 3;
    uint32_t bits = (c.lit[sym] >> 16) + eb;
    if (dist) bits += c.dist[dist == 1 ? 0 : 2] >> 16;
    return bits;
}

// bit count of every slice, exclusive prefix within its row and the row total
__global__ void __launch_bounds__(TOK_LANES) png_bits_kernel(const uint32_t* __restrict__ tokens,
                                                             const uint32_t* __restrict__ ntok, int n,
                                                             const CodeTables* __restrict__ codes,
                                                             uint32_t* __restrict__ slice_prefix,
                                                             uint32_t* __restrict__ row_bits) {
    __shared__ CodeTables c;
    __shared__ uint32_t warp_sum[TOK_LANES / 32];
    for (int i = threadIdx.x; i < NLIT + NDIST; i += blockDim.x) (&c.lit[0])[i] = (&codes->lit[0])[i];
    __syncthreads();
    const size_t s = (size_t)blockIdx.x * TOK_LANES + threadIdx.x;
    const uint32_t* tk = tokens + s * tok_slice_max(n);
    uint32_t bits = 0;
    for (uint32_t k = 0; k < ntok[s]; k++) bits += token_bits(c, tk[k]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = bits;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; w++) before += warp_sum[w];
    slice_prefix[s] = before + incl - bits;
    if (threadIdx.x == blockDim.x - 1) row_bits[blockIdx.x] = before + incl;
}

__global__ void __launch_bounds__(TOK_LANES) png_emit_kernel(const uint32_t* __restrict__ tokens,
                                                             const uint32_t* __restrict__ ntok, int n,
                                                             const CodeTables* __restrict__ codes,
                                                             const unsigned long long* __restrict__ row_offsets,
                                                             const uint32_t* __restrict__ slice_prefix,
                                                             uint64_t header_bits, uint32_t* __restrict__ words) {
    __shared__ CodeTables c;
    for (int i = threadIdx.x; i < NLIT + NDIST; i += blockDim.x) (&c.lit[0])[i] = (&codes->lit[0])[i];
    __syncthreads();
    const size_t s = (size_t)blockIdx.x * TOK_LANES + threadIdx.x;
    const uint32_t* tk = tokens + s * tok_slice_max(n);
    BitSink bs{words, header_bits + row_offsets[blockIdx.x] + slice_prefix[s]};
    bs.begin();
    for (uint32_t k = 0; k < ntok[s]; k++) {
        const uint32_t t = tk[k];
        const int sym = t & 511, eb = (t >> 9) & 7, ev = (t >> 12) & 31, dist = (t >> 17) & 3;
        bs.put(c.lit[sym] & 0xFFFF, (int)(c.lit[sym] >> 16));
        bs.put((uint32_t)ev, eb);
        if (dist) {
            const uint32_t dc = c.dist[dist == 1 ? 0 : 2];
            bs.put(dc & 0xFFFF, (int)(dc >> 16));
        }
    }
    bs.finish();
}

// end of block after the last slice; the stream's byte length
__global__ void png_eob_kernel(const unsigned long long* __restrict__ offsets, int nslices, uint64_t header_bits,
                               const CodeTables* __restrict__ codes, uint32_t* __restrict__ words,
                               unsigned long long* __restrict__ total_bytes) {
    BitSink bs{words, header_bits + offsets[nslices]};
    bs.begin();
    bs.put(codes->lit[256] & 0xFFFF, (int)(codes->lit[256] >> 16));
    bs.finish();
    *total_bytes = (bs.pos + 7) >> 3;
}

// exclusive scan of the row bit counts (one block); offsets[count] = total
__global__ void png_scan_kernel(const uint32_t* __restrict__ vals, int count,
                                unsigned long long* __restrict__ offsets) {
    __shared__ unsigned long long part[1024];
    const int t = threadIdx.x;
    const int per = (count + blockDim.x - 1) / blockDim.x;
    unsigned long long s = 0;
    for (int i = t * per; i < min(count, (t + 1) * per); i++) s += vals[i];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < (int)blockDim.x; i++) {
            const unsigned long long v = part[i];
            part[i] = run;
            run += v;
        }
        offsets[count] = run;
    }
    __syncthreads();
    unsigned long long run = part[t];
    for (int i = t * per; i < min(count, (t + 1) * per); i++) {
        offsets[i] = run;
        run += vals[i];
    }
}

// ---- CRC-32 (PNG / zlib polynomial, reflected 0xEDB88320) on the device --
// a * b in GF(2)[x] / P, reflected bit order (zlib's multmodp)
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

// The raw CRC (register starting at 0, no final xor) is linear, raw(A||B) =
// raw(A) * x^(8|B|) ^ raw(B), and leading zero bytes do not change it.  So
// the stream is virtually front-padded with zeros to a power-of-two number
// of CRC_BLOCK-byte blocks: every pair in both combine trees (8-byte thread
// chunks inside a block, then blocks) has a full right half, and each level
// multiplies by one fixed power x^(2^k) -- one multmodp per pair.  The host
// turns the raw value into the PNG CRC: raw ^ 0xFFFFFFFF * x^(8 n) ^
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

using vc::NDIST;
using vc::NLIT;

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

uint32_t crc32_combine_host(uint32_t c1, uint32_t c2, unsigned long long len2) { return shift_host(c1, len2) ^ c2; }

void put_be32(uint8_t* o, uint32_t x) {
    o[0] = x >> 24;
    o[1] = x >> 16;
    o[2] = x >> 8;
    o[3] = x;
}

// ---- Huffman code construction (host) ---------------------------------
// Optimal code lengths limited to maxlen: package-merge in its prefix form.
// List j is merge(leaves, pairs of list j-1) by weight; the first 2m-2
// items of list maxlen are selected, and a selected prefix of list j holds
// p packages, which select the first 2p items of list j-1; every selected
// leaf adds one to its symbol's length.  O(maxlen * m), no per-item symbol
// sets.  A single used symbol gets length 1.
std::vector<int> limited_lengths(const std::vector<unsigned long long>& freq, int maxlen) {
    const int n = (int)freq.size();
    std::vector<int> len(n, 0);
    struct Item {
        unsigned long long w;
        int sym;  // >= 0 leaf, -1 package
    };
    std::vector<Item> leaves;
    for (int i = 0; i < n; i++)
        if (freq[i]) leaves.push_back({freq[i], i});
    const int m = (int)leaves.size();
    if (m == 0) return len;
    if (m == 1) {
        len[leaves[0].sym] = 1;
        return len;
    }
    std::stable_sort(leaves.begin(), leaves.end(), [](const Item& a, const Item& b) { return a.w < b.w; });
    std::vector<std::vector<Item>> lists(maxlen + 1);
    lists[1] = leaves;
    for (int j = 2; j <= maxlen; j++) {
        const std::vector<Item>& prev = lists[j - 1];
        std::vector<Item> pk;
        pk.reserve(prev.size() / 2);
        for (size_t i = 0; i + 1 < prev.size(); i += 2) pk.push_back({prev[i].w + prev[i + 1].w, -1});
        std::vector<Item>& cur = lists[j];
        cur.reserve(leaves.size() + pk.size());
        std::merge(leaves.begin(), leaves.end(), pk.begin(), pk.end(), std::back_inserter(cur),
                   [](const Item& a, const Item& b) { return a.w < b.w; });
    }
    size_t take = 2 * (size_t)m - 2;
    for (int j = maxlen; j >= 1 && take > 0; j--) {
        size_t npk = 0;
        for (size_t i = 0; i < take && i < lists[j].size(); i++) {
            if (lists[j][i].sym >= 0) len[lists[j][i].sym]++;
            else npk++;
        }
        take = 2 * npk;
    }
    return len;
}

// canonical codes (RFC 1951 3.2.2), bit-reversed for LSB-first output;
// code in the low 16 bits, length in the high 16
std::vector<uint32_t> canonical(const std::vector<int>& len) {
    int bl_count[16] = {0}, next_code[16] = {0};
    for (int l : len)
        if (l) bl_count[l]++;
    int code = 0;
    for (int b = 1; b < 16; b++) {
        code = (code + bl_count[b - 1]) << 1;
        next_code[b] = code;
    }
    std::vector<uint32_t> out(len.size(), 0);
    for (size_t s = 0; s < len.size(); s++) {
        const int l = len[s];
        if (!l) continue;
        uint32_t c = (uint32_t)next_code[l]++, r = 0;
        for (int i = 0; i < l; i++) r |= ((c >> i) & 1u) << (l - 1 - i);
        out[s] = r | ((uint32_t)l << 16);
    }
    return out;
}

struct HostBits {
    std::vector<uint8_t> bytes;
    uint64_t pos = 0;
    void put(uint32_t v, int n) {
        for (int i = 0; i < n; i++, pos++) {
            if ((pos >> 3) >= bytes.size()) bytes.push_back(0);
            if ((v >> i) & 1u) bytes[pos >> 3] |= (uint8_t)(1u << (pos & 7));
        }
    }
    void code(uint32_t c) { put(c & 0xFFFF, (int)(c >> 16)); }
};

// The dynamic block: tables for the symbols in `hist` and the block header
// (BFINAL = 1, BTYPE = 2, HLIT / HDIST / HCLEN, code-length code, run-length
// coded code lengths), RFC 1951 3.2.7.
void build_block(const unsigned int* hist, vc::CodeTables& tabs, HostBits& hdr) {
    std::vector<unsigned long long> lf(NLIT), df(NDIST);
    for (int i = 0; i < NLIT; i++) lf[i] = hist[i];
    for (int i = 0; i < NDIST; i++) df[i] = hist[NLIT + i];
    lf[256] = 1;  // end of block
    int nused = 0;
    for (auto f : lf) nused += f != 0;
    if (nused < 2) lf[0] = std::max<unsigned long long>(lf[0], 1);  // a complete literal code
    const std::vector<int> ll = limited_lengths(lf, 15), dl = limited_lengths(df, 15);
    const std::vector<uint32_t> lc = canonical(ll), dc = canonical(dl);
    for (int i = 0; i < NLIT; i++) tabs.lit[i] = lc[i];
    for (int i = 0; i < NDIST; i++) tabs.dist[i] = dc[i];
    int hlit = NLIT, hdist = NDIST;
    while (hlit > 257 && ll[hlit - 1] == 0) hlit--;
    while (hdist > 1 && dl[hdist - 1] == 0) hdist--;
    std::vector<int> seq(ll.begin(), ll.begin() + hlit);
    seq.insert(seq.end(), dl.begin(), dl.begin() + hdist);
    // run-length code the lengths: (symbol, extra bits, extra value)
    struct Rl {
        int sym, eb, ev;
    };
    std::vector<Rl> rl;
    for (size_t i = 0; i < seq.size();) {
        size_t j = i;
        while (j < seq.size() && seq[j] == seq[i]) j++;
        int run = (int)(j - i);
        if (seq[i] == 0) {
            while (run >= 11) {
                const int r = std::min(run, 138);
                rl.push_back({18, 7, r - 11});
                run -= r;
            }
            if (run >= 3) {
                rl.push_back({17, 3, run - 3});
                run = 0;
            }
            while (run-- > 0) rl.push_back({0, 0, 0});
        } else {
            rl.push_back({seq[i], 0, 0});
            run--;
            while (run >= 3) {
                const int r = std::min(run, 6);
                rl.push_back({16, 2, r - 3});
                run -= r;
            }
            while (run-- > 0) rl.push_back({seq[i], 0, 0});
        }
        i = j;
    }
    std::vector<unsigned long long> cf(19, 0);
    for (const Rl& r : rl) cf[r.sym]++;
    const std::vector<int> cl = limited_lengths(cf, 7);
    const std::vector<uint32_t> cc = canonical(cl);
    static const int order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    int hclen = 19;
    while (hclen > 4 && cl[order[hclen - 1]] == 0) hclen--;
    hdr.put(1, 1);  // BFINAL
    hdr.put(2, 2);  // BTYPE = 10: dynamic Huffman
    hdr.put((uint32_t)(hlit - 257), 5);
    hdr.put((uint32_t)(hdist - 1), 5);
    hdr.put((uint32_t)(hclen - 4), 4);
    for (int i = 0; i < hclen; i++) hdr.put((uint32_t)cl[order[i]], 3);
    for (const Rl& r : rl) {
        hdr.code(cc[r.sym]);
        hdr.put((uint32_t)r.ev, r.eb);
    }
}

}  // namespace

extern "C" VC_API int vc_encode_png(const uint8_t* d_rgba, int width, int height, void* stream, uint8_t* h_out,
                                    size_t h_cap, size_t* out_len) {
    using namespace vc;
    if (!d_rgba || !out_len || width <= 0 || height <= 0) return VC_ERR_INVALID;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int n = 1 + 3 * width;
    const int nslices = height * TOK_LANES;
    const size_t tok_cap = (size_t)nslices * tok_slice_max(n);
    // bound of the block: every byte a literal of <= 15 bits, + header
    const size_t max_bytes = (size_t)height * ((size_t)n * 15 / 8 + 8) + 4096;
    uint32_t *tokens = nullptr, *ntok = nullptr, *slice_bits = nullptr, *row_bits = nullptr, *block_crc = nullptr,
             *tables = nullptr;
    unsigned int* hist = nullptr;
    unsigned long long *adler = nullptr, *offsets = nullptr, *total_bytes = nullptr;
    uint32_t* words = nullptr;
    CodeTables* codes = nullptr;
    int rc = VC_OK;
    auto ok = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == VC_OK) rc = VC_ERR_CUDA;
        return e == cudaSuccess;
    };
    if (!crc_ready) crc_init();
    size_t max_blocks = 1;  // power of two >= the stream's CRC block count (upper bound)
    while (max_blocks * CRC_BLOCK < max_bytes) max_blocks <<= 1;
    const size_t words_bytes = (max_bytes + 8) & ~(size_t)3;
    ok(cudaMallocAsync((void**)&tokens, tok_cap * 4, s));
    ok(cudaMallocAsync((void**)&ntok, 4 * (size_t)nslices, s));
    ok(cudaMallocAsync((void**)&slice_bits, 4 * (size_t)nslices, s));
    ok(cudaMallocAsync((void**)&row_bits, 4 * (size_t)height, s));
    ok(cudaMallocAsync((void**)&hist, 4 * (NLIT + NDIST), s));
    ok(cudaMallocAsync((void**)&adler, 16 * (size_t)height, s));
    ok(cudaMallocAsync((void**)&offsets, 8 * ((size_t)height + 1), s));
    ok(cudaMallocAsync((void**)&total_bytes, 8, s));
    ok(cudaMallocAsync((void**)&words, words_bytes, s));
    ok(cudaMallocAsync((void**)&codes, sizeof(CodeTables), s));
    ok(cudaMallocAsync((void**)&tables, 4 * (256 + 32), s));
    ok(cudaMallocAsync((void**)&block_crc, 4 * max_blocks + 4, s));
    std::vector<unsigned int> hhist(NLIT + NDIST, 0);
    std::vector<unsigned long long> hadler(2 * (size_t)height);
    unsigned long long total = 0;
    uint32_t raw_crc = 0;
    HostBits hdr;
    CodeTables tabs{};
    if (rc == VC_OK) {  // pass 1: filter, tokenize, histogram
        ok(cudaMemsetAsync(hist, 0, 4 * (NLIT + NDIST), s));
        const size_t smem = ((size_t)n + 15) & ~(size_t)15;
        if (smem > 40 * 1024)
            ok(cudaFuncSetAttribute(png_tokenize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        png_tokenize_kernel<<<height, TOK_LANES, smem, s>>>(d_rgba, width, height, tokens, ntok, hist, adler);
        ok(cudaGetLastError());
        ok(cudaMemcpyAsync(hhist.data(), hist, 4 * (NLIT + NDIST), cudaMemcpyDeviceToHost, s));
        ok(cudaStreamSynchronize(s));
    }
    if (rc == VC_OK) {  // the code and the block header; pass 2: bit counts, offsets, emission, CRC
        build_block(hhist.data(), tabs, hdr);
        const size_t hdr_words = (hdr.bytes.size() + 3) / 4;
        std::vector<uint32_t> hw(hdr_words, 0);
        memcpy(hw.data(), hdr.bytes.data(), hdr.bytes.size());
        ok(cudaMemsetAsync(words, 0, words_bytes, s));
        ok(cudaMemcpyAsync(words, hw.data(), hdr_words * 4, cudaMemcpyHostToDevice, s));
        ok(cudaMemcpyAsync(codes, &tabs, sizeof(CodeTables), cudaMemcpyHostToDevice, s));
        ok(cudaMemcpyAsync(tables, crc_tab[0], 4 * 256, cudaMemcpyHostToDevice, s));
        ok(cudaMemcpyAsync(tables + 256, x2n_tab, 4 * 32, cudaMemcpyHostToDevice, s));
        png_bits_kernel<<<height, TOK_LANES, 0, s>>>(tokens, ntok, n, codes, slice_bits, row_bits);
        png_scan_kernel<<<1, 1024, 0, s>>>(row_bits, height, offsets);
        png_emit_kernel<<<height, TOK_LANES, 0, s>>>(tokens, ntok, n, codes, offsets, slice_bits, hdr.pos, words);
        png_eob_kernel<<<1, 1, 0, s>>>(offsets, height, hdr.pos, codes, words, total_bytes);
        png_crc_blocks_kernel<<<(unsigned)max_blocks, 256, 0, s>>>(reinterpret_cast<const uint8_t*>(words),
                                                                   total_bytes, tables, tables + 256, block_crc);
        png_crc_tree_kernel<<<1, 1024, 0, s>>>(block_crc, total_bytes, tables + 256, block_crc + max_blocks);
        ok(cudaGetLastError());
        ok(cudaMemcpyAsync(&total, total_bytes, 8, cudaMemcpyDeviceToHost, s));
        ok(cudaMemcpyAsync(&raw_crc, block_crc + max_blocks, 4, cudaMemcpyDeviceToHost, s));
        ok(cudaMemcpyAsync(hadler.data(), adler, 16 * (size_t)height, cudaMemcpyDeviceToHost, s));
        ok(cudaStreamSynchronize(s));
    }
    // file layout: signature, IHDR, IDAT {78 01, deflate block, Adler-32}, IEND
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
        // the deflate block goes straight from HBM into the caller's buffer
        ok(cudaMemcpyAsync(id + 10, words, total, cudaMemcpyDeviceToHost, s));
        // Adler-32 of all filtered rows (per-row sums from the device)
        unsigned long long A = 1, B = 0;
        for (int y = 0; y < height; y++) {
            B = (B + ((unsigned long long)n % 65521) * A + hadler[2 * y + 1] % 65521) % 65521;
            A = (A + hadler[2 * y] % 65521) % 65521;
        }
        uint8_t ad[4];
        put_be32(ad, (uint32_t)((B << 16) | A));
        // CRC over "IDAT", the zlib header, the block (device) and the Adler
        const uint32_t block_std = raw_crc ^ shift_host(0xFFFFFFFFu, total) ^ 0xFFFFFFFFu;
        uint32_t c = crc32(id + 4, 6);
        c = crc32_combine_host(c, block_std, total);
        c = crc32(ad, 4, c);
        ok(cudaStreamSynchronize(s));
        memcpy(id + 10 + total, ad, 4);
        put_be32(id + 10 + total + 4, c);
        const uint8_t iend[12] = {0, 0, 0, 0, 'I', 'E', 'N', 'D', 0xAE, 0x42, 0x60, 0x82};
        memcpy(id + 10 + total + 8, iend, 12);
    }
    cudaFreeAsync(tokens, s);
    cudaFreeAsync(ntok, s);
    cudaFreeAsync(slice_bits, s);
    cudaFreeAsync(row_bits, s);
    cudaFreeAsync(hist, s);
    cudaFreeAsync(adler, s);
    cudaFreeAsync(offsets, s);
    cudaFreeAsync(total_bytes, s);
    cudaFreeAsync(words, s);
    cudaFreeAsync(codes, s);
    cudaFreeAsync(tables, s);
    cudaFreeAsync(block_crc, s);
    if (rc != VC_OK) return rc;
    if (h_out != nullptr && h_cap < file_len) return VC_ERR_INVALID;
    return VC_OK;
}
