// im2col front-end: convolution layers run as the
// network-derived GEMMs the selectors were trained on.
//   cols[M, K] with M = B*Ho*Wo (row = b*Ho*Wo + oh*Wo + ow) and
//   K = Cin*kh*kw (col = c*kh*kw + r*kw + s), zero for padded taps;
//   y[M, Cout] (NHWC) = cols @ W^T, W stored [Cout, K] row-major -> the GEMM
//   is the NT variant (trans_b), dispatched through the compiled selector.
// The gather is HBM-bound byte movement (the cols write dominates; see the
// tiled kernel below), not GEMM-shaped work.
#include <cuda_bf16.h>

#include <algorithm>

#include "kp_internal.cuh"

namespace kp {

// Unsigned 32-bit division by a run-time constant as a multiply-high + shift
// (valid for dividends < 2^31): the gather's index decomposition would
// otherwise be dominated by integer divides.
struct FastDiv {
    uint32_t d, magic, shift;
    FastDiv() = default;
    explicit FastDiv(uint32_t div) : d(div) {
        shift = 0;
        while ((1ull << shift) < div) ++shift;
        magic = uint32_t(((1ull << 32) * ((1ull << shift) - div)) / div + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return (__umulhi(n, magic) + n) >> shift;
    }
};

struct Im2colGeom {
    FastDiv hwo, wo, khw, kw;
    int32_t c_in, h, w, kh, stride_h, stride_w, pad_h, pad_w;
};

// Tiled gather: a CTA owns 64 consecutive output pixels (cols rows) and walks
// K in chunks of 64 taps.  Gather phase: lanes run along pixels, so for every
// tap (c, r, s) a warp reads consecutive input columns (coalesced for stride
// 1; neighbouring pixels' receptive fields overlap, so most re-reads hit
// L1/L2), 16 independent loads in flight per thread; the chunk's tap table is
// decoded once into shared memory.  Write phase: the tile is read back
// transposed (padded rows, <= 2-way conflicts) and stored as 16-byte vectors
// along K (VEC: K a multiple of 16/sizeof(T) and a 16-byte aligned cols),
// otherwise as coalesced scalars.  Both HBM streams are coalesced; the kernel
// is bound by the cols write (x is re-read from L2).
constexpr int kIm2colPix = 64;
constexpr int kIm2colKC = 64;

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) im2col_tiled_kernel(const T* __restrict__ x,
                                                           T* __restrict__ cols, Im2colGeom g,
                                                           uint32_t rows, uint32_t K,
                                                           uint32_t ldk) {
    constexpr int KC = kIm2colKC, PIX = kIm2colPix;
    __shared__ T tile[KC][PIX + 1];
    __shared__ int32_t tab_off[KC], tab_r[KC], tab_s[KC];
    const int t = threadIdx.x;
    const int p = t & (PIX - 1), grp = t >> 6;
    const uint32_t row0 = blockIdx.x * PIX;
    const uint32_t prow = row0 + p;
    const bool pvalid = prow < rows;
    const uint32_t b = g.hwo.div(prow);
    const uint32_t pix = prow - b * g.hwo.d;
    const uint32_t oh = g.wo.div(pix), ow = pix - oh * g.wo.d;
    const int32_t ih0 = int32_t(oh) * g.stride_h - g.pad_h;
    const int32_t iw0 = int32_t(ow) * g.stride_w - g.pad_w;
    const T* xp = x + int64_t(b) * g.c_in * g.h * g.w + int64_t(ih0) * g.w + iw0;
    // columns [K, ldk) of a padded pitch are written as zeros (taps past K
    // gather nothing)
    for (uint32_t k0 = blockIdx.y * KC; k0 < ldk; k0 += gridDim.y * KC) {
        if (t < KC && k0 + t < K) {
            const uint32_t k = k0 + t;
            const uint32_t c = g.khw.div(k);
            const uint32_t rs = k - c * g.khw.d;
            const uint32_t r = g.kw.div(rs);
            const uint32_t sc = rs - r * g.kw.d;
            tab_off[t] = int32_t((c * g.h + r) * g.w + sc);
            tab_r[t] = int32_t(r);
            tab_s[t] = int32_t(sc);
        }
        __syncthreads();
        // Branch-free gather: every lane issues all KC/4 loads back to back
        // (out-of-range taps read a valid dummy address and are zeroed
        // after), so their latencies overlap instead of serialising behind
        // per-tap branches.
        T v[KC / 4];
        bool in[KC / 4];
#pragma unroll
        for (int i = 0; i < KC / 4; ++i) {
            const int j = grp + 4 * i;
            const int32_t ih = ih0 + tab_r[j], iw = iw0 + tab_s[j];
            in[i] = pvalid && k0 + j < K && unsigned(ih) < unsigned(g.h) &&
                    unsigned(iw) < unsigned(g.w);
            v[i] = __ldg(in[i] ? xp + tab_off[j] : x);
        }
#pragma unroll
        for (int i = 0; i < KC / 4; ++i) tile[grp + 4 * i][p] = in[i] ? v[i] : T(0.0f);
        __syncthreads();
        if constexpr (VEC) {
            constexpr int VW = 16 / int(sizeof(T));  // elements per 16-byte store
            constexpr int LPR = KC / VW;             // threads per row segment
            constexpr int RPP = 256 / LPR;           // rows per pass
            const int q = t % LPR;
            const uint32_t kk = k0 + q * VW;
#pragma unroll
            for (int pass = 0; pass < PIX / RPP; ++pass) {
                const int pr = t / LPR + pass * RPP;
                const uint32_t row = row0 + pr;
                if (row < rows && kk < ldk) {
                    union { uint4 u; T e[VW]; } out;
#pragma unroll
                    for (int e = 0; e < VW; ++e) out.e[e] = tile[q * VW + e][pr];
                    *reinterpret_cast<uint4*>(cols + int64_t(row) * ldk + kk) = out.u;
                }
            }
        } else {
#pragma unroll 4
            for (int idx = t; idx < PIX * KC; idx += 256) {
                const int pr = idx / KC, j = idx % KC;
                const uint32_t row = row0 + pr;
                if (row < rows && k0 + j < ldk) cols[int64_t(row) * ldk + k0 + j] = tile[j][pr];
            }
        }
        __syncthreads();
    }
}

template <typename T, bool VEC>
static void launch_im2col_tiled(const T* x, T* cols, const Im2colGeom& g, int64_t rows,
                                int64_t K, int64_t ldk, int sms, cudaStream_t s) {
    const int64_t gx = (rows + kIm2colPix - 1) / kIm2colPix;
    const int64_t kchunks = (ldk + kIm2colKC - 1) / kIm2colKC;
    const int64_t gy = std::min<int64_t>(
        std::min<int64_t>(kchunks, 65535), std::max<int64_t>(1, (int64_t(sms) * 8 + gx - 1) / gx));
    im2col_tiled_kernel<T, VEC><<<dim3(unsigned(gx), unsigned(gy)), 256, 0, s>>>(
        x, cols, g, uint32_t(rows), uint32_t(K), uint32_t(ldk));
    note_launch();
}

static kp_status conv_shape(const kp_conv_desc* d, int64_t* ho, int64_t* wo) {
    if (!d) return fail(KP_ERR_INVALID_ARG, "null conv descriptor");
    if (d->batch < 1 || d->c_in < 1 || d->h < 1 || d->w < 1 || d->c_out < 1 || d->kh < 1 ||
        d->kw < 1 || d->stride_h < 1 || d->stride_w < 1 || d->pad_h < 0 || d->pad_w < 0)
        return fail(KP_ERR_BAD_SHAPE, "conv dims must be >= 1 (pads >= 0)");
    *ho = (d->h + 2 * d->pad_h - d->kh) / d->stride_h + 1;
    *wo = (d->w + 2 * d->pad_w - d->kw) / d->stride_w + 1;
    if (*ho < 1 || *wo < 1) return fail(KP_ERR_BAD_SHAPE, "conv output is empty");
    return KP_OK;
}

}  // namespace kp

using namespace kp;

extern "C" kp_status kp_conv_output_shape(const kp_conv_desc* d, int64_t* ho, int64_t* wo) {
    if (!ho || !wo) return fail(KP_ERR_INVALID_ARG, "null output");
    return conv_shape(d, ho, wo);
}

// K pitch of the im2col matrix kp_conv2d_auto uses: K itself, rounded up to
// 16 bytes for the tcgen05 families (TMA needs 16-byte row pitches; the
// padding columns are zeros and the GEMM still sees k = K).
static int64_t conv_pitch(kp_family family, int64_t K) {
    if (family == KP_TF32_TC) return (K + 3) / 4 * 4;
    if (family == KP_BF16_TC) return (K + 7) / 8 * 8;
    return K;
}

extern "C" kp_status kp_im2col_pitched(kp_family family, const kp_conv_desc* d, const void* x,
                                       void* cols, int64_t ldk, void* stream) {
    int64_t ho, wo;
    kp_status st = conv_shape(d, &ho, &wo);
    if (st != KP_OK) return st;
    if (!x || !cols) return fail(KP_ERR_INVALID_ARG, "null tensor");
    const int64_t K = d->c_in * d->kh * d->kw, hwo = ho * wo;
    if (ldk < K) return fail(KP_ERR_BAD_SHAPE, "im2col pitch smaller than c_in*kh*kw");
    if (ldk >= (1ll << 30) || hwo >= (1ll << 30) || d->c_in * d->h * d->w >= (1ll << 31))
        return fail(KP_ERR_BAD_SHAPE, "conv dims exceed the 2^31 gather range");
    const bool bf16 = family == KP_BF16_TC;
    const int esz = bf16 ? 2 : 4;
    const bool vec = ldk % (16 / esz) == 0 && aligned16(cols);
    Im2colGeom g;
    g.hwo = FastDiv(uint32_t(hwo));
    g.wo = FastDiv(uint32_t(wo));
    g.khw = FastDiv(uint32_t(d->kh * d->kw));
    g.kw = FastDiv(uint32_t(d->kw));
    g.c_in = int32_t(d->c_in); g.h = int32_t(d->h); g.w = int32_t(d->w); g.kh = int32_t(d->kh);
    g.stride_h = int32_t(d->stride_h); g.stride_w = int32_t(d->stride_w);
    g.pad_h = int32_t(d->pad_h); g.pad_w = int32_t(d->pad_w);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Rows per launch stay below 2^31 (FastDiv's range): split over images.
    const int64_t imgs = std::max<int64_t>(1, ((1ll << 31) - 2 * kIm2colPix) / hwo);
    for (int64_t b0 = 0; b0 < d->batch; b0 += imgs) {
        const int64_t nb = std::min(imgs, d->batch - b0);
        const int64_t xoff = b0 * d->c_in * d->h * d->w, coff = b0 * hwo * ldk;
        if (bf16) {
            auto xp = static_cast<const __nv_bfloat16*>(x) + xoff;
            auto cp = static_cast<__nv_bfloat16*>(cols) + coff;
            if (vec) launch_im2col_tiled<__nv_bfloat16, true>(xp, cp, g, nb * hwo, K, ldk, sms, s);
            else launch_im2col_tiled<__nv_bfloat16, false>(xp, cp, g, nb * hwo, K, ldk, sms, s);
        } else {
            auto xp = static_cast<const float*>(x) + xoff;
            auto cp = static_cast<float*>(cols) + coff;
            if (vec) launch_im2col_tiled<float, true>(xp, cp, g, nb * hwo, K, ldk, sms, s);
            else launch_im2col_tiled<float, false>(xp, cp, g, nb * hwo, K, ldk, sms, s);
        }
        if ((st = check_launch("im2col_kernel")) != KP_OK) return st;
    }
    return KP_OK;
}

extern "C" kp_status kp_im2col(kp_family family, const kp_conv_desc* d, const void* x, void* cols,
                               void* stream) {
    if (!d) return fail(KP_ERR_INVALID_ARG, "null conv descriptor");
    return kp_im2col_pitched(family, d, x, cols, d->c_in * d->kh * d->kw, stream);
}

extern "C" kp_status kp_conv_workspace_elems(kp_family family, const kp_conv_desc* d,
                                             int64_t* elems) {
    int64_t ho, wo;
    if (!elems) return fail(KP_ERR_INVALID_ARG, "null output");
    kp_status st = conv_shape(d, &ho, &wo);
    if (st != KP_OK) return st;
    *elems = d->batch * ho * wo * conv_pitch(family, d->c_in * d->kh * d->kw);
    return KP_OK;
}

extern "C" kp_status kp_conv2d_auto(kp_family family, const kp_conv_desc* d, const void* x,
                                    const void* w, float* y, void* cols, void* stream,
                                    kp_config* chosen) {
    int64_t ho, wo;
    kp_status st = conv_shape(d, &ho, &wo);
    if (st != KP_OK) return st;
    const int64_t m = d->batch * ho * wo, k = d->c_in * d->kh * d->kw, n = d->c_out;
    const int64_t ldk = conv_pitch(family, k);
    if ((st = kp_im2col_pitched(family, d, x, cols, ldk, stream)) != KP_OK) return st;
    // the weights' K pitch may still be unaligned: tc::launch stages them
    kp_gemm_desc g = {1, m, k, n, 0, 1, ldk, k, n, 0, 0, m * n, 1.0f, 0.0f};
    return kp_gemm_auto(family, &g, cols, w, y, stream, chosen);
}
