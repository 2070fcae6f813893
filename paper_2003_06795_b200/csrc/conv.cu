// im2col front-end: convolution layers run as the
// network-derived GEMMs the selectors were trained on.
//   cols[M, K] with M = B*Ho*Wo (row = b*Ho*Wo + oh*Wo + ow) and
//   K = Cin*kh*kw (col = c*kh*kw + r*kw + s), zero for padded taps;
//   y[M, Cout] (NHWC) = cols @ W^T, W stored [Cout, K] row-major -> the GEMM
//   is the NT variant (trans_b), dispatched through the compiled selector.
// The gather is HBM/L2-bound integer work: one thread per cols element,
// consecutive threads along K (coalesced 4-byte stores), grid-stride loop
// sized to a multiple of the SM count.
#include <cuda_bf16.h>

#include <algorithm>

#include "kp_internal.cuh"

namespace kp {

template <typename T>
__global__ void __launch_bounds__(256) im2col_kernel(const T* __restrict__ x, T* __restrict__ cols,
                                                     kp_conv_desc d, int64_t ho, int64_t wo,
                                                     int64_t total) {
    const int64_t K = d.c_in * d.kh * d.kw;
    const int64_t khw = d.kh * d.kw;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = idx / K, col = idx - row * K;
        const int64_t b = row / (ho * wo);
        const int64_t pix = row - b * ho * wo;
        const int64_t oh = pix / wo, ow = pix - oh * wo;
        const int64_t c = col / khw;
        const int64_t rs = col - c * khw;
        const int64_t r = rs / d.kw, s = rs - r * d.kw;
        const int64_t ih = oh * d.stride_h - d.pad_h + r;
        const int64_t iw = ow * d.stride_w - d.pad_w + s;
        T v = T(0.0f);
        if (ih >= 0 && ih < d.h && iw >= 0 && iw < d.w)
            v = x[((b * d.c_in + c) * d.h + ih) * d.w + iw];
        cols[idx] = v;
    }
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

extern "C" kp_status kp_im2col(kp_family family, const kp_conv_desc* d, const void* x, void* cols,
                               void* stream) {
    int64_t ho, wo;
    kp_status st = conv_shape(d, &ho, &wo);
    if (st != KP_OK) return st;
    if (!x || !cols) return fail(KP_ERR_INVALID_ARG, "null tensor");
    const int64_t total = d->batch * ho * wo * d->c_in * d->kh * d->kw;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, int64_t(sms) * 16);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (family == KP_BF16_TC)
        im2col_kernel<__nv_bfloat16><<<unsigned(blocks), 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(cols), *d, ho, wo, total);
    else
        im2col_kernel<float><<<unsigned(blocks), 256, 0, s>>>(
            static_cast<const float*>(x), static_cast<float*>(cols), *d, ho, wo, total);
    note_launch();
    return check_launch("im2col_kernel");
}

extern "C" kp_status kp_conv2d_auto(kp_family family, const kp_conv_desc* d, const void* x,
                                    const void* w, float* y, void* cols, void* stream,
                                    kp_config* chosen) {
    int64_t ho, wo;
    kp_status st = conv_shape(d, &ho, &wo);
    if (st != KP_OK) return st;
    if ((st = kp_im2col(family, d, x, cols, stream)) != KP_OK) return st;
    const int64_t m = d->batch * ho * wo, k = d->c_in * d->kh * d->kw, n = d->c_out;
    kp_gemm_desc g = {1, m, k, n, 0, 1, k, k, n, 0, 0, m * n, 1.0f, 0.0f};
    return kp_gemm_auto(family, &g, cols, w, y, stream, chosen);
}
