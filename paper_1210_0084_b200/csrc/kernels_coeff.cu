// Coefficient processing on the device (paper §VI):
// masking, the sliCQ spectrogram |s^0 + s^1|^2 and transposition by whole CQ bins, as
// kernels over the slice-major coefficient layout [batch][S][C] (channel k at off_k).
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "fft_dev.cuh"
#include "slicq_internal.h"

namespace slicq {
namespace {
using namespace slicq::dev;

// c[r][i] *= a(mask), a = m (linear) or 10^(-5 (1 - m)) (dB) -- the amplitude the
// fused masked synthesis applies (kernels_dev.cuh mask_coef), so both give equal products
__global__ void mask_kernel(float2 *c, const float *mask, int64_t total, int64_t C, int full,
                            int db) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float mv = mask[full ? i : i % C];
    const float amp = db ? exp10f(-5.0f * (1.0f - mv)) : mv;
    const float2 v = c[i];
    c[i] = make_float2(v.x * amp, v.y * amp);
  }
}

// |s^0 + s^1|^2 of channel k at p = m h + n' (h = M/2, n' < h): slice m's entry n' + h plus
// slice m+1's entry n' (two-layer array of Alg. 3; slices circular);
// out[b][S off_k / 2 + p]
__global__ void spectrogram_kernel(const ChanDev *ch, const float2 *c, float *out, int S,
                                   int64_t C) {
  const int k = blockIdx.x;
  const int64_t b = blockIdx.y;
  const ChanDev d = ch[k];
  const int h = d.M / 2;
  const int64_t W = (int64_t)S * h;
  const float2 *cb = c + b * S * C + d.off;
  float *o = out + b * (S * C / 2) + (int64_t)S * d.off / 2;
  for (int64_t p = blockIdx.z * (int64_t)blockDim.x + threadIdx.x; p < W;
       p += (int64_t)gridDim.z * blockDim.x) {
    const int m = (int)(p / h), np = (int)(p - (int64_t)m * h);
    const int m1 = m + 1 == S ? 0 : m + 1;
    const float2 a = cb[(int64_t)m * C + np + h], e = cb[(int64_t)m1 * C + np];
    const float re = a.x + e.x, im = a.y + e.y;
    o[p] = re * re + im * im;
  }
}

// CQ channel k takes channel (k - shift)'s coefficients modulated by e^{2 pi i d n / M},
// d = round(centre_k - centre_src) (centre = lo + (len - 1)/2, half to even as Python's
// round); vacated CQ channels are zero, the plateaus are copied
__global__ void transpose_kernel(const ChanDev *ch, const float2 *twM, const float2 *c,
                                 float2 *out, int64_t C, int K, int shift) {
  const int64_t row = blockIdx.x;
  const int k = blockIdx.y;
  const ChanDev d = ch[k];
  const float2 *ci = c + row * C;
  float2 *co = out + row * C + d.off;
  if (k == 0 || k == K + 1) {
    for (int n = threadIdx.x; n < d.M; n += blockDim.x) co[n] = ci[d.off + n];
    return;
  }
  const int src = k - shift;
  if (src < 1 || src > K) {
    for (int n = threadIdx.x; n < d.M; n += blockDim.x) co[n] = make_float2(0.f, 0.f);
    return;
  }
  const ChanDev s = ch[src];
  const int d2 = 2 * (d.lo - s.lo) + (d.len - s.len);
  const int dd = (int)rint(0.5 * (double)d2);
  const int M = d.M;
  const int dm = ((dd % M) + M) % M;
  const float2 *tw = twM + d.twoff;
  for (int n = threadIdx.x; n < M; n += blockDim.x)
    co[n] = cmul(ci[s.off + n], tw[(int)(((int64_t)dm * n) % M)]);
}

int cuda_err(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return SLICQ_OK;
  return set_error(SLICQ_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

int launch_mask(const slicq_plan *p, slicq_c32 *c, const float *mask, int64_t rows, int full,
                int db, void *stream) {
  const int64_t total = rows * p->C;
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  mask_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float2 *>(c), mask, total, p->C, full, db);
  return cuda_err(cudaGetLastError(), "mask launch");
}

int launch_spectrogram(const slicq_plan *p, const slicq_c32 *c, int64_t nslices, int64_t batch,
                       float *out, void *stream) {
  if (batch > 65535) return set_error(SLICQ_ESHAPE, "batch too large");
  const int64_t per = nslices * p->C / 2 / (p->K + 2);  // mean entries per channel
  const unsigned z = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, per / 4096));
  spectrogram_kernel<<<dim3((unsigned)(p->K + 2), (unsigned)batch, z), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      p->d.chan, reinterpret_cast<const float2 *>(c), out, (int)nslices, p->C);
  return cuda_err(cudaGetLastError(), "spectrogram launch");
}

int launch_transpose(const slicq_plan *p, const slicq_c32 *c, slicq_c32 *out, int64_t rows,
                     int shift, void *stream) {
  transpose_kernel<<<dim3((unsigned)rows, (unsigned)(p->K + 2)), 128, 0,
                     static_cast<cudaStream_t>(stream)>>>(
      p->d.chan, reinterpret_cast<const float2 *>(p->d.twM), reinterpret_cast<const float2 *>(c),
      reinterpret_cast<float2 *>(out), p->C, p->K, shift);
  return cuda_err(cudaGetLastError(), "transpose launch");
}

}  // namespace slicq
