// Complex-input sliCQ (Alg. 3/4 on f in C^L over all 2K+2 channels of Table 1)
// through the real-input kernels.  By linearity c(f) = c(Re f) + i c(Im f) for every channel,
// and for a real input the mirror channel 2K+2-k of CQ channel k is
//   c_{n,2K+2-k} = w_n conj(c_{n,k}),  w_n = e^{2 pi i 2N n / M_k}      (C15)
// so the forward runs the real transform on the 2B rows (Re f_b, Im f_b) and combines:
//   stored k:  c_k = a_k + i b_k,   mirror of k:  w (conj a_k + i conj b_k)
// The synthesis splits the 2K+2-channel coefficients into two real-consistent sets
//   u_k = (c_k + z_k) / 2,  v_k = (c_k - z_k) / (2i),  z_k = w conj(c_{mirror(k)})
// (mirror(0) = 0 with w = 1: the DC plateau of a real input is real; mirror(K+1) = K+1:
// the Nyquist plateau is its own mirror), runs the real synthesis on the 2B rows (u_b, v_b)
// (exact on real-consistent sets, C15) and interleaves y = y_u + i y_v.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "fft_dev.cuh"
#include "slicq_internal.h"

namespace slicq {
namespace {
using namespace slicq::dev;

__global__ void cx_split_rows(const float2 *x, int64_t n, float *r) {  // [B][n] -> [2B][n]
  const int64_t b = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = x[b * n + i];
    r[(2 * b) * n + i] = v.x;
    r[(2 * b + 1) * n + i] = v.y;
  }
}

__global__ void cx_join_rows(const float *r, int64_t n, float2 *y) {  // [2B][n] -> [B][n]
  const int64_t b = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[b * n + i] = make_float2(r[(2 * b) * n + i], r[(2 * b + 1) * n + i]);
}

// out[b][m][j] over the full layout from the Re / Im rows T[2b][m], T[2b+1][m] ([C] each):
// stored column: a + i b; mirror column: w (conj a + i conj b) = w (a.x + b.y, b.x - a.y)
__global__ void cx_combine(const uint2 *cxf, const float2 *twM, const float2 *T, float2 *out,
                           int64_t S, int64_t C, int64_t Cf, int64_t row0) {
  const int64_t row = row0 + blockIdx.y, b = row / S, m = row - b * S;
  const float2 *ta = T + ((2 * b) * S + m) * C, *tb = T + ((2 * b + 1) * S + m) * C;
  float2 *o = out + row * Cf;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < Cf;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint2 e = __ldg(cxf + j);
    const float2 av = ta[e.x], bv = tb[e.x];
    o[j] = (e.y & 1u) ? cmul(__ldg(twM + (e.y >> 1)), make_float2(av.x + bv.y, bv.x - av.y))
                      : make_float2(av.x - bv.y, av.y + bv.x);
  }
}

// c: [B][S][Cf] -> U: [2B][S][C] (rows u_b, v_b): z = w conj(c_mirror) (DC: conj c),
// u = (c + z) / 2, v = (c - z) / (2i)
__global__ void cx_split(const uint2 *cxs, const float2 *twM, const float2 *cf, float2 *U,
                         int64_t S, int64_t C, int64_t Cf, int64_t row0) {
  const int64_t row = row0 + blockIdx.y, b = row / S, m = row - b * S;
  const float2 *cr = cf + row * Cf;
  float2 *u = U + ((2 * b) * S + m) * C, *v = U + ((2 * b + 1) * S + m) * C;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < C;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint2 e = __ldg(cxs + j);
    const float2 w = (e.y & 1u) ? make_float2(1.f, 0.f) : __ldg(twM + (e.y >> 1));
    const float2 z = cmul(w, cconj(cr[e.x]));
    const float2 x = cr[j];
    u[j] = make_float2(0.5f * (x.x + z.x), 0.5f * (x.y + z.y));
    v[j] = make_float2(0.5f * (x.y - z.y), -0.5f * (x.x - z.x));  // (x - z) / (2i)
  }
}

int cuda_err(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return SLICQ_OK;
  return set_error(SLICQ_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

int64_t coeffs_full(const slicq_plan *p) {
  int64_t c = p->C;
  for (int k = 1; k <= p->K; ++k) c += p->M[k];
  return c;
}

// workspace: [real-path workspace for 2B rows][real buffer 2B x n][coefficients 2B x S x C]
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
size_t workspace_bytes_complex(const slicq_plan *p, int64_t nslices, int64_t batch, int64_t n) {
  return al(workspace_bytes(p, nslices, 2 * batch)) + al(sizeof(float) * 2 * batch * n) +
         sizeof(float2) * (size_t)(2 * batch * nslices * p->C);
}

// nsgt = 1: the full-length CQ-NSGT of the whole signal (one frame per row, n <= sl_len)
int launch_forward_complex(const slicq_plan *p, const slicq_c32 *x, int64_t n, int64_t batch,
                           slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream,
                           int nsgt) {
  const int64_t L = nsgt ? p->sl_len : (n + p->sl_len - 1) / p->sl_len * p->sl_len;
  const int64_t S = nsgt ? 1 : L / p->N;
  if (ws_bytes < workspace_bytes_complex(p, S, batch, n))
    return set_error(SLICQ_ESHAPE, "workspace too small");
  if (batch > 65535) return set_error(SLICQ_ESHAPE, "batch too large");
  char *w = static_cast<char *>(ws);
  const size_t wr = al(workspace_bytes(p, S, 2 * batch));
  float *R = reinterpret_cast<float *>(w + wr);
  float2 *T = reinterpret_cast<float2 *>(w + wr + al(sizeof(float) * 2 * batch * n));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cx_split_rows<<<dim3((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)batch), 256, 0, s>>>(
      reinterpret_cast<const float2 *>(x), n, R);
  int rc = cuda_err(cudaGetLastError(), "complex split");
  if (rc) return rc;
  rc = nsgt ? launch_forward(p, R, n, n, 0, L, 0, 1, 1, 2 * batch,
                             reinterpret_cast<slicq_c32 *>(T), ws, wr, stream, 1)
            : launch_forward(p, R, n, n, 0, L, 1, 0, S, 2 * batch,
                             reinterpret_cast<slicq_c32 *>(T), ws, wr, stream);
  if (rc) return rc;
  {
    const int64_t Cf = coeffs_full(p), rows = batch * S;
    const unsigned gx = (unsigned)std::min<int64_t>((Cf + 255) / 256, 64);
    for (int64_t r0 = 0; r0 < rows; r0 += 65535)  // grid y <= 65535 rows per launch
      cx_combine<<<dim3(gx, (unsigned)std::min<int64_t>(65535, rows - r0)), 256, 0, s>>>(
          p->d.cxf, reinterpret_cast<const float2 *>(p->d.twM), T,
          reinterpret_cast<float2 *>(coeffs), S, p->C, Cf, r0);
  }
  return cuda_err(cudaGetLastError(), "complex combine");
}

int launch_inverse_complex(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n,
                           int64_t batch, slicq_c32 *y, void *ws, size_t ws_bytes, void *stream,
                           int nsgt) {
  const int64_t L = nsgt ? p->sl_len : (n + p->sl_len - 1) / p->sl_len * p->sl_len;
  const int64_t S = nsgt ? 1 : L / p->N;
  if (ws_bytes < workspace_bytes_complex(p, S, batch, n))
    return set_error(SLICQ_ESHAPE, "workspace too small");
  if (batch > 65535) return set_error(SLICQ_ESHAPE, "batch too large");
  char *w = static_cast<char *>(ws);
  const size_t wr = al(workspace_bytes(p, S, 2 * batch));
  float *Y = reinterpret_cast<float *>(w + wr);
  float2 *U = reinterpret_cast<float2 *>(w + wr + al(sizeof(float) * 2 * batch * n));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  {
    const int64_t rows = batch * S;
    const unsigned gx = (unsigned)std::min<int64_t>((p->C + 255) / 256, 64);
    for (int64_t r0 = 0; r0 < rows; r0 += 65535)
      cx_split<<<dim3(gx, (unsigned)std::min<int64_t>(65535, rows - r0)), 256, 0, s>>>(
          p->d.cxs, reinterpret_cast<const float2 *>(p->d.twM),
          reinterpret_cast<const float2 *>(coeffs), U, S, p->C, coeffs_full(p), r0);
  }
  int rc = cuda_err(cudaGetLastError(), "complex split");
  if (rc) return rc;
  rc = nsgt ? launch_inverse(p, reinterpret_cast<const slicq_c32 *>(U), 1, 1, 2, 2 * batch, 0, n,
                             L, Y, n, 0, nullptr, 0, ws, wr, stream, nullptr, 0, 1)
            : launch_inverse(p, reinterpret_cast<const slicq_c32 *>(U), 0, S, S, 2 * batch, 1, n,
                             L, Y, n, 0, nullptr, 0, ws, wr, stream);
  if (rc) return rc;
  cx_join_rows<<<dim3((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)batch), 256, 0, s>>>(
      Y, n, reinterpret_cast<float2 *>(y));
  return cuda_err(cudaGetLastError(), "complex join");
}

}  // namespace slicq
