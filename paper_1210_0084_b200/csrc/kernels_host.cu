// Host side of the kernels: plan-time kernel configuration (packets, element tables, the
// inverse gather list, shared-memory budgets, staging chunking), device-table upload and the
// launch sequences.  Device code: kernels_dev.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#define SLICQ_DEFINE_CHAN_KERNELS
#include "kernels_dev.cuh"
#include "kernels_fused.cuh"
#include "kernels_ring.cuh"
#include "kernels_chan2.cuh"
#include "kernels_tb.cuh"
#include "kernels_large.cuh"
#include "kernels_long_api.h"

namespace slicq {
namespace {
using namespace slicq::kern;

// y += spill (the right neighbour's overlap-add spill, multi-GPU slice ranges)
__global__ void overlap_add_kernel(float *y, int64_t y_stride, const float *spill, int64_t count) {
  const int64_t row = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    y[row * y_stride + i] += spill[row * count + i];
}

// Prop. 4 sums (slicq_approx_error): one CTA per (stored channel, row).  c_P4 = c sqrt(M^L)/L,
// s_P4 = s sqrt(M)/(2N) (reading C22); (s^0 + s^1)[m h + n'] = c^m[n' + h] + c^{m+1}[n'],
// h = M/2 = N/a_k (two-layer array of Alg. 3, slices circular).
// full = 1 (complex input): the layouts of slicq_forward_complex / slicq_nsgt_forward_complex,
// channel index k' over all 2K+2 channels (mirror k' = 2K+2-k: M_k, after the stored ones)
__device__ __forceinline__ int64_t full_off(const ChanDev *ch, int kk, int K, int64_t C) {
  if (kk <= K + 1) return ch[kk].off;
  const int k = 2 * K + 2 - kk;
  return C + ch[K + 1].off - (ch[k].off + ch[k].M);
}
__global__ void __launch_bounds__(256) approx_kernel(const ChanDev *chs, const ChanDev *chl,
                                                     const float2 *s, const float2 *c, int64_t Cs,
                                                     int64_t Cl, int S, float scs, float scl_num,
                                                     double *out, int full, int K, int64_t Cs0,
                                                     int64_t Cl0) {
  const int kk = blockIdx.x, K2 = gridDim.x;
  const int k = kk <= K + 1 ? kk : 2 * K + 2 - kk;
  const int64_t b = blockIdx.y;
  const ChanDev a = chs[k], l = chl[k];
  const int64_t aoff = full ? full_off(chs, kk, K, Cs0) : a.off;
  const int64_t loff = full ? full_off(chl, kk, K, Cl0) : l.off;
  const int h = a.M / 2;
  const float ss = sqrtf((float)a.M) * scs, sl = sqrtf((float)l.M) * scl_num;
  const float2 *srow = s + b * (int64_t)S * Cs + aoff;
  const float2 *crow = c + b * Cl + loff;
  double e0 = 0.0, e1 = 0.0;
  for (int n = threadIdx.x; n < l.M; n += 256) {
    const int m = n / h, np = n - m * h;
    const int m1 = m + 1 == S ? 0 : m + 1;
    const float2 v0 = srow[(int64_t)m * Cs + np + h], v1 = srow[(int64_t)m1 * Cs + np];
    const float2 cv = crow[n];
    const float cr = cv.x * sl, ci = cv.y * sl;
    const float dr = cr - (v0.x + v1.x) * ss, di = ci - (v0.y + v1.y) * ss;
    e0 += (double)cr * cr + (double)ci * ci;
    e1 += (double)dr * dr + (double)di * di;
  }
  __shared__ double r0[256], r1[256];
  r0[threadIdx.x] = e0;
  r1[threadIdx.x] = e1;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      r0[threadIdx.x] += r0[threadIdx.x + w];
      r1[threadIdx.x] += r1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[(b * K2 + kk) * 2 + 0] = r0[0];
    out[(b * K2 + kk) * 2 + 1] = r1[0];
  }
}

const int kSizes[] = {1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 18, 20, 24, 25, 27, 30, 32};
const int kSmall[] = {4, 6, 8, 10, 12, 16, 18, 20, 24, 30, 32};

bool in_list(const int *l, int n, int v) {
  for (int i = 0; i < n; ++i)
    if (l[i] == v) return true;
  return false;
}
bool in_sizes(int v) { return in_list(kSizes, sizeof(kSizes) / sizeof(int), v); }
bool in_small(int v) { return in_list(kSmall, sizeof(kSmall) / sizeof(int), v); }

// M = M1 * M2 with both register-DFT sizes, minimising max(M1, M2) then padding.
bool factor_m(int M, int &M1, int &M2) {
  int best = 1 << 30, bp = 1 << 30;
  bool ok = false;
  for (int s : kSizes) {
    if (M % s) continue;
    const int o = M / s;
    if (!in_sizes(o)) continue;
    const int mx = std::max(s, o);
    const int pad = s * (o | 1);
    if (mx < best || (mx == best && pad < bp)) {
      best = mx;
      bp = pad;
      M1 = s;
      M2 = o;
      ok = true;
    }
  }
  return ok;
}

int threads_for(int logN) {
  switch (logN) {
    case 11: return Big<11>::T;
    case 12: return Big<12>::T;
    case 13: return Big<13>::T;
    case 14: return Big<14>::T;
  }
  return 0;
}

size_t spec_smem_for(int logN, int tr) {
  switch (logN) {
    case 11: return spec_smem_bytes<11>(tr);
    case 12: return spec_smem_bytes<12>(tr);
    case 13: return spec_smem_bytes<13>(tr);
    case 14: return spec_smem_bytes<14>(tr);
  }
  return 0;
}

constexpr size_t kSmemCap = 227 * 1024;  // per CTA
#ifndef SLICQ_SMALL_CAP
#define SLICQ_SMALL_CAP 640
#endif
constexpr int kSmallCap = SLICQ_SMALL_CAP;  // float2 scratch entries a small packet may use
#ifndef SLICQ_SMALL_MAX
#define SLICQ_SMALL_MAX 32
#endif
constexpr int kSmallMax = SLICQ_SMALL_MAX;  // channels with M <= this: one lane per channel
// channel-kernel variants: <largest DFT size, CTAs per SM (register budget)>
#ifndef SLICQ_LITE_MAX
#define SLICQ_LITE_MAX 16
#endif
#ifndef SLICQ_LITE_MINB
#define SLICQ_LITE_MINB 3
#endif
#ifndef SLICQ_MICRO_MAX
#define SLICQ_MICRO_MAX 0  // 0: no micro variant (8: measured within +-0.5 %, cfg2 -7 %)
#endif
#ifndef SLICQ_MICRO_MINB
#define SLICQ_MICRO_MINB 4
#endif
#ifndef SLICQ_LITE_MINB_INV
#define SLICQ_LITE_MINB_INV SLICQ_LITE_MINB
#endif
constexpr int kLiteMax = SLICQ_LITE_MAX, kLiteMinB = SLICQ_LITE_MINB, kFullMax = 32, kFullMinB = 2;
constexpr int kLiteMinBInv = SLICQ_LITE_MINB_INV;  // the inverse lite variant's CTAs per SM
constexpr int kMicroMax = SLICQ_MICRO_MAX, kMicroMinB = SLICQ_MICRO_MINB;
constexpr int kVariants = 3;  // micro (DFT sizes <= kMicroMax), lite (<= kLiteMax), full
using ChanFn = void (*)(const KArgs);
template <int MK>
static ChanFn inv_fn(int variant) {
  if (variant == 0) return slicq_inv_chan_kernel<(kMicroMax ? kMicroMax : 1), kMicroMinB, MK>;
  return variant == 1 ? slicq_inv_chan_kernel<kLiteMax, kLiteMinBInv, MK>
                      : slicq_inv_chan_kernel<kFullMax, kFullMinB, MK>;
}
// variant 0 micro, 1 lite, 2 full; mask: inverse with a fused coefficient mask (0 none,
// 1 linear, 2 dB)
static ChanFn chan_fn(bool fwd, int variant, int mask = 0) {
  if (fwd) {
    if (variant == 0) return slicq_fwd_chan_kernel<(kMicroMax ? kMicroMax : 1), kMicroMinB>;
    return variant == 1 ? slicq_fwd_chan_kernel<kLiteMax, kLiteMinB>
                        : slicq_fwd_chan_kernel<kFullMax, kFullMinB>;
  }
  switch (mask) {
    case 1: return inv_fn<1>(variant);
    case 2: return inv_fn<2>(variant);
  }
  return inv_fn<0>(variant);
}
// TMA-staged channel kernels (kernels_tb.cuh); variant 0 (micro) runs as lite
static ChanFn tb_fn(bool fwd, int variant) {
  if (fwd)
    return variant <= 1 ? slicq_fwd_chan_tb_kernel<kLiteMax, kLiteMinB>
                        : slicq_fwd_chan_tb_kernel<kFullMax, kFullMinB>;
  return variant <= 1 ? slicq_inv_chan_tb_kernel<kLiteMax, kLiteMinBInv>
                      : slicq_inv_chan_tb_kernel<kFullMax, kFullMinB>;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int64_t env_int(const char *name, int64_t dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoll(v);
}

}  // namespace

// logN 11..16: sliCQ (and full-length CQ-NSGT) slices; 17..21: full-length CQ-NSGT only
int device_supports(int logN) { return logN >= 11 && logN <= 21; }

namespace {
// Long mode (sl_len = 2^18 .. 2^22): the full-length CQ-NSGT of kernels_long.cuh.  No
// packets or element tables: per-channel fp32 weights and, for the synthesis, the list of
// channel terms of every half-spectrum bin (Hermitian rule C15, plan order).
int configure_long(slicq_plan *p, int logN) {
  KernelConfig &kc = p->kc;
  kc.logN = logN;
  kc.large = false;
  kc.longmode = true;
  kc.npackets = kc.nlite = 0;
  const int K2 = p->K + 2;
  const int64_t N = p->N, N2 = 2 * N;
  // channels by size class (kernels_long_api.h); the class list replaces the packet list
  p->pchans.clear();
  p->lm1.assign(K2, 0);
  int maxm[kLongClasses] = {};
  for (int c = 0; c < kLongClasses; ++c) {
    kc.lcls.off[c] = (int)p->pchans.size();
    for (int k = 0; k < K2; ++k) {
      const int M = p->M[k];
      int cls = 0;
      while (cls + 1 < kLongClasses && M > long_class_maxm(cls)) ++cls;
      if (cls != c) continue;
      int Msm = M;  // the shared-memory DFT size of the channel
      if (c == kLongClasses - 1) {  // four-step M1 x M2 (kernels_long.cuh)
        for (int m1 : {2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16})
          if (M % m1 == 0 && M / m1 <= kLongSmemMax) {
            p->lm1[k] = m1;
            break;
          }
        if (!p->lm1[k])
          return set_error(SLICQ_EUNSUPPORTED, "channel length M_k = " + std::to_string(M) +
                                                   " has no factor M1 <= 16 with M_k / M1 <= " +
                                                   std::to_string(kLongSmemMax));
        Msm = M / p->lm1[k];
      }
      p->pchans.push_back(k);
      maxm[c] = std::max(maxm[c], Msm);
    }
    kc.lcls.smem[c] = maxm[c] ? sizeof(float2) * (size_t)(padi(maxm[c]) + 1 +
                                                          long_twiddle_entries(maxm[c]) +
                                                          kDifPlanEntries)
                              : 0;
  }
  kc.lcls.off[kLongClasses] = (int)p->pchans.size();
  const int64_t nterms = (int64_t)p->g.size();
  if (nterms >= (int64_t(1) << 31)) return set_error(SLICQ_EUNSUPPORTED, "too many filter terms");
  p->lgw.assign(nterms, 0.f);
  p->lgdw.assign(nterms, 0.f);
  std::vector<uint32_t> cnt(N + 2, 0u);
  auto bins = [&](int64_t j, int64_t &b1, int64_t &b2) {  // direct bin, conjugate bin (or -1)
    int64_t p1 = j % N2;
    if (p1 < 0) p1 += N2;
    const int64_t p2 = p1 == 0 ? 0 : N2 - p1;
    b1 = p1 <= N ? p1 : -1;
    b2 = p2 <= N ? p2 : -1;
  };
  for (int k = 0; k < K2; ++k) {
    const double sc = 1.0 / std::sqrt((double)p->M[k]);
    const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;  // self-mirrored plateaus (C15)
    for (int dd = 0; dd < p->len[k]; ++dd) {
      const int64_t e = p->goff[k] + dd;
      p->lgw[e] = (float)(p->g[e] * sc);
      p->lgdw[e] = (float)(p->gdual[e] * sc * half);
      int64_t b1, b2;
      bins(p->lo[k] + dd, b1, b2);
      if (b1 >= 0) ++cnt[b1];
      if (b2 >= 0) ++cnt[b2];
    }
  }
  p->lrow.assign(N + 2, 0u);
  for (int64_t b = 0; b <= N; ++b) {
    if (!cnt[b]) return set_error(SLICQ_EINTERNAL, "half-spectrum bin without a channel term");
    p->lrow[b + 1] = p->lrow[b] + cnt[b];
  }
  p->lent.assign(p->lrow[N + 1], 0u);
  std::vector<uint32_t> fill(p->lrow.begin(), p->lrow.end() - 1);
  for (int k = 0; k < K2; ++k)
    for (int dd = 0; dd < p->len[k]; ++dd) {
      const uint32_t e = (uint32_t)(p->goff[k] + dd);
      int64_t b1, b2;
      bins(p->lo[k] + dd, b1, b2);
      if (b1 >= 0) p->lent[fill[b1]++] = e;
      if (b2 >= 0) p->lent[fill[b2]++] = e | 0x80000000u;
    }
  // staging per row: X[0..N] then the four-step intermediate (forward); the channel terms
  // then the packed spectrum W (inverse)
  kc.toff_f = (N + 2) & ~int64_t(1);
  kc.xs = kc.toff_f + N;
  kc.toff_i = (nterms + 1) & ~int64_t(1);
  kc.zs = kc.toff_i + N;
  // four-step channels: their M_k-entry scratch after both layouts (same offset per channel
  // in the forward and the inverse row)
  p->lsoff.assign(K2, 0);
  {
    int64_t so = std::max(kc.xs, kc.zs);
    bool any = false;
    for (int k = 0; k < K2; ++k)
      if (p->lm1[k]) {
        p->lsoff[k] = so;
        so += (p->M[k] + 1) & ~1;
        any = true;
      }
    if (any) {
      if (so >= (int64_t(1) << 31)) return set_error(SLICQ_EUNSUPPORTED, "staging row too long");
      kc.xs = kc.zs = so;
    }
  }
  kc.zso = 0;
  kc.nover = 0;
  kc.tile = 1;
  const int64_t per_unit = sizeof(float2) * std::max(kc.xs, kc.zs);
  const int64_t budget = env_int("SLICQ_STAGE_MB", 8192) << 20;
  kc.chunk_units = std::min<int64_t>(65535, std::max<int64_t>(1, budget / per_unit));
  return SLICQ_OK;
}
}  // namespace

// generic-length spectrum kernels: the in-place mixed-radix DIT plan of N (radices 16, 8, 4,
// 2, 3, 5; r_1 the outermost factor), its digit-reversal map and twiddle table
static int configure_generic(slicq_plan *p) {
  const int N = (int)p->N;
  std::vector<int> R;
  int m = N;
  for (int r : {16, 8, 4, 2, 3, 5})
    while (m % r == 0 && (r != 16 || m >= 256)) {
      R.push_back(r);
      m /= r;
    }
  for (int r : {4, 2})
    while (m % r == 0) {
      R.push_back(r);
      m /= r;
    }
  if (m != 1 || (int)R.size() > kGenericMaxPasses)
    return set_error(SLICQ_EUNSUPPORTED, "slice length is not 2/3/5-smooth");
  KernelConfig &kc = p->kc;
  kc.gargs = GArgs{};
  kc.gargs.N = N;
  kc.gargs.np = (int)R.size();
  int S = 1;
  for (int i = (int)R.size() - 1, q = 0; i >= 0; --i, ++q) {  // innermost factor first
    kc.gargs.pass[q] = GPass{R[i], S};
    S *= R[i];
  }
  p->gperm.assign(N, 0);
  for (int n = 0; n < N; ++n) {
    int rem = n, prod = 1, pos = 0;
    for (int r : R) {
      const int j = rem % r;
      rem /= r;
      prod *= r;
      pos += j * (N / prod);
    }
    p->gperm[n] = pos;
  }
  p->gtw.resize(2 * (size_t)N);
  for (int t = 0; t < N; ++t) {
    const double a = -2.0 * 3.14159265358979323846 * (double)t / (double)N;
    p->gtw[2 * t] = (float)std::cos(a);
    p->gtw[2 * t + 1] = (float)std::sin(a);
  }
  return SLICQ_OK;
}

int configure_kernels(slicq_plan *p) {
  int logN = 0;
  while ((int64_t(1) << logN) < p->N) ++logN;
  const bool pow2 = (int64_t(1) << logN) == p->N;
  const bool generic = (!pow2 || env_int("SLICQ_GENERIC", 0) != 0) && p->N <= kGenericMaxN &&
                       p->N >= 64 && p->sampled_from == 0;
  if (!generic && (!pow2 || !device_supports(logN)))
    return set_error(SLICQ_EUNSUPPORTED,
                     "CUDA path implements sl_len = 2^12 .. 2^17 and any 2/3/5-smooth sl_len "
                     "<= " + std::to_string(2 * kGenericMaxN) + " (sliCQ), up to 2^22 "
                     "(full-length CQ-NSGT)");
  if (!generic && logN >= 17) return configure_long(p, logN);
  if (!p->painless)  // the element tables hold one term per fold position
    return set_error(SLICQ_EUNSUPPORTED, "a system with M_k < L_k (sampled_from) needs "
                                         "sl_len >= 2^18 on the device");
  KernelConfig &kc = p->kc;
  kc.generic = generic;
  if (generic) {
    const int rc = configure_generic(p);
    if (rc != SLICQ_OK) return rc;
    logN = 0;
  }
  kc.logN = logN;
  kc.large = !generic && logN >= 15;
  kc.threads = generic ? 512 : kc.large ? LT : threads_for(logN);
  kc.spec_smem = generic ? generic_smem_bytes((int)p->N)
                 : kc.large ? (logN == 15 ? large_smem_bytes<15>() : large_smem_bytes<16>())
                            : spec_smem_for(logN, (int)p->tr);
  if (kc.spec_smem > kSmemCap)
    return set_error(SLICQ_EUNSUPPORTED, "spectrum kernel shared memory exceeds 227 KB");
  if (!kc.large && !kc.generic) {
    switch (logN) {
      case 11: kc.spec_smem_p = spec_persist_smem_bytes<11>((int)p->tr); break;
      case 12: kc.spec_smem_p = spec_persist_smem_bytes<12>((int)p->tr); break;
      case 13: kc.spec_smem_p = spec_persist_smem_bytes<13>((int)p->tr); break;
      case 14: kc.spec_smem_p = spec_persist_smem_bytes<14>((int)p->tr); break;
    }
    kc.inv_persist = env_int("SLICQ_INV_PERSIST", 1) != 0 && kc.spec_smem_p <= kSmemCap;
    kc.fwd_persist = env_int("SLICQ_FWD_PERSIST", 1) != 0;
  }
  const int K2 = p->K + 2;
  const int N = (int)p->N, N2 = 2 * N;
  std::map<int, std::pair<int, int>> fac;
  for (int k = 0; k < K2; ++k) {
    const int M = p->M[k];
    if (fac.count(M)) continue;
    int m1 = 0, m2 = 0;
    if (M <= 32 && in_small(M)) {
      fac[M] = {M, 1};
      continue;
    }
    if (M > 1024 || !factor_m(M, m1, m2)) {
      // too long for the register-DFT packets: one CTA per (channel, unit) with a
      // shared-memory mixed-radix DFT (the long-mode channel kernels, kernels_long.cuh)
      if (M > long_class_maxm(kLongClasses - 2))
        return set_error(SLICQ_EUNSUPPORTED, "channel length M_k = " + std::to_string(M) +
                                                 " exceeds the sliCQ channel kernels (26000)");
      fac[M] = {0, 0};
      continue;
    }
    fac[M] = {m1, m2};
  }
  // big channels (fac = {0, 0}) by size class; their fp32 weights
  p->pbig.clear();
  kc.nbig = 0;
  {
    int maxm[kLongClasses] = {};
    for (int c = 0; c < kLongClasses - 1; ++c) {
      kc.bcls.off[c] = (int)p->pbig.size();
      for (int k = 0; k < K2; ++k) {
        const int M = p->M[k];
        if (fac[M].first != 0) continue;
        int cls = 0;
        while (cls + 1 < kLongClasses - 1 && M > long_class_maxm(cls)) ++cls;
        if (cls != c) continue;
        p->pbig.push_back(k);
        maxm[c] = std::max(maxm[c], M);
      }
      kc.bcls.smem[c] = maxm[c] ? sizeof(float2) * (size_t)(padi(maxm[c]) + 1 +
                                                            long_twiddle_entries(maxm[c]) +
                                                            kDifPlanEntries)
                                : 0;
    }
    kc.bcls.off[kLongClasses - 1] = kc.bcls.off[kLongClasses] = (int)p->pbig.size();
    kc.bcls.smem[kLongClasses - 1] = 0;
    kc.nbig = (int)p->pbig.size();
    if (kc.nbig && p->lgw.size() != p->g.size()) {
      p->lgw.assign(p->g.size(), 0.f);
      p->lgdw.assign(p->g.size(), 0.f);
      for (int k = 0; k < K2; ++k) {
        const double sc = 1.0 / std::sqrt((double)p->M[k]);
        const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;
        for (int d = 0; d < p->len[k]; ++d) {
          const int64_t e = p->goff[k] + d;
          p->lgw[e] = (float)(p->g[e] * sc);
          p->lgdw[e] = (float)(p->gdual[e] * sc * half);
        }
      }
    }
  }

  // X(j) = X[b] or conj(X[b]) for real input
  auto bin_of = [&](int j, int &conj) {
    int jj = j % N2;
    if (jj < 0) jj += N2;
    conj = jj > N;
    return jj > N ? N2 - jj : jj;
  };
  // TMA-staged channel kernels (kernels_tb.cuh): a warp task's operand block (forward: the
  // packet's bins for nu units; inverse: its coefficient columns for nu units) must fit the
  // per-warp buffer; nu is capped so that it does (SLICQ_TB_CAP entries)
  kc.tb = env_int("SLICQ_TB", 0) != 0;  // opt-in: measured slower
  const int tb_cap = (int)env_int("SLICQ_TB_CAP", 600);
  kc.tbe_f = kc.tbe_i = 0;

  // ---------------- packets: runs of consecutive channels of one length
  struct Pk {
    PacketDev d;
    std::vector<int> ks;
    int M, scr;
  };
  std::vector<Pk> pks;
  for (int k = 0; k < K2;) {
    const int M = p->M[k];
    if (fac[M].first == 0) {  // big channel (above)
      ++k;
      continue;
    }
    const bool small = M <= kSmallMax && in_small(M);
    const int m1 = fac[M].first, m2 = fac[M].second;
    const int nch = small ? std::min(32, kSmallCap / M) : std::max(1, 32 / std::max(m1, m2));
    Pk pk;
    pk.d = PacketDev{};
    pk.M = M;
    pk.d.m1m2 = m1 | (m2 << 8) | ((small ? 1 : 0) << 17);
    pk.d.mag1 = (uint32_t)((65536 + m1 - 1) / m1);
    pk.d.mag2 = (uint32_t)((65536 + m2 - 1) / m2);
    while (k < K2 && p->M[k] == M && (int)pk.ks.size() < nch) pk.ks.push_back(k++);
    const int r = (int)pk.ks.size();
    pk.d.nch = r;
    // units per warp task: fill the lanes (short runs of one M would leave them idle)
    int nu = small ? std::max(1, std::min(32 / r, kSmallCap / (r * M)))
                   : std::max(1, 32 / (r * std::max(m1, m2)));
    if (kc.tb) {
      int bl = N, bh = 0;
      for (int kk : pk.ks)
        for (int dd = 0; dd < p->len[kk]; ++dd) {
          int cj = 0;
          const int b = bin_of(p->lo[kk] + dd, cj);
          bl = std::min(bl, b);
          bh = std::max(bh, b);
        }
      const int wf = ((bh + 2) & ~1) - (bl & ~1);
      const int wi = (int)(((p->off[pk.ks.back()] + M + 1) & ~int64_t(1)) - (p->off[pk.ks[0]] & ~int64_t(1)));
      while (nu > 1 && nu * std::max(wf, wi) > tb_cap) --nu;
      kc.tbe_f = std::max(kc.tbe_f, nu * wf);
      kc.tbe_i = std::max(kc.tbe_i, nu * wi);
    }
    pk.d.nu = nu;
    pk.d.magc = (uint32_t)((65536 + r - 1) / r);
    pk.d.ustride = small ? r : r * m1 * (m2 | 1);
    // small packets: scratch q * nvp + vc with the odd stride nvp = (nu r) | 1, so that the
    // inverse term scatter (a warp reads consecutive q of one channel) is bank-conflict free
    pk.scr = small ? ((nu * r) | 1) * M : nu * pk.d.ustride;
    pks.push_back(std::move(pk));
  }
  // shape-sorted (the warps of a channel-kernel CTA run the same code), longer first, by
  // channel-kernel variant: packets whose DFT sizes are all <= kMicroMax / kLiteMax run in
  // the variants with the smaller register budgets (more resident warps), the rest in full
  auto variant = [](const Pk &x) {
    const int m1 = x.d.m1m2 & 255, m2 = (x.d.m1m2 >> 8) & 255, mx = std::max(m1, m2);
    return mx <= kMicroMax ? 0 : mx <= kLiteMax ? 1 : 2;
  };
  std::stable_sort(pks.begin(), pks.end(), [&](const Pk &x, const Pk &y) {
    const int vx = variant(x), vy = variant(y);
    return vx != vy ? vx < vy : x.M > y.M;
  });
  for (int v = 0; v <= kVariants; ++v) kc.voff[v] = 0;
  for (const Pk &x : pks) ++kc.voff[variant(x) + 1];
  for (int v = 0; v < kVariants; ++v) kc.voff[v + 1] += kc.voff[v];
  kc.nlite = kc.voff[2];

  // ---------------- inverse destinations (I3b gather without index tables): every channel
  // contribution Z_k[d] goes to half-spectrum bin b by the Hermitian rule of C15 (term at
  // j mod 2N if <= N, conjugate at -j mod 2N if <= N).  The staging row of a unit holds two
  // slot arrays [slot][N+1] (slot preferred = channel parity: with the Hann filters' 50%
  // overlap almost every bin has exactly two terms, one from an even and one from an odd
  // channel) and an overflow area for the rare deeper bins (ordered by bin, summed in order).
  // Unused slots receive an explicit zero.  The IA kernel reads slot0[b] + slot1[b] (+ the
  // overflow run dpos[b]), coalesced and table-free for regular bins.
  struct Dst {
    int d;
    uint32_t dst;
    int conj;
    bool zero;
  };
  std::vector<std::vector<Dst>> dsts(K2);
  {
    const int64_t zso = (N + 2) & ~int64_t(1);
    std::vector<uint8_t> used(N + 1, 0);
    std::vector<std::vector<std::pair<int, int>>> ovf(N + 1);  // (k, index into dsts[k])
    std::vector<std::pair<int, int>> first(N + 1, std::make_pair(-1, -1));
    for (int k = 0; k < K2; ++k)
      for (int dd = 0; dd < p->len[k]; ++dd) {
        const int j = p->lo[k] + dd;
        int p1 = j % N2;
        if (p1 < 0) p1 += N2;
        const int p2 = p1 == 0 ? 0 : N2 - p1;
        for (int t = 0; t < 2; ++t) {
          const int b = t == 0 ? p1 : p2;
          if (b > N) continue;
          if (first[b].first < 0) first[b] = std::make_pair(k, dd);
          const int pref = k & 1;
          int slot = 2;
          if (!((used[b] >> pref) & 1)) slot = pref;
          else if (!((used[b] >> (pref ^ 1)) & 1)) slot = pref ^ 1;
          if (slot < 2) {
            used[b] |= (uint8_t)(1 << slot);
            dsts[k].push_back(Dst{dd, (uint32_t)(slot * zso + b), t, false});
          } else {
            ovf[b].push_back(std::make_pair(k, (int)dsts[k].size()));
            dsts[k].push_back(Dst{dd, 0u, t, false});
          }
        }
      }
    p->dpos.assign(N + 2, 0u);  // N + 2: the kernels read bin pairs
    int64_t start = 0;
    for (int b = 0; b <= N; ++b) {
      if (first[b].first < 0)
        return set_error(SLICQ_EINTERNAL, "half-spectrum bin without a channel term");
      for (int sl = 0; sl < 2; ++sl)  // explicit zeros for unused slots
        if (!((used[b] >> sl) & 1))
          dsts[first[b].first].push_back(Dst{first[b].second, (uint32_t)(sl * zso + b), 0, true});
      if (ovf[b].empty()) continue;
      const int64_t cnt = (int64_t)ovf[b].size();
      if (start >= (1 << 20) || cnt >= (1 << 11))
        return set_error(SLICQ_EUNSUPPORTED, "inverse overflow list too long");
      p->dpos[b] = (uint32_t)start | ((uint32_t)cnt << 20);
      for (int64_t i = 0; i < cnt; ++i)
        dsts[ovf[b][i].first][ovf[b][i].second].dst = (uint32_t)(2 * zso + start + i);
      start += cnt;
    }
    kc.zso = zso;
    kc.nover = start;
    // the overflow bins as a list (the persistent inverse spectrum kernel sums them in a
    // pre-pass spread over all threads of the CTA, kernels_dev.cuh inv_unit)
    // ovbins[i] = (first term, term count) of the i-th overflow bin in the flat term list
    // ovterm (offsets into a unit's staging row: slot 0, slot 1, then the overflow run, the
    // order of the sum)
    p->ovbins.clear();
    p->ovterm.clear();
    p->dord.assign(N + 2, 0u);
    for (int b = 0; b <= N; ++b)
      if (p->dpos[b]) {
        const uint32_t st = p->dpos[b] & 0xfffffu, cnt = p->dpos[b] >> 20;
        p->ovbins.push_back(make_uint2((uint32_t)p->ovterm.size(), 2u + cnt));
        p->ovterm.push_back((uint32_t)b);
        p->ovterm.push_back((uint32_t)(zso + b));
        for (uint32_t k = 0; k < cnt; ++k) p->ovterm.push_back((uint32_t)(2 * zso + st + k));
        p->dord[b] = (uint32_t)p->ovbins.size();
      }
    // the persistent inverse spectrum kernel stages the terms and keeps the sums in shared
    // memory
    kc.spec_smem_p += sizeof(float2) * (p->ovbins.size() + p->ovterm.size());
    if (kc.spec_smem_p > kSmemCap) kc.inv_persist = false;
    if (2 * zso + start >= (int64_t(1) << 18))
      return set_error(SLICQ_EUNSUPPORTED, "slice too long for the inverse element tables");
  }

  // ---------------- big channels: their terms' destinations (kernels_long.cuh
  // long_chan_inv_slots): (dst | conj << 31, d | zero << 31)
  p->bent.clear();
  p->bentoff.assign(K2, 0);
  p->bentn.assign(K2, 0);
  for (int k : p->pbig) {
    p->bentoff[k] = (int)p->bent.size();
    for (const Dst &ds : dsts[k])
      p->bent.push_back(make_uint2(ds.dst | ((uint32_t)ds.conj << 31),
                                   (uint32_t)ds.d | ((ds.zero ? 1u : 0u) << 31)));
    p->bentn[k] = (int)p->bent.size() - p->bentoff[k];
  }

  // ---------------- element tables
  auto fbits = [](double v) {
    const float f = (float)v;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
  };
  for (double gv : p->g)  // the element tables carry the conjugation flag in the sign bit
    if (!(gv >= 0.0)) return set_error(SLICQ_EUNSUPPORTED, "negative filter value");
  p->packets.clear();
  p->pchans.clear();
  p->fent.clear();
  p->ient.clear();
  int need = 8, need_f = 8;
  for (Pk &pk : pks) {
    PacketDev &d = pk.d;
    const int M = pk.M;
    const bool small = (d.m1m2 >> 17) & 1;
    const int m1 = d.m1m2 & 255, S2 = ((d.m1m2 >> 8) & 255) | 1;
    {  // bins the fold reads (X(j) or conj X(2N - j) for real input)
      int bl = N, bh = 0;
      for (int k : pk.ks)
        for (int dd = 0; dd < p->len[k]; ++dd) {
          int conj = 0;
          const int b = bin_of(p->lo[k] + dd, conj);
          bl = std::min(bl, b);
          bh = std::max(bh, b);
        }
      d.xlo = bl;
      d.xhi = bh;
    }
    // zero-padding entries of the fold tables (weight 0) point at xlo: a bin of the packet's
    // band, which the TMA-staged kernels hold in shared memory (kernels_tb.cuh)
    const uint32_t padbin = (uint32_t)d.xlo;
    d.chan_off = (int)p->pchans.size();
    d.fent_off = (int)p->fent.size();
    d.ient_off = (int)p->ient.size();
    const double sc = 1.0 / std::sqrt((double)M);  // Alg. 1 sqrt(M) IFFT (1/M); Alg. 2 FFT/sqrt(M)
    // forward fold table: bin | scratch position << 18, weight g_k/sqrt(M_k) whose sign bit
    // marks the conjugated (mirrored) bins (g >= 0); weight 0 and bin 0 for the zero padding
    if (small) {
      std::vector<uint2> t(32 * M, make_uint2(padbin, 0u));
      for (int c = 0; c < d.nch; ++c) {
        const int k = pk.ks[c];
        const int lo_mod = ((p->lo[k] % M) + M) % M;
        for (int q = 0; q < M; ++q) {
          int dd = q - lo_mod;
          if (dd < 0) dd += M;
          if (dd >= p->len[k]) continue;
          int conj = 0;
          const int b = bin_of(p->lo[k] + dd, conj);
          t[q * 32 + c] = make_uint2((uint32_t)b, fbits(conj ? -(p->g[p->goff[k] + dd] * sc)
                                                          : p->g[p->goff[k] + dd] * sc));
        }
      }
      p->fent.insert(p->fent.end(), t.begin(), t.end());
    } else {
      for (int c = 0; c < d.nch; ++c) {
        const int k = pk.ks[c];
        const int lo_mod = ((p->lo[k] % M) + M) % M;
        for (int q = 0; q < M; ++q) {
          int dd = q - lo_mod;
          if (dd < 0) dd += M;
          const uint32_t pos = (uint32_t)(c * m1 * S2 + q);
          uint2 e = make_uint2(padbin | (pos << 18), 0u);
          if (dd < p->len[k]) {
            int conj = 0;
            const int b = bin_of(p->lo[k] + dd, conj);
            const double w = p->g[p->goff[k] + dd] * sc;
            e = make_uint2((uint32_t)b | (pos << 18), fbits(conj ? -w : w));
          }
          p->fent.push_back(e);
        }
      }
    }
    // inverse entry table: e over (channel, destination): scratch position | dst << 14,
    // weight g~_k[j]/sqrt(M_k) (plateaus x 1/2, C15) with the conjugation flag in bit 31
    int nz = 0;
    for (int c = 0; c < d.nch; ++c) {
      const int k = pk.ks[c];
      const int lo_mod = ((p->lo[k] % M) + M) % M;
      const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;  // self-mirrored plateaus (C15)
      for (const Dst &ds : dsts[k]) {
        int q = lo_mod + ds.d;
        if (q >= M) q -= M;
        // small: scratch q * ((nu * nch) | 1) + vc; big: vc * M1 * S2 + q (+ u * ustride in-kernel)
        const uint32_t pos = small ? (uint32_t)(q * ((d.nu * d.nch) | 1) + c) : (uint32_t)(c * m1 * S2 + q);
        const double w = ds.zero ? 0.0 : p->gdual[p->goff[k] + ds.d] * sc * half;
        if (!(w >= 0.0)) return set_error(SLICQ_EUNSUPPORTED, "negative dual filter value");
        p->ient.push_back(make_uint2(pos | (ds.dst << 14), fbits(w) | ((uint32_t)ds.conj << 31)));
        ++nz;
      }
    }
    d.nz = nz;
    for (int k : pk.ks) p->pchans.push_back(k);
    p->packets.push_back(d);
    need = std::max(need, pk.scr);
    if (!small) need_f = std::max(need_f, pk.scr);
  }
  kc.npackets = (int)p->packets.size();
  kc.scr = (need + 7) & ~7;
  kc.chan_smem = sizeof(float2) * (size_t)kc.scr * (CHAN_T / 32);
  kc.scr_f = (need_f + 7) & ~7;
  kc.tbe_f = (kc.tbe_f + 7) & ~7;
  kc.tbe_i = (kc.tbe_i + 7) & ~7;
  // [scratch][buffers][mbarriers][cursors] (kernels_tb.cuh)
  kc.tb_smem_f = sizeof(float2) * (size_t)(kc.scr_f + kc.tbe_f + 1) * (CHAN_T / 32) +
                 2 * sizeof(kern::TbCursor) * (CHAN_T / 32);
  kc.tb_smem_i = sizeof(float2) * (size_t)(kc.scr + kc.tbe_i + 1) * (CHAN_T / 32) +
                 2 * sizeof(kern::TbCursor) * (CHAN_T / 32);
  if (kc.tb && std::max(kc.tb_smem_f, kc.tb_smem_i) > kSmemCap) kc.tb = false;
  // element encoding: bin < 2^17, scratch position < 2^14 (fold table, kernels_dev.cuh)
  if (N > (1 << 17) - 1 || kc.scr > (1 << 14))
    return set_error(SLICQ_EUNSUPPORTED, "slice or channel too long for the element tables");
  if (kc.chan_smem > kSmemCap)
    return set_error(SLICQ_EUNSUPPORTED, "channel scratch does not fit in shared memory");

  // ---------------- staging: X spectra (N+1) and inverse slots + overflow per unit
  kc.xs = (p->N + 2) & ~int64_t(1);
  kc.zs = (2 * kc.zso + kc.nover + 1) & ~int64_t(1);
  if (kc.large) {  // the four-step intermediate (N per unit) follows X / the contributions
    kc.toff_f = kc.xs;
    kc.toff_i = kc.zs;
    kc.xs += p->N;
    kc.zs += p->N;
  }
  kc.tile = (int)std::max<int64_t>(1, env_int("SLICQ_TILE", 128));
  kc.stiles = (int)std::max<int64_t>(0, env_int("SLICQ_STILES", 0));
  kc.pf = (int)env_int("SLICQ_INV_PF", 0);
  kc.chan_per_sm = (int)env_int("SLICQ_CHAN_PER_SM", 0);  // dev override: 0 = occupancy
  // staging is sized for one chunk of units; calls with more units run chunk by chunk
  // (each chunk costs kernel tails, so the default budget keeps every BASELINE config in a
  // single chunk: 8 GB of staging = 61 K slices of 2N = 16384)
  const int64_t per_unit = sizeof(float2) * std::max(kc.xs, kc.zs);
  const int64_t budget = env_int("SLICQ_STAGE_MB", 8192) << 20;
  int64_t cu = env_int("SLICQ_CHUNK_UNITS", std::max<int64_t>(1, budget / per_unit));
  // chunk pipelining (Pipe below): calls of >= pipe_min units run as pipe_parts chunks
  kc.pipe = env_int("SLICQ_PIPE", 1) != 0;
  kc.pdl = env_int("SLICQ_PDL", 1) != 0;  // programmatic dependent launch between kernels
  kc.pipe_min = env_int("SLICQ_PIPE_MIN_UNITS", 8192);
  kc.pipe_parts = std::max<int64_t>(2, env_int("SLICQ_PIPE_PARTS", 4));
  cu = std::min<int64_t>(cu, 0x7fffffff);  // grid x dimension of the spectrum kernels
  cu = std::max<int64_t>(kc.tile, cu / kc.tile * kc.tile);
  kc.chunk_units = cu;
  int rc = configure_fused(p);
  if (rc == SLICQ_OK) rc = configure_ring(p);
  if (rc == SLICQ_OK) rc = configure_fwd2(p);
  return rc;
}

int upload(slicq_plan *p) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  p->device = dev;
  const int K2 = p->K + 2;
  const int64_t N = p->N, N2 = 2 * N;
  // channel twiddle tables e^{+2 pi i t / M}, one per distinct M
  std::map<int, int> twoff;
  std::vector<float> twM;
  for (int k = 0; k < K2; ++k) {
    const int M = p->M[k];
    if (twoff.count(M)) continue;
    twoff[M] = (int)(twM.size() / 2);
    for (int t = 0; t < M; ++t) {
      const double ang = 2.0 * 3.14159265358979323846 * (double)t / (double)M;
      twM.push_back((float)std::cos(ang));
      twM.push_back((float)std::sin(ang));
    }
  }
  for (std::vector<FChan> *v : {&p->fchf, &p->fchi, &p->f2ch})  // channel index -> twiddle table
    for (FChan &f : *v) f.twoff = twoff[p->M[f.twoff]];
  std::vector<ChanDev> ch(K2);
  for (int k = 0; k < K2; ++k) {
    ChanDev &c = ch[k];
    c.lo = p->lo[k];
    c.len = p->len[k];
    c.M = p->M[k];
    c.goff = (int32_t)p->goff[k];
    c.off = (int32_t)p->off[k];
    c.twoff = twoff[c.M];
    c.scale = (float)(1.0 / std::sqrt((double)c.M));
    c.lo_mod = ((c.lo % c.M) + c.M) % c.M;
    if (p->kc.longmode) {
      c.m1 = p->lm1[k];
      c.soff = (int32_t)p->lsoff[k];
    } else if (!p->bentn.empty() && p->bentn[k]) {  // big sliCQ channel: its term destinations
      c.m1 = p->bentn[k];
      c.soff = p->bentoff[k];
    }
  }
  std::vector<float> h0(N2), h0d(N2);
  for (int64_t i = 0; i < N2; ++i) {
    h0[i] = (float)p->h0[i];
    h0d[i] = (float)p->h0dual[i];
  }
  // e^{-i pi t/N}: t < 64, then t = 64 h
  std::vector<float> tw;
  for (int t = 0; t < 64; ++t) {
    const double a = -3.14159265358979323846 * t / (double)N;
    tw.push_back((float)std::cos(a));
    tw.push_back((float)std::sin(a));
  }
  for (int64_t h = 0; h < N2 / 64; ++h) {
    const double a = -3.14159265358979323846 * (double)(64 * h) / (double)N;
    tw.push_back((float)std::cos(a));
    tw.push_back((float)std::sin(a));
  }
  // complex-input column maps (kernels_complex.cu): full layout (stored 0..K+1, then the
  // mirrors of K..1) -> (source stored column, e^{2 pi i 2N n/M} table index << 1 | mirror);
  // stored column -> (its mirror's full-layout column, table index << 1 | (DC ? no phase))
  {
    const int K2 = p->K + 2;
    int64_t Cf = p->C;
    for (int k = 1; k <= p->K; ++k) Cf += p->M[k];
    p->cxf.assign(Cf, make_uint2(0u, 0u));
    p->cxs.assign(p->C, make_uint2(0u, 0u));
    for (int64_t j = 0; j < p->C; ++j) p->cxf[j] = make_uint2((uint32_t)j, 0u);
    int64_t mo = p->C;
    for (int k = p->K; k >= 1; --k) {  // mirror of k: full channel 2K+2-k, after the stored
      const int M = p->M[k];
      const int64_t n2m = (2 * N) % M;
      for (int n = 0; n < M; ++n) {
        const uint32_t t = (uint32_t)(twoff[M] + (int)((n2m * n) % M));
        p->cxf[mo + n] = make_uint2((uint32_t)(p->off[k] + n), (t << 1) | 1u);
        p->cxs[p->off[k] + n] = make_uint2((uint32_t)(mo + n), t << 1);
      }
      mo += M;
    }
    for (int k : {0, K2 - 1}) {  // self-mirrored plateaus
      const int M = p->M[k];
      const int64_t n2m = (2 * N) % M;
      for (int n = 0; n < M; ++n) {
        const uint32_t t = (uint32_t)(twoff[M] + (int)((n2m * n) % M));
        p->cxs[p->off[k] + n] = make_uint2((uint32_t)(p->off[k] + n), k == 0 ? 1u : (t << 1));
      }
    }
  }
  struct Part {
    const void *src;
    size_t bytes;
    size_t off;
  };
  std::vector<Part> parts = {
      {ch.data(), sizeof(ChanDev) * ch.size(), 0},
      {p->packets.data(), sizeof(PacketDev) * p->packets.size(), 0},
      {p->pchans.data(), sizeof(int32_t) * p->pchans.size(), 0},
      {p->fent.data(), sizeof(uint2) * p->fent.size(), 0},
      {p->ient.data(), sizeof(uint2) * p->ient.size(), 0},
      {p->dpos.data(), sizeof(uint32_t) * p->dpos.size(), 0},
      {h0.data(), sizeof(float) * h0.size(), 0},
      {h0d.data(), sizeof(float) * h0d.size(), 0},
      {tw.data(), sizeof(float) * tw.size(), 0},
      {twM.data(), sizeof(float) * twM.size(), 0},
      {p->lgw.data(), sizeof(float) * p->lgw.size(), 0},
      {p->lgdw.data(), sizeof(float) * p->lgdw.size(), 0},
      {p->lrow.data(), sizeof(uint32_t) * p->lrow.size(), 0},
      {p->lent.data(), sizeof(uint32_t) * p->lent.size(), 0},
      {p->cxf.data(), sizeof(uint2) * p->cxf.size(), 0},
      {p->cxs.data(), sizeof(uint2) * p->cxs.size(), 0},
      {p->fchf.data(), sizeof(FChan) * p->fchf.size(), 0},
      {p->fchi.data(), sizeof(FChan) * p->fchi.size(), 0},
      {p->ftf.data(), sizeof(FTask) * p->ftf.size(), 0},
      {p->fti.data(), sizeof(FTask) * p->fti.size(), 0},
      {p->ovb.data(), sizeof(int2) * p->ovb.size(), 0},
      {p->ovl.data(), sizeof(int32_t) * p->ovl.size(), 0},
      {p->rband.data(), sizeof(RBand) * p->rband.size(), 0},
      {p->rtask.data(), sizeof(RTask) * p->rtask.size(), 0},
      {p->rfch.data(), sizeof(FChan) * p->rfch.size(), 0},
      {p->rbtw.data(), sizeof(float) * p->rbtw.size(), 0},
      {p->rround.data(), sizeof(int32_t) * p->rround.size(), 0},
      {p->f2pk.data(), sizeof(P2Dev) * p->f2pk.size(), 0},
      {p->f2ch.data(), sizeof(FChan) * p->f2ch.size(), 0},
      {p->gtw.data(), sizeof(float) * p->gtw.size(), 0},
      {p->gperm.data(), sizeof(int32_t) * p->gperm.size(), 0},
      {p->pbig.data(), sizeof(int32_t) * p->pbig.size(), 0},
      {p->bent.data(), sizeof(uint2) * p->bent.size(), 0},
      {p->ovbins.data(), sizeof(uint2) * p->ovbins.size(), 0},
      {p->dord.data(), sizeof(uint32_t) * p->dord.size(), 0},
      {p->ovterm.data(), sizeof(uint32_t) * p->ovterm.size(), 0},
  };
  size_t o = 0;
  for (Part &pt : parts) {
    pt.off = o;
    o = align_up(o + pt.bytes + 16);
  }
  void *blk = nullptr;
  e = cudaMalloc(&blk, o);
  if (e != cudaSuccess)
    return set_error(SLICQ_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  p->d.block = blk;
  p->d.bytes = o;
  std::vector<char> host(o, 0);
  for (const Part &pt : parts)
    if (pt.bytes) std::memcpy(host.data() + pt.off, pt.src, pt.bytes);
  char *b = static_cast<char *>(blk);
  p->d.chan = reinterpret_cast<ChanDev *>(b + parts[0].off);
  p->d.packets = reinterpret_cast<PacketDev *>(b + parts[1].off);
  p->d.pchans = reinterpret_cast<int32_t *>(b + parts[2].off);
  p->d.fent = reinterpret_cast<uint2 *>(b + parts[3].off);
  p->d.ient = reinterpret_cast<uint2 *>(b + parts[4].off);
  p->d.dpos = reinterpret_cast<uint32_t *>(b + parts[5].off);
  p->d.h0 = reinterpret_cast<float *>(b + parts[6].off);
  p->d.h0dual = reinterpret_cast<float *>(b + parts[7].off);
  p->d.tw2n = reinterpret_cast<float *>(b + parts[8].off);
  p->d.twM = reinterpret_cast<float *>(b + parts[9].off);
  p->d.gw = reinterpret_cast<float *>(b + parts[10].off);
  p->d.gdw = reinterpret_cast<float *>(b + parts[11].off);
  p->d.lrow = reinterpret_cast<uint32_t *>(b + parts[12].off);
  p->d.lent = reinterpret_cast<uint32_t *>(b + parts[13].off);
  p->d.cxf = reinterpret_cast<uint2 *>(b + parts[14].off);
  p->d.cxs = reinterpret_cast<uint2 *>(b + parts[15].off);
  p->d.fchf = reinterpret_cast<FChan *>(b + parts[16].off);
  p->d.fchi = reinterpret_cast<FChan *>(b + parts[17].off);
  p->d.ftf = reinterpret_cast<FTask *>(b + parts[18].off);
  p->d.fti = reinterpret_cast<FTask *>(b + parts[19].off);
  p->d.ovb = reinterpret_cast<int2 *>(b + parts[20].off);
  p->d.ovl = reinterpret_cast<int32_t *>(b + parts[21].off);
  p->d.rband = reinterpret_cast<RBand *>(b + parts[22].off);
  p->d.rtask = reinterpret_cast<RTask *>(b + parts[23].off);
  p->d.rfch = reinterpret_cast<FChan *>(b + parts[24].off);
  p->d.rbtw = reinterpret_cast<float2 *>(b + parts[25].off);
  p->d.rround = reinterpret_cast<int32_t *>(b + parts[26].off);
  p->d.f2pk = reinterpret_cast<P2Dev *>(b + parts[27].off);
  p->d.f2ch = reinterpret_cast<FChan *>(b + parts[28].off);
  p->kc.gargs.twN = reinterpret_cast<const float2 *>(b + parts[29].off);
  p->kc.gargs.perm = reinterpret_cast<const int *>(b + parts[30].off);
  p->d.pbig = reinterpret_cast<int32_t *>(b + parts[31].off);
  p->d.bent = reinterpret_cast<uint2 *>(b + parts[32].off);
  p->d.ovbins = reinterpret_cast<uint2 *>(b + parts[33].off);
  p->d.dord = reinterpret_cast<uint32_t *>(b + parts[34].off);
  p->d.ovterm = reinterpret_cast<uint32_t *>(b + parts[35].off);
  e = cudaMemcpy(blk, host.data(), o, cudaMemcpyHostToDevice);
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  // (the dynamic shared-memory limit: the device cap, allow_max_dyn_smem)
  int rc = 0;
  if (rc == 0 && p->kc.nbig) rc = slice_big_attrs();
  if (p->kc.generic) rc = rc ? rc : generic_set_attrs();
  else switch (p->kc.logN) {
    case 11: rc = set_attrs<11>(kSmemCap); break;
    case 12: rc = set_attrs<12>(kSmemCap); break;
    case 13: rc = set_attrs<13>(kSmemCap); break;
    case 14: rc = set_attrs<14>(kSmemCap); break;
    case 15: rc = large_set_attrs<15>(); break;
    case 16: rc = large_set_attrs<16>(); break;
    default: rc = long_set_attrs(p->kc.logN, p->kc.lcls); break;
  }
  // 2N = 131072: the four-step slice FFT on a 16-CTA cluster (DSMEM transpose) when the
  // device can co-schedule it; SLICQ_LCLUSTER bit 0 forward, bit 1 inverse (0: the split
  // column / row kernels through the staging buffer)
  p->kc.lcluster = 0;
  if (rc == 0 && !p->kc.generic && p->kc.logN == 16 && large_cluster_ok<16>())
    p->kc.lcluster = (int)(env_int("SLICQ_LCLUSTER", 3) & 3);
  if (rc == 0 && p->kc.ftables) rc = fused_set_attrs(p);
  if (rc == 0 && p->kc.fwd2) {
    rc = (int)allow_max_dyn_smem((const void *)slicq_fwd_chan2_kernel<kLiteMax, kLiteMinB>);
    if (rc == 0) rc = (int)allow_max_dyn_smem((const void *)slicq_fwd_chan2_kernel<kFullMax, kFullMinB>);
  }
  for (int v = 0; v < 2 * kVariants * 3 && rc == 0 && !p->kc.longmode; ++v)  // fwd, variant, mask
    rc = (int)allow_max_dyn_smem((const void *)chan_fn(v & 1, (v >> 1) % kVariants, v / (2 * kVariants)));
  for (int v = 0; v < 4 && rc == 0 && !p->kc.longmode; ++v)  // fwd, lite / full
    rc = (int)allow_max_dyn_smem((const void *)tb_fn(v & 1, 1 + (v >> 1)));
  if (rc != 0)
    return set_error(SLICQ_ECUDA, std::string("cudaFuncSetAttribute: ") +
                                      cudaGetErrorString((cudaError_t)rc));
  if (p->kc.pipe) {
    for (cudaStream_t &st : p->d.pipe)
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return set_error(SLICQ_ECUDA, "cudaStreamCreate");
    for (cudaEvent_t &ev : p->d.pev)
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
        return set_error(SLICQ_ECUDA, "cudaEventCreate");
  }
  p->has_device = true;
  return SLICQ_OK;
}

void free_device(slicq_plan *p) {
  if (p) {
    for (cudaStream_t &st : p->d.pipe)
      if (st) cudaStreamDestroy(st), st = nullptr;
    for (cudaEvent_t &ev : p->d.pev)
      if (ev) cudaEventDestroy(ev), ev = nullptr;
  }
  if (p && p->d.block) {
    cudaFree(p->d.block);
    p->d.block = nullptr;
  }
  if (p) p->has_device = false;
}

namespace {
// workspace layout: [pairing counters][boundary halves][staging for one chunk of units]
struct WsLayout {
  size_t cnt, bnd, stage, total;
  int64_t chunk;
  bool pipe;  // chunks alternate between the plan's two streams (two staging buffers)
};
WsLayout ws_layout(const slicq_plan *p, int64_t nslices, int64_t batch) {
  WsLayout w{};
  const int64_t units = nslices * batch;
  w.chunk = std::min<int64_t>(units, p->kc.chunk_units);
  w.pipe = p->kc.pipe && !p->kc.longmode && units >= p->kc.pipe_min;
  if (w.pipe) {  // pipe_parts chunks (rounded up to the channel-kernel tile)
    const int64_t t = p->kc.tile;
    w.chunk = std::min(w.chunk, ((units + p->kc.pipe_parts - 1) / p->kc.pipe_parts + t - 1) / t * t);
    w.pipe = units > w.chunk;
  }
  w.cnt = 0;
  w.bnd = align_up(sizeof(unsigned) * (size_t)units);
  w.stage = align_up(w.bnd + sizeof(float) * (size_t)(units * 2 * p->tr));
  w.total = w.stage + (w.pipe ? 2 : 1) * sizeof(float2) *
                         (size_t)(w.chunk * std::max(p->kc.xs, p->kc.zs));
  return w;
}

// chunk pipelining: chunks alternate between the plan's two streams (forked from and joined
// back into the caller's stream) with ping-pong staging, so that one chunk's kernel tails
// overlap the next chunk's first kernels (measured +1.5 % on cfg4; the results are
// bit-identical: same kernels, deterministic boundary pairing)
struct Pipe {
  const slicq_plan *p;
  cudaStream_t s;
  bool on, joined = false;
  cudaError_t err = cudaSuccess;    // first failure of the fork / join
  std::unique_lock<std::mutex> lk;  // held from the fork to the join (shared streams / events)
  Pipe(const slicq_plan *p_, cudaStream_t s_, const WsLayout &w)
      : p(p_), s(s_), on(w.pipe) {
    if (!on) return;
    lk = std::unique_lock<std::mutex>(p->pipe_mu);
    note(cudaEventRecord(p->d.pev[0], s));
    note(cudaStreamWaitEvent(p->d.pipe[0], p->d.pev[0], 0));
    note(cudaStreamWaitEvent(p->d.pipe[1], p->d.pev[0], 0));
  }
  // every exit path (including a launch failure part-way) joins the plan streams back into
  // the caller's stream, so the caller never reuses buffers that queued chunks still use
  ~Pipe() { join(); }
  void note(cudaError_t e) {
    if (err == cudaSuccess && e != cudaSuccess) err = e;
  }
  cudaStream_t stream(int64_t i) const { return on ? p->d.pipe[i & 1] : s; }
  float2 *stage(float2 *base, int64_t i, int64_t chunk, int64_t row) const {
    return on ? base + (i & 1) * chunk * row : base;
  }
  cudaError_t join() {
    if (!on || joined) return err;
    joined = true;
    note(cudaEventRecord(p->d.pev[1], p->d.pipe[0]));
    note(cudaEventRecord(p->d.pev[2], p->d.pipe[1]));
    note(cudaStreamWaitEvent(s, p->d.pev[1], 0));
    note(cudaStreamWaitEvent(s, p->d.pev[2], 0));
    return err;
  }
};
}  // namespace

int kernel_launches(const slicq_plan *p, int direction, int64_t nslices, int64_t batch) {
  const WsLayout w = ws_layout(p, nslices, batch);
  const int64_t chunks = (nslices * batch + w.chunk - 1) / w.chunk;
  if (p->kc.longmode) return (int)(chunks * (direction == 0 ? 3 : 4));
  if ((p->kc.fused || p->kc.cluster || p->kc.ring) && direction == 0)
    return (int)((nslices * batch + 0x7fffffef) / 0x7ffffff0);
  if (p->kc.band && direction == 0 && !p->kc.large) return (int)(chunks * 2);
  int nchan = 0;
  for (int v = 0; v < 3; ++v) nchan += p->kc.voff[v + 1] > p->kc.voff[v];
  for (int c = 0; c + 1 < kLongClasses; ++c) nchan += p->kc.bcls.off[c + 1] > p->kc.bcls.off[c];
  const int nspec = !p->kc.large ? 1
                    : direction == 0 ? ((p->kc.lcluster & 1) ? 1 : 2)
                                     : ((p->kc.lcluster & 2) ? 2 : 4);
  return (int)(chunks * (nchan + nspec));
}

// ring kernels: [ring slots][ready, done flags, error word][dev stats: 1024 CTAs x 4 u64]
constexpr size_t kRingStatsBytes = 1024 * 4 * sizeof(unsigned long long);
static size_t ring_ws_bytes(const slicq_plan *p) {
  if (!p->kc.ring) return 0;
  return align_up(sizeof(float2) * (size_t)p->kc.rR * p->kc.rslot) +
         align_up(sizeof(unsigned) * (size_t)(2 * p->kc.rR + 4)) + kRingStatsBytes;
}

size_t workspace_bytes(const slicq_plan *p, int64_t nslices, int64_t batch) {
  if (!p->has_device) return 0;  // the layout depends on the device configuration
  return std::max(ws_layout(p, nslices, batch).total, ring_ws_bytes(p));
}

static KArgs base_args(const slicq_plan *p) {
  KArgs a{};
  a.tr = (int)p->tr;
  a.C = p->C;
  a.chan = p->d.chan;
  a.packets = p->d.packets;
  a.pchans = p->d.pchans;
  a.npackets = p->kc.npackets;
  a.scr = p->kc.scr;
  a.fent = p->d.fent;
  a.ient = p->d.ient;
  a.dpos = p->d.dpos;
  a.ovbins = p->d.ovbins;
  a.dord = p->d.dord;
  a.novbins = (int)p->ovbins.size();
  a.ovterm = p->d.ovterm;
  a.novterm = (int)p->ovterm.size();
  a.zso = p->kc.zso;
  a.h0 = p->d.h0;
  a.h0dual = p->d.h0dual;
  a.tw2n = reinterpret_cast<const float2 *>(p->d.tw2n);
  a.twM = reinterpret_cast<const float2 *>(p->d.twM);
  a.xs = p->kc.xs;
  a.zs = p->kc.zs;
  a.tile = p->kc.tile;
  a.stiles = p->kc.stiles;
  a.pf = p->kc.pf;
  a.Nh = (int)p->N;
  a.bent = p->d.bent;
  a.gw = p->d.gw;
  a.gdw = p->d.gdw;
  a.lrow = p->d.lrow;
  a.lent = p->d.lent;
  return a;
}

static int check_device(const slicq_plan *p) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != p->device)
    return set_error(SLICQ_EINVAL, "current CUDA device differs from the plan's device");
  return SLICQ_OK;
}

// resident CTAs (occupancy x SMs) of a persistent kernel with `smem` dynamic shared memory
static int64_t chan_capacity_smem(ChanFn fn, size_t smem) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, CHAN_T, smem) != cudaSuccess || occ <= 0)
    occ = 2;
  return (int64_t)occ * nsm;
}

// persistent channel-kernel grid: resident CTAs (occupancy x SMs), capped by the work items
static int64_t chan_capacity(const slicq_plan *p, ChanFn fn, size_t smem) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int per_sm = 2;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, CHAN_T, smem) ==
          cudaSuccess && occ > 0)
    per_sm = occ;
  if (p->kc.chan_per_sm > 0) per_sm = std::min(per_sm, p->kc.chan_per_sm);
  return (int64_t)per_sm * nsm;
}

// the channel kernels of one direction: one launch per non-empty variant (micro, lite, full)
static cudaError_t launch_chan(bool fwd, const slicq_plan *p, KArgs a, cudaStream_t s) {
  for (int v = 0; v < kVariants; ++v) {
    a.packets = p->d.packets + p->kc.voff[v];
    a.npackets = p->kc.voff[v + 1] - p->kc.voff[v];
    if (a.npackets == 0) continue;
    // TMA-staged variant (kernels_tb.cuh): unmasked calls whose operand rows are 16-byte
    // aligned (bulk copies)
    const bool tb = p->kc.tb && (fwd ? (reinterpret_cast<uintptr_t>(a.stage) % 16 == 0 && a.xs % 2 == 0)
                                     : (!a.mask && reinterpret_cast<uintptr_t>(a.coef_in) % 16 == 0 &&
                                        a.C % 2 == 0));
    const ChanFn fn = tb ? tb_fn(fwd, v) : chan_fn(fwd, v, fwd || !a.mask ? 0 : (a.mask_db ? 2 : 1));
    const size_t smem = tb ? (fwd ? p->kc.tb_smem_f : p->kc.tb_smem_i) : p->kc.chan_smem;
    a.scr = tb && fwd ? p->kc.scr_f : p->kc.scr;
    a.tbe = fwd ? p->kc.tbe_f : p->kc.tbe_i;
    // small calls (e.g. the ranges of the streaming executor): shrink the tile until there
    // are >= 4 work items per resident CTA (load balance of the persistent grid)
    const int64_t cap = chan_capacity(p, fn, smem);
    a.tile = p->kc.tile;
    while (a.tile > 8 && (int64_t)a.npackets * ((a.nunits + a.tile - 1) / a.tile) < 4 * cap)
      a.tile /= 2;
    const int64_t items = (int64_t)a.npackets * ((a.nunits + a.tile - 1) / a.tile);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(items, cap)));
    cfg.blockDim = dim3(CHAN_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = p->kc.pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// the forward channel kernel v2 (kernels_chan2.cuh): one launch per non-empty variant
static cudaError_t launch_chan2(const slicq_plan *p, KArgs a, cudaStream_t s) {
  for (int v = 0; v < 2; ++v) {
    C2Args c2{};
    c2.pk = p->d.f2pk + p->kc.f2voff[v];
    c2.npk = p->kc.f2voff[v + 1] - p->kc.f2voff[v];
    c2.fch = p->d.f2ch;
    if (c2.npk == 0) continue;
    const ChanFn fn0 = reinterpret_cast<ChanFn>(v == 0 ? slicq_fwd_chan2_kernel<kLiteMax, kLiteMinB>
                                                       : slicq_fwd_chan2_kernel<kFullMax, kFullMinB>);
    a.scr = p->kc.f2scr;
    const size_t smem = sizeof(float2) * (size_t)p->kc.f2scr * (CHAN_T / 32);
    const int64_t cap = chan_capacity_smem(fn0, smem);
    a.tile = p->kc.tile;
    while (a.tile > 8 && (int64_t)c2.npk * ((a.nunits + a.tile - 1) / a.tile) < 4 * cap) a.tile /= 2;
    const int64_t items = (int64_t)c2.npk * ((a.nunits + a.tile - 1) / a.tile);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(items, cap)));
    cfg.blockDim = dim3(CHAN_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = p->kc.pdl ? 1 : 0;
    const cudaError_t e =
        v == 0 ? cudaLaunchKernelEx(&cfg, slicq_fwd_chan2_kernel<kLiteMax, kLiteMinB>, a, c2)
               : cudaLaunchKernelEx(&cfg, slicq_fwd_chan2_kernel<kFullMax, kFullMinB>, a, c2);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static cudaError_t launch_spec(bool fwd, const slicq_plan *p, const KArgs &a, dim3 grid,
                               cudaStream_t s, int mode) {
  const size_t sm = p->kc.spec_smem;
  switch (p->kc.logN) {
#define CASE_(L)                                                                           \
  case L:                                                                                  \
    return fwd ? launch_fwd_spec<L>(a, grid, sm, s, p->kc.pdl, mode)                       \
               : launch_inv_spec<L>(a, grid, sm, s, p->kc.pdl, mode);
    CASE_(11)
    CASE_(12)
    CASE_(13)
    CASE_(14)
#undef CASE_
  }
  return cudaErrorInvalidValue;
}

static cudaError_t launch_fused(bool fwd, const slicq_plan *p, const KArgs &a, dim3 grid,
                                cudaStream_t s) {
  switch (p->kc.logN) {
#define CASE_(L)                                                                           \
  case L:                                                                                  \
    return !fwd ? cudaErrorInvalidValue                                                   \
           : p->kc.cluster ? launch_fwd_cluster<L>(a, p->kc.cluster, p->kc.fsmem_f, s, p->kc.pdl) \
                           : launch_fwd_fused<L>(a, grid, p->kc.fsmem_f, s, p->kc.pdl);
    CASE_(11)
    CASE_(12)
    CASE_(13)
    CASE_(14)
#undef CASE_
  }
  return cudaErrorInvalidValue;
}

static cudaError_t launch_fwd_persist(const slicq_plan *p, const KArgs &a, cudaStream_t s) {
  const size_t sm = p->kc.spec_smem;
  switch (p->kc.logN) {
#define CASE_(L) \
  case L: return launch_fwd_spec_persist<L>(a, sm, s, p->kc.pdl);
    CASE_(11)
    CASE_(12)
    CASE_(13)
    CASE_(14)
#undef CASE_
  }
  return cudaErrorInvalidValue;
}

// the band / ring tables of RArgs (the ring buffers and flags are set by the ring launch)
static RArgs band_args(const slicq_plan *p) {
  RArgs r{};
  r.nb = p->kc.rnb;
  r.bt = p->kc.rbt;
  r.la = p->kc.rla;
  r.grp = p->kc.rgroup;
  r.meta = p->kc.rmeta;
  r.band = p->d.rband;
  r.task = p->d.rtask;
  r.fch = p->d.rfch;
  r.btw = p->d.rbtw;
  r.round = p->d.rround;
  r.xstride = p->kc.rxstride;
  r.wmax = p->kc.rwmax;
  r.twmax = p->kc.rtwmax;
  r.iscr = p->kc.rfscr;
  return r;
}

int launch_forward(const slicq_plan *p, const float *x, int64_t x_len, int64_t x_stride,
                   int64_t base_off, int64_t L, int wrap, int64_t slice0, int64_t nslices,
                   int64_t batch, slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream,
                   int mode) {
  int rc = check_device(p);
  if (rc) return rc;
  if (nslices > 0x7fffffff) return set_error(SLICQ_ESHAPE, "too many slices");
  const WsLayout w = ws_layout(p, nslices, batch);
  if (!ws || ws_bytes < std::max(w.total, ring_ws_bytes(p)))
    return set_error(SLICQ_ESHAPE, "workspace too small");
  if ((uintptr_t)ws % 16) return set_error(SLICQ_ESHAPE, "workspace must be 16-byte aligned");
  KArgs a = base_args(p);
  a.x = x;
  a.x_len = x_len;
  a.x_stride = x_stride;
  a.base_off = base_off;
  a.L = L;
  a.wrap = wrap;
  a.slice0 = slice0;
  a.nslices = (int)nslices;
  a.coef_out = reinterpret_cast<float2 *>(coeffs);
  a.stage = reinterpret_cast<float2 *>(static_cast<char *>(ws) + w.stage);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t units = nslices * batch;
  a.toff = p->kc.toff_f;
  if (p->kc.longmode) {  // full-length CQ-NSGT only (kernels_long.cuh)
    if (mode != 1 || nslices != 1)
      return set_error(SLICQ_EUNSUPPORTED, "sl_len > 2^17: only the full-length CQ-NSGT "
                                           "(slicq_nsgt_forward / slicq_nsgt_inverse)");
    for (int64_t u0 = 0; u0 < units; u0 += w.chunk) {
      a.unit0 = u0;
      a.nunits = (int)std::min<int64_t>(w.chunk, units - u0);
      const cudaError_t e = long_forward(p->kc.logN, a, p->kc.lcls, s);
      if (e != cudaSuccess)
        return set_error(SLICQ_ECUDA, std::string("forward launch: ") + cudaGetErrorString(e));
    }
    return SLICQ_OK;
  }
  if (p->kc.ring && mode == 0 && units <= 0x7fffffff) {  // ring kernel (kernels_ring.cuh)
    a.vec16 = (reinterpret_cast<uintptr_t>(coeffs) % 16 == 0) ? 1 : 0;
    a.unit0 = 0;
    a.nunits = (int)units;
    RArgs r = band_args(p);
    char *wb = static_cast<char *>(ws);
    r.ring = reinterpret_cast<float2 *>(wb);
    r.slot_entries = p->kc.rslot;
    unsigned *flags = reinterpret_cast<unsigned *>(wb + align_up(sizeof(float2) * (size_t)p->kc.rR * p->kc.rslot));
    r.ready = flags;
    r.done = flags + p->kc.rR;
    r.err = flags + 2 * p->kc.rR;
    r.R = p->kc.rR;
    r.qctr = reinterpret_cast<unsigned long long *>(flags + 2 * p->kc.rR + 2);
    r.ngrid = p->kc.rnspec;
    const size_t fl_bytes = align_up(sizeof(unsigned) * (size_t)(2 * p->kc.rR + 4));
    r.qctr = reinterpret_cast<unsigned long long *>(flags + 2 * p->kc.rR + 2);
    r.la = p->kc.rla;
    r.ngrid = p->kc.rnspec;
    r.stats = std::getenv("SLICQ_RING_STATS")
                  ? reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(flags) + fl_bytes)
                  : nullptr;
    cudaError_t e = cudaMemsetAsync(flags, 0, fl_bytes + (r.stats ? kRingStatsBytes : 0), s);
    if (e == cudaSuccess) {
      switch (p->kc.logN) {
        case 12: e = launch_fwd_ring<12>(a, r, p->kc.rsmem, s); break;
        case 13: e = launch_fwd_ring<13>(a, r, p->kc.rsmem, s); break;
        default: e = cudaErrorInvalidValue;
      }
    }
    if (e != cudaSuccess)
      return set_error(SLICQ_ECUDA, std::string("forward ring launch: ") + cudaGetErrorString(e));
    return SLICQ_OK;
  }
  if ((p->kc.fused || p->kc.cluster) && mode == 0) {  // one fused kernel: no staging (kernels_fused.cuh)
    a.fch = p->d.fchf;
    a.ftask = p->d.ftf;
    a.nftask = p->kc.nftf;
    a.fscr = p->kc.fscr;
    a.vec16 = (reinterpret_cast<uintptr_t>(coeffs) % 16 == 0) ? 1 : 0;
    for (int64_t u0 = 0; u0 < units; u0 += 0x7ffffff0) {  // (grid rounded up to the cluster)
      a.unit0 = u0;
      a.nunits = (int)std::min<int64_t>(0x7ffffff0, units - u0);
      const cudaError_t e = launch_fused(true, p, a, dim3((unsigned)a.nunits), s);
      if (e != cudaSuccess)
        return set_error(SLICQ_ECUDA, std::string("forward launch: ") + cudaGetErrorString(e));
    }
    return SLICQ_OK;
  }
  Pipe pp(p, s, w);
  if (pp.err != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("stream fork: ") + cudaGetErrorString(pp.err));
  float2 *stage0 = a.stage;
  for (int64_t u0 = 0, i = 0; u0 < units; u0 += w.chunk, ++i) {
    a.unit0 = u0;
    a.nunits = (int)std::min<int64_t>(w.chunk, units - u0);
    a.stage = pp.stage(stage0, i, w.chunk, std::max(p->kc.xs, p->kc.zs));
    const cudaStream_t st = pp.stream(i);
    cudaError_t e = p->kc.generic ? launch_generic(true, a, p->kc.gargs, a.nunits, st, p->kc.pdl, mode)
                    : !p->kc.large && mode == 0 && p->kc.fwd_persist
                        ? launch_fwd_persist(p, a, st)
                    : !p->kc.large ? launch_spec(true, p, a, dim3((unsigned)a.nunits), st, mode)
                    : p->kc.logN == 15 ? large_forward<15>(a, st, mode)
                                       : large_forward<16>(a, st, mode, p->kc.lcluster & 1);
    if (e == cudaSuccess && p->kc.band && !p->kc.large) {
      // band-major channel kernel (kernels_ring.cuh): claim counter per chunk in the
      // (forward-unused) pairing-counter area of the workspace
      RArgs r = band_args(p);
      r.qctr = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + w.cnt) + i;
      a.vec16 = (reinterpret_cast<uintptr_t>(coeffs) % 16 == 0) ? 1 : 0;
      e = cudaMemsetAsync(r.qctr, 0, sizeof(unsigned long long), st);
      if (e == cudaSuccess) {
        static int nsm = 0;
        if (!nsm) {
          int dev = 0;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
          if (nsm <= 0) nsm = 148;
        }
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(2 * nsm, a.nunits));
        e = p->kc.logN == 12 ? launch_fwd_band<12>(a, r, p->kc.rchsmem, grid, st, p->kc.pdl)
            : launch_fwd_band<13>(a, r, p->kc.rchsmem, grid, st, p->kc.pdl);
      }
    } else if (e == cudaSuccess && p->kc.fwd2 && !p->kc.large) {
      a.vec16 = (reinterpret_cast<uintptr_t>(coeffs) % 16 == 0) ? 1 : 0;
      e = launch_chan2(p, a, st);
    } else if (e == cudaSuccess) {
      e = launch_chan(true, p, a, st);
    }
    if (e == cudaSuccess && p->kc.nbig) e = slice_big_launch(true, a, p->d.pbig, p->kc.bcls, st);
    if (e != cudaSuccess)
      return set_error(SLICQ_ECUDA, std::string("forward launch: ") + cudaGetErrorString(e));
  }
  if (pp.join() != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("stream join: ") + cudaGetErrorString(pp.err));
  return SLICQ_OK;
}

static cudaError_t launch_inv_persist(const slicq_plan *p, const KArgs &a, cudaStream_t s) {
  const size_t sm = p->kc.spec_smem_p;
  switch (p->kc.logN) {
#define CASE_(L) \
  case L: return launch_inv_spec_persist<L>(a, sm, s, p->kc.pdl, nullptr);
    CASE_(11)
    CASE_(12)
    CASE_(13)
    CASE_(14)
#undef CASE_
  }
  return cudaErrorInvalidValue;
}

int launch_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t slice0, int64_t nslices,
                   int64_t total_slices, int64_t batch, int circular, int64_t n_valid, int64_t L,
                   float *y, int64_t y_stride, int64_t y_base, float *left_spill, int64_t halo,
                   void *ws, size_t ws_bytes, void *stream, const float *mask, int mask_db,
                   int mode) {
  (void)total_slices;
  int rc = check_device(p);
  if (rc) return rc;
  if (nslices > 0x7fffffff) return set_error(SLICQ_ESHAPE, "too many slices");
  const WsLayout w = ws_layout(p, nslices, batch);
  if (!ws || ws_bytes < w.total) return set_error(SLICQ_ESHAPE, "workspace too small");
  if ((uintptr_t)ws % 16) return set_error(SLICQ_ESHAPE, "workspace must be 16-byte aligned");
  KArgs a = base_args(p);
  a.coef_in = reinterpret_cast<const float2 *>(coeffs);
  a.vec16 = (reinterpret_cast<uintptr_t>(coeffs) % 16 == 0 && p->C % 2 == 0) ? 1 : 0;
  a.mask = mask;
  a.mask_db = mask_db;
  a.y = y;
  a.y_len = n_valid;
  a.y_stride = y_stride;
  a.y_base = y_base;
  a.spill = left_spill;
  a.halo = halo;
  a.L = L;
  a.circular = circular;
  a.slice0 = slice0;
  a.nslices = (int)nslices;
  char *wb = static_cast<char *>(ws);
  a.cnt = reinterpret_cast<unsigned *>(wb + w.cnt);
  // the boundary-pairing counters start every call at zero: the workspace layout depends on
  // the call's unit count, so a workspace reused by calls of different sizes (the streaming
  // executor's ranges) would otherwise read an earlier call's boundary halves as counters
  {
    const cudaError_t e = cudaMemsetAsync(a.cnt, 0, sizeof(unsigned) * (size_t)(nslices * batch),
                                          static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess)
      return set_error(SLICQ_ECUDA, std::string("counter reset: ") + cudaGetErrorString(e));
  }
  a.bnd = reinterpret_cast<float *>(wb + w.bnd);
  a.stage = reinterpret_cast<float2 *>(wb + w.stage);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t units = nslices * batch;
  a.toff = p->kc.toff_i;
  if (!p->painless)
    return set_error(SLICQ_EUNSUPPORTED, "synthesis needs a painless system (M_k >= L_k, P:170)");
  if (p->kc.longmode) {  // full-length CQ-NSGT only (kernels_long.cuh)
    if (mode != 1 || nslices != 1 || mask)
      return set_error(SLICQ_EUNSUPPORTED, "sl_len > 2^17: only the full-length CQ-NSGT "
                                           "(slicq_nsgt_forward / slicq_nsgt_inverse)");
    for (int64_t u0 = 0; u0 < units; u0 += w.chunk) {
      a.unit0 = u0;
      a.nunits = (int)std::min<int64_t>(w.chunk, units - u0);
      const cudaError_t e = long_inverse(p->kc.logN, a, p->kc.lcls, s);
      if (e != cudaSuccess)
        return set_error(SLICQ_ECUDA, std::string("inverse launch: ") + cudaGetErrorString(e));
    }
    return SLICQ_OK;
  }
  Pipe pp(p, s, w);
  if (pp.err != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("stream fork: ") + cudaGetErrorString(pp.err));
  float2 *stage0 = a.stage;
  for (int64_t u0 = 0, i = 0; u0 < units; u0 += w.chunk, ++i) {
    a.unit0 = u0;
    a.nunits = (int)std::min<int64_t>(w.chunk, units - u0);
    a.stage = pp.stage(stage0, i, w.chunk, std::max(p->kc.xs, p->kc.zs));
    const cudaStream_t st = pp.stream(i);
    cudaError_t e = launch_chan(false, p, a, st);
    if (e == cudaSuccess && p->kc.nbig) e = slice_big_launch(false, a, p->d.pbig, p->kc.bcls, st);
    if (e == cudaSuccess && p->kc.generic)
      e = launch_generic(false, a, p->kc.gargs, a.nunits, st, p->kc.pdl, mode);
    else if (e == cudaSuccess && !p->kc.large && mode == 0 && p->kc.inv_persist)
      e = launch_inv_persist(p, a, st);
    else if (e == cudaSuccess)
      e = !p->kc.large ? launch_spec(false, p, a, dim3((unsigned)a.nunits), st, mode)
          : p->kc.logN == 15 ? large_inverse_spec<15>(a, st, mode)
                             : large_inverse_spec<16>(a, st, mode, (p->kc.lcluster & 2) != 0);
    if (e != cudaSuccess)
      return set_error(SLICQ_ECUDA, std::string("inverse launch: ") + cudaGetErrorString(e));
  }
  if (pp.join() != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("stream join: ") + cudaGetErrorString(pp.err));
  return SLICQ_OK;
}

int launch_approx(const slicq_plan *ps, const slicq_plan *pl, const slicq_c32 *s,
                  const slicq_c32 *c, int64_t batch, double *out, void *stream, int full) {
  int rc = check_device(ps);
  if (!rc) rc = check_device(pl);
  if (rc) return rc;
  if (batch > 65535) return set_error(SLICQ_ESHAPE, "batch too large");
  const int S = (int)(pl->sl_len / ps->N);
  const int nch = full ? 2 * ps->K + 2 : ps->K + 2;
  approx_kernel<<<dim3((unsigned)nch, (unsigned)batch), 256, 0,
                  static_cast<cudaStream_t>(stream)>>>(
      ps->d.chan, pl->d.chan, reinterpret_cast<const float2 *>(s),
      reinterpret_cast<const float2 *>(c), full ? coeffs_full(ps) : ps->C,
      full ? coeffs_full(pl) : pl->C, S, (float)(1.0 / (double)ps->sl_len),
      (float)(1.0 / (double)pl->sl_len), out, full, ps->K, ps->C, pl->C);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("approx launch: ") + cudaGetErrorString(e));
  return SLICQ_OK;
}

int launch_overlap_add(float *y, int64_t y_stride, const float *spill, int64_t count,
                       int64_t batch, void *stream) {
  if (batch > 65535) return set_error(SLICQ_ESHAPE, "batch too large");
  const int T = 256;
  const unsigned blocks = (unsigned)std::min<int64_t>((count + T - 1) / T, 1024);
  overlap_add_kernel<<<dim3(blocks, (unsigned)batch), T, 0, static_cast<cudaStream_t>(stream)>>>(
      y, y_stride, spill, count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("overlap_add launch: ") + cudaGetErrorString(e));
  return SLICQ_OK;
}

}  // namespace slicq

// Debug only (not part of include/slicq.h): the ring kernels' configuration and the byte
// offset of their dev statistics in the workspace (tools/ring_stats.py).
extern "C" __attribute__((visibility("default"))) int slicq_debug_ring_info(const slicq_plan *p,
                                                                           long long *out) {
  if (!p || !p->kc.ring) return -1;
  out[0] = p->kc.rR;
  out[1] = p->kc.rslot;
  out[2] = p->kc.rnb;
  out[3] = p->kc.rq;
  out[4] = p->kc.rbt;
  out[5] = p->kc.rnspec;
  out[6] = (long long)(slicq::align_up(sizeof(float2) * (size_t)p->kc.rR * p->kc.rslot) +
                       slicq::align_up(sizeof(unsigned) * (size_t)(2 * p->kc.rR + 4)));
  out[7] = (long long)p->kc.rsmem;
  return 0;
}

// Debug only (not part of include/slicq.h): accumulated per-phase clock64 cycles of the
// forward [0..15] and inverse [16..31] spectrum kernels, in a library built with
// -DSLICQ_PHASE_TIMING (tools/phase_timing.py).  Returns -1 in the product build.
extern "C" __attribute__((visibility("default"))) int slicq_debug_phase_times(
    int logN, unsigned long long *out32, int reset) {
  switch (logN) {
    case 11: return slicq::kern::phase_times<11>(out32, reset);
    case 12: return slicq::kern::phase_times<12>(out32, reset);
    case 13: return slicq::kern::phase_times<13>(out32, reset);
    case 14: return slicq::kern::phase_times<14>(out32, reset);
  }
  return -1;
}
