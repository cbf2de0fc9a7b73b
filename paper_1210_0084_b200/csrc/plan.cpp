// Host side of the sliCQ library: the float64 plan (Table 1 layout, sampled filters,
// coefficient counts, painless dual, slicing windows) and the C ABI entry points.
//
// Written from the paper (arXiv 1210.0084), cited as P:<line>, under the readings
// C<n> listed in DESIGN.md.  Independent of the Python oracle (no shared code).
#include <cmath>
#include <cstring>
#include <limits>
#include <new>
#include <string>

#include "slicq_internal.h"

namespace {
thread_local std::string g_last_error;
constexpr double kEdgeEps = 1e-9;  // C7/C18 support-edge guard
constexpr double kKEps = 1e-12;    // C4/C18 guard on B log2(.)
constexpr double kPi = 3.14159265358979323846;

bool smooth235(int64_t m) {
  if (m < 1) return false;
  for (int q : {2, 3, 5})
    while (m % q == 0) m /= q;
  return m == 1;
}

// C9: smallest even 2/3/5-smooth integer >= L.
int64_t even_smooth_ge(int64_t L) {
  int64_t m = L < 2 ? 2 : L;
  while (!(m % 2 == 0 && smooth235(m))) ++m;
  return m;
}

// H(x) = cos^2(pi x) on |x| <= 1/2 (reading C7 of P:262's H).
double hann(double x) {
  if (std::fabs(x) > 0.5) return 0.0;
  double c = std::cos(kPi * x);
  return c * c;
}
// 4-term Blackman-Harris centred on [-1/2, 1/2] (reading C20)
double blackman_harris(double x) {
  if (std::fabs(x) > 0.5) return 0.0;
  return 0.35875 + 0.48829 * std::cos(2.0 * kPi * x) + 0.14128 * std::cos(4.0 * kPi * x) +
         0.01168 * std::cos(6.0 * kPi * x);
}

struct Filt {
  int64_t lo;
  std::vector<double> v;
  double at(int64_t j) const {  // 0 off the support
    int64_t i = j - lo;
    return (i >= 0 && i < (int64_t)v.size()) ? v[i] : 0.0;
  }
};
}  // namespace

namespace slicq {
int set_error(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
}  // namespace slicq

using slicq::set_error;

// Filters of the stored channels 0..K+1 on a length-Ls DFT grid (reading C7):
// fractional centre omega = xi Ls/fs, width W = max(Omega Ls/fs, min_width) bins,
// J = [ceil(omega - W/2 - eps), floor(omega + W/2 + eps)], g[j] = H((j - omega)/W), then the
// plateaus (C8).  grid = 2N' > 0 (Prop. 4, reading C21): omega = s (xi 2N'/fs),
// W = s max(Omega 2N'/fs, min_width), s = Ls/2N' -- sampled every s bins this is the 2N'
// system's filter.
static int cq_filters(const slicq_plan *p, int64_t Ls, int64_t grid, std::vector<Filt> &f) {
  const double fs = p->fs;
  const int64_t K = p->K;
  double (*H)(double) = p->window == SLICQ_WINDOW_BLACKMAN_HARRIS ? blackman_harris : hann;
  f.assign(K + 2, Filt{});
  std::vector<double> omega(K + 2, 0.0);
  for (int64_t k = 1; k <= K; ++k) {
    const double xi = p->xi[k - 1], Om = xi / p->Q;
    double om, W;
    if (grid) {
      const double sc = (double)(Ls / grid);
      om = sc * (xi * grid / fs);
      W = sc * std::max(Om * grid / fs, p->min_width);
    } else {
      om = xi * Ls / fs;
      W = std::max(Om * Ls / fs, p->min_width);
    }
    const int64_t lo = (int64_t)std::ceil(om - W / 2 - kEdgeEps);
    const int64_t hi = (int64_t)std::floor(om + W / 2 + kEdgeEps);
    if (hi < lo) return set_error(SLICQ_ENOTFRAME, "empty filter support");
    f[k].lo = lo;
    f[k].v.resize(hi - lo + 1);
    for (int64_t j = lo; j <= hi; ++j) f[k].v[j - lo] = H(((double)j - om) / W);
    omega[k] = om;
  }
  // plateaus (Table 1 rows 0 and K+1; reading C8)
  const int64_t a = (int64_t)std::floor(omega[1]);
  f[0].lo = -a;
  f[0].v.resize(2 * a + 1);
  for (int64_t j = -a; j <= a; ++j) f[0].v[j + a] = 1.0 - f[1].at(j < 0 ? -j : j);
  const int64_t b0 = (int64_t)std::ceil(omega[K]);
  const int64_t b1 = (int64_t)std::floor((double)Ls - omega[K]);
  if (b1 < b0) return set_error(SLICQ_ENOTFRAME, "empty filter support");
  f[K + 1].lo = b0;
  f[K + 1].v.resize(b1 - b0 + 1);
  for (int64_t j = b0; j <= b1; ++j) {
    double v = 1.0 - f[K].at(j) - f[K].at(Ls - j);
    f[K + 1].v[j - b0] = v > 0.0 ? v : 0.0;
  }
  return SLICQ_OK;
}

// M_k = L/a_k >= L_k (readings C9, C10)
static int channel_counts(const slicq_plan *p, const std::vector<Filt> &f, std::vector<int64_t> &M) {
  const int64_t K = p->K, B = p->B;
  M.assign(K + 2, 0);
  auto len = [&](int64_t k) { return (int64_t)f[k].v.size(); };
  if (p->raster == SLICQ_RASTER_NONE) {
    for (int64_t k = 0; k < K + 2; ++k) M[k] = even_smooth_ge(len(k));
  } else if (p->raster == SLICQ_RASTER_FULL) {
    int64_t mx = 0;
    for (int64_t k = 0; k < K + 2; ++k) mx = std::max(mx, len(k));
    for (int64_t k = 0; k < K + 2; ++k) M[k] = even_smooth_ge(mx);
  } else {  // per octave: groups {0}, {K+1}, CQ octaves floor((k-1)/B)
    M[0] = even_smooth_ge(len(0));
    M[K + 1] = even_smooth_ge(len(K + 1));
    for (int64_t k0 = 1; k0 <= K; k0 += B) {
      const int64_t k1 = std::min(k0 + B - 1, K);
      int64_t mx = 0;
      for (int64_t k = k0; k <= k1; ++k) mx = std::max(mx, len(k));
      for (int64_t k = k0; k <= k1; ++k) M[k] = even_smooth_ge(mx);
    }
  }
  return SLICQ_OK;
}

static int build_host_plan(slicq_plan *p) {
  const double fs = p->fs, fmin = p->fmin, fmax = p->fmax;
  const int B = p->B;
  const int64_t Ls = p->sl_len, N = p->N, tr = p->tr;
  // ---- Table 1; K per reading C4: the paper's xi_max <= xi_K < fs/2 is
  // impossible for fmax >= fs/2, so K = min(first k covering fmax, last k below Nyquist).
  const double y = B * std::log2(fmax / fmin);
  const int64_t k_cover = (int64_t)std::ceil(y - kKEps) + 1;
  const double x = B * std::log2((fs / 2.0) / fmin);
  const int64_t k_nyq = (int64_t)std::ceil(x - kKEps);
  const int64_t K = k_cover < k_nyq ? k_cover : k_nyq;
  if (K < 1) return set_error(SLICQ_EINVAL, "K < 1: no constant-Q channel below Nyquist");
  if (K > 100000) return set_error(SLICQ_EINVAL, "too many channels");
  p->K = (int)K;
  p->Q = 1.0 / (std::pow(2.0, 1.0 / B) - std::pow(2.0, -1.0 / B));
  p->xi.resize(K);
  for (int64_t k = 1; k <= K; ++k) p->xi[k - 1] = fmin * std::pow(2.0, (double)(k - 1) / B);

  // ---- CQ filters and plateaus (readings C7, C8); coefficient counts (C9, C10)
  std::vector<Filt> f;
  std::vector<int64_t> Mk;
  int rc = cq_filters(p, Ls, p->sampled_from, f);
  if (rc) return rc;
  if (!p->sampled_from) {
    rc = channel_counts(p, f, Mk);
  } else {  // Prop. 4 (reading C21): the counts of the 2N' system times L/2N'
    std::vector<Filt> f0;
    rc = cq_filters(p, p->sampled_from, 0, f0);
    if (!rc) rc = channel_counts(p, f0, Mk);
    for (int64_t &m : Mk) m *= Ls / p->sampled_from;
  }
  if (rc) return rc;
  p->lo.resize(K + 2);
  p->len.resize(K + 2);
  p->M.resize(K + 2);
  for (int64_t k = 0; k < K + 2; ++k) {
    p->lo[k] = (int32_t)f[k].lo;
    p->len[k] = (int32_t)f[k].v.size();
    if (Mk[k] > INT32_MAX) return set_error(SLICQ_EINVAL, "channel length overflows int32");
    p->M[k] = (int32_t)Mk[k];
  }
  p->off.assign(K + 3, 0);
  p->goff.assign(K + 2, 0);
  int64_t gl = 0;
  p->painless = true;
  for (int64_t k = 0; k < K + 2; ++k) {
    if (p->M[k] < p->len[k]) {
      // a sampled_from system keeps the slice system's hops (Prop. 4, reading C21): only
      // its analysis is defined (Alg. 1 folds); everything else must be painless
      if (!p->sampled_from)
        return set_error(SLICQ_ENOTFRAME, "painless condition M_k >= L_k violated (P:170)");
      p->painless = false;
    }
    p->off[k + 1] = p->off[k] + p->M[k];
    p->goff[k] = gl;
    gl += p->len[k];
  }
  p->C = p->off[K + 2];
  // ---- frame diagonal over all 2K+2 channels (Prop. 2; weights per C1/C16).
  // The mirror of CQ channel k (Table 1 row 2K+2-k) has g[Ls - j]: it adds g_k[j]^2
  // at bin (-j) mod Ls.  The plateaus are their own mirrors.
  std::vector<double> D(Ls, 0.0);
  auto md = [Ls](int64_t j) { int64_t r = j % Ls; return r < 0 ? r + Ls : r; };
  for (int64_t k = 0; k < K + 2; ++k)
    for (int64_t i = 0; i < p->len[k]; ++i) {
      const int64_t j = f[k].lo + i;
      const double g2 = f[k].v[i] * f[k].v[i];
      D[md(j)] += g2;
      if (k >= 1 && k <= K) D[md(-j)] += g2;
    }
  for (int64_t j = 0; j < Ls; ++j)
    if (!(D[j] > 0.0)) return set_error(SLICQ_ENOTFRAME, "frame diagonal vanishes (P:221)");
  // canonical dual g~_k = g_k / D
  p->g.resize(gl);
  p->gdual.resize(gl);
  for (int64_t k = 0; k < K + 2; ++k)
    for (int64_t i = 0; i < p->len[k]; ++i) {
      const int64_t j = f[k].lo + i;
      p->g[p->goff[k] + i] = f[k].v[i];
      p->gdual[p->goff[k] + i] = f[k].v[i] / D[md(j)];
    }
  // ---- slicing window h_0 (Tukey, essential length N, transitions tr, zero-padded to 2N;
  // P:372-374, reading C11) and its canonical dual h_0 / sum_m T_{mN} h_0^2 (dualwincond
  // P:354-356, reading C12)
  p->h0.assign(2 * N, 0.0);
  p->h0dual.assign(2 * N, 0.0);
  const double A = (double)(N - tr) / 2.0, Bw = (double)(N + tr) / 2.0;
  for (int64_t i = 0; i < 2 * N; ++i) {
    const double t = std::fabs((double)(i - N));
    if (t <= A) p->h0[i] = 1.0;
    else if (t < Bw) {
      const double c = std::cos(kPi * (t - A) / (2.0 * (double)tr));
      p->h0[i] = c * c;
    }
  }
  std::vector<double> per(N, 0.0);
  for (int64_t i = 0; i < 2 * N; ++i) per[(i - N + 2 * N) % N] += p->h0[i] * p->h0[i];
  for (int64_t i = 0; i < 2 * N; ++i)
    if (p->h0[i] != 0.0) p->h0dual[i] = p->h0[i] / per[(i - N + 2 * N) % N];
  return SLICQ_OK;
}

extern "C" {

int plan_create_ex(double fs, double fmin, double fmax, int bins_per_octave, int64_t sl_len,
                   int64_t tr_area, int rasterize, unsigned flags, slicq_plan **out) {
  return plan_create_ex2(fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize, flags,
                         SLICQ_WINDOW_HANN, 4.0, 0, out);
}

int plan_create_ex2(double fs, double fmin, double fmax, int bins_per_octave, int64_t sl_len,
                    int64_t tr_area, int rasterize, unsigned flags, int window, double min_width,
                    int64_t sampled_from, slicq_plan **out) {
  if (!out) return set_error(SLICQ_EINVAL, "out is NULL");
  *out = nullptr;
  if (window != SLICQ_WINDOW_HANN && window != SLICQ_WINDOW_BLACKMAN_HARRIS)
    return set_error(SLICQ_EINVAL, "window must be SLICQ_WINDOW_HANN or _BLACKMAN_HARRIS");
  if (!(min_width >= 1.0) || !std::isfinite(min_width))
    return set_error(SLICQ_EINVAL, "min_width must be >= 1 bin");
  if (sampled_from < 0 || (sampled_from > 0 && (sampled_from % 4 != 0 || sl_len % sampled_from != 0)))
    return set_error(SLICQ_EINVAL, "sampled_from must be 0 or a multiple of 4 dividing sl_len");
  *out = nullptr;
  if (!(fs > 0) || !std::isfinite(fs)) return set_error(SLICQ_EINVAL, "fs must be > 0");
  if (!(fmin > 0) || !(fmin < fs / 2)) return set_error(SLICQ_EINVAL, "need 0 < fmin < fs/2");
  if (!(fmax > fmin) || !std::isfinite(fmax)) return set_error(SLICQ_EINVAL, "need fmax > fmin");
  if (bins_per_octave < 1) return set_error(SLICQ_EINVAL, "bins_per_octave must be >= 1");
  if (sl_len < 8 || sl_len % 4 != 0 || !smooth235(sl_len) || sl_len > (int64_t(1) << 26))
    return set_error(SLICQ_EINVAL, "sl_len must be divisible by 4, 2/3/5-smooth, 8..2^26");
  if (tr_area < 2 || tr_area % 2 != 0 || tr_area >= sl_len / 2)
    return set_error(SLICQ_EINVAL, "tr_area must be even, >= 2 and < sl_len/2 (P:373)");
  if (rasterize < 0 || rasterize > 2) return set_error(SLICQ_EINVAL, "rasterize must be 0, 1, 2");
  if (fmax > fs / 2) fmax = fs / 2;  // C4: cap at Nyquist
  slicq_plan *p = new (std::nothrow) slicq_plan();
  if (!p) return set_error(SLICQ_ENOMEM, "host allocation failed");
  p->fs = fs;
  p->fmin = fmin;
  p->fmax = fmax;
  p->B = bins_per_octave;
  p->sl_len = sl_len;
  p->N = sl_len / 2;
  p->tr = tr_area;
  p->raster = rasterize;
  p->window = window;
  p->min_width = min_width;
  p->sampled_from = sampled_from;
  int rc = build_host_plan(p);
  if (rc == SLICQ_OK && !(flags & SLICQ_PLAN_HOST_ONLY)) {
    rc = slicq::configure_kernels(p);
    if (rc == SLICQ_OK) rc = slicq::upload(p);
  }
  if (rc != SLICQ_OK) {
    slicq::free_device(p);
    delete p;
    return rc;
  }
  *out = p;
  return SLICQ_OK;
}

int plan_create(double fs, double fmin, double fmax, int bins_per_octave, int64_t sl_len,
                int64_t tr_area, int rasterize, slicq_plan **out) {
  return plan_create_ex(fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize, 0u, out);
}

void plan_destroy(slicq_plan *p) {
  if (!p) return;
  slicq::free_device(p);
  delete p;
}

int slicq_num_channels(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return p->K + 2;
}
int slicq_num_cq_channels(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return p->K;
}
int slicq_channel_lengths(const slicq_plan *p, int32_t *M) {
  if (!p || !M) return set_error(SLICQ_EINVAL, "NULL argument");
  std::memcpy(M, p->M.data(), sizeof(int32_t) * p->M.size());
  return SLICQ_OK;
}
int slicq_channel_offsets(const slicq_plan *p, int64_t *off) {
  if (!p || !off) return set_error(SLICQ_EINVAL, "NULL argument");
  std::memcpy(off, p->off.data(), sizeof(int64_t) * p->off.size());
  return SLICQ_OK;
}
int64_t slicq_coeffs_per_slice(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return p->C;
}
int64_t slicq_sl_len(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return p->sl_len;
}
int64_t slicq_padded_length(const slicq_plan *p, int64_t n) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  if (n < 1) return set_error(SLICQ_ESHAPE, "n must be >= 1");
  return (n + p->sl_len - 1) / p->sl_len * p->sl_len;
}
int64_t slicq_num_slices(const slicq_plan *p, int64_t n) {
  int64_t L = slicq_padded_length(p, n);
  if (L < 0) return L;
  return L / p->N;
}
int64_t slicq_halo(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return (p->N + p->tr) / 2;
}
size_t slicq_workspace_bytes(const slicq_plan *p, int64_t nslices, int64_t batch) {
  if (!p || nslices < 1 || batch < 1) return 0;
  return slicq::workspace_bytes(p, nslices, batch);
}
int slicq_kernel_launches(const slicq_plan *p, int direction, int64_t nslices, int64_t batch) {
  if (!p || !p->has_device || nslices < 1 || batch < 1 || (direction != 0 && direction != 1))
    return 0;
  return slicq::kernel_launches(p, direction, nslices, batch);
}
int64_t slicq_filter_total_length(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return (int64_t)p->g.size();
}
int slicq_plan_export(const slicq_plan *p, int32_t *lo, int32_t *len, double *g, double *gdual,
                      double *h0, double *h0dual, double *xi) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  if (lo) std::memcpy(lo, p->lo.data(), sizeof(int32_t) * p->lo.size());
  if (len) std::memcpy(len, p->len.data(), sizeof(int32_t) * p->len.size());
  if (g) std::memcpy(g, p->g.data(), sizeof(double) * p->g.size());
  if (gdual) std::memcpy(gdual, p->gdual.data(), sizeof(double) * p->gdual.size());
  if (h0) std::memcpy(h0, p->h0.data(), sizeof(double) * p->h0.size());
  if (h0dual) std::memcpy(h0dual, p->h0dual.data(), sizeof(double) * p->h0dual.size());
  if (xi) std::memcpy(xi, p->xi.data(), sizeof(double) * p->xi.size());
  return SLICQ_OK;
}
const char *slicq_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ hot path entry points
static int check_dev_plan(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  if (!p->has_device) return set_error(SLICQ_EINVAL, "plan was created host-only");
  return SLICQ_OK;
}

int slicq_forward(const slicq_plan *p, const float *x, int64_t n, int64_t batch,
                  slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1) return set_error(SLICQ_ESHAPE, "n and batch must be >= 1");
  if (!x || !coeffs) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)x % 4 || (uintptr_t)coeffs % 8) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  const int64_t L = slicq_padded_length(p, n);
  const int64_t S = L / p->N;
  return slicq::launch_forward(p, x, n, n, 0, L, 1, 0, S, batch, coeffs, ws, ws_bytes, stream);
}

int slicq_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n, int64_t batch,
                  float *y, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1) return set_error(SLICQ_ESHAPE, "n and batch must be >= 1");
  if (!y || !coeffs) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)y % 4 || (uintptr_t)coeffs % 8) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  const int64_t L = slicq_padded_length(p, n);
  const int64_t S = L / p->N;
  return slicq::launch_inverse(p, coeffs, 0, S, S, batch, 1, n, L, y, n, 0, nullptr, 0, ws,
                               ws_bytes, stream);
}

int slicq_nsgt_forward(const slicq_plan *p, const float *x, int64_t n, int64_t batch,
                       slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1 || n > 2 * p->N)
    return set_error(SLICQ_ESHAPE, "need 1 <= n <= sl_len and batch >= 1");
  if (!x || !coeffs) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)x % 4 || (uintptr_t)coeffs % 8) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  // one frame per row: "slice" 1 of a 2-slice stream starts at sample 0, no wrap, no window
  return slicq::launch_forward(p, x, n, n, 0, 2 * p->N, 0, 1, 1, batch, coeffs, ws, ws_bytes,
                               stream, 1);
}

int slicq_nsgt_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n, int64_t batch,
                       float *y, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1 || n > 2 * p->N)
    return set_error(SLICQ_ESHAPE, "need 1 <= n <= sl_len and batch >= 1");
  if (!y || !coeffs) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)y % 4 || (uintptr_t)coeffs % 8) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_inverse(p, coeffs, 1, 1, 2, batch, 0, n, 2 * p->N, y, n, 0, nullptr, 0, ws,
                               ws_bytes, stream, nullptr, 0, 1);
}

int slicq_inverse_masked(const slicq_plan *p, const slicq_c32 *coeffs, const float *mask,
                         int mask_db, int64_t n, int64_t batch, float *y, void *ws,
                         size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1) return set_error(SLICQ_ESHAPE, "n and batch must be >= 1");
  if (!y || !coeffs || !mask) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)y % 4 || (uintptr_t)coeffs % 8 || (uintptr_t)mask % 4)
    return set_error(SLICQ_ESHAPE, "misaligned buffer");
  const int64_t L = slicq_padded_length(p, n);
  const int64_t S = L / p->N;
  return slicq::launch_inverse(p, coeffs, 0, S, S, batch, 1, n, L, y, n, 0, nullptr, 0, ws,
                               ws_bytes, stream, mask, mask_db ? 1 : 0);
}

int slicq_forward_range(const slicq_plan *p, const float *x_local, int64_t x_len,
                        int64_t x_stride, int64_t halo, int64_t slice0, int64_t nslices,
                        int64_t total_slices, int64_t batch, slicq_c32 *coeffs_local,
                        void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (nslices < 1 || batch < 1 || slice0 < 0 || slice0 + nslices > total_slices || x_len < 0 ||
      x_stride < x_len || total_slices < 2 || total_slices % 2)
    return set_error(SLICQ_ESHAPE, "bad slice range / shape");
  if (halo < slicq_halo(p) - 1 || halo % 2) return set_error(SLICQ_ESHAPE, "halo too small or odd");
  if (!x_local || !coeffs_local) return set_error(SLICQ_ESHAPE, "NULL buffer");
  const int64_t L = total_slices * p->N;
  return slicq::launch_forward(p, x_local, x_len, x_stride, slice0 * p->N - halo, L, 0, slice0,
                               nslices, batch, coeffs_local, ws, ws_bytes, stream);
}

int slicq_inverse_range(const slicq_plan *p, const slicq_c32 *coeffs_local, int64_t slice0,
                        int64_t nslices, int64_t total_slices, int64_t batch, float *y_local,
                        int64_t y_stride, float *left_spill, int64_t halo, void *ws,
                        size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (nslices < 1 || batch < 1 || slice0 < 0 || slice0 + nslices > total_slices ||
      y_stride < nslices * p->N || total_slices < 2)
    return set_error(SLICQ_ESHAPE, "bad slice range / shape");
  if (halo < slicq_halo(p) - 1) return set_error(SLICQ_ESHAPE, "halo too small");
  if (!coeffs_local || !y_local || !left_spill) return set_error(SLICQ_ESHAPE, "NULL buffer");
  const int64_t L = total_slices * p->N;
  return slicq::launch_inverse(p, coeffs_local, slice0, nslices, total_slices, batch, 0,
                               nslices * p->N, L, y_local, y_stride, slice0 * p->N, left_spill,
                               halo, ws, ws_bytes, stream);
}

int64_t slicq_coeffs_per_slice_full(const slicq_plan *p) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  return slicq::coeffs_full(p);
}

size_t slicq_workspace_bytes_complex(const slicq_plan *p, int64_t nslices, int64_t batch,
                                     int64_t n) {
  if (!p || !p->has_device || nslices < 1 || batch < 1 || n < 1) return 0;
  return slicq::workspace_bytes_complex(p, nslices, batch, n);
}

int slicq_forward_complex(const slicq_plan *p, const slicq_c32 *x, int64_t n, int64_t batch,
                          slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1) return set_error(SLICQ_ESHAPE, "n and batch must be >= 1");
  if (!x || !coeffs || !ws) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)x % 8 || (uintptr_t)coeffs % 8 || (uintptr_t)ws % 256)
    return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_forward_complex(p, x, n, batch, coeffs, ws, ws_bytes, stream);
}

int slicq_inverse_complex(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n, int64_t batch,
                          slicq_c32 *y, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1) return set_error(SLICQ_ESHAPE, "n and batch must be >= 1");
  if (!y || !coeffs || !ws) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)y % 8 || (uintptr_t)coeffs % 8 || (uintptr_t)ws % 256)
    return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_inverse_complex(p, coeffs, n, batch, y, ws, ws_bytes, stream);
}

int slicq_apply_mask(const slicq_plan *p, slicq_c32 *coeffs, const float *mask, int64_t rows,
                     int mask_full, int mask_db, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (rows < 1) return set_error(SLICQ_ESHAPE, "rows must be >= 1");
  if (!coeffs || !mask) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)coeffs % 8 || (uintptr_t)mask % 4) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_mask(p, coeffs, mask, rows, mask_full ? 1 : 0, mask_db ? 1 : 0, stream);
}

int slicq_spectrogram(const slicq_plan *p, const slicq_c32 *coeffs, int64_t nslices,
                      int64_t batch, float *out, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (nslices < 2 || nslices % 2 || batch < 1)
    return set_error(SLICQ_ESHAPE, "need an even number of slices >= 2 and batch >= 1");
  if (!coeffs || !out) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)coeffs % 8 || (uintptr_t)out % 4) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_spectrogram(p, coeffs, nslices, batch, out, stream);
}

int slicq_transpose_bins(const slicq_plan *p, const slicq_c32 *coeffs, slicq_c32 *out,
                         int64_t rows, int shift, void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (rows < 1) return set_error(SLICQ_ESHAPE, "rows must be >= 1");
  if (!coeffs || !out || coeffs == out) return set_error(SLICQ_ESHAPE, "NULL or aliased buffer");
  if ((uintptr_t)coeffs % 8 || (uintptr_t)out % 8) return set_error(SLICQ_ESHAPE, "misaligned buffer");
  for (int k = 2; k <= p->K; ++k)
    if (p->M[k] != p->M[1])
      return set_error(SLICQ_EINVAL, "transposition needs equal M_k over the CQ channels "
                                     "(rasterize = SLICQ_RASTER_FULL)");
  return slicq::launch_transpose(p, coeffs, out, rows, shift, stream);
}

int slicq_nsgt_forward_complex(const slicq_plan *p, const slicq_c32 *x, int64_t n,
                               int64_t batch, slicq_c32 *coeffs, void *ws, size_t ws_bytes,
                               void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1 || n > p->sl_len)
    return set_error(SLICQ_ESHAPE, "need 1 <= n <= sl_len and batch >= 1");
  if (!x || !coeffs || !ws) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)x % 8 || (uintptr_t)coeffs % 8 || (uintptr_t)ws % 256)
    return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_forward_complex(p, x, n, batch, coeffs, ws, ws_bytes, stream, 1);
}

int slicq_nsgt_inverse_complex(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n,
                               int64_t batch, slicq_c32 *y, void *ws, size_t ws_bytes,
                               void *stream) {
  int rc = check_dev_plan(p);
  if (rc) return rc;
  if (n < 1 || batch < 1 || n > p->sl_len)
    return set_error(SLICQ_ESHAPE, "need 1 <= n <= sl_len and batch >= 1");
  if (!y || !coeffs || !ws) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)y % 8 || (uintptr_t)coeffs % 8 || (uintptr_t)ws % 256)
    return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_inverse_complex(p, coeffs, n, batch, y, ws, ws_bytes, stream, 1);
}

static int approx_common(const slicq_plan *ps, const slicq_plan *pl, const slicq_c32 *s,
                         const slicq_c32 *c, int64_t batch, double *out, void *stream,
                         int full) {
  int rc = check_dev_plan(ps);
  if (!rc) rc = check_dev_plan(pl);
  if (rc) return rc;
  const int64_t N2 = ps->sl_len, L = pl->sl_len;
  if (pl->sampled_from != N2 || L % N2 || ps->K != pl->K || ps->B != pl->B)
    return set_error(SLICQ_EINVAL, "pl must be created with sampled_from = sl_len of ps");
  for (int k = 0; k < ps->K + 2; ++k)
    if ((int64_t)pl->M[k] != (L / N2) * ps->M[k] || ps->M[k] % 2)
      return set_error(SLICQ_EINVAL, "channel counts are not (L/2N) M_k");
  if (batch < 1) return set_error(SLICQ_ESHAPE, "batch must be >= 1");
  if (!s || !c || !out) return set_error(SLICQ_ESHAPE, "NULL buffer");
  if ((uintptr_t)s % 8 || (uintptr_t)c % 8 || (uintptr_t)out % 8)
    return set_error(SLICQ_ESHAPE, "misaligned buffer");
  return slicq::launch_approx(ps, pl, s, c, batch, out, stream, full);
}

int slicq_approx_error_complex(const slicq_plan *ps, const slicq_plan *pl, const slicq_c32 *s,
                               const slicq_c32 *c, int64_t batch, double *out, void *stream) {
  return approx_common(ps, pl, s, c, batch, out, stream, 1);
}

int slicq_approx_error(const slicq_plan *ps, const slicq_plan *pl, const slicq_c32 *s,
                       const slicq_c32 *c, int64_t batch, double *out, void *stream) {
  return approx_common(ps, pl, s, c, batch, out, stream, 0);
}

int slicq_overlap_add(float *y, int64_t y_stride, const float *spill, int64_t count,
                      int64_t batch, void *stream) {
  if (!y || !spill || count < 0 || batch < 1 || y_stride < count)
    return set_error(SLICQ_ESHAPE, "bad overlap_add arguments");
  if (count == 0) return SLICQ_OK;
  return slicq::launch_overlap_add(y, y_stride, spill, count, batch, stream);
}

}  // extern "C"
