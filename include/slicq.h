/*
 * slicq.h — C ABI of the B200-native sliCQ library (libslicq.so).
 *
 * The sliCQ transform of Holighaus, Dörfler, Velasco, Grill, "A framework for
 * invertible, real-time constant-Q transforms" (arXiv 1210.0084).  References
 * "P:<line>" are lines of that paper's text; "C<n>" are the readings
 * of ambiguous passages listed in DESIGN.md ("Readings of the paper").
 *
 * What the library computes
 *   slicq_forward  = Alg. 3 "sliCQ analysis" with Alg. 1 "NSG analysis"
 *                     applied to every slice of length 2N = sl_len,
 *                    for REAL fp32 input; coefficients of the channels
 *                    k = 0 (DC plateau), 1..K (constant-Q), K+1 (Nyquist plateau)
 *                    of Table 1.  The mirror channels K+2..2K+1 are
 *                    redundant for real input (C15) and are not stored.
 *   slicq_inverse  = Alg. 4 "sliCQ synthesis" with Alg. 2 "NSG
 *                    synthesis" and the canonical duals of Prop. 2
 *                     and of dualwincond.
 *
 * Normalisation (C1): FFT_n unnormalised, IFFT_n with 1/n, so channel k of slice m is
 *     c^m_k = sqrt(M_k) * IFFT_{M_k}( fold_{M_k}( FFT_{2N}(f^m) * g_k ) ),
 *     f^m[j] = f[((m-1)N + j) mod L] * h_0[j-N]
 * where M_k = L/a_k is channel k's coefficient count per slice (C9/C10).
 *
 * Layouts (all contiguous, row-major, caller-owned, device memory unless stated)
 *   x, y    : float32 [batch][n]   (one row per mono signal / audio channel)
 *   coeffs  : slicq_c32 [batch][S][C] with S = slicq_num_slices(p, n) and
 *             C = slicq_coeffs_per_slice(p) = sum_k M_k; channel k occupies
 *             columns [off_k, off_k + M_k) (slicq_channel_offsets), entry n of
 *             channel k is coefficient c^m_{n,k} (slice-local time n*2N/M_k).
 *             The paper's two-layer array s is the index view
 *             s^{m mod 2}_k[((m-1) M_k/2 + n) mod (L M_k / 2N)] = c^m_k[n].
 *   L       : padded length ceil(n / 2N) * 2N, zero padding at the end (C13);
 *             y is trimmed back to n.
 *
 * Execution model
 *   plan_create runs on the host (float64) and uploads read-only tables once.
 *   The hot-path calls are asynchronous and stream-ordered on `stream` (a
 *   cudaStream_t passed as void*; NULL = legacy default stream), perform no
 *   allocation and no host synchronisation.  A plan is immutable: concurrent
 *   calls on different streams are safe if they use distinct workspaces.  Calls of
 *   >= 8192 (row, slice) units run their chunks on two streams owned by the plan (forked
 *   from and joined back into `stream`); such calls on one plan are serialised on those
 *   streams -- use one plan per stream for concurrent large calls.
 *   Device faults surface at the caller's next synchronisation (CUDA semantics).
 *
 * Errors: every int-returning call returns SLICQ_OK (0) or a negative code and
 * sets a thread-local message readable with slicq_last_error().
 */
#ifndef SLICQ_H
#define SLICQ_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SLICQ_API __attribute__((visibility("default")))
#else
#define SLICQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct slicq_plan slicq_plan;       /* opaque */
typedef struct { float re, im; } slicq_c32;  /* interleaved complex64 (torch.complex64 layout) */

enum {
  SLICQ_RASTER_NONE = 0,   /* M_k = smallest even 2/3/5-smooth >= L_k per channel (C9)    */
  SLICQ_RASTER_OCTAVE = 1, /* one M per CQ octave, DC and Nyquist separate (C10)           */
  SLICQ_RASTER_FULL = 2    /* one M for all channels: "L/a_k constant" (C10)    */
};

enum {
  SLICQ_OK = 0,
  SLICQ_EINVAL = -1,        /* invalid parameter (SPEC InvalidParams)                     */
  SLICQ_ENOTFRAME = -2,     /* frame diagonal not positive / M_k < L_k (Prop. 2)   */
  SLICQ_ESHAPE = -3,        /* n, batch, pointer alignment, workspace size                */
  SLICQ_ECUDA = -4,         /* CUDA runtime error (no device, launch failure, ...)        */
  SLICQ_ENOMEM = -5,        /* host or device allocation failed                           */
  SLICQ_EINTERNAL = -6,     /* broken internal invariant                                  */
  SLICQ_EUNSUPPORTED = -7   /* valid plan the CUDA path has no kernel for (see plan_create) */
};

enum { SLICQ_PLAN_HOST_ONLY = 1 }; /* plan_create_ex flag: host tables only, no device */
/* filter shape H of P:262: Hann (C7) or the 4-term Blackman-Harris of the paper's
 * approximation experiments (reading C20) */
enum { SLICQ_WINDOW_HANN = 0, SLICQ_WINDOW_BLACKMAN_HARRIS = 1 };

/* ------------------------------------------------------------------ plans
 * plan_create: build the CQ-NSGT system for slices of length sl_len = 2N.
 *   fs               sampling rate xi_s in Hz (> 0)
 *   fmin, fmax       xi_min, xi_max in Hz: 0 < fmin < fs/2, fmax > fmin; fmax >= fs/2 is
 *                    allowed and caps K at the last centre below Nyquist (C4)
 *   bins_per_octave  B >= 1
 *   sl_len           2N: divisible by 4 and 2/3/5-smooth.  The CUDA path implements
 *                    2N = 2^12 .. 2^17 (4096 .. 131072; 2N >= 65536 use a four-step FFT
 *                    through the workspace) and every other 2/3/5-smooth 2N from 128 to
 *                    53248 (a mixed-radix in-place FFT in one CTA's shared memory,
 *                    kernels_generic.cu; e.g. the paper's 12288, 24000, 50000) for
 *                    every entry point, and 2N = 2^18 .. 2^22 for the full-length CQ-NSGT
 *                    (slicq_nsgt_*) only; other valid values give SLICQ_EUNSUPPORTED unless
 *                    SLICQ_PLAN_HOST_ONLY is set.  Channel lengths: M_k <= 1024 run in the
 *                    register-DFT channel kernels, 1024 < M_k <= 26000 in one CTA per
 *                    (channel, unit) with a shared-memory mixed-radix DFT.
 *   tr_area          Tukey transition length (the paper's M): even, 2 <= tr < N
 *   rasterize        SLICQ_RASTER_*
 *   out              receives the plan (NULL on failure)
 * The plan allocates its device tables (a few MB; up to ~100 MB for 2N = 2^22) on the device
 * current at the call.
 * Returns SLICQ_EINVAL, SLICQ_ENOTFRAME, SLICQ_EUNSUPPORTED, SLICQ_ECUDA, SLICQ_ENOMEM. */
SLICQ_API int plan_create(double fs, double fmin, double fmax, int bins_per_octave, int64_t sl_len,
                int64_t tr_area, int rasterize, slicq_plan **out);
SLICQ_API int plan_create_ex(double fs, double fmin, double fmax, int bins_per_octave, int64_t sl_len,
                   int64_t tr_area, int rasterize, unsigned flags, slicq_plan **out);
/* plan_create_ex2: plan_create_ex with the filter options of the paper's approximation
 * experiments (Sec. V-A; Prop. 4):
 *   window        SLICQ_WINDOW_HANN (plan_create_ex) or SLICQ_WINDOW_BLACKMAN_HARRIS
 *   min_width     lower bound on the filter width in bins, >= 1 (plan_create_ex: 4; the x
 *                 axis of Fig. CoeffQual)
 *   sampled_from  0, or 2N' (a multiple of 4 dividing sl_len): build the full-length system
 *                 G(g^L, a) of Prop. 4 -- filters whose samples every sl_len/2N' bins are the
 *                 2N' system's (g_k[j] = g^L_k[j sl_len/2N'], the width clamp acting on the
 *                 2N' grid) and counts M_k = (sl_len/2N') M'_k (the same hops a_k; reading
 *                 C21).  Such a system need not be painless (M_k < L_k where the support is
 *                 longer than the hops allow): only slicq_nsgt_forward is defined on it
 *                 (other calls return SLICQ_EUNSUPPORTED), and its device path requires
 *                 sl_len >= 2^18 (the fold of the long path sums aliased bins).
 * Errors as plan_create_ex; SLICQ_EINVAL for a bad window / min_width / sampled_from. */
SLICQ_API int plan_create_ex2(double fs, double fmin, double fmax, int bins_per_octave,
                              int64_t sl_len, int64_t tr_area, int rasterize, unsigned flags,
                              int window, double min_width, int64_t sampled_from,
                              slicq_plan **out);
/* NULL-safe; frees the plan-owned device tables.  No call may be in flight on the plan. */
SLICQ_API void plan_destroy(slicq_plan *p);

/* ------------------------------------------------------------------ queries (host, cheap)
 * Channel order 0 = DC plateau, 1..K = ascending CQ channels, K+1 = Nyquist plateau. */
SLICQ_API int slicq_num_channels(const slicq_plan *p);                      /* K+2, or <0 on error  */
SLICQ_API int slicq_num_cq_channels(const slicq_plan *p);                   /* K                    */
SLICQ_API int slicq_channel_lengths(const slicq_plan *p, int32_t *M);       /* host out [K+2]: M_k  */
SLICQ_API int slicq_channel_offsets(const slicq_plan *p, int64_t *off);     /* host out [K+3]       */
SLICQ_API int64_t slicq_coeffs_per_slice(const slicq_plan *p);              /* sum_k M_k            */
SLICQ_API int64_t slicq_sl_len(const slicq_plan *p);                        /* 2N                   */
SLICQ_API int64_t slicq_padded_length(const slicq_plan *p, int64_t n);      /* L = ceil(n/2N)*2N    */
SLICQ_API int64_t slicq_num_slices(const slicq_plan *p, int64_t n);         /* S = L/N      */
SLICQ_API int64_t slicq_halo(const slicq_plan *p);                          /* (N+tr)/2: one-sided reach of h_0 */
/* Workspace bytes needed by the hot-path calls for `nslices` slices of `batch` rows (0 for
 * host-only plans).  One workspace serves both directions: it holds the inverse's overlap-add
 * pairing counters and boundary halves, and a staging area for the spectra / channel
 * contributions of one chunk of slices (by default at most 8 GB of staging: larger calls
 * run chunk by chunk with identical results).  No initialisation is needed (each inverse
 * call resets its boundary-pairing counters on its stream); a workspace may be reused by
 * calls of any size, one workspace per concurrently running call. */
SLICQ_API size_t slicq_workspace_bytes(const slicq_plan *p, int64_t nslices, int64_t batch);
/* Number of CUDA kernels one slicq_forward (direction 0) or slicq_inverse (direction 1) call
 * (or the _range variant) launches for nslices x batch slices -- for launch accounting.
 * Returns 0 for a host-only plan or invalid arguments. */
SLICQ_API int slicq_kernel_launches(const slicq_plan *p, int direction, int64_t nslices,
                                    int64_t batch);
/* Plan export for parity tests (host out-params, any may be NULL):
 *   lo[K+2], len[K+2]   unwrapped support J_k = [lo_k, lo_k + len_k) in 2N-bins (C5)
 *   g[sum len], gdual[sum len]   g_k and canonical dual g_k / sum_l |g_l|^2 on J_k
 *   h0[2N], h0dual[2N]  slicing window and its dual at t = -N..N-1 (index t+N)
 *   layout[K]           centre frequencies xi_1..xi_K in Hz (Table 1)          */
SLICQ_API int slicq_plan_export(const slicq_plan *p, int32_t *lo, int32_t *len, double *g, double *gdual,
                      double *h0, double *h0dual, double *xi);
SLICQ_API int64_t slicq_filter_total_length(const slicq_plan *p);           /* sum_k len_k          */
SLICQ_API const char *slicq_last_error(void);                               /* thread-local message */

/* ------------------------------------------------------------------ hot path
 * slicq_forward: coeffs[b][m][:] = sliCQ analysis of x[b][0..n) for all S slices.
 *   x       device float32 [batch][n], rows contiguous, 4-byte aligned (8-byte gives
 *           vector loads)
 *   coeffs  device slicq_c32 [batch][S][C], 8-byte aligned
 *   ws      >= slicq_workspace_bytes(p, S, batch) bytes, 16-byte aligned (see above)
 * Returns SLICQ_ESHAPE on n < 1, batch < 1, NULL/misaligned pointers, small workspace;
 * SLICQ_ECUDA if a launch fails. */
SLICQ_API int slicq_forward(const slicq_plan *p, const float *x, int64_t n, int64_t batch,
                  slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream);

/* slicq_inverse: y[b][0..n) = sliCQ synthesis of coeffs[b] (any coefficients: modified
 * ones are synthesised with the Hermitian projection of C15, i.e. the real part of the
 * full 2K+2-channel Alg. 2).  ws: >= slicq_workspace_bytes(p, S, batch) bytes, see above.
 * y is fully overwritten (no need to zero it). */
SLICQ_API int slicq_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n, int64_t batch,
                  float *y, void *ws, size_t ws_bytes, void *stream);

/* slicq_inverse_masked: slicq_inverse of (coeffs * a), the coefficient mask fused into the
 * inverse's coefficient loads (paper §VI masking):
 *   mask  device float32 [batch][S][C], the layout of coeffs, 4-byte aligned
 *   mask_db  0: a = mask (linear amplitude); 1: dB-scaled, a = 10^(-5 (1 - mask)), i.e.
 *            0 -> -100 dB, 1 -> 0 dB, linear in dB in between
 * Errors as slicq_inverse (NULL mask -> SLICQ_ESHAPE). */
SLICQ_API int slicq_inverse_masked(const slicq_plan *p, const slicq_c32 *coeffs, const float *mask,
                                   int mask_db, int64_t n, int64_t batch, float *y, void *ws,
                                   size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ full-length CQ-NSGT
 * slicq_nsgt_forward / slicq_nsgt_inverse: the CQ-NSGT of Alg. 1 / Alg. 2 of a
 * whole signal of length L = sl_len (L = 2^12 .. 2^22 — plans with
 * sl_len = 2^18 .. 2^22 serve only these two calls, the sliCQ calls on them return
 * SLICQ_EUNSUPPORTED; channel lengths up to 16 x 26000):
 * the frame is x itself (zero padded from n to L), no slicing window, no overlap; the plan's
 * channels are the CQ-NSGT's at length L.
 *   x, y    device float32 [batch][n], 1 <= n <= sl_len
 *   coeffs  device slicq_c32 [batch][C] (C = slicq_coeffs_per_slice, channel k at
 *           slicq_channel_offsets[k]; mirror channels not stored, C15)
 *   ws      >= slicq_workspace_bytes(p, 1, batch) bytes, as for slicq_forward
 * Errors as slicq_forward / slicq_inverse; n > sl_len gives SLICQ_ESHAPE. */
SLICQ_API int slicq_nsgt_forward(const slicq_plan *p, const float *x, int64_t n, int64_t batch,
                                 slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream);
SLICQ_API int slicq_nsgt_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n,
                                 int64_t batch, float *y, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ complex input
 * slicq_forward_complex / slicq_inverse_complex: the sliCQ of complex signals f in C^L
 * (Alg. 3/4) over all 2K+2 channels of Table 1: no Hermitian
 * reduction, the mirror channels K+2..2K+1 are stored.
 *   x, y    device slicq_c32 [batch][n] (interleaved re, im), 8-byte aligned
 *   coeffs  device slicq_c32 [batch][S][Cf], Cf = slicq_coeffs_per_slice_full(p): channels
 *           in Table-1 order -- 0..K+1 at slicq_channel_offsets[k] as in the real layout,
 *           then the mirrors of channels K, K-1, .., 1 (M_{2K+2-k} = M_k)
 *   ws      >= slicq_workspace_bytes_complex(p, S, batch, n) bytes, 256-byte aligned
 * Computed through the real-input kernels by linearity (f = Re f + i Im f; the mirror
 * channels of a real input are e^{2 pi i 2N n/M_k} conj(c_{n,k}), C15): forward = real
 * transform of the 2 batch rows (Re, Im) + a combine kernel; inverse = split into two
 * real-consistent coefficient sets + real synthesis of 2 batch rows + interleave.  Errors
 * as slicq_forward / slicq_inverse. */
SLICQ_API int64_t slicq_coeffs_per_slice_full(const slicq_plan *p);  /* sum over 2K+2 M_k */
SLICQ_API size_t slicq_workspace_bytes_complex(const slicq_plan *p, int64_t nslices,
                                               int64_t batch, int64_t n);
SLICQ_API int slicq_forward_complex(const slicq_plan *p, const slicq_c32 *x, int64_t n,
                                    int64_t batch, slicq_c32 *coeffs, void *ws,
                                    size_t ws_bytes, void *stream);
SLICQ_API int slicq_inverse_complex(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n,
                                    int64_t batch, slicq_c32 *y, void *ws, size_t ws_bytes,
                                    void *stream);
/* slicq_nsgt_forward_complex / slicq_nsgt_inverse_complex: the full-length CQ-NSGT (Alg. 1/2)
 * of complex signals, 1 <= n <= sl_len, coefficients [batch][Cf] in the layout above;
 * ws >= slicq_workspace_bytes_complex(p, 1, batch, n).  Same construction as the sliced
 * calls; plans with M_k < L_k (sampled_from) serve only the forward. */
SLICQ_API int slicq_nsgt_forward_complex(const slicq_plan *p, const slicq_c32 *x, int64_t n,
                                         int64_t batch, slicq_c32 *coeffs, void *ws,
                                         size_t ws_bytes, void *stream);
SLICQ_API int slicq_nsgt_inverse_complex(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n,
                                         int64_t batch, slicq_c32 *y, void *ws, size_t ws_bytes,
                                         void *stream);

/* ------------------------------------------------------------------ coefficient processing
 * Device kernels on the slice-major coefficient layout [rows][C] (rows = batch x S; paper
 * §VI).  All enqueue on `stream` and return
 * SLICQ_ESHAPE for NULL / misaligned buffers or bad counts.
 *
 * slicq_apply_mask: coeffs[r][i] *= a, a = m (mask_db = 0) or 10^(-5 (1 - m)) (mask_db = 1:
 *   0 -> -100 dB, 1 -> 0 dB), m = mask[i] (mask_full = 0: one float32 per column,
 *   [C]) or mask[r][i] (mask_full = 1: float32 [rows][C]).  In place.
 * slicq_spectrogram: the sliCQ spectrogram |s^0 + s^1|^2 of coefficients
 *   [batch][nslices][C] (nslices even): out float32 [batch][nslices C / 2], channel k at
 *   nslices off_k / 2, entry p = m M_k/2 + n' = |c^m_k[n' + M_k/2] + c^{m+1}_k[n']|^2 (the
 *   two-layer array of Alg. 3; slices circular), hop 2N / M_k samples.
 * slicq_transpose_bins: out = coeffs with every CQ channel k taking channel k - shift's
 *   coefficients (B bins = one octave), modulated by e^{2 pi i d n / M}
 *   (d = round(centre_k - centre_{k-shift}) in bins: the library's coefficients carry
 *   absolute phase, C6); vacated CQ channels are zero, the plateaus copied.  Needs equal
 *   M_k over the CQ channels (SLICQ_RASTER_FULL) else SLICQ_EINVAL; out must not alias. */
SLICQ_API int slicq_apply_mask(const slicq_plan *p, slicq_c32 *coeffs, const float *mask,
                               int64_t rows, int mask_full, int mask_db, void *stream);
SLICQ_API int slicq_spectrogram(const slicq_plan *p, const slicq_c32 *coeffs, int64_t nslices,
                                int64_t batch, float *out, void *stream);
SLICQ_API int slicq_transpose_bins(const slicq_plan *p, const slicq_c32 *coeffs, slicq_c32 *out,
                                   int64_t rows, int shift, void *stream);

/* ------------------------------------------------------------------ Prop. 4 / Sec. V-A
 * slicq_approx_error: the sliCQ's approximation of the full-length CQ-NSGT (Prop. 4,
 * P:377-391; the experiment of P:475-497).  Per row b and stored
 * channel k, in the Prop. 4 normalisation c_{n,k} = <f, T_{n a_k} g^L_k-check> (reading C22:
 * the library's Alg. 1 coefficients divided by sqrt(L a_k), slices by sqrt(2N a_k)):
 *   out[b][k][0] = sum_n |c_{n,k}|^2
 *   out[b][k][1] = sum_n |c_{n,k} - (s^0_{n,k} + s^1_{n,k})|^2,  n < L/a_k,
 * with s^0 + s^1 at n = m N/a_k + n' (n' < N/a_k) = c^m_{n' + N/a_k, k} + c^{m+1}_{n', k}
 * (the two-layer array of Alg. 3; slices circular).  SNR = 10 log10(sum [0] /
 * sum [1]).
 *   ps   sliCQ plan (slices 2N); pl: plan_create_ex2(..., sampled_from = 2N) with sl_len
 *        L, a multiple of 2N, and the same CQ parameters
 *   s    device slicq_c32 [batch][S][C_ps], S = L/N: slicq_forward(ps, x, n = L)
 *   c    device slicq_c32 [batch][C_pl]: slicq_nsgt_forward(pl, x, n = L)
 *   out  device double [batch][K+2][2], fully overwritten
 * Enqueued on `stream`.  SLICQ_EINVAL if (ps, pl) is not such a pair; SLICQ_ESHAPE for
 * NULL / misaligned buffers or batch < 1. */
SLICQ_API int slicq_approx_error(const slicq_plan *ps, const slicq_plan *pl, const slicq_c32 *s,
                                 const slicq_c32 *c, int64_t batch, double *out, void *stream);
/* slicq_approx_error_complex: the same sums for complex signals over all 2K+2 channels:
 *   s    [batch][S][Cf_ps] from slicq_forward_complex(ps, x, n = L)
 *   c    [batch][Cf_pl]    from slicq_nsgt_forward_complex(pl, x, n = L)
 *   out  device double [batch][2K+2][2] (Table-1 channel order) */
SLICQ_API int slicq_approx_error_complex(const slicq_plan *ps, const slicq_plan *pl,
                                         const slicq_c32 *s, const slicq_c32 *c, int64_t batch,
                                         double *out, void *stream);

/* ------------------------------------------------------------------ slice-range shards
 * Multi-GPU partition of one long stream: a rank owns slices
 * [slice0, slice0 + nslices) of total_slices = S and input samples
 * [slice0*N, (slice0 + nslices)*N).
 *
 * slicq_forward_range: x_local holds `x_len` samples of each row (row stride x_stride
 *   floats) where x_local[i] is global sample slice0*N - halo + i; the caller places the
 *   left neighbour's samples (circularly wrapped for slice0 = 0) in the first
 *   `halo` entries and zeros for padding positions >= n.  halo must be even and
 *   >= slicq_halo(p) - 1; slicq_halo(p) = (N + tr)/2 is itself odd when tr = 2 mod 4, so
 *   callers use slicq_halo(p) rounded up to even (paper_1210_0084_b200/dist.py LibBackend);
 *   positions outside [0, x_len) read as 0.
 *   coeffs_local: [batch][nslices][C]; ws as for slicq_forward with S = nslices.
 * slicq_inverse_range: y_local [batch][nslices*N] (row stride y_stride) receives the
 *   overlap-added output of samples [slice0*N, (slice0+nslices)*N) from these slices
 *   only; left_spill [batch][halo] receives the part of slice0's output that falls on
 *   samples [slice0*N - halo, slice0*N) (the left neighbour adds it with
 *   slicq_overlap_add).  ws as for slicq_inverse with S = nslices. */
SLICQ_API int slicq_forward_range(const slicq_plan *p, const float *x_local, int64_t x_len,
                        int64_t x_stride, int64_t halo, int64_t slice0, int64_t nslices,
                        int64_t total_slices, int64_t batch, slicq_c32 *coeffs_local,
                        void *ws, size_t ws_bytes, void *stream);
SLICQ_API int slicq_inverse_range(const slicq_plan *p, const slicq_c32 *coeffs_local, int64_t slice0,
                        int64_t nslices, int64_t total_slices, int64_t batch, float *y_local,
                        int64_t y_stride, float *left_spill, int64_t halo, void *ws,
                        size_t ws_bytes, void *stream);
/* y[b][i] += spill[b][i] for i < count (rows: y stride y_stride, spill stride count). */
SLICQ_API int slicq_overlap_add(float *y, int64_t y_stride, const float *spill, int64_t count,
                      int64_t batch, void *stream);

/* ------------------------------------------------------------------ streaming executor
 * slicq_process_host: host-to-host round trip y = inverse(fn(forward(x))) of a long signal,
 * pipelined over `pieces` contiguous slice ranges (native executor, csrc/stream_exec.cpp):
 * per range a host -> device copy of its samples plus the left halo (circular for the first
 * range), slicq_forward_range, the optional hook, slicq_inverse_range, the
 * overlap-add of its left spill into the previous range (slicq_overlap_add), and a device
 * -> host copy of the completed range, on three streams forked from `stream` so that the
 * copies of one range overlap the kernels of another.  The arithmetic is exactly that of
 * slicq_forward + slicq_inverse.
 *   x_host, y_host  host float32 [batch][n] (pinned for overlap; pageable works, slower);
 *                   y_host is fully overwritten
 *   fn (may be NULL) is called on the host while the work is being enqueued, once per
 *     range, with the device coefficients [batch][nslices][C] of slices [slice0,
 *     slice0 + nslices) and the stream its device work must be enqueued on (in-place
 *     coefficient processing, e.g. masking); a nonzero return aborts with SLICQ_EINVAL
 *   ws  device, >= slicq_process_host_workspace_bytes(p, n, batch, pieces) bytes,
 *       256-byte aligned (a ring of 4 range buffers; its size does not grow with n beyond
 *       one range).  No initialisation is needed: every inverse call resets its own
 *       overlap-add pairing counters.
 * Asynchronous with respect to the host: synchronise `stream` before reading y_host.
 * One call per workspace at a time. */
typedef int (*slicq_coeff_fn)(void *user, slicq_c32 *coeffs, int64_t slice0, int64_t nslices,
                              int64_t batch, void *stream);
SLICQ_API size_t slicq_process_host_workspace_bytes(const slicq_plan *p, int64_t n, int64_t batch,
                                                    int pieces);
SLICQ_API int slicq_process_host(const slicq_plan *p, const float *x_host, float *y_host, int64_t n,
                                 int64_t batch, int pieces, slicq_coeff_fn fn, void *user, void *ws,
                                 size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SLICQ_H */
