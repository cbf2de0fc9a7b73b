// Register-resident mixed-radix (2/3/4/5) DFT building blocks for sm_100a.
//
// dft<R, SIGN>(v): in-place DFT of R complex values held in registers,
//   Y[n] = sum_p v[p] * exp(SIGN * 2 pi i p n / R),   output in natural order.
// SIGN = -1 is the (unnormalised) forward FFT, SIGN = +1 the unnormalised inverse.
// Composite R = r * s is split four-step style (input p = s p1 + p2, output
// n = n1 + r n2) with compile-time twiddles computed in double precision by
// constexpr code, so every twiddle is an FMUL/FFMA immediate — no tables, no
// fast-math trigonometry (reading C18).
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

namespace slicq {
namespace dev {

// ---------------------------------------------------------------- constexpr trig
constexpr double kPiD = 3.14159265358979323846264338327950288;

constexpr double taylor_sin(double x) {  // |x| <= pi/4
  double x2 = x * x, term = x, sum = x;
  for (int i = 1; i < 14; ++i) {
    term *= -x2 / ((2.0 * i) * (2.0 * i + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double taylor_cos(double x) {  // |x| <= pi/4
  double x2 = x * x, term = 1.0, sum = 1.0;
  for (int i = 1; i < 14; ++i) {
    term *= -x2 / ((2.0 * i - 1.0) * (2.0 * i));
    sum += term;
  }
  return sum;
}
// cos(pi * num / den) for 0 <= num/den <= 1/2.
constexpr double cos_pi_frac(long num, long den) {
  if (4 * num > den) return taylor_sin(kPiD * (double)(den - 2 * num) / (2.0 * (double)den));
  return taylor_cos(kPiD * (double)num / (double)den);
}
// cos(2 pi t / R) with the octant reduction done on the integers (t, R).
constexpr double cos2pi(long t, long R) {
  t %= R;
  if (t < 0) t += R;
  if (2 * t > R) t = R - t;                        // cos is even and R-periodic
  if (4 * t > R) return -cos_pi_frac(R - 2 * t, R);  // cos(a) = -cos(pi - a)
  return cos_pi_frac(2 * t, R);
}
// sin(2 pi t / R) = cos(2 pi (4t - R) / (4R))
constexpr double sin2pi(long t, long R) { return cos2pi(4 * t - R, 4 * R); }

// ---------------------------------------------------------------- complex helpers
// SLICQ_F32X2 = 1 (default): complex arithmetic on sm_100a's packed FP32 pair instructions
// (FADD2 / FMUL2 / FFMA2: one issue slot for the real and the imaginary lane; the swap of
// the two lanes, a per-lane sign and a scalar or immediate broadcast are operand modifiers
// in SASS, so a complex add is one instruction, a complex multiply two, and a rotation by
// +-i folds into its consumer).  The kernels are bound by instruction issue, not by the FP32
// pipe, so halving the FP issue slots is what counts.  = 0 keeps the
// scalar FADD/FMUL/FFMA forms (same values up to the order of the roundings in cmul).
#ifndef SLICQ_F32X2
#define SLICQ_F32X2 1
#endif
#if SLICQ_F32X2
__device__ __forceinline__ float2 bcast2(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(-a.y, a.x), bcast2(b.y), __fmul2_rn(a, bcast2(b.x)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, bcast2(s)); }
// a * s + b with a real scalar s
__device__ __forceinline__ float2 cfma_s(float2 a, float s, float2 b) { return __ffma2_rn(a, bcast2(s), b); }
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cfma_s(float2 a, float s, float2 b) {
  return make_float2(fmaf(a.x, s, b.x), fmaf(a.y, s, b.y));
}
#endif
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// multiply by SIGN * i
template <int SIGN>
__device__ __forceinline__ float2 mul_si(float2 a) {
  return SIGN > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// v * exp(SIGN * 2 pi i * T / R) with T, R compile-time; trivial cases specialised.
template <int T, int R, int SIGN>
__device__ __forceinline__ float2 twiddle_c(float2 v) {
  constexpr int t = ((T % R) + R) % R;
  if constexpr (t == 0) {
    return v;
  } else if constexpr (4 * t == R) {
    return mul_si<SIGN>(v);
  } else if constexpr (2 * t == R) {
    return make_float2(-v.x, -v.y);
  } else if constexpr (4 * t == 3 * R) {
    return mul_si<-SIGN>(v);
  } else {
    constexpr float c = (float)cos2pi(t, R);
    constexpr float s = (float)(SIGN * sin2pi(t, R));
#if SLICQ_F32X2
    return cmul(v, make_float2(c, s));
#else
    return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
#endif
  }
}

constexpr int first_factor(int R) {
  return (R % 4 == 0 && R != 8) ? 4 : (R % 2 == 0 ? 2 : (R % 3 == 0 ? 3 : 5));
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(float2 (&v)[R]);

template <int SIGN>
__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    dft2<SIGN>(v[0], v[1]);
  } else if constexpr (R == 3) {
    constexpr float h = 0.86602540378443864676f;  // sin(2 pi/3)
    float2 t1 = cadd(v[1], v[2]);
    float2 t2 = csub(v[1], v[2]);
    float2 y0 = cadd(v[0], t1);
    float2 a = cfma_s(t1, -0.5f, v[0]);
    float2 b = mul_si<SIGN>(cscale(t2, h));
    v[0] = y0;
    v[1] = cadd(a, b);
    v[2] = csub(a, b);
  } else if constexpr (R == 4) {
    float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    float2 b0 = cadd(v[1], v[3]), b1 = mul_si<SIGN>(csub(v[1], v[3]));
    v[0] = cadd(a0, b0);
    v[2] = csub(a0, b0);
    v[1] = cadd(a1, b1);
    v[3] = csub(a1, b1);
  } else if constexpr (R == 5) {
    constexpr float c1 = 0.30901699437494742410f;   // cos(2 pi/5)
    constexpr float c2 = -0.80901699437494742410f;  // cos(4 pi/5)
    constexpr float s1 = 0.95105651629515357212f;   // sin(2 pi/5)
    constexpr float s2 = 0.58778525229247312917f;   // sin(4 pi/5)
    float2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    float2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    float2 y0 = cadd(v[0], cadd(t1, t2));
#if SLICQ_F32X2
    float2 a1 = cfma_s(t2, c2, cfma_s(t1, c1, v[0]));
    float2 a2 = cfma_s(t2, c1, cfma_s(t1, c2, v[0]));
    float2 b1 = cfma_s(t4, s2, cscale(t3, s1));
    float2 b2 = cfma_s(t4, -s1, cscale(t3, s2));
#else
    float2 a1 = make_float2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    float2 a2 = make_float2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    float2 b1 = make_float2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
    float2 b2 = make_float2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
#endif
    b1 = mul_si<SIGN>(b1);
    b2 = mul_si<SIGN>(b2);
    v[0] = y0;
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
  } else {
    constexpr int r = first_factor(R);
    constexpr int s = R / r;
    static_assert(r * s == R, "R must be 2/3/5-smooth");
    float2 b[s][r];
    static_for<0, s>([&](auto P2c) {
      constexpr int p2 = decltype(P2c)::value;
      float2 a[r];
#pragma unroll
      for (int p1 = 0; p1 < r; ++p1) a[p1] = v[s * p1 + p2];
      dft<r, SIGN>(a);
      static_for<0, r>([&](auto N1c) {
        constexpr int n1 = decltype(N1c)::value;
        b[p2][n1] = twiddle_c<p2 * n1, R, SIGN>(a[n1]);
      });
    });
#pragma unroll
    for (int n1 = 0; n1 < r; ++n1) {
      float2 c[s];
#pragma unroll
      for (int p2 = 0; p2 < s; ++p2) c[p2] = b[p2][n1];
      dft<s, SIGN>(c);
#pragma unroll
      for (int n2 = 0; n2 < s; ++n2) v[n1 + r * n2] = c[n2];
    }
  }
}

}  // namespace dev
}  // namespace slicq
