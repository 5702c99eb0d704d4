// Register-resident small DFTs (radix butterflies) for the ILS FFT engine.
//
// Replaces the inner arithmetic of scipy.fft.fft2/ifft2 that the reference
// calls through solver.py:24-30.  Everything here is compile-time shaped:
// a radix-R DFT over R complex values held in registers, with every twiddle
// a constexpr folded into the instruction stream.  Composite radices with
// coprime factors use the prime-factor algorithm (no internal twiddles),
// prime powers Cooley-Tukey from 2, 4 and odd primes (3, 5, 7, 11, 13).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include <utility>

namespace ils {

template <typename T>
struct alignas(2 * sizeof(T)) cx {
  T x, y;
};

template <typename T>
__host__ __device__ __forceinline__ cx<T> operator+(cx<T> a, cx<T> b) { return {a.x + b.x, a.y + b.y}; }
template <typename T>
__host__ __device__ __forceinline__ cx<T> operator-(cx<T> a, cx<T> b) { return {a.x - b.x, a.y - b.y}; }
template <typename T>
__host__ __device__ __forceinline__ cx<T> cmul(cx<T> a, cx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// a * conj(b)
template <typename T>
__host__ __device__ __forceinline__ cx<T> cmulc(cx<T> a, cx<T> b) {
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> conj(cx<T> a) { return {a.x, -a.y}; }
template <typename T>
__host__ __device__ __forceinline__ cx<T> scale(cx<T> a, T s) { return {a.x * s, a.y * s}; }

// fp32 complex arithmetic on sm_100's packed FP32x2 pipe (FADD2 / FMUL2 /
// FFMA2): one instruction per complex add, two per complex multiply, with
// swaps, sign flips and scalar broadcasts folded into operand modifiers.
// Each lane computes exactly the scalar operations (same IEEE roundings),
// at half the issued instructions.  Enabled per translation unit
// (-DILS_PACKED_F32X2, build.py): the column kernels and the compile-time row
// plans (FFT, stencil and real packing all packed: 1080p fused row pass
// 19.7 M -> 15.2 M warp instructions, +6% frames/s).
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000) && defined(ILS_PACKED_F32X2)
#define ILS_F32X2 1
__device__ __forceinline__ float2 f2_(cx<float> a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ cx<float> c2_(float2 a) { return cx<float>{a.x, a.y}; }
__device__ __forceinline__ cx<float> operator+(cx<float> a, cx<float> b) { return c2_(__fadd2_rn(f2_(a), f2_(b))); }
__device__ __forceinline__ cx<float> operator-(cx<float> a, cx<float> b) {
  return c2_(__fadd2_rn(f2_(a), make_float2(-b.x, -b.y)));
}
// a w = w.x a + w.y (i a)
__device__ __forceinline__ cx<float> cmul(cx<float> a, cx<float> w) {
  const float2 t = __fmul2_rn(f2_(a), make_float2(w.x, w.x));
  return c2_(__ffma2_rn(make_float2(-a.y, a.x), make_float2(w.y, w.y), t));
}
// a conj(w) = w.x a - w.y (i a)
__device__ __forceinline__ cx<float> cmulc(cx<float> a, cx<float> w) {
  const float2 t = __fmul2_rn(f2_(a), make_float2(w.x, w.x));
  return c2_(__ffma2_rn(make_float2(a.y, -a.x), make_float2(w.y, w.y), t));
}
__device__ __forceinline__ cx<float> scale(cx<float> a, float s) { return c2_(__fmul2_rn(f2_(a), make_float2(s, s))); }
// acc + x * s (real s)
__device__ __forceinline__ cx<float> fma_cs(cx<float> x, float s, cx<float> acc) {
  return c2_(__ffma2_rn(f2_(x), make_float2(s, s), f2_(acc)));
}
#else
#define ILS_F32X2 0
#endif
template <typename T>
__host__ __device__ __forceinline__ cx<T> fma_cs(cx<T> x, T s, cx<T> acc) {
  return {acc.x + x.x * s, acc.y + x.y * s};
}

// ------------------------------------------------------------ constexpr trig
constexpr double kPi = 3.141592653589793238462643383279502884;

struct sc_t {
  double s, c;
};

__host__ __device__ constexpr double ct_sin_small(double x) {
  double x2 = x * x, term = x, sum = x;
  for (int n = 1; n < 14; ++n) {
    term *= -x2 / double((2 * n) * (2 * n + 1));
    sum += term;
  }
  return sum;
}
__host__ __device__ constexpr double ct_cos_small(double x) {
  double x2 = x * x, term = 1.0, sum = 1.0;
  for (int n = 1; n < 14; ++n) {
    term *= -x2 / double((2 * n - 1) * (2 * n));
    sum += term;
  }
  return sum;
}
// sin/cos of 2*pi*num/den with exact integer octant reduction (|arg| <= pi/4
// for the series), so table entries are correct to ~1 ulp in double.
__host__ __device__ constexpr sc_t sincos2pi(long long num, long long den) {
  long long m = ((num % den) + den) % den;
  long long q = (4 * m) / den;       // quadrant
  long long r = 4 * m - q * den;     // angle inside quadrant = (pi/2) r / den
  bool swap = 2 * r > den;
  double x = swap ? (kPi / 2) * double(den - r) / double(den) : (kPi / 2) * double(r) / double(den);
  double sx = ct_sin_small(x), cx_ = ct_cos_small(x);
  double s0 = swap ? cx_ : sx, c0 = swap ? sx : cx_;
  sc_t out{0.0, 0.0};
  if (q == 0) out = {s0, c0};
  else if (q == 1) out = {c0, -s0};
  else if (q == 2) out = {-s0, -c0};
  else out = {-c0, s0};
  return out;
}

// ------------------------------------------------------------ static for
template <int... Is, class F>
__device__ __forceinline__ void sfor_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (N > 0) sfor_impl(std::make_integer_sequence<int, N>{}, static_cast<F&&>(f));
}
#define ILS_CV(I) (decltype(I)::value)

// ------------------------------------------------------------ radix helpers
template <int R>
constexpr bool ct_is_prime() {
  if (R < 2) return false;
  for (int d = 2; d * d <= R; ++d)
    if (R % d == 0) return false;
  return true;
}
constexpr int split_of(int r) {
  int best = r;
  if (r % 4 == 0 && r > 4) {
    best = 4;
  } else {
    int p = 2;
    while (p < r && r % p != 0) ++p;
    best = p;
  }
  return best;
}
template <int R>
constexpr int ct_split() {
  return split_of(R);
}

constexpr int gcd_i(int a, int b) { return b == 0 ? a : gcd_i(b, a % b); }
constexpr int modinv_i(int a, int m) {  // a^-1 mod m (gcd(a, m) = 1)
  int r = 1;
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) r = x;
  return r;
}
// Coprime split for the prime-factor (Good-Thomas) algorithm: the power-of-
// two part of r, else the first odd prime power; 0 when r is a prime power.
constexpr int pfa_split(int r) {
  const int p2 = r & -r;
  if (p2 > 1 && p2 < r) return p2;
  for (int p = 3; p <= r; p += 2) {
    if (r % p) continue;
    int a = 1;
    while (r % (a * p) == 0) a *= p;
    return a < r ? a : 0;
  }
  return 0;
}

// Multiply by w = exp(DIR * 2*pi*i * K / R), specialised for quarter turns.
template <int K, int R, int DIR, typename T>
__device__ __forceinline__ cx<T> twc(cx<T> a) {
  constexpr int k = ((K % R) + R) % R;
  if constexpr (k == 0) {
    return a;
  } else if constexpr ((4 * k) % R == 0) {
    constexpr int q = (4 * k) / R;
    constexpr int qq = (DIR > 0) ? q : (4 - q) % 4;
    if constexpr (qq == 1) return cx<T>{-a.y, a.x};
    else if constexpr (qq == 2) return cx<T>{-a.x, -a.y};
    else return cx<T>{a.y, -a.x};
  } else {
    constexpr sc_t w = sincos2pi(DIR * k, R);
    const T c = T(w.c), s = T(w.s);
#if ILS_F32X2
    if constexpr (std::is_same<T, float>::value) {  // c a + s (i a): FMUL2 + FFMA2, immediates
      const float2 t = __fmul2_rn(f2_(a), make_float2(c, c));
      return c2_(__ffma2_rn(make_float2(-a.y, a.x), make_float2(s, s), t));
    }
#endif
    return cx<T>{a.x * c - a.y * s, a.x * s + a.y * c};
  }
}

template <int R, int DIR, typename T>
__device__ __forceinline__ void dft(cx<T>* v);

// Odd prime: symmetric direct form, (R-1)^2/2 real FMAs per component.
template <int R, int DIR, typename T>
__device__ __forceinline__ void dft_prime(cx<T>* v) {
  constexpr int h = (R - 1) / 2;
  cx<T> s[h], d[h];
  sfor<h>([&](auto I) {
    constexpr int n = ILS_CV(I) + 1;
    s[ILS_CV(I)] = v[n] + v[R - n];
    d[ILS_CV(I)] = v[n] - v[R - n];
  });
  const cx<T> x0 = v[0];
  cx<T> X0 = x0;
  sfor<h>([&](auto I) { X0 = X0 + s[ILS_CV(I)]; });
  cx<T> out[R];
  out[0] = X0;
  sfor<h>([&](auto K) {
    constexpr int k = ILS_CV(K) + 1;
    cx<T> a = x0, b{T(0), T(0)};
    sfor<h>([&](auto I) {
      constexpr int n = ILS_CV(I) + 1;
      constexpr sc_t w = sincos2pi((long long)(n * k) % R, R);
      const T c = T(w.c), sn = T(w.s);
      a = fma_cs(s[ILS_CV(I)], c, a);
      b = fma_cs(d[ILS_CV(I)], sn, b);
    });
    const cx<T> ib = (DIR > 0) ? cx<T>{-b.y, b.x} : cx<T>{b.y, -b.x};
    out[k] = a + ib;
    out[R - k] = a - ib;
  });
  sfor<R>([&](auto I) { v[ILS_CV(I)] = out[ILS_CV(I)]; });
}

// Composite: R = A*B, n = B*n1 + n2, k = k1 + A*k2.
template <int R, int DIR, typename T>
__device__ __forceinline__ void dft_ct(cx<T>* v) {
  constexpr int A = ct_split<R>(), B = R / A;
  sfor<B>([&](auto N2) {
    constexpr int n2 = ILS_CV(N2);
    cx<T> t[A];
    sfor<A>([&](auto N1) { t[ILS_CV(N1)] = v[B * ILS_CV(N1) + n2]; });
    dft<A, DIR>(t);
    sfor<A>([&](auto K1) {
      constexpr int k1 = ILS_CV(K1);
      v[B * k1 + n2] = twc<n2 * k1, R, DIR>(t[k1]);
    });
  });
  sfor<A>([&](auto K1) { dft<B, DIR>(v + B * ILS_CV(K1)); });
  cx<T> o[R];
  sfor<A>([&](auto K1) {
    sfor<B>([&](auto K2) { o[ILS_CV(K1) + A * ILS_CV(K2)] = v[B * ILS_CV(K1) + ILS_CV(K2)]; });
  });
  sfor<R>([&](auto I) { v[ILS_CV(I)] = o[ILS_CV(I)]; });
}

// Prime-factor algorithm, R = A*B with gcd(A, B) = 1: no internal twiddles.
// n = (n1 B + n2 A) mod R, k = (k1 B (B^-1 mod A) + k2 A (A^-1 mod B)) mod R.
template <int R, int DIR, typename T>
__device__ __forceinline__ void dft_pfa(cx<T>* v) {
  constexpr int A = pfa_split(R), B = R / A;
  constexpr int Ai = modinv_i(A % B, B), Bi = modinv_i(B % A, A);
  cx<T> y[R];
  sfor<B>([&](auto N2) {
    constexpr int n2 = ILS_CV(N2);
    cx<T> t[A];
    sfor<A>([&](auto N1) { t[ILS_CV(N1)] = v[(ILS_CV(N1) * B + n2 * A) % R]; });
    dft<A, DIR>(t);
    sfor<A>([&](auto K1) { y[ILS_CV(K1) * B + n2] = t[ILS_CV(K1)]; });
  });
  sfor<A>([&](auto K1) { dft<B, DIR>(y + ILS_CV(K1) * B); });
  sfor<A>([&](auto K1) {
    sfor<B>([&](auto K2) {
      v[(ILS_CV(K1) * B * Bi + ILS_CV(K2) * A * Ai) % R] = y[ILS_CV(K1) * B + ILS_CV(K2)];
    });
  });
}

// X[k] = sum_n v[n] exp(DIR * 2*pi*i*n*k/R), unnormalised, in place.
template <int R, int DIR, typename T>
__device__ __forceinline__ void dft(cx<T>* v) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const cx<T> a = v[0], b = v[1];
    v[0] = a + b;
    v[1] = a - b;
  } else if constexpr (R == 4) {
    const cx<T> a0 = v[0] + v[2], a1 = v[0] - v[2], a2 = v[1] + v[3];
    const cx<T> d = v[1] - v[3];
    const cx<T> a3 = (DIR > 0) ? cx<T>{-d.y, d.x} : cx<T>{d.y, -d.x};
    v[0] = a0 + a2;
    v[2] = a0 - a2;
    v[1] = a1 + a3;
    v[3] = a1 - a3;
  } else if constexpr (ct_is_prime<R>()) {
    dft_prime<R, DIR>(v);
  } else if constexpr (pfa_split(R) > 0) {
    dft_pfa<R, DIR>(v);
  } else {
    dft_ct<R, DIR>(v);
  }
}

}  // namespace ils
