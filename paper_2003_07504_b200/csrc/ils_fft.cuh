// Shared-memory mixed-radix Stockham FFT engine (one line per thread group).
//
// Replaces scipy.fft.fft2/ifft2 (reference solver.py:24-30, called at
// solver.py:75 and 127-130).  A group of G threads (G = 32: one warp,
// synchronised with __syncwarp; G > 32: a named barrier) owns one line of
// length n in shared memory and runs every pass on it.  Each pass is a
// radix-R Stockham step:
//
//     v[r] = x[j + r*n/R] * w_{Ns R}^{r (j mod Ns)}      (r = 0..R-1)
//     v    = DFT_R(v)                                    (registers, ils_dft.cuh)
//     x[(j - j mod Ns) R + j mod Ns + r Ns] = v[r]
//
// A thread holds KM = MAXE/R butterflies in registers across the group
// barrier, so the pass runs in place and the output is in natural order.
// Register need depends on n/G only, never on how many lines a CTA holds.
// Element e of a line lives at pad(e) = e + (e >> PADSH): one spare slot per
// 128 bytes, which makes the stride-R stores of early passes conflict-free.
// Twiddles come from a per-pass table [m][r-1] computed on the host in double
// with exact integer angle reduction.  Radices 2..16 are unrolled; odd primes
// 17..61 use a looped direct DFT (generic sizes only).
#pragma once

#include "ils_dft.cuh"

namespace ils {

constexpr int kMaxPass = 16;
constexpr int kMaxGenericPrime = 61;

template <typename T>
struct FftDev {
  int n;
  int npass;
  int G;  // threads per line group
  int radix[kMaxPass];
  int tw_off[kMaxPass];   // pass twiddles: Ns*(R-1) entries, layout [m][r-1]
  int gen_off[kMaxPass];  // generic primes: R entries w_R^q
  const cx<T>* tw;
};

template <typename T>
struct PadOf {
  static constexpr int SH = sizeof(T) == 4 ? 4 : 3;  // 16 x 8 B or 8 x 16 B per 128 B
};
template <typename T>
__host__ __device__ __forceinline__ constexpr int pad(int e) {
  return e + (e >> PadOf<T>::SH);
}
// complex slots a padded line of n elements occupies
template <typename T>
__host__ __device__ constexpr int padded_len(int n) {
  return n > 0 ? pad<T>(n - 1) + 1 : 1;
}

template <typename T>
struct MaxElems {
  static constexpr int value = (sizeof(T) == 4) ? 16 : 8;
};
template <int R, int MAXE>
struct KmOf {
  static constexpr int value = (MAXE / R) > 0 ? (MAXE / R) : 1;
};

struct Group {
  int id;    // group index inside the CTA (named barrier id + 1)
  int size;  // threads in the group (multiple of 32)
  int rank;  // thread index inside the group
  __device__ __forceinline__ void sync() const {
    if (size == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(size) : "memory");
  }
};

template <typename T>
__device__ __forceinline__ cx<T> ldg_cx(const cx<T>* p) {
  if constexpr (sizeof(T) == 4) {
    float2 v = __ldg(reinterpret_cast<const float2*>(p));
    return cx<T>{v.x, v.y};
  } else {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    return cx<T>{v.x, v.y};
  }
}

// Twiddle load pinned between the pass barriers: a plain __ldg of read-only
// data may be hoisted by the compiler above every barrier of the whole
// transform, which keeps all passes' twiddles live at once.
template <typename T>
__device__ __forceinline__ cx<T> ldtw(const cx<T>* p) {
  cx<T> v;
  if constexpr (sizeof(T) == 4)
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  else
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <typename T, int R, int KM, int DIR>
__device__ __forceinline__ void fft_pass(cx<T>* __restrict__ x, int nb, int Ns, const cx<T>* __restrict__ tw,
                                         const Group& g) {
  // Idle slots (j >= nb) recompute the last butterfly instead of skipping it:
  // conditionally-defined register arrays become loop-carried live ranges in
  // the caller's line loop and triple the register footprint.
  cx<T> v[KM][R];
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const int j = min(g.rank + k * g.size, nb - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) v[k][r] = x[pad<T>(j + r * nb)];
    if (Ns > 1) {
      const cx<T>* w = tw + (j % Ns) * (R - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cx<T> ww = ldtw(w + r - 1);
        if (DIR > 0) ww.y = -ww.y;
        v[k][r] = cmul(v[k][r], ww);
      }
    }
    dft<R, DIR>(v[k]);
  }
  g.sync();
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const int j = g.rank + k * g.size;
    if (j < nb) {
      const int m = j % Ns;
      const int base = (j - m) * R + m;
#pragma unroll
      for (int r = 0; r < R; ++r) x[pad<T>(base + r * Ns)] = v[k][r];
    }
  }
  g.sync();
}

// Generic odd prime R (17..61): one butterfly per thread, looped direct DFT.
template <typename T, int DIR>
__device__ __noinline__ void fft_pass_generic(cx<T>* __restrict__ x, int n, int Ns, int R,
                                              const cx<T>* __restrict__ tw, const cx<T>* __restrict__ wr,
                                              const Group& g) {
  const int nb = n / R;
  cx<T> in[kMaxGenericPrime], out[kMaxGenericPrime];
  const int j = g.rank;
  const bool act = j < nb;  // host guarantees nb <= G
  if (act) {
    const int m = j % Ns;
    for (int r = 0; r < R; ++r) {
      cx<T> a = x[pad<T>(j + r * nb)];
      if (Ns > 1 && r > 0) {
        cx<T> ww = ldg_cx(tw + m * (R - 1) + r - 1);
        if (DIR > 0) ww.y = -ww.y;
        a = cmul(a, ww);
      }
      in[r] = a;
    }
    for (int k = 0; k < R; ++k) {
      cx<T> acc{T(0), T(0)};
      int q = 0;
      for (int r = 0; r < R; ++r) {
        cx<T> w = ldg_cx(wr + q);
        if (DIR > 0) w.y = -w.y;
        acc = acc + cmul(in[r], w);
        q += k;
        if (q >= R) q -= R;
      }
      out[k] = acc;
    }
  }
  g.sync();
  if (act) {
    const int m = j % Ns;
    const int base = (j - m) * R + m;
    for (int r = 0; r < R; ++r) x[pad<T>(base + r * Ns)] = out[r];
  }
  g.sync();
}

// Runtime-planned path (any supported n): each radix pass is its own
// non-inlined function so the register allocator sees one radix at a time
// (inlining all cases into one body blows up live ranges and spills).
template <typename T, int R, int DIR>
__device__ __noinline__ void fft_pass_rt(cx<T>* __restrict__ x, int nb, int Ns, const cx<T>* __restrict__ tw,
                                         const Group g) {
  fft_pass<T, R, KmOf<R, MaxElems<T>::value>::value, DIR>(x, nb, Ns, tw, g);
}

// Full n-point transform of one padded line (DIR = -1 forward, +1 inverse,
// unnormalised) from a runtime radix plan.  Every thread of the group must
// call it.
template <typename T, int DIR>
__device__ __forceinline__ void fft_line_rt(cx<T>* __restrict__ x, const FftDev<T>& P, const Group& g) {
  int Ns = 1;
  for (int p = 0; p < P.npass; ++p) {
    const int R = P.radix[p];
    const int nb = P.n / R;
    const cx<T>* tw = P.tw + P.tw_off[p];
    switch (R) {
#define ILS_FFT_CASE(RR)                                                  \
  case RR:                                                                \
    fft_pass_rt<T, RR, DIR>(x, nb, Ns, tw, g);                            \
    break;
      ILS_FFT_CASE(2)
      ILS_FFT_CASE(3)
      ILS_FFT_CASE(4)
      ILS_FFT_CASE(5)
      ILS_FFT_CASE(6)
      ILS_FFT_CASE(7)
      ILS_FFT_CASE(8)
      ILS_FFT_CASE(9)
      ILS_FFT_CASE(10)
      ILS_FFT_CASE(11)
      ILS_FFT_CASE(12)
      ILS_FFT_CASE(13)
      ILS_FFT_CASE(15)
      ILS_FFT_CASE(16)
#undef ILS_FFT_CASE
      default:
        fft_pass_generic<T, DIR>(x, P.n, Ns, R, tw, P.tw + P.gen_off[p], g);
        break;
    }
    Ns *= R;
  }
}

// ------------------------------------------------------------ compile-time plans
// The hot sizes get a compile-time radix list: straight-line passes with n,
// Ns and every index constant-folded.  FftRt selects the runtime path.
struct FftRt {
  static constexpr int n = 0;
};
template <int N, int... Rs>
struct FftCt {
  static constexpr int n = N;
  static constexpr int npass = sizeof...(Rs);
  static_assert((Rs * ... * 1) == N, "radix product must equal N");
};

template <typename T, int DIR, int N, int... Rs>
__device__ __forceinline__ void fft_line_ct(cx<T>* __restrict__ x, const FftDev<T>& P, const Group& g,
                                            FftCt<N, Rs...>) {
  constexpr int ME = MaxElems<T>::value;
  int Ns = 1, p = 0;
  ((fft_pass<T, Rs, KmOf<Rs, ME>::value, DIR>(x, N / Rs, Ns, P.tw + P.tw_off[p], g), Ns *= Rs, ++p), ...);
}

template <typename T, int DIR, class S>
__device__ __forceinline__ void fft_line(cx<T>* __restrict__ x, const FftDev<T>& P, const Group& g) {
  if constexpr (S::n == 0) fft_line_rt<T, DIR>(x, P, g);
  else fft_line_ct<T, DIR>(x, P, g, S{});
}

}  // namespace ils
