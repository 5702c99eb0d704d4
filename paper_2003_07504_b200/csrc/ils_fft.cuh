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
//
// Shared-memory layout: between passes, element e of a line lives at slot
// L(e), either the identity or an XOR swizzle of e's position inside its
// 128-byte block by e's block index (L(e) = e ^ ((e >> SH) & MASK)); the
// host planner simulates the bank traffic of both and picks per plan.  The
// line is identity-laid at both ends of every transform: the first pass
// reads j + r*n/R and the last pass writes j + r*Ns (both unit-stride across
// the group, conflict-free), so whole lines can move with TMA bulk copies
// and vector loads while the interior passes still avoid the stride-R
// conflicts of the first pass's stores.
//
// Twiddles: one table entry w_{Ns R}^m per butterfly class, computed on the
// host in double with exact integer angle reduction; powers in registers.
// Radices 2..16 are unrolled; odd primes 17..61 use a looped direct DFT per
// butterfly, larger primes a direct DFT per output (generic sizes only).
#pragma once

#include "ils_dft.cuh"

namespace ils {

constexpr int kMaxPass = 16;
constexpr int kMaxGenericPrime = 61;

template <typename T>
struct FftDev {
  int n;
  int npass;
  int G;        // threads per line group
  int laykind;  // interior-pass line layout (0 identity, 1/2 XOR swizzles)
  int radix[kMaxPass];
  int tw_off[kMaxPass];   // pass twiddles: unrolled R: Ns entries w^m; generic R: Ns*(R-1), [m][r-1]
  int gen_off[kMaxPass];  // generic primes: R entries w_R^q
  const cx<T>* tw;
};

// complex elements per 128 bytes = 1 << SwzShift<T>
template <typename T>
struct SwzShift {
  static constexpr int value = sizeof(T) == 4 ? 4 : 3;
};
template <typename T>
constexpr int kSwzMask = (1 << SwzShift<T>::value) - 1;

// Line layouts: kind 0 identity, 1 XOR by the 128-byte block index, 2 XOR
// by (block index ^ block index >> 1) -- the latter suits radix-32 first
// passes.  Kind 3 (compile-time two-pass 32 x R plans only) pads one slot
// per 32 elements, L(e) = e + e/32: the radix-32 pass stores 32 j + r at
// 33 j + r and the second pass loads j + 32 r from j + 33 r, so both are
// conflict-free and every address is a per-thread base plus an immediate --
// no XOR index arithmetic at all (the line needs n + n/32 slots).
// LayoutCt: compile-time kind (hot sizes); LayoutRt: runtime (kinds 0-2).
template <typename T, int KIND>
struct LayoutCt {
  __device__ __forceinline__ int operator()(int e) const {
    constexpr int SH = SwzShift<T>::value, M = kSwzMask<T>;
    if constexpr (KIND == 0) return e;
    else if constexpr (KIND == 1) return e ^ ((e >> SH) & M);
    else if constexpr (KIND == 2) return e ^ (((e >> SH) ^ (e >> (SH + 1))) & M);
    else return e + (e >> 5);
  }
};
template <typename T>
struct LayoutRt {
  int kind;
  __device__ __forceinline__ int operator()(int e) const {
    constexpr int SH = SwzShift<T>::value, M = kSwzMask<T>;
    const int s = kind == 1 ? (e >> SH) : (e >> SH) ^ (e >> (SH + 1));
    return kind == 0 ? e : e ^ (s & M);
  }
};

template <typename T>
struct MaxElems {
  static constexpr int value = (sizeof(T) == 4) ? 16 : 8;
};
template <int R, int MAXE>
struct KmOf {
  static constexpr int value = (MAXE / R) > 0 ? (MAXE / R) : 1;
};

// Group of G threads owning one line.  GC > 0 makes the size compile-time.
template <int GC>
struct GroupT {
  static constexpr int kSize = GC;  // compile-time group size (0: runtime)
  int id;     // group index inside the CTA (named barrier id - 1)
  int size_;  // runtime size (GC == 0)
  int rank;   // thread index inside the group
  __device__ __forceinline__ int size() const { return GC > 0 ? GC : size_; }
  __device__ __forceinline__ void sync() const {
    if (size() == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(size()) : "memory");
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

// An optimisation barrier on a value: the compiler must assume it changes
// here, so nothing computed from it can be hoisted above this point.
template <typename T>
__device__ __forceinline__ void opaque(cx<T>& w) {
  if constexpr (sizeof(T) == 4)
    asm volatile("" : "+f"(w.x), "+f"(w.y));
  else
    asm volatile("" : "+d"(w.x), "+d"(w.y));
}

// Twiddle load pinned between the pass barriers (a plain __ldg of read-only
// data may be hoisted above every barrier of the transform).
template <typename T>
__device__ __forceinline__ cx<T> ldtw(const cx<T>* p) {
  cx<T> v;
  if constexpr (sizeof(T) == 4)
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  else
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// ---- asynchronous global -> shared copies (LDGSTS), no register staging
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct LayoutId {
  __device__ __forceinline__ int operator()(int e) const { return e; }
};

// Pointwise map applied to elements as a transform's first pass loads them
// (e.g. the column pass's 1/(H W denom) multiply, fused into the inverse).
struct NoPre {
  template <typename C>
  __device__ __forceinline__ C operator()(int, C v) const {
    return v;
  }
};

template <typename T, int R, int KM, int DIR, class Grp, class LayI, class LayO, class Pre = NoPre>
__device__ __forceinline__ void fft_pass(cx<T>* __restrict__ x, int nb, int Ns, const cx<T>* __restrict__ tw,
                                         const Grp& g, const LayI& lay_in, const LayO& lay_out,
                                         const Pre& pre = Pre{}, const cx<T>* wcache = nullptr) {
  // Idle slots (j >= nb) recompute the last butterfly instead of skipping it:
  // conditionally-defined register arrays become loop-carried live ranges in
  // the caller's line loop and triple the register footprint.
  cx<T> v[KM][R];
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const int j = min(g.rank + k * g.size(), nb - 1);
    // warps whose lanes all fall past the last butterfly skip the work (a
    // warp-uniform branch); the array stays defined so the allocator sees no
    // loop-carried undefined values
    if (((g.rank & ~31) + k * g.size()) >= nb) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[k][r] = cx<T>{T(0), T(0)};
      continue;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) v[k][r] = pre(j + r * nb, x[lay_in(j + r * nb)]);
    if (Ns > 1) {
      // one table load per butterfly: w = w_{Ns R}^(j mod Ns); the powers
      // w^r by running product (<= 15 roundings) for R <= 16, and for larger
      // radices w^(8a+b) = (w^8)^a w^b (two short chains instead of one long).
      // Loading all R-1 powers measured slower (load latency on the critical
      // path of every pass).
      // base twiddle: from the per-thread cache (compile-time plans: it only
      // depends on the thread's rank, so it is loaded once per kernel) or the table
      cx<T> w1 = wcache ? wcache[k] : ldtw(tw + (j % Ns));
#ifndef ILS_TW_HOIST
      // a cached base is the same for every line the thread transforms: left
      // visible, nvcc hoists the whole chain of powers out of the caller's
      // line loop and keeps R-1 complex values per pass live across the
      // kernel -- spilled to local memory at 3840 / 7680 wide (300 bytes per
      // thread, reloaded through L2 in every butterfly).  Recomputing the
      // chain per line is a few FFMA2 per power.
      if (wcache) opaque(w1);
#endif
      if (DIR > 0) w1.y = -w1.y;
      if constexpr (R <= 16) {
        cx<T> w = w1;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          v[k][r] = cmul(v[k][r], w);
          if (r + 1 < R) w = cmul(w, w1);
        }
      } else {
        cx<T> wb[8];
        wb[1] = w1;
#pragma unroll
        for (int b = 2; b < 8; ++b) wb[b] = cmul(wb[b - 1], w1);
        const cx<T> w8 = cmul(wb[4], wb[4]);
        cx<T> wa = w8;
#pragma unroll
        for (int a = 0; a * 8 < R; ++a) {
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const int r = 8 * a + b;
            if (r == 0 || r >= R) continue;
            v[k][r] = cmul(v[k][r], a == 0 ? wb[b] : (b == 0 ? wa : cmul(wa, wb[b])));
          }
          if (a > 0) wa = cmul(wa, w8);
        }
      }
    }
    dft<R, DIR>(v[k]);
  }
  g.sync();
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const int j = g.rank + k * g.size();
    if (j < nb) {
      const int m = j % Ns;
      const int base = (j - m) * R + m;
#pragma unroll
      for (int r = 0; r < R; ++r) x[lay_out(base + r * Ns)] = v[k][r];
    }
  }
  g.sync();
}

// Generic odd prime R (17..61): one butterfly per thread, looped direct DFT.
template <typename T, int DIR, class Grp, class Lay>
__device__ __noinline__ void fft_pass_generic(cx<T>* __restrict__ x, int n, int Ns, int R,
                                              const cx<T>* __restrict__ tw, const cx<T>* __restrict__ wr,
                                              const Grp g, const Lay lay_in, const Lay lay_out) {
  const int nb = n / R;
  cx<T> in[kMaxGenericPrime], out[kMaxGenericPrime];
  const int j = g.rank;
  const bool act = j < nb;  // host guarantees nb <= G
  if (act) {
    const int m = j % Ns;
    for (int r = 0; r < R; ++r) {
      cx<T> a = x[lay_in(j + r * nb)];
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
    for (int r = 0; r < R; ++r) x[lay_out(base + r * Ns)] = out[r];
  }
  g.sync();
}

// Large prime R (> 61, or a 17..61 prime with more butterflies than group
// threads): outputs are spread over the group instead of butterflies, so
// register need is MAXE accumulators whatever R is (the line must satisfy
// n <= MAXE * G).  Output slot o = (j - m) R + m + k Ns of butterfly j
// (m = j mod Ns) is the direct R-point sum over that butterfly's twiddled
// inputs, O(R) per output -- the reference (scipy.fft, solver.py:24-30)
// accepts every length, and these lengths are correctness cases, not hot.
template <typename T, int DIR, int MAXE, class Grp, class Lay>
__device__ __noinline__ void fft_pass_bigprime(cx<T>* __restrict__ x, int n, int Ns, int R,
                                               const cx<T>* __restrict__ tw, const cx<T>* __restrict__ wr,
                                               const Grp g, const Lay lay_in, const Lay lay_out) {
  const int nb = n / R;
  cx<T> acc[MAXE];
#pragma unroll
  for (int i = 0; i < MAXE; ++i) {
    const int o = g.rank + i * g.size();
    acc[i] = cx<T>{T(0), T(0)};
    if (o < n) {
      const int m = o % Ns, q = o / Ns;
      const int k = q % R, j = (q / R) * Ns + m;
      int e = 0;  // r k mod R
      for (int r = 0; r < R; ++r) {
        cx<T> a = x[lay_in(j + r * nb)];
        if (Ns > 1 && r > 0) {
          cx<T> ww = ldg_cx(tw + m * (R - 1) + r - 1);
          if (DIR > 0) ww.y = -ww.y;
          a = cmul(a, ww);
        }
        cx<T> w = ldg_cx(wr + e);
        if (DIR > 0) w.y = -w.y;
        acc[i] = acc[i] + cmul(a, w);
        e += k;
        if (e >= R) e -= R;
      }
    }
  }
  g.sync();
#pragma unroll
  for (int i = 0; i < MAXE; ++i) {
    const int o = g.rank + i * g.size();
    if (o < n) x[lay_out(o)] = acc[i];
  }
  g.sync();
}

// Runtime-planned path (any supported n): each radix pass is its own
// non-inlined function so the register allocator sees one radix at a time
// (inlining all cases into one body blows up live ranges and spills).
template <typename T, int R, int DIR, class Grp, class Lay>
__device__ __noinline__ void fft_pass_rt(cx<T>* __restrict__ x, int nb, int Ns, const cx<T>* __restrict__ tw,
                                         const Grp g, const Lay lay_in, const Lay lay_out) {
  fft_pass<T, R, KmOf<R, MaxElems<T>::value>::value, DIR>(x, nb, Ns, tw, g, lay_in, lay_out);
}

template <typename T, int DIR, class Grp>
__device__ __forceinline__ void fft_line_rt(cx<T>* __restrict__ x, const FftDev<T>& P, const Grp& g) {
  int Ns = 1;
  for (int p = 0; p < P.npass; ++p) {
    const int R = P.radix[p];
    const int nb = P.n / R;
    const cx<T>* tw = P.tw + P.tw_off[p];
    const LayoutRt<T> lay_in{p == 0 ? 0 : P.laykind}, lay_out{p == P.npass - 1 ? 0 : P.laykind};
    switch (R) {
#define ILS_FFT_CASE(RR)                            \
  case RR:                                          \
    fft_pass_rt<T, RR, DIR>(x, nb, Ns, tw, g, lay_in, lay_out); \
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
        if (R <= kMaxGenericPrime && nb <= g.size())
          fft_pass_generic<T, DIR>(x, P.n, Ns, R, tw, P.tw + P.gen_off[p], g, lay_in, lay_out);
        else
          fft_pass_bigprime<T, DIR, MaxElems<T>::value>(x, P.n, Ns, R, tw, P.tw + P.gen_off[p], g, lay_in,
                                                        lay_out);
        break;
    }
    Ns *= R;
  }
}

template <bool FIRST, class Pre>
__device__ __forceinline__ std::conditional_t<FIRST, Pre, NoPre> pick_pre(const Pre& p) {
  if constexpr (FIRST) return p;
  else return NoPre{};
}

// ------------------------------------------------------------ plans as types
// FftRt: runtime plan (FftDev), runtime group size and layout.
// FftCt<SWZ, G, N, radices...>: the hot sizes -- group size, layout, n, Ns
// and every index are compile-time constants.
struct FftRt {
  static constexpr int swz = 0;  // runtime layout (kinds 0-2, FftDev::laykind)
  static constexpr int n = 0;
  static constexpr int G = 0;
  static constexpr int ME = 1;  // no twiddle cache for runtime plans
  static constexpr int npass = 0;
};
// FftRtWide: a runtime plan whose column lines need a 512-thread group
// (H > 4096 fp32 / 2048 fp64 elements at <= MAXE per thread): k_col runs it
// with 512 threads and a 1-CTA/SM register budget
struct FftRtWide : FftRt {};
template <int SWZ, int GG, int ME_, int N, int... Rs>
struct FftCt {
  static constexpr int n = N;
  static constexpr int G = GG;
  static constexpr int ME = ME_;  // register budget: complex elements per thread per pass
  static constexpr int swz = SWZ;
  static constexpr int npass = sizeof...(Rs);
  static_assert((Rs * ... * 1) == N, "radix product must equal N");
};

template <int... Rs>
struct RadixList {
  static constexpr int r[sizeof...(Rs)] = {Rs...};
  static constexpr int ns(int p) {  // product of the radices before pass p
    int v = 1;
    for (int q = 0; q < p; ++q) v *= r[q];
    return v;
  }
};

// Per-thread base twiddles of a compile-time plan: pass p, slot k holds
// w_{Ns R}^(j mod Ns) for j = min(rank + k G, n/R - 1) -- the same for every
// line the thread transforms, so a kernel loads them once (fill_twcache).
template <typename T, class S>
struct TwCache {
  static constexpr int NP = S::npass > 0 ? S::npass : 1;
  static constexpr int KX = S::ME;  // >= KM of every pass
  cx<T> w[NP][KX];
};

template <typename T, int SWZ, int GG, int MEX, int N, int... Rs, class Grp, int... Is>
__device__ __forceinline__ void fill_twcache_impl(TwCache<T, FftCt<SWZ, GG, MEX, N, Rs...>>& c, const FftDev<T>& P,
                                                  const Grp& g, std::integer_sequence<int, Is...>) {
  using RL = RadixList<Rs...>;
  auto one = [&](auto I) {
    constexpr int p = ILS_CV(I);
    constexpr int R = RL::r[p], nb = N / R, Ns = RL::ns(p), KM = KmOf<R, MEX>::value;
    if constexpr (Ns > 1) {
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        const int j = min(g.rank + k * g.size(), nb - 1);
        c.w[p][k] = ldg_cx(P.tw + P.tw_off[p] + (j % Ns));
      }
    }
  };
  (one(std::integral_constant<int, Is>{}), ...);
}

template <typename T, class S, class Grp>
__device__ __forceinline__ void fill_twcache(TwCache<T, S>& c, const FftDev<T>& P, const Grp& g) {
  if constexpr (S::n > 0) fill_twcache_impl(c, P, g, std::make_integer_sequence<int, S::npass>{});
}

template <typename T, int DIR, int SWZ, int GG, int MEX, int N, int... Rs, class Grp, class Pre, int... Is>
__device__ __forceinline__ void fft_line_ct_impl(cx<T>* __restrict__ x, const FftDev<T>& P, const Grp& g,
                                                 const Pre& pre, const TwCache<T, FftCt<SWZ, GG, MEX, N, Rs...>>* tc,
                                                 std::integer_sequence<int, Is...>) {
  constexpr int ME = MEX;
  using RL = RadixList<Rs...>;
  constexpr int NP = sizeof...(Rs);
  using LaySw = LayoutCt<T, SWZ>;
  (fft_pass<T, RL::r[Is], KmOf<RL::r[Is], ME>::value, DIR>(
       x, N / RL::r[Is], RL::ns(Is), P.tw + P.tw_off[Is], g,
       std::conditional_t<Is == 0, LayoutId, LaySw>{}, std::conditional_t<Is == NP - 1, LayoutId, LaySw>{},
       std::conditional_t<Is == 0, Pre, NoPre>(pick_pre<Is == 0>(pre)), tc ? tc->w[Is] : nullptr),
   ...);
}

template <typename T, int DIR, int SWZ, int GG, int MEX, int N, int... Rs, class Grp, class Pre>
__device__ __forceinline__ void fft_line_ct(cx<T>* __restrict__ x, const FftDev<T>& P, const Grp& g, const Pre& pre,
                                            const TwCache<T, FftCt<SWZ, GG, MEX, N, Rs...>>* tc,
                                            FftCt<SWZ, GG, MEX, N, Rs...>) {
  fft_line_ct_impl<T, DIR, SWZ, GG, MEX, N, Rs...>(x, P, g, pre, tc,
                                                   std::make_integer_sequence<int, sizeof...(Rs)>{});
}

// Full transform of one identity-laid line (DIR = -1 forward, +1 inverse,
// unnormalised).  Every thread of the group must call it.
template <typename T, int DIR, class S, class Grp, class Pre = NoPre>
__device__ __forceinline__ void fft_line(cx<T>* __restrict__ x, const FftDev<T>& P, const Grp& g,
                                         const Pre& pre = Pre{}, const TwCache<T, S>* tc = nullptr) {
  if constexpr (S::n == 0) {
    if constexpr (!std::is_same<Pre, NoPre>::value) {  // runtime plans: apply the map as its own sweep
      for (int e = g.rank; e < P.n; e += g.size()) x[e] = pre(e, x[e]);
      g.sync();
    }
    fft_line_rt<T, DIR>(x, P, g);
  } else {
    fft_line_ct<T, DIR>(x, P, g, pre, tc, S{});
  }
}

}  // namespace ils
