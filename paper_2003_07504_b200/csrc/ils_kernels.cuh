// ILS hot-path kernels (sm_100a): the fused row pass and the column pass.
//
// One ILS iteration (reference smoother.py:162-169 -> penalty.py:117-126,
// solver.py:33-49 and solver.py:109-134) is two launches over a half
// spectrum S[B][H][Sp] (complex, row-major, the layout of rfft2):
//
//   k_row  (band of rows + 1 halo row each side):
//          S rows --c2r--> u rows (smem) --stencil--> rhs = f + lam/2 D^T mu
//          --r2c--> S rows          (mu = c*Du - phi'(Du), never materialised)
//   k_col  (strip of columns): forward column FFT, * 1/(H W denom), inverse
//          column FFT, in place.  denom = 1 + c lam/2 (wy[ky] + wx[kx]) is
//          evaluated from two 1-D tables (solver.py:100-102).
//
// Iteration 0 reads f directly (u0 = f); the final row pass (k_row with
// MODE_FIN) writes u.  F(f) is never needed: f is added in the spatial
// domain (linearity), so every iteration moves (S in, f in, S out) + (S in,
// S out) = 20 bytes per pixel for fp32.
#pragma once

#include "ils_fft.cuh"

#include <mutex>
#include <unordered_map>

namespace ils {

enum RowMode : int {
  MODE_F0 = 0,   // u = f                     -> stencil -> r2c -> S
  MODE_IT = 1,   // u = c2r(S_in)             -> stencil -> r2c -> S_out
  MODE_MU = 2,   // rhs = f + lam/2 D^T(mu_x, mu_y) (solve_ls) -> r2c -> S
  MODE_FIN = 3,  // u = c2r(S_in) -> u_out
  MODE_R2C = 4,  // rhs = f -> r2c -> S  (rfft2)
};

enum ColMode : int { COL_SOLVE = 0, COL_FWD = 1, COL_INV = 2 };

constexpr int kStatusClean = 0x7f7f7f7f;  // cudaMemset(0x7f) pattern
constexpr int kMaxBandLines = 32;        // band + 2 halo lines per row CTA (mbarriers)

template <typename T>
struct PenaltyDev {
  int kind;   // 0 Charbonnier, 1 Welsch, 2 soft threshold (HQS field step)
  T p;        // Charbonnier exponent
  T pe;       // p/2 - 1
  T ph;       // p/2
  T eps;
  T wk;       // Welsch: -log2(e) / (2 g^2)   (exp via exp2)
  T g2x2;     // Welsch: 2 g^2
  T c;        // curvature
  T lam;
  T lam2;     // lam / 2
  // branch-free mu = x * max(c + coef * 2^(E * Lg), floor), Lg = log2(x^2 + eps0)
  // (Charbonnier, soft threshold) or x^2 (Welsch): one code path for all
  // three.  floor = -inf for the ILS penalties (c >= c0 keeps the factor
  // >= 0 anyway); 0 for the soft threshold x * max(1 - alpha/|x|, 0).
  T eps0, E, coef, floor;
};

constexpr int kMaxSeg = 8;  // ranks of a slab-decomposed (distributed) transform
constexpr int kMaxPlaneLam = 4;  // planes of a launch with their own lambda

// Spectrum rows split into column segments: the row-pass side of the
// distributed FFT transpose.  Segment q holds columns
// [c0[q], c0[q+1]) of every row at base + off[q] + row * pitch[q], i.e. the
// all-to-all blocks [q][rows][cols_q], so the row pass reads what the
// all-to-all delivered and writes what it sends, with no pack/unpack pass.
// n = 0: plain rows (base + row * S_rp).
struct SegRows {
  int n;
  int c0[kMaxSeg + 1];
  long long off[kMaxSeg];
  int pitch[kMaxSeg];  // even (16-byte rows for bulk copies)
};

template <typename T>
struct RowArgs {
  int mode;  // RowMode
  int wrap;  // 1: rows periodic in [0, H); 0: slab rows, halo rows -1 and H present
  int B, H, W, N, Wc, band, LP;
  const T* f;
  long long f_ps;
  int f_rp;
  const T* mux;
  const T* muy;
  const cx<T>* Sin;
  cx<T>* Sout;
  long long S_ps;
  int S_rp;
  SegRows sin_seg, sout_seg;
  T* u;
  long long u_ps;
  int u_rp;
  PenaltyDev<T> pen;
  int iter;          // iteration index of the u held by this pass
  int* status;       // atomicMin(first bad iteration); 0 = non-finite input
  double* epart;     // energy partials [B][gridDim.x] or nullptr
  FftDev<T> fft;     // row transform (length N = W/2 packed, W otherwise)
  const cx<T>* wreal;  // exp(-2 pi i k / W), k = 0..N/2 (packed only)
  // 8-bit interleaved frames (kernels specialised with SMODE >= kU8Modes):
  // plane b is channel b % ch of frame b / ch in [frames][H][W][ch] bytes.
  // k_u8_planar turns f8 into the planar fcopy (v / 255, formats.py read
  // side) every row pass reads as f; FIN writes u8 = floor(clip01(u) 255 + 0.5)
  // (formats.py:25-27).
  const unsigned char* f8;
  unsigned char* u8;
  int ch;
  T* fcopy;
  // FIN epilogue (applications.py): epi = 1 writes clip01(u + k (f - u))
  // (detail_enhance, :80-93; k = 0 is the clip01 of clipart/texture presets)
  int epi;
  T epi_k;
  // per-plane lambda (tonemap_multi's three scales in one batched launch,
  // applications.py:165-168): nlam > 0 replaces pen.lam2 by lam2_tab[min(b, nlam-1)]
  int nlam;
  T lam2_tab[kMaxPlaneLam];
};

template <typename T>
struct ColArgs {
  int B, H, Wc, C, CS;
  cx<T>* S;
  long long S_ps;
  int S_rp;
  // distributed: scatter the result into per-destination blocks
  // [rows of p plus its two halo rows][ncols] (the reverse all-to-all's send
  // buffer) instead of writing it back in place.  P = 0: in place.
  int P;
  int r0[kMaxSeg + 1];
  long long dst_off[kMaxSeg];
  cx<T>* dst;
  const T* wx;  // 2 - 2 cos(2 pi kx / W), kx < Wc
  const T* wy;  // 2 - 2 cos(2 pi ky / H)
  const cx<T>* tw2;  // exp(-2 pi i m / H), m < H (two-stage column kernel)
  T cl2;        // c * lam / 2
  T inv_hw;     // 1 / (H W)
  int mode;
  FftDev<T> fft;
  int nlam;                   // > 0: plane b uses cl2_tab[min(b, nlam-1)] (see RowArgs::nlam)
  T cl2_tab[kMaxPlaneLam];
  __device__ __forceinline__ T cl2_of(int b) const { return nlam > 0 ? cl2_tab[min(b, nlam - 1)] : cl2; }
};

// ------------------------------------------------------------ penalty math
// fp32 uses the SFU directly (lg2/ex2.approx.ftz: ~2 ulp); fp64 uses libm.
__device__ __forceinline__ float lg2_(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double lg2_(double x) { return log2(x); }
__device__ __forceinline__ double ex2_(double x) { return exp2(x); }

// Explicitly rounded primitives: the compiler never contracts these, so the
// same pixel computes bit-identical mu wherever it sits in a band (placement
// invariance, the multi-GPU / batch-size bitwise-equality contract).
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// mu = c x - phi'(x) (penalty.py:117-126) with phi' from penalty.py:64-66
// (Charbonnier: p x (x^2+eps)^(p/2-1)) or 93-96 (Welsch: 2x exp(-x^2/2g^2)),
// written as x * (c + coef * 2^(E * Lg)).
// SOFT: kernels that may run the soft threshold (kind 2) apply the floor;
// the specialised ILS kernels never see kind 2 (launch_row_impl routes HQS
// plans to the generic kernel) and skip it.
template <bool SOFT, typename T>
__device__ __forceinline__ T aux(T x, const PenaltyDev<T>& P) {
  const T q = fma_rn(x, x, P.eps0);
  const T lg = P.kind != 1 ? lg2_(q) : q;
  const T t = ex2_(mul_rn(P.E, lg));
  T v = fma_rn(P.coef, t, P.c);
  if constexpr (SOFT) v = fmax(v, P.floor);
  return mul_rn(x, v);
}
#if ILS_F32X2
// aux on two columns at once on the packed FP32x2 pipe: each lane performs
// exactly aux<false>'s roundings, so results are bitwise the scalar ones
__device__ __forceinline__ float2 aux2(float2 x, const PenaltyDev<float>& P) {
  const float2 q = __ffma2_rn(x, x, make_float2(P.eps0, P.eps0));
  const float2 lg = P.kind != 1 ? make_float2(lg2_(q.x), lg2_(q.y)) : q;
  const float2 m = __fmul2_rn(make_float2(P.E, P.E), lg);
  const float2 t = make_float2(ex2_(m.x), ex2_(m.y));
  const float2 v = __ffma2_rn(make_float2(P.coef, P.coef), t, make_float2(P.c, P.c));
  return __fmul2_rn(x, v);
}
#endif
// phi(x): penalty.py:60-62, 88-91 (energy trace only)
template <typename T>
__device__ __forceinline__ T phi(T x, const PenaltyDev<T>& P) {
  if (P.kind == 0) return ex2_(P.ph * lg2_(x * x + P.eps));
  return P.g2x2 * (T(1) - ex2_(x * x * P.wk));
}

template <typename T>
__device__ __forceinline__ bool finite_(T v) { return isfinite(v); }

__device__ __forceinline__ float fast_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fast_div(double a, double b) { return a / b; }

// ------------------------------------------------------------ line access
// Line i of a row CTA starts at lines + i*LP (complex slots).  Outside the
// FFT passes lines are identity-laid: in a packed line real sample x is the
// x-th scalar of the line.
template <typename T, bool PACKED>
struct Lines {
  cx<T>* base;
  int LP;
  __device__ __forceinline__ cx<T>* line(int i) const { return base + (size_t)i * LP; }
  __device__ __forceinline__ T get(int i, int x) const {
    if (PACKED) return reinterpret_cast<const T*>(line(i))[x];
    return line(i)[x].x;
  }
  __device__ __forceinline__ void set(int i, int x, T v) const {
    if (PACKED) reinterpret_cast<T*>(line(i))[x] = v;
    else line(i)[x] = cx<T>{v, T(0)};
  }
  // QW consecutive reals from x0 (QW | x0) of a packed line: vector loads
  template <int QW>
  __device__ __forceinline__ void get_strip(int i, int x0, T (&v)[QW]) const {
    const T* z = reinterpret_cast<const T*>(line(i)) + x0;
    if constexpr (sizeof(T) == 4 && QW % 4 == 0) {
#pragma unroll
      for (int q = 0; q < QW; q += 4) {
        const float4 a = *reinterpret_cast<const float4*>(z + q);
        v[q] = a.x;
        v[q + 1] = a.y;
        v[q + 2] = a.z;
        v[q + 3] = a.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < QW; ++q) v[q] = z[q];
    }
  }
  template <int QW>
  __device__ __forceinline__ void set_strip(int i, int x0, const T (&v)[QW]) const {
    T* z = reinterpret_cast<T*>(line(i)) + x0;
    if constexpr (sizeof(T) == 4 && QW % 4 == 0) {
#pragma unroll
      for (int q = 0; q < QW; q += 4)
        *reinterpret_cast<float4*>(z + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < QW; ++q) z[q] = v[q];
    }
  }
};

__device__ __forceinline__ int wrapi(int x, int n) { return x < 0 ? x + n : (x >= n ? x - n : x); }

// Deterministic block sum (fixed shuffle tree + fixed warp order).
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
  }
  __syncthreads();
  return s;
}

// Wait until at most `keep` of this thread's cp.async groups are pending.
__device__ __forceinline__ void cp_async_wait_keep(int keep) {
  switch (keep) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
  }
}

// ------------------------------------------------------------ programmatic dependent launch
// The passes are launched with programmatic stream serialisation: each CTA
// lets the next pass launch as soon as it is resident (every CTA of this
// grid has started), the next pass stages its constant tables / twiddle
// cache, then waits for this grid's completion (and memory flush) before it
// touches the data this pass produces.  Both are no-ops in a normal launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------ TMA bulk copies
// 1-D bulk copies (cp.async.bulk, SASS UBLKCP) of whole rows between global
// memory and shared memory, completion tracked by an mbarrier (loads) or a
// bulk group (stores).  16-byte aligned addresses, sizes multiple of 16.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, whole 16-byte units)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// L2 eviction policies for bulk copies: data that is dead after this use
// (the spectrum a row pass consumes, the output u) is marked evict-first so it
// does not push the frame's live working set (f, the next spectrum) out of L2
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, unsigned bytes, unsigned long long policy) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(policy)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> async proxy
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_reads() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ------------------------------------------------------------ real <-> half-complex packing
// Packing twiddles w^k = exp(-2 pi i k / W) for the loops below, which visit
// k = rank + size * m:
//   TwTab<SMEM>  the host table, staged in shared memory (SMEM) or read
//                through L1 from global memory
//   TwSplit      w^rank (a register, loaded once) * w^(32 m) (a 16-entry
//                shared table): the 32-thread-group plans whose padded line
//                layout leaves no room for the full table; one complex
//                multiply (about 2 ulp) instead of an L2 load per twiddle
template <bool SMEM, typename T>
__device__ __forceinline__ cx<T> ldw(const cx<T>* w, int k) {
  if constexpr (SMEM) return w[k];
  else return ldg_cx(w + k);
}
template <typename T, bool SMEM>
struct TwTab {
  const cx<T>* w;
  __device__ __forceinline__ cx<T> operator()(int k, int) const { return ldw<SMEM>(w, k); }
};
template <typename T>
struct TwSplit {
  cx<T> lo;         // w^rank
  const cx<T>* hi;  // hi[m] = w^(32 m), shared memory
  __device__ __forceinline__ cx<T> operator()(int, int m) const { return cmul(lo, hi[m]); }
};
constexpr int kTwSplitMax = 32;  // entries of the w^(32 m) table (N/2 < 32 * 32)

// Forward post-process of one packed line: Z = FFT_N(x[2n] + i x[2n+1]) ->
// X[k] = E + w^k O, X[N-k] = conj(E - w^k O), E = (Z_k + conj Z_{N-k})/2,
// O = -i (Z_k - conj Z_{N-k})/2, w = exp(-2 pi i/W).  X[N] goes to element N.
// (complex operations: the packed FP32x2 forms in fp32 translation units)
// (compile-time plans: N and the group size are constants and the loop
// unrolls, the k == 0 / k == N/2 cases folded -- 1080p IT pass 30.7 -> 29.5 us,
// 3840-wide IT 172 -> 158 us, 7680-wide IT 695 -> 652 us)

template <typename T, class TW, class Grp>
__device__ __forceinline__ void r2c_post(cx<T>* z, int N, const TW& tw, const Grp& g) {
  const int M = (N / 2) / g.size() + 1;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int k = g.rank + m * g.size();
    if (k > N / 2) break;
    if (k == 0) {
      const cx<T> z0 = z[0];
      z[0] = cx<T>{z0.x + z0.y, T(0)};
      z[N] = cx<T>{z0.x - z0.y, T(0)};
    } else {
      const cx<T> zk = z[k], zm = z[N - k];
      const cx<T> E = scale(zk + conj(zm), T(0.5));
      const cx<T> d = scale(zk - conj(zm), T(0.5));  // (zk - conj zm)/2
      const cx<T> O{d.y, -d.x};                      // -i * d
      const cx<T> wO = cmul(tw(k, m), O);
      z[k] = E + wO;
      if (N - k != k) z[N - k] = conj(E - wO);
    }
  }
  g.sync();
}

// Inverse pre-process: Z_k = E + iO, Z_{N-k} = conj(E) + i conj(O) with
// E = X_k + conj X_{N-k}, O = (X_k - conj X_{N-k}) conj(w^k).  An inverse
// N-point FFT of Z then yields W * (x[2n] + i x[2n+1]) of the c2r of X/W.
template <typename T, class TW, class Grp>
__device__ __forceinline__ void c2r_pre(cx<T>* z, int N, const TW& tw, const Grp& g) {
  const int M = (N / 2) / g.size() + 1;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int k = g.rank + m * g.size();
    if (k > N / 2) break;
    if (k == 0) {
      const T a = z[0].x, c = z[N].x;  // DC / Nyquist: imaginary parts ignored (as irfft)
      z[0] = cx<T>{a + c, a - c};
    } else {
      const cx<T> xk = z[k], xm = z[N - k];
      const cx<T> E = xk + conj(xm);
      const cx<T> D = xk - conj(xm);
      const cx<T> O = cmulc(D, tw(k, m));
      z[k] = E + cx<T>{-O.y, O.x};
      if (N - k != k) z[N - k] = conj(E) + cx<T>{O.y, O.x};
    }
  }
  g.sync();
}

// ------------------------------------------------------------ row pass
template <typename T>
struct AddPair {  // element e of a packed line += (f[2e], f[2e+1])
  const cx<T>* f;
  __device__ __forceinline__ cx<T> operator()(int e, cx<T> v) const { return v + ldg_cx(f + e); }
};

constexpr int kRowThreads = 256;
// threads per row CTA of a compile-time plan (the 960-point line plan of
// 1920-wide rows is a tuning point: ILS_ROW_THREADS_960)
#ifndef ILS_ROW_THREADS_960
#define ILS_ROW_THREADS_960 256
#endif
template <class FS>
constexpr int kRowThreadsOf = FS::n == 960 ? ILS_ROW_THREADS_960 : kRowThreads;
constexpr int kColThreads = 256;
constexpr int kColMinBlocks = 3;  // k_col register budget: 3 CTAs / SM
constexpr int kNarrowMaxW = 4 * 4 * kRowThreads;  // stencil: 4 strips x 4 columns per thread
constexpr int kWideMaxW = 4 * 8 * kRowThreads;

// Whole-row TMA bulk copies need 16-byte granularity: compile-time plans of
// widths W = 2n with W % 8 == 0 (f / u rows of W*4 bytes, spectrum rows of
// round16((n+1)*8) bytes inside 32-byte aligned, 4-element padded rows).
template <typename T, class FS>
constexpr bool kBulkRows = sizeof(T) == 4 && FS::n > 0 && (2 * FS::n) % 8 == 0;

// SMODE >= 0: kernel specialised for that mode without trace (the hot
// kernels; dead phases compiled out keeps the code inside the I-cache);
// SMODE = -1: any mode from A.mode, optional energy trace.
// Register budget: compile-time plans budget for 3 resident CTAs per SM (80 for
// the 32 x 30 plan, no spills): with a band of 6 the row pass then leaves
// room on every SM for the other lane's column-pass CTAs, which is worth more
// than the band-12 CTA's lower halo overhead (4993 -> 5859 frames/s);
// runtime plans for 2
#ifndef ILS_ROW_MINB  // (tuning override: resident row CTAs per SM the registers are budgeted for)
// (the 1920- and 3840-point line plans -- 3840 / 7680-wide rows -- fit one
// CTA per SM in shared memory, so they get the whole register file: at 80
// registers the 7680-wide pass spilled 1.1 KB per thread, IT 1285 -> 751 us,
// and the 3840-wide final pass 136 bytes, 75 -> 57 us)
template <class FS>
constexpr int kRowBlocksOf = FS::n > 0 ? (FS::n >= 1920 ? 1 : 3) : 2;
#else
template <class FS>
constexpr int kRowBlocksOf = ILS_ROW_MINB;
#endif

// u8 value -> T exactly as the reference's v / 255.0 rounded to T
// (correctly rounded division; equal to float(double(v) / 255) for all 256 v)
// one Newton correction of v * (1/255): equal to the correctly rounded
// v / 255 for all 256 inputs (checked exhaustively), 3 FP instructions
// instead of a full-precision division
__device__ __forceinline__ float u8_to(unsigned v, float) {
  const float x = float(v), r = 1.0f / 255.0f;
  const float q = __fmul_rn(x, r);
  return __fmaf_rn(__fmaf_rn(-q, 255.0f, x), r, q);
}
__device__ __forceinline__ double u8_to(unsigned v, double) { return double(v) / 255.0; }
// formats.py:25-27: floor(clip01(u) * 255 + 0.5) with the reference's two roundings
__device__ __forceinline__ unsigned char quant8(float v) {
  const float c = fminf(fmaxf(v, 0.f), 1.f);
  return (unsigned char)floorf(__fadd_rn(__fmul_rn(c, 255.f), 0.5f));
}
__device__ __forceinline__ unsigned char quant8(double v) {
  const double c = fmin(fmax(v, 0.0), 1.0);
  return (unsigned char)floor(__dadd_rn(__dmul_rn(c, 255.0), 0.5));
}

// applications.py:80-93 / image.clip01: clip01(u + k (f - u)) with the
// reference's roundings (no contraction); k = 0 is clip01(u).
template <typename T>
__device__ __forceinline__ T detail_epilogue(T u, T f, T k) {
  T v = u;
  if (k != T(0)) v = v + mul_rn(k, f - u);
  return fmin(fmax(v, T(0)), T(1));
}

constexpr int kU8Modes = 8;
// stencil rows per barrier (rhs of that many rows held in registers)
#ifndef ILS_STENCIL_ROWS
#define ILS_STENCIL_ROWS 3
#endif
constexpr int kStencilRows = ILS_STENCIL_ROWS;  // SMODE = kU8Modes + MODE_FIN: 8-bit frame egress

// resident CTAs per SM the registers are budgeted for, per pass kind
#ifndef ILS_FIN_MINB  // (the 3840 / 7680-wide final pass: 2 CTAs per SM, 114-127 registers, no spills)
#define ILS_FIN_MINB 2
#endif
template <class FS, int SMODE>
constexpr int kRowBlocksOfMode =
    (FS::n >= 1920 && (SMODE == MODE_FIN || SMODE == kU8Modes + MODE_FIN)) ? ILS_FIN_MINB : kRowBlocksOf<FS>;

template <typename T, bool PACKED, class FS, bool WIDE, int SMODE>
#ifdef ILS_ROW_MAXREG  // (tuning override: explicit register cap for the row kernels)
__global__ void __maxnreg__(ILS_ROW_MAXREG) k_row(const RowArgs<T> A) {
#else
__global__ void __launch_bounds__(kRowThreadsOf<FS>, kRowBlocksOfMode<FS, SMODE>) k_row(const RowArgs<T> A) {
#endif
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ unsigned long long bars[kMaxBandLines];
  using Grp = GroupT<FS::G>;
  constexpr bool BULK = kBulkRows<T, FS> && PACKED;
  constexpr bool U8 = SMODE >= kU8Modes;
  constexpr bool BULKIN = BULK;
  // specialised fp32 final pass (no trace, no 8-bit egress): each line group
  // checks and stores its own row as soon as its transform is done
  constexpr bool FINLINE8 = SMODE == kU8Modes + MODE_FIN && BULK && sizeof(T) == 4;  // same, 8-bit egress
  // 8-bit ingest fused into the first pass: each line's interleaved byte row
  // arrives by TMA in the tail of its line slot and is widened in place
  constexpr bool INGEST8 = SMODE == kU8Modes + MODE_F0 && BULK && sizeof(T) == 4;
  constexpr bool FINLINE = (SMODE == MODE_FIN && BULK && sizeof(T) == 4) || FINLINE8;
  constexpr bool SOFTOK = SMODE < 0 || U8;  // kernels that accept the soft-threshold penalty
  const int MODE = U8 ? SMODE - kU8Modes : (SMODE >= 0 ? SMODE : A.mode);  // block-uniform
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int G = FS::G > 0 ? FS::G : A.fft.G;
  const Grp g{tid / G, G, tid % G};
  const int ngroups = nthr / G;
  const int b = blockIdx.y;
  const int r0 = blockIdx.x * A.band;
  const int nb = min(A.band, A.H - r0);
  // compile-time plans fix the width (W = 2n packed): every strip bound and
  // wrap in the stencil folds, so its per-element guards compile away
  constexpr int WCT = (FS::n > 0 && PACKED) ? 2 * FS::n : 0;
  const int W = WCT > 0 ? WCT : A.W, H = A.H;
  const bool trace = SMODE < 0 && A.epart != nullptr;
  const bool halo = (MODE == MODE_F0 || MODE == MODE_IT || (MODE == MODE_FIN && trace));
  const int nl = halo ? nb + 2 : nb;
  const int y0 = halo ? r0 - 1 : r0;
  const int off = halo ? 1 : 0;
  const Lines<T, PACKED> L{reinterpret_cast<cx<T>*>(smem_raw), A.LP};
  const PenaltyDev<T>& P = A.pen;
  const T lam2 = A.nlam > 0 ? A.lam2_tab[min(b, A.nlam - 1)] : P.lam2;  // block-uniform
  const T* fpl = A.f ? A.f + (size_t)b * A.f_ps : nullptr;
  // real-packing twiddles staged in shared memory after the band's lines
#ifndef ILS_WREAL_SMEM  // kind-3 plans read the packing twiddles from global memory through L1
  constexpr bool WSMEM = FS::swz != 3;
#else  // (tuning: a shared-memory table for every plan -- faster passes alone, but the
       // 4 KB larger row CTAs co-reside worse with the column pass: bench 5879 -> 5353)
  constexpr bool WSMEM = true;
#endif
  // (after the band's line slots: band + 2 with halo rows, band without --
  // the final pass runs a band 2 rows taller in the same shared memory)
  cx<T>* swreal = WSMEM ? reinterpret_cast<cx<T>*>(smem_raw) + (size_t)(A.band + (halo ? 2 : 0)) * A.LP
                        : const_cast<cx<T>*>(A.wreal);
  // kind-3 plans without the table in shared memory: split twiddles
  constexpr bool WSPLIT = !WSMEM && FS::G == 32 && FS::n / 2 / 32 < kTwSplitMax;
  __shared__ cx<T> s_whi[WSPLIT ? kTwSplitMax : 1];
  // the packing twiddles by one bulk copy (whole 16-byte pairs; the host
  // sizes the region so), waited for after the PDL wait
  __shared__ unsigned long long wbar;
  if (PACKED && WSMEM) {
    if (tid == 0) {
      const unsigned wb = (unsigned)(((A.N / 2 + 2) & ~1) * sizeof(cx<T>));
      mbar_init(&wbar, 1);
      mbar_fence_init();
      mbar_expect_tx(&wbar, wb);
      bulk_g2s(swreal, A.wreal, wb, &wbar);
    }
    __syncthreads();  // publishes wbar's initialisation
  }
  if (PACKED && WSPLIT) {
    if (tid * 32 <= A.N / 2) s_whi[tid] = A.wreal[32 * tid];
    __syncthreads();
  }
  const int NPK = (FS::n > 0 && PACKED) ? FS::n : A.N;  // packed line length (compile-time for specs)
  using TwT = std::conditional_t<WSPLIT, TwSplit<T>, TwTab<T, WSMEM>>;
  TwT twp;
  if constexpr (WSPLIT) twp = TwSplit<T>{ldg_cx(A.wreal + (tid % 32)), s_whi};
  else twp = TwTab<T, WSMEM>{swreal};
  TwCache<T, FS> twc;
  fill_twcache(twc, A.fft, g);
  const unsigned spec_bytes = (unsigned)((A.Wc * sizeof(cx<T>) + 15) & ~size_t(15));
#ifndef ILS_PDL_LATE
  pdl_trigger();
#endif
  if (MODE == MODE_IT && tid < nb && (W * sizeof(T)) % 16 == 0 && (A.f_rp * sizeof(T)) % 16 == 0) {
    // the stencil reads f one row at a time: pull the band's rows into L2 now
    // (f is the call's input, written before the first pass: no need to wait
    // for the previous pass before the prefetch)
    const T* row = fpl + (size_t)(r0 + tid) * A.f_rp;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"((unsigned)(W * sizeof(T))) : "memory");
  }
  pdl_wait();  // the previous pass's spectrum / the caller's f from here on
  if (PACKED && WSMEM) mbar_wait(&wbar, 0);

  if (MODE == MODE_MU || MODE == MODE_R2C) {
    // rhs rows straight from global memory; each group owns whole lines.
    bool bf = false, bx = false, by = false;
    const T* mx = A.mux ? A.mux + (size_t)b * A.f_ps : nullptr;
    const T* my = A.muy ? A.muy + (size_t)b * A.f_ps : nullptr;
    for (int i = g.id; i < nb; i += ngroups) {
      const int r = r0 + i;
      for (int x = g.rank; x < W; x += g.size()) {
        const size_t o = (size_t)r * A.f_rp + x;
        T v = fpl[o];
        bf |= !finite_(v);
        if (MODE == MODE_MU) {
          // rhs = f + lam/2 (mu_x[r,x-1] - mu_x[r,x] + mu_y[r-1,x] - mu_y[r,x]): solver.py:43-49, 127-129
          const T mxc = mx[o], myc = my[o];
          const T mxl = mx[(size_t)r * A.f_rp + wrapi(x - 1, W)];
          const T myu = my[(size_t)wrapi(r - 1, H) * A.f_rp + x];
          bx |= !finite_(mxc);
          by |= !finite_(myc);
          v = v + lam2 * ((mxl - mxc) + (myu - myc));
        }
        L.set(i, x, v);
      }
    }
    if (MODE == MODE_MU) {
      // solve_ls checks f, mu_x, mu_y in that order (solver.py:119-125)
      const int fb = __syncthreads_or(bf), xb = __syncthreads_or(bx), yb = __syncthreads_or(by);
      if (tid == 0) {
        if (fb) atomicMin(A.status, 1);
        if (xb) atomicMin(A.status, 2);
        if (yb) atomicMin(A.status, 3);
      }
    } else {
      __syncthreads();
    }
  } else {
    // ---------------- phase A: u rows into shared memory (group per line)
    // Rows arrive asynchronously: one TMA bulk copy per row (compile-time
    // plans) or per-element cp.async (runtime plans), issued for every line
    // up front; each group then transforms its lines while later ones land.
    const int mine = (nl - g.id + ngroups - 1) / ngroups;  // lines owned by this group
    if constexpr (BULKIN) {
      // thread i arms line i's barrier and issues its copy (parallel issue)
      if (tid < nl) {
        mbar_init(&bars[tid], 1);
        mbar_fence_init();
        {
          const int i = tid;
          const int y = A.wrap ? wrapi(y0 + i, H) : y0 + i;
          if (INGEST8) {
            const unsigned bytes = (unsigned)(W * A.ch);
            const unsigned char* src = A.f8 + ((size_t)(b / A.ch) * H + y) * (size_t)W * A.ch;
            unsigned char* dst = reinterpret_cast<unsigned char*>(L.line(i)) + (size_t)A.LP * sizeof(cx<T>) - bytes;
            mbar_expect_tx(&bars[i], bytes);
            bulk_g2s(dst, src, bytes, &bars[i]);
          } else if (MODE == MODE_F0) {
            const unsigned bytes = (unsigned)(W * sizeof(T));
            mbar_expect_tx(&bars[i], bytes);
            bulk_g2s(L.line(i), fpl + (size_t)y * A.f_rp, bytes, &bars[i]);
          } else if (A.sin_seg.n == 0) {
            mbar_expect_tx(&bars[i], spec_bytes);
            bulk_g2s_hint(L.line(i), A.Sin + (size_t)b * A.S_ps + (size_t)y * A.S_rp, spec_bytes, &bars[i],
                          l2_evict_first());
          } else {
            const SegRows& sg = A.sin_seg;
            unsigned total = 0;
            for (int q = 0; q < sg.n; ++q) total += (unsigned)(((sg.c0[q + 1] - sg.c0[q] + 1) & ~1) * sizeof(cx<T>));
            mbar_expect_tx(&bars[i], total);
            for (int q = 0; q < sg.n; ++q)
              bulk_g2s(L.line(i) + sg.c0[q], A.Sin + (size_t)b * A.S_ps + sg.off[q] + (long long)y * sg.pitch[q],
                       (unsigned)(((sg.c0[q + 1] - sg.c0[q] + 1) & ~1) * sizeof(cx<T>)), &bars[i]);
          }
        }
      }
      __syncthreads();
    } else if (MODE != MODE_F0 || PACKED) {
      for (int i = g.id; i < nl; i += ngroups) {
        const int y = A.wrap ? wrapi(y0 + i, H) : y0 + i;
        cx<T>* z = L.line(i);
        if (MODE == MODE_F0) {
          const cx<T>* src = reinterpret_cast<const cx<T>*>(fpl + (size_t)y * A.f_rp);
          for (int q = g.rank; q < W / 2; q += g.size()) cp_async<sizeof(cx<T>)>(z + q, src + q);
        } else if (A.sin_seg.n == 0) {
          const cx<T>* src = A.Sin + (size_t)b * A.S_ps + (size_t)y * A.S_rp;
          for (int k = g.rank; k < A.Wc; k += g.size()) cp_async<sizeof(cx<T>)>(z + k, src + k);
        } else {
          const SegRows& sg = A.sin_seg;
          for (int q = 0; q < sg.n; ++q) {
            const cx<T>* src = A.Sin + (size_t)b * A.S_ps + sg.off[q] + (long long)y * sg.pitch[q] - sg.c0[q];
            for (int k = sg.c0[q] + g.rank; k < sg.c0[q + 1]; k += g.size()) cp_async<sizeof(cx<T>)>(z + k, src + k);
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    }
    bool bad = false;
    T chkf = T(0);  // FINLINE finiteness accumulator
    int li = 0;
    for (int i = g.id; i < nl; i += ngroups, ++li) {
      const int y = A.wrap ? wrapi(y0 + i, H) : y0 + i;
      cx<T>* z = L.line(i);
      if constexpr (BULKIN) {
        mbar_wait(&bars[i], 0);
      } else if (MODE != MODE_F0 || PACKED) {
        cp_async_wait_keep(mine - 1 - li);
        g.sync();
      }
      if constexpr (INGEST8) {
        // widen channel b % C of the byte row (3 bytes per pixel, 4 pixels per
        // lane and round) to v / 255 floats at the front of the slot, and
        // write the band's own rows to the planar f the later passes add.
        // Rounds go front to back: round k's float stores end below round
        // k+1's byte loads (the host only fuses when the slot's byte tail
        // starts at >= W bytes), so one warp barrier per round suffices.
        const int C = A.ch, c = b % C;
        const unsigned char* src8 =
            reinterpret_cast<const unsigned char*>(z) + (size_t)A.LP * sizeof(cx<T>) - (size_t)W * C;
        float* zf = reinterpret_cast<float*>(z);
        T* fc = (i >= 1 && i <= nb) ? A.fcopy + (size_t)b * A.f_ps + (size_t)(y0 + i) * A.f_rp : nullptr;
        for (int q0 = 0; q0 < W / 4; q0 += g.size()) {
          const int q = q0 + g.rank;
          unsigned wd[3] = {0u, 0u, 0u};
          if (q < W / 4) {
            const unsigned* w = reinterpret_cast<const unsigned*>(src8 + 12 * q);
            wd[0] = w[0];
            wd[1] = w[1];
            wd[2] = w[2];
          }
          g.sync();
          if (q < W / 4) {
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int pos = 3 * k + c;  // byte of pixel k, channel c (C == 3)
              v[k] = u8_to((wd[pos >> 2] >> (8 * (pos & 3))) & 0xffu, T{});
            }
            const float4 o = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4*>(zf + 4 * q) = o;
            if (fc) *reinterpret_cast<float4*>(fc + 4 * q) = o;
          }
        }
      } else if (MODE == MODE_F0) {
        if (!PACKED)
          for (int x = g.rank; x < W; x += g.size()) L.set(i, x, fpl[(size_t)y * A.f_rp + x]);
      } else {
        if (PACKED) {
          c2r_pre<T>(z, NPK, twp, g);
        } else {
          // Hermitian completion X[W-k] = conj X[k]; DC imaginary part dropped
          for (int k = A.Wc + g.rank; k < W; k += g.size()) z[k] = conj(z[W - k]);
          if (g.rank == 0) z[0].y = T(0);
          g.sync();
        }
        fft_line<T, +1, FS>(z, A.fft, g, NoPre{}, &twc);
        if constexpr (FINLINE) {
          // the group finishes its own row: finiteness (smoother.py:166-167),
          // the optional detail/clip epilogue, and its bulk store -- no block
          // barrier between the transforms and the stores
          T* zr = reinterpret_cast<T*>(z);
          if constexpr (FINLINE8) {
            // quantised bytes straight to channel ch of the interleaved frame row
            const int C = A.ch;
            unsigned char* row = A.u8 + ((size_t)(b / C) * H + (r0 + i)) * (size_t)W * C + (b % C);
            for (int x = 4 * g.rank; x < W; x += 4 * g.size()) {
              const float4 q = *reinterpret_cast<const float4*>(zr + x);
              chkf = fma_rn(q.x, T(0), chkf);
              chkf = fma_rn(q.y, T(0), chkf);
              chkf = fma_rn(q.z, T(0), chkf);
              chkf = fma_rn(q.w, T(0), chkf);
              row[(size_t)x * C] = quant8(q.x);
              row[(size_t)(x + 1) * C] = quant8(q.y);
              row[(size_t)(x + 2) * C] = quant8(q.z);
              row[(size_t)(x + 3) * C] = quant8(q.w);
            }
            continue;
          }
          const T* fr = fpl ? fpl + (size_t)(r0 + i) * A.f_rp : nullptr;
          for (int x = 4 * g.rank; x < W; x += 4 * g.size()) {
            float4 q = *reinterpret_cast<const float4*>(zr + x);
            chkf = fma_rn(q.x, T(0), chkf);
            chkf = fma_rn(q.y, T(0), chkf);
            chkf = fma_rn(q.z, T(0), chkf);
            chkf = fma_rn(q.w, T(0), chkf);
            if (A.epi) {
              const bool kf = A.epi_k != T(0);
              q.x = detail_epilogue(q.x, kf ? fr[x] : T(0), A.epi_k);
              q.y = detail_epilogue(q.y, kf ? fr[x + 1] : T(0), A.epi_k);
              q.z = detail_epilogue(q.z, kf ? fr[x + 2] : T(0), A.epi_k);
              q.w = detail_epilogue(q.w, kf ? fr[x + 3] : T(0), A.epi_k);
              *reinterpret_cast<float4*>(zr + x) = q;
            }
          }
          g.sync();
          if (g.rank == 0)
            bulk_s2g_hint(A.u + (size_t)b * A.u_ps + (size_t)(r0 + i) * A.u_rp, z, (unsigned)(W * sizeof(T)),
                          l2_evict_first());
        }
      }
    }
    if constexpr (FINLINE) {
      bad = !finite_(chkf);
      if (__syncthreads_or(bad) && tid == 0) atomicMin(A.status, A.iter);
      bulk_wait_reads();
      return;
    }
    __syncthreads();

    // ---------------- final pass: write u (and its energy)
    if (MODE == MODE_FIN) {
      if constexpr (U8) {
        // 8-bit egress: quantised, interleaved into channel ch of the frame
        const int C = A.ch;
        unsigned char* dst = A.u8 + (size_t)(b / C) * H * W * C + (b % C);
        T chk = T(0);
        for (int j = 0; j < nb; ++j) {
          unsigned char* row = dst + (size_t)(r0 + j) * W * C;
          for (int x = tid; x < W; x += nthr) {
            const T v = L.get(j + off, x);
            chk = fma_rn(v, T(0), chk);
            row[(size_t)x * C] = quant8(v);
          }
        }
        bad = !finite_(chk);
        if (__syncthreads_or(bad) && tid == 0) atomicMin(A.status, A.iter);
        return;
      }
      double e = 0.0;
      T* upl = A.u + (size_t)b * A.u_ps;
      if (PACKED && !trace) {
        // finiteness (smoother.py:166-167): fma(x, 0, c) is NaN iff some x is not finite
        T chk = T(0);
        for (int j = 0; j < nb; ++j) {
          T* z = reinterpret_cast<T*>(L.line(j + off));
          const T* fr = fpl ? fpl + (size_t)(r0 + j) * A.f_rp : nullptr;
          for (int x = tid; x < W; x += nthr) {
            chk = fma_rn(z[x], T(0), chk);
            if (A.epi) z[x] = detail_epilogue(z[x], A.epi_k != T(0) ? fr[x] : T(0), A.epi_k);
          }
        }
        if constexpr (BULK) {
          __syncthreads();
          if (tid < nb)
            bulk_s2g_hint(upl + (size_t)(r0 + tid) * A.u_rp, L.line(tid + off), (unsigned)(W * sizeof(T)),
                          l2_evict_first());
        } else {
          const int np = W / 2;
          if (A.epi) __syncthreads();  // pairs below span other threads' epilogue elements
          for (int j = 0; j < nb; ++j) {
            cx<T>* dst = reinterpret_cast<cx<T>*>(upl + (size_t)(r0 + j) * A.u_rp);
            const cx<T>* z = L.line(j + off);
            for (int q = tid; q < np; q += nthr) dst[q] = z[q];
          }
        }
        bad = !finite_(chk);
        if (__syncthreads_or(bad) && tid == 0) atomicMin(A.status, A.iter);
        if constexpr (BULK) bulk_wait_reads();
        return;
      }
      for (int t = tid; t < nb * W; t += nthr) {
        const int j = t / W, x = t - j * W;
        const T uc = L.get(j + off, x);
        bad |= !finite_(uc);
        upl[(size_t)(r0 + j) * A.u_rp + x] =
            A.epi ? detail_epilogue(uc, A.epi_k != T(0) ? fpl[(size_t)(r0 + j) * A.f_rp + x] : T(0), A.epi_k) : uc;
        if (trace) {
          const T gx = L.get(j + off, wrapi(x + 1, W)) - uc;
          const T gy = L.get(j + off + 1, x) - uc;
          const T d = uc - fpl[(size_t)(r0 + j) * A.f_rp + x];
          e += double(d) * double(d) + double(P.lam) * (double(phi(gx, P)) + double(phi(gy, P)));
        }
      }
      if (__syncthreads_or(bad) && tid == 0) atomicMin(A.status, A.iter);
      if (trace) {
        const double s = block_sum(e, red);
        if (tid == 0) A.epart[(size_t)b * gridDim.x + blockIdx.x] = s;
      }
      return;
    }

    // ---------------- phase B: fused stencil -> rhs rows (lines 0..nb-1)
    // Each thread walks down a QW-column strip carrying mu_y of the row above
    // in registers.  Line j+1 holds row r0+j; rhs of row r0+j is written into
    // line j once every thread is past row r0+j-1.  f of the next row is
    // prefetched into registers one row ahead.
    constexpr int QW = WIDE ? 8 : 4;
    // every strip is whole when the compile-time width is a multiple of QW
    constexpr bool ALLFULL = WCT > 0 && WCT % QW == 0;
    // strips per thread: exact for compile-time plans, 4 (W <= 16 * 256) otherwise
    constexpr int GMAX = FS::n > 0 ? (2 * FS::n / QW + kRowThreadsOf<FS> - 1) / kRowThreadsOf<FS> : 4;
    const int ng = (W + QW - 1) / QW;
    const bool is_it = MODE == MODE_IT;
    T chk = T(0);  // fma(x, 0, chk) turns NaN on any non-finite x
    double e = 0.0;
    auto band = [&](auto trace_tag) {
      constexpr bool TR = decltype(trace_tag)::value;
      // packed FP32x2 stencil (column pairs) for whole-strip fp32 plans
      constexpr bool PKS = ILS_F32X2 && std::is_same<T, float>::value && !TR && !SOFTOK && ALLFULL;
      float2 chk2 = make_float2(0.f, 0.f);
      T myup[GMAX][QW];
      T fcur[GMAX][QW];
#pragma unroll
      for (int gi = 0; gi < GMAX; ++gi) {
        const int gg = tid + gi * nthr;
        if (gg < ng) {
#pragma unroll
          for (int q = 0; q < QW; ++q) {
            const int x = gg * QW + q;
            myup[gi][q] = x < W ? aux<SOFTOK>(L.get(1, x) - L.get(0, x), P) : T(0);
            fcur[gi][q] = (TR && is_it && x < W) ? __ldg(fpl + (size_t)r0 * A.f_rp + x) : T(0);
          }
        }
      }
      // rows in blocks of KB: the rhs of a block stays in registers until one
      // barrier shows every thread is past the block (a row reads its own
      // line and the one below, so lines <= jb + KB are free to take rhs)
      constexpr int KB = TR ? 1 : kStencilRows;
      for (int jb = 0; jb < nb; jb += KB) {
        T rhs[KB][GMAX][QW];
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int j = jb + kk;
          if (j >= nb) break;  // block-uniform
          const int i = j + 1;
          T fnext[GMAX][QW];
#pragma unroll
          for (int gi = 0; gi < GMAX; ++gi) {
            const int gg = tid + gi * nthr;
            if (gg < ng) {
              const int x0 = gg * QW;
              const bool full = ALLFULL || (PACKED && x0 + QW <= W);
              if (TR && is_it) {
                const T* fr = fpl + (size_t)(r0 + min(j + 1, nb - 1)) * A.f_rp + x0;
#pragma unroll
                for (int q = 0; q < QW; ++q) fnext[gi][q] = (full || x0 + q < W) ? __ldg(fr + q) : T(0);
              }
              T uc[QW], ud[QW];
              if (full) {
                L.template get_strip<QW>(i, x0, uc);
                L.template get_strip<QW>(i + 1, x0, ud);
              } else {
#pragma unroll
                for (int q = 0; q < QW; ++q) {
                  const int x = x0 + q;
                  uc[q] = x < W ? L.get(i, x) : T(0);
                  ud[q] = x < W ? L.get(i + 1, x) : T(0);
                }
              }
              T mxp = aux<SOFTOK>(uc[0] - L.get(i, wrapi(x0 - 1, W)), P);
              const T uright = L.get(i, wrapi(full ? x0 + QW : min(x0 + QW, W), W));
#if ILS_F32X2
              if constexpr (PKS) {
                // the scalar loop below, two columns per instruction
                float gxs[QW], mx[QW], my[QW];
#pragma unroll
                for (int q = 0; q < QW; ++q) gxs[q] = (q + 1 < QW ? uc[q + 1] : uright) - uc[q];
#pragma unroll
                for (int p2 = 0; p2 < QW; p2 += 2) {
                  const float2 gy2 = __fadd2_rn(make_float2(ud[p2], ud[p2 + 1]), make_float2(-uc[p2], -uc[p2 + 1]));
                  const float2 m = aux2(make_float2(gxs[p2], gxs[p2 + 1]), P);
                  const float2 n = aux2(gy2, P);
                  mx[p2] = m.x;
                  mx[p2 + 1] = m.y;
                  my[p2] = n.x;
                  my[p2 + 1] = n.y;
                }
#pragma unroll
                for (int p2 = 0; p2 < QW; p2 += 2) {
                  const float ax0 = (p2 == 0 ? mxp : mx[p2 - 1]) - mx[p2], ax1 = mx[p2] - mx[p2 + 1];
                  const float2 ay = __fadd2_rn(make_float2(myup[gi][p2], myup[gi][p2 + 1]),
                                               make_float2(-my[p2], -my[p2 + 1]));
                  const float2 a = __fadd2_rn(make_float2(ax0, ax1), ay);
                  const float2 l2 = make_float2(lam2, lam2);
                  const float2 r = is_it ? __fmul2_rn(l2, a) : __ffma2_rn(l2, a, make_float2(uc[p2], uc[p2 + 1]));
                  rhs[kk][gi][p2] = r.x;
                  rhs[kk][gi][p2 + 1] = r.y;
                  chk2 = __ffma2_rn(make_float2(uc[p2], uc[p2 + 1]), make_float2(0.f, 0.f), chk2);
                }
#pragma unroll
                for (int q = 0; q < QW; ++q) myup[gi][q] = my[q];
                continue;
              }
#endif
#pragma unroll
              for (int q = 0; q < QW; ++q) {
                if (full || x0 + q < W) {
                  const T ur = (q + 1 < QW && (full || x0 + q + 1 < W)) ? uc[q + 1] : uright;
                  const T gx = ur - uc[q];
                  const T gy = ud[q] - uc[q];
                  const T mxq = aux<SOFTOK>(gx, P);
                  const T myq = aux<SOFTOK>(gy, P);
                  const T a = (mxp - mxq) + (myup[gi][q] - myq);
                  // iteration >= 1: rhs holds lam/2 D^T mu only; f is added as the
                  // r2c's first pass loads each element (phase C), off the
                  // stencil's critical path
                  const T fv = is_it ? fcur[gi][q] : uc[q];
                  rhs[kk][gi][q] = is_it ? mul_rn(lam2, a) : fma_rn(lam2, a, fv);
                  chk = fma_rn(uc[q], T(0), chk);
                  if constexpr (TR) {
                    const T d = uc[q] - fv;
                    e += double(d) * double(d) + double(P.lam) * (double(phi(gx, P)) + double(phi(gy, P)));
                  }
                  myup[gi][q] = myq;
                  mxp = mxq;
                } else {
                  rhs[kk][gi][q] = T(0);
                }
              }
              if constexpr (TR) {
#pragma unroll
                for (int q = 0; q < QW; ++q) fcur[gi][q] = fnext[gi][q];
              }
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int j = jb + kk;
          if (j >= nb) break;
#pragma unroll
          for (int gi = 0; gi < GMAX; ++gi) {
            const int gg = tid + gi * nthr;
            if (gg < ng) {
              const int x0 = gg * QW;
              if (ALLFULL || (PACKED && x0 + QW <= W)) {
                L.template set_strip<QW>(j, x0, rhs[kk][gi]);
              } else {
#pragma unroll
                for (int q = 0; q < QW; ++q)
                  if (x0 + q < W) L.set(j, x0 + q, rhs[kk][gi][q]);
              }
            }
          }
        }
      }
      chk = chk + (chk2.x + chk2.y);  // 0, or NaN when a packed lane saw a non-finite u
    };
    if (trace) band(std::true_type{});
    else band(std::false_type{});
    // the stencil read every band row of u once: flag the first non-finite
    // iterate (0 = non-finite input plane), smoother.py:166-167 / image.py:43-44
    bad = !finite_(chk);
    if (__syncthreads_or(bad) && tid == 0) atomicMin(A.status, MODE == MODE_F0 ? 0 : A.iter);
    if (trace) {
      const double s = block_sum(e, red);
      if (tid == 0) A.epart[(size_t)b * gridDim.x + blockIdx.x] = s;
    }
  }

#ifdef ILS_PDL_LATE  // (tuning: let the next pass launch only once this one reaches its last phase)
  pdl_trigger();
#endif
  // ---------------- phase C: r2c of rhs rows -> S_out (group per line)
  for (int i = g.id; i < nb; i += ngroups) {
    cx<T>* z = L.line(i);
    if (MODE == MODE_IT && PACKED) {
      // rhs = f + lam/2 D^T mu: the f row is added as the first pass loads
      // (independent coalesced loads, latency overlapped with the butterflies)
      const AddPair<T> pre{reinterpret_cast<const cx<T>*>(fpl + (size_t)(r0 + i) * A.f_rp)};
      fft_line<T, -1, FS>(z, A.fft, g, pre, &twc);
    } else {
      if (MODE == MODE_IT) {  // unpacked (odd W): add f as its own sweep
        for (int x = g.rank; x < W; x += g.size()) z[x].x += fpl[(size_t)(r0 + i) * A.f_rp + x];
        g.sync();  // the first pass reads other threads' elements
      }
      fft_line<T, -1, FS>(z, A.fft, g, NoPre{}, &twc);
    }
    if (PACKED) r2c_post<T>(z, NPK, twp, g);
    else g.sync();
    if (A.sout_seg.n == 0) {
      cx<T>* dst = A.Sout + (size_t)b * A.S_ps + (size_t)(r0 + i) * A.S_rp;
      if constexpr (BULK) {
        if (g.rank == 0) bulk_s2g(dst, z, spec_bytes);
      } else {
        for (int k = g.rank; k < A.Wc; k += g.size()) dst[k] = z[k];
      }
    } else {
      // fused pack: each column segment goes straight into its destination's
      // all-to-all block
      const SegRows& sg = A.sout_seg;
      for (int q = 0; q < sg.n; ++q) {
        cx<T>* dst = A.Sout + (size_t)b * A.S_ps + sg.off[q] + (long long)(r0 + i) * sg.pitch[q];
        if constexpr (BULK) {
          if (g.rank == 0)
            bulk_s2g(dst, z + sg.c0[q], (unsigned)(((sg.c0[q + 1] - sg.c0[q] + 1) & ~1) * sizeof(cx<T>)));
        } else {
          for (int k = sg.c0[q] + g.rank; k < sg.c0[q + 1]; k += g.size()) dst[k - sg.c0[q]] = z[k];
        }
      }
    }
  }
  if constexpr (BULK) bulk_wait_reads();
}

// ------------------------------------------------------------ column pass
template <typename T>
struct DenomScale {  // v * inv_hw / (1 + c lam/2 (wx[kx] + wy[ky]))
  const T* wy;
  T base, cl2, inv_hw;
  __device__ __forceinline__ cx<T> operator()(int y, cx<T> v) const {
    return scale(v, fast_div(inv_hw, base + cl2 * wy[y]));
  }
};
template <typename T>
struct UniformScale {
  T s;
  __device__ __forceinline__ cx<T> operator()(int, cx<T> v) const { return scale(v, s); }
};

// A strip of C columns is loaded transposed into C lines (line pitch CS
// chosen so the transposing copies are bank-conflict-free); a group owns one
// column at a time: forward FFT, * 1/(H W denom), inverse FFT.
// plans holding more than 16 elements per thread get the 2-CTA register budget
template <class FS>
constexpr int kColBlocksOf = FS::ME > 16 ? 2 : kColMinBlocks;

template <class FS>
constexpr int kColThreadsOf = std::is_same<FS, FftRtWide>::value ? 2 * kColThreads : kColThreads;
template <class FS>
constexpr int kColLaunchBlocksOf = std::is_same<FS, FftRtWide>::value ? 1 : kColBlocksOf<FS>;

template <typename T, class FS>
__global__ void __launch_bounds__(kColThreadsOf<FS>, kColLaunchBlocksOf<FS>) k_col(const ColArgs<T> A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cx<T>* tile = reinterpret_cast<cx<T>*>(smem_raw);
  T* swy = reinterpret_cast<T*>(tile + A.C * A.CS);  // wy[0..H) staged once per CTA
  using Grp = GroupT<FS::G>;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int G = FS::G > 0 ? FS::G : A.fft.G;
  const Grp g{tid / G, G, tid % G};
  const int ngroups = nthr / G;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * A.C;
  const int nc = min(A.C, A.Wc - c0);
  const int H = A.H;
  cx<T>* Spl = A.S + (size_t)b * A.S_ps + c0;
  TwCache<T, FS> twc;
  fill_twcache(twc, A.fft, g);
  pdl_trigger();
  pdl_wait();
  // transposing copies: thread -> (column cc, first row y0), rows step ystep
  const int ystep = nthr / nc, cc = tid % nc, y0 = tid / nc;
  const bool copier = tid < ystep * nc;
  if (copier)
    for (int y = y0; y < H; y += ystep) cp_async<sizeof(cx<T>)>(tile + cc * A.CS + y, Spl + (size_t)y * A.S_rp + cc);
  if (A.mode == COL_SOLVE)
    for (int y = tid; y < H; y += nthr) swy[y] = __ldg(A.wy + y);
  cp_async_wait_all();
  __syncthreads();
  for (int c = g.id; c < nc; c += ngroups) {
    cx<T>* z = tile + c * A.CS;
    if (A.mode != COL_INV) fft_line<T, -1, FS>(z, A.fft, g, NoPre{}, &twc);
    if (A.mode == COL_SOLVE) {
      // / denom (solver.py:100-102, 130) and the 1/(H W) of both inverses,
      // applied as the inverse transform's first pass loads each element
      const T cl2 = A.cl2_of(b);
      const T base = T(1) + cl2 * __ldg(A.wx + c0 + c);
      const DenomScale<T> pre{swy, base, cl2, A.inv_hw};
      fft_line<T, +1, FS>(z, A.fft, g, pre, &twc);
    } else if (A.mode == COL_INV) {
      const UniformScale<T> pre{A.inv_hw};
      fft_line<T, +1, FS>(z, A.fft, g, pre, &twc);
    }
  }
  __syncthreads();
  if (A.P == 0) {
    if (copier)
      for (int y = y0; y < H; y += ystep) Spl[(size_t)y * A.S_rp + cc] = tile[cc * A.CS + y];
    return;
  }
  // distributed: row y goes to its owner p (block row y - r0[p] + 1) and, when
  // it is p's first / last row, also to p-1 / p+1 as their bottom / top halo
  // (periodic across ranks): the reverse transpose plus the halo exchange in
  // one scatter (fused pack)
  if (copier) {
    cx<T>* dpl = A.dst + (size_t)b * A.S_ps + c0 + cc;
    int p = 0;
    for (int y = y0; y < H; y += ystep) {
      while (y >= A.r0[p + 1]) ++p;
      const cx<T> v = tile[cc * A.CS + y];
      dpl[A.dst_off[p] + (long long)(y - A.r0[p] + 1) * A.S_rp] = v;
      if (y == A.r0[p]) {
        const int q = p == 0 ? A.P - 1 : p - 1;
        dpl[A.dst_off[q] + (long long)(A.r0[q + 1] - A.r0[q] + 1) * A.S_rp] = v;
      }
      if (y == A.r0[p + 1] - 1) {
        const int q = p == A.P - 1 ? 0 : p + 1;
        dpl[A.dst_off[q]] = v;
      }
    }
  }
}

// ------------------------------------------------------------ small kernels
// energies[b] = sum of partials in fixed order (deterministic)
static __global__ void k_energy_reduce(const double* __restrict__ part, int nparts, int B, double* __restrict__ out) {
  const int b = blockIdx.x;
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[(size_t)b * nparts + i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[b] = s;
}

// BT.601 (image.py:110-128): planes [frame][3][H*W] in place
template <typename T>
__global__ void k_rgb_yuv(T* __restrict__ p, long long plane_stride, long long npx, int nframes, int inverse) {
  const long long n = npx * nframes;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long fr = t / npx, i = t - fr * npx;
    T* q = p + fr * 3 * plane_stride + i;
    const T a = q[0], b = q[plane_stride], c = q[2 * plane_stride];
    if (!inverse) {
      const T y = T(0.299) * a + T(0.587) * b + T(0.114) * c;
      q[0] = y;
      q[plane_stride] = T(0.492) * (c - y);
      q[2 * plane_stride] = T(0.877) * (a - y);
    } else {
      const T r = a + c / T(0.877);
      const T bb = a + b / T(0.492);
      q[0] = r;
      q[plane_stride] = (a - T(0.299) * r - T(0.114) * bb) / T(0.587);
      q[2 * plane_stride] = bb;
    }
  }
}

// 8-bit interleaved frames [frames][H][W][ch] -> planar planes [frames][ch][H W]
// holding v / 255 (formats.py read side, u8_to), so the first row pass reads
// f with whole-row TMA copies like any fp32 plane.  ch = 3: one thread per 4
// pixels -- 3 coalesced 32-bit loads, one 16-byte store per plane.
template <typename T>
__global__ void k_u8_planar(const unsigned char* __restrict__ f8, T* __restrict__ f, int ch, int npx) {
  // blockIdx.y = frame; 32-bit indices inside a frame (no 64-bit division)
  const size_t fr = blockIdx.y;
  const int stride = gridDim.x * blockDim.x;
  if (ch == 3 && (npx & 3) == 0) {
    const int nq = npx / 4;
    const unsigned* w = reinterpret_cast<const unsigned*>(f8 + fr * 3 * (size_t)npx);
    T* out = f + fr * 3 * (size_t)npx;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const unsigned wd[3] = {__ldg(w + 3 * q), __ldg(w + 3 * q + 1), __ldg(w + 3 * q + 2)};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        T v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int pos = 3 * k + c;  // byte of pixel k, channel c
          v[k] = u8_to((wd[pos >> 2] >> (8 * (pos & 3))) & 0xffu, T{});
        }
        T* o = out + (size_t)c * npx + 4 * q;
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = v[k];
        }
      }
    }
    return;
  }
  const unsigned char* src = f8 + fr * (size_t)ch * npx;
  T* out = f + fr * (size_t)ch * npx;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < npx * ch; t += stride) {
    const int i = t / ch, c = t - i * ch;
    out[(size_t)c * npx + i] = u8_to(__ldg(src + t), T{});
  }
}

// ------------------------------------------------------------ applications
// gaussian_blur (applications.py:210-222): separable, radius ceil(3 sigma),
// replicate ("nearest") edges, axis 0 then axis 1.  Sums follow scipy's
// symmetric correlate: w[r] x[i] + sum_j w[r+j] (x[i+j] + x[i-j]).
constexpr int kMaxGaussRadius = 128;
template <typename T>
struct GaussW {
  int r;
  T w[kMaxGaussRadius + 1];  // w[j] = weight at offset j (symmetric)
};

template <typename T>
__global__ void k_gauss_cols(const T* __restrict__ x, T* __restrict__ y, int H, int W, long long ps, GaussW<T> g) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r0 = blockIdx.y * 32;
  if (c >= W) return;
  const T* xp = x + (size_t)blockIdx.z * ps;
  T* yp = y + (size_t)blockIdx.z * ps;
  for (int r = r0; r < min(r0 + 32, H); ++r) {
    T acc = g.w[0] * xp[(size_t)r * W + c];
    for (int j = 1; j <= g.r; ++j) {
      const int a = min(r + j, H - 1), b = max(r - j, 0);
      acc = acc + g.w[j] * (xp[(size_t)a * W + c] + xp[(size_t)b * W + c]);
    }
    yp[(size_t)r * W + c] = acc;
  }
}

template <typename T>
__global__ void k_gauss_rows(const T* __restrict__ x, T* __restrict__ y, int W, long long ps, GaussW<T> g) {
  extern __shared__ __align__(16) unsigned char gsm[];
  T* row = reinterpret_cast<T*>(gsm);  // [r halo][W][r halo], replicate edges
  const int rr = blockIdx.x;
  const T* xp = x + (size_t)blockIdx.y * ps + (size_t)rr * W;
  T* yp = y + (size_t)blockIdx.y * ps + (size_t)rr * W;
  for (int i = threadIdx.x; i < W + 2 * g.r; i += blockDim.x) row[i] = xp[min(max(i - g.r, 0), W - 1)];
  __syncthreads();
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    const T* q = row + c + g.r;
    T acc = g.w[0] * q[0];
    for (int j = 1; j <= g.r; ++j) acc = acc + g.w[j] * (q[j] + q[-j]);
    yp[c] = acc;
  }
}

// ------------------------------------------------------------ launchers
// Compile-time FFT plans for the hot sizes (fp32).  Everything else runs the
// runtime-planned path (FftRt).  The host planner (ils_api.cu) uses exactly
// these radix lists when n matches, so twiddle tables and kernels agree.
// X(id, swizzle, group threads, elements per thread, n, radices...)
#define ILS_ROW_SPECS(X) X(0, 1, 32, 16, 256, 16, 16) X(1, 3, 32, 32, 960, 32, 30) X(2, 1, 128, 16, 1920, 16, 15, 8) X(3, 1, 256, 16, 3840, 16, 16, 15) X(4, 1, 32, 16, 512, 16, 8, 4)
// row specs with a rolling-band first / fused pass (ils_rowroll.cuh): the wide
// rows (3840, 7680) whose halo lines cost 40% of k_row's inverse transforms
#define ILS_ROW_SPEC_ROLL(ID) ((ID) == 2 || (ID) == 3)
// row specs whose width 2n exceeds 4 * kRowThreads * 4 need the WIDE stencil (8-column strips)
#ifndef ILS_ROW_SPEC_WIDE  // (tuning override: which row specs use 8-column stencil strips)
#define ILS_ROW_SPEC_WIDE(ID) ((ID) == 3)
#endif
#define ILS_COL_SPECS(X) X(0, 1, 32, 16, 512, 16, 8, 4) X(1, 0, 128, 16, 1080, 9, 12, 10) X(2, 1, 256, 16, 2160, 16, 15, 9) X(3, 1, 32, 16, 256, 16, 16) X(4, 1, 128, 16, 720, 16, 9, 5) X(5, 1, 256, 24, 4320, 24, 18, 10)

template <int ID>
struct RowSpec;
template <int ID>
struct ColSpec;
#define ILS_DEF_ROW_SPEC(ID, ...) \
  template <>                     \
  struct RowSpec<ID> {            \
    using type = FftCt<__VA_ARGS__>; \
  };
#define ILS_DEF_COL_SPEC(ID, ...) \
  template <>                     \
  struct ColSpec<ID> {            \
    using type = FftCt<__VA_ARGS__>; \
  };
ILS_ROW_SPECS(ILS_DEF_ROW_SPEC)
ILS_COL_SPECS(ILS_DEF_COL_SPEC)

template <typename T, bool PACKED, class FS, bool WIDE = false>
cudaError_t launch_row_impl(const RowArgs<T>& a, dim3 grid, int threads, size_t smem, cudaStream_t s);
template <typename T, class FS>
cudaError_t launch_col_impl(const ColArgs<T>& a, dim3 grid, int threads, size_t smem, cudaStream_t s);

// Launch a pass with programmatic stream serialisation (see pdl_wait);
// ILS_NO_PDL=1 launches plainly (A/B comparisons).
template <class K, class Args>
cudaError_t launch_pdl(K kernel, dim3 grid, int threads, size_t smem, cudaStream_t s, const Args& a) {
  static const bool off = [] {
    const char* v = getenv("ILS_NO_PDL");
    return v && atoi(v) != 0;
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

// Raise a kernel's dynamic shared-memory limit once per (kernel, device)
// instead of on every launch (a driver call in the per-batch host path).
inline cudaError_t smem_attr(const void* k, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, size_t> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long key = reinterpret_cast<unsigned long long>(k) * 64ull + (unsigned)dev;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[key] = smem;
  return e;
}

#ifdef ILS_DEFINE_LAUNCHERS
template <typename T, bool PACKED, class FS, bool WIDE>
cudaError_t launch_row_impl(const RowArgs<T>& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  // generic kernel (SMODE -1): energy trace, or the HQS soft threshold (kind 2)
  auto k = k_row<T, PACKED, FS, WIDE, -1>;
  if (a.f8 || a.u8) {
    if (a.epart) return cudaErrorInvalidValue;  // no energy trace on the 8-bit path
    if (a.mode == MODE_F0 && a.f8) k = k_row<T, PACKED, FS, WIDE, kU8Modes + MODE_F0>;
    if (a.mode == MODE_FIN && a.u8) k = k_row<T, PACKED, FS, WIDE, kU8Modes + MODE_FIN>;
  } else if (a.epart == nullptr && (a.pen.kind != 2 || a.mode == MODE_FIN)) {
    if (a.mode == MODE_F0) k = k_row<T, PACKED, FS, WIDE, MODE_F0>;
    if (a.mode == MODE_IT) k = k_row<T, PACKED, FS, WIDE, MODE_IT>;
    if (a.mode == MODE_FIN) k = k_row<T, PACKED, FS, WIDE, MODE_FIN>;
  }
  cudaError_t e = smem_attr(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, threads, smem, s, a);
}
template <typename T, class FS>
cudaError_t launch_col_impl(const ColArgs<T>& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  auto k = k_col<T, FS>;
  cudaError_t e = smem_attr(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, threads, smem, s, a);
}
#endif

}  // namespace ils
