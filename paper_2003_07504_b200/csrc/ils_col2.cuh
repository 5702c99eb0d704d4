// Two-stage register-resident column solve (sm_100a), H = N1 * N2.
//
// The column half of one ILS iteration (reference solver.py:127-130: fft2 of
// the right-hand side, / denom, ifft2) on a strip of CW spectrum columns.
// Instead of a Stockham sweep per radix through shared memory (k_col), each
// column's H-point transform is split once, n = n2 + N2 n1, k = k1 + N1 k2:
//
//   stage A  thread (n2, c): N1 strided rows straight from global memory
//            (a warp reads CW adjacent columns of a row), DFT_N1 over n1 in
//            registers, twiddle w_H^(n2 k1), one store per k1 to shared memory
//   stage B  thread (k1, c): the N2 values of its k1, DFT_N2 -> X[k1 + N1 k2]
//            in registers, * 1/(H W denom(k1 + N1 k2, c)), inverse DFT_N2 on
//            the same registers (the spectrum never leaves them in between),
//            conjugate twiddle, back to the same shared-memory slots
//   stage C  thread (n2, c): inverse DFT_N1 over k1, N1 rows straight back to
//            global memory (in place, or scattered to the reverse all-to-all
//            blocks of a slab plan)
//
// Two barriers and two shared-memory round trips per strip (k_col: ~7), no
// running twiddle products (one table load per element), and 36 independent
// global loads in flight per thread.  Shared memory is laid out so that both
// access patterns are conflict-free: element (k1, n2, c) sits at
// k1 * KS + n2 * CW + c with KS = N2 CW + PAD, PAD = CW (1 - N2) mod 16, so in
// either stage a warp's addresses are its thread indices plus a constant,
// modulo 16 complex (128 bytes).
#pragma once

#include "ils_kernels.cuh"

namespace ils {

template <int N1, int N2, int CW, int MINB>
struct Col2Shape {
  static constexpr int H = N1 * N2;
  static constexpr int R = N1 > N2 ? N1 : N2;
  static constexpr int NT = (CW * R + 31) / 32 * 32;
  static constexpr int PAD = ((CW * (1 - N2)) % 16 + 16) % 16;
  static constexpr int KS = N2 * CW + PAD;
  static constexpr int TILE = (N1 * KS + 1) & ~1;  // complex elements (whole 16-byte pairs: the tables follow)
  // the constant tables stay in global memory (read through L1) when staging
  // them would keep MINB strips from sharing an SM: the 4320-row strip of 2
  // columns, 69 KB of tile, then fits 2 CTAs per SM with 118 KB of L1 left
  static constexpr bool TG = ((size_t)TILE * 8 + (size_t)H * 12) * MINB > 227 * 1024;
  static constexpr size_t SMEM = (size_t)TILE * 8 + (TG ? 0 : (size_t)H * 12);
  static_assert(H % 4 == 0, "the tables arrive by bulk copy: whole 16-byte rows");
};

// (__launch_bounds__ leaves the 288-thread 30 x 36 strip at 96 registers with
// 100 bytes of L1-resident spills; an explicit 112-register cap removes them
// but measured slower, 23.5 vs 19.8 us per 1080p RGB pass)
template <int N1, int N2, int CW, int MINB>
__global__ void __launch_bounds__(Col2Shape<N1, N2, CW, MINB>::NT, MINB) k_col2(const ColArgs<float> A) {
  using S = Col2Shape<N1, N2, CW, MINB>;
  constexpr int H = S::H, KS = S::KS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cx<float>* buf = reinterpret_cast<cx<float>*>(smem_raw);
  cx<float>* stw = buf + S::TILE;                  // w_H^m = exp(-2 pi i m / H), m < H
  float* swy = reinterpret_cast<float*>(stw + H);  // 2 - 2 cos(2 pi ky / H)
  // table reads: shared memory, or global through L1 (S::TG)
#define ILS_C2_TW(m) (S::TG ? ldg_cx(A.tw2 + (m)) : stw[m])
#define ILS_C2_WY(m) (S::TG ? __ldg(A.wy + (m)) : swy[m])
  const int t = threadIdx.x;
  const int c = t % CW, r = t / CW;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * CW;
  const bool colok = c0 + c < A.Wc;
  cx<float>* Spl = A.S + (size_t)b * A.S_ps + c0 + c;
  const bool actA = r < N2;  // stages A and C: r = n2

  // ---------------- stage A: strided rows -> DFT_N1 -> twiddle -> smem
#ifndef ILS_PDL_LATE
  pdl_trigger();
#endif
  // the constant tables: two bulk copies issued before the wait on the
  // previous pass, landing while the strip's rows load (a per-thread
  // load -> store loop costs H / NT serial L2 round trips per CTA: 10% of
  // the 8K pass)
  __shared__ unsigned long long tbar;
  if (!S::TG && t == 0) {
    mbar_init(&tbar, 1);
    mbar_fence_init();
    mbar_expect_tx(&tbar, (unsigned)(H * 12));
    bulk_g2s(stw, A.tw2, (unsigned)(H * 8), &tbar);
    bulk_g2s(swy, A.wy, (unsigned)(H * 4), &tbar);
  }
  pdl_wait();
  cx<float> v[N1];
  if (actA) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1)
      v[n1] = colok ? ldg_cx(Spl + (size_t)(r + N2 * n1) * A.S_rp) : cx<float>{0.f, 0.f};
  }
  __syncthreads();  // (also publishes tbar's initialisation)
  if (!S::TG) mbar_wait(&tbar, 0);
  if (actA) {
    dft<N1, -1>(v);
    cx<float>* d = buf + r * CW + c;
    d[0] = v[0];
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) d[k1 * KS] = cmul(v[k1], ILS_C2_TW(r * k1));
  }
  __syncthreads();

  // ---------------- stage B: DFT_N2, / denom, inverse DFT_N2, conj twiddle
  if (r < N1) {
    cx<float> w[N2];
    cx<float>* d = buf + r * KS + c;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) w[n2] = d[n2 * CW];
    dft<N2, -1>(w);
    // / denom (solver.py:100-102, 130) with the 1/(H W) of both inverses:
    // the same expression as k_col's DenomScale, so the scale is bit-identical
    const float cl2 = A.cl2_of(b);
    const float base = 1.f + cl2 * __ldg(A.wx + min(c0 + c, A.Wc - 1));
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) w[k2] = scale(w[k2], fast_div(A.inv_hw, base + cl2 * ILS_C2_WY(r + N1 * k2)));
    dft<N2, +1>(w);
    d[0] = w[0];
#pragma unroll
    for (int n2 = 1; n2 < N2; ++n2) d[n2 * CW] = cmulc(w[n2], ILS_C2_TW(n2 * r));
  }
  __syncthreads();

#ifdef ILS_PDL_LATE
  pdl_trigger();
#endif
  // ---------------- stage C: inverse DFT_N1 -> rows
  if (actA) {
    const cx<float>* d = buf + r * CW + c;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) v[k1] = d[k1 * KS];
    dft<N1, +1>(v);
    if (!colok) return;
    if (A.P == 0) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) Spl[(size_t)(r + N2 * n1) * A.S_rp] = v[n1];
      return;
    }
    // slab plan: row y to its owner p (block row y - r0[p] + 1) and, as the
    // first / last row of p, to p-1 / p+1 as their bottom / top halo (k_col's
    // fused reverse-transpose scatter)
    cx<float>* dpl = A.dst + c0 + c;
    int p = 0;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int y = r + N2 * n1;
      while (y >= A.r0[p + 1]) ++p;
      dpl[A.dst_off[p] + (long long)(y - A.r0[p] + 1) * A.S_rp] = v[n1];
      if (y == A.r0[p]) {
        const int q = p == 0 ? A.P - 1 : p - 1;
        dpl[A.dst_off[q] + (long long)(A.r0[q + 1] - A.r0[q] + 1) * A.S_rp] = v[n1];
      }
      if (y == A.r0[p + 1] - 1) {
        const int q = p == A.P - 1 ? 0 : p + 1;
        dpl[A.dst_off[q]] = v[n1];
      }
    }
  }
#undef ILS_C2_TW
#undef ILS_C2_WY
}

// (id, N1, N2, CW, min CTAs per SM); a plan takes the first entry with N1 N2 = H
// (ILS_COL2_SPEC=id overrides, for sweeps: tools/gpu_sweep_col2.sh,
// tools/gpu_sweep_band_col2.sh, tools/gpu_col2_resweep.sh -- with the tables
// bulk-copied, 30 x 36 runs a 1080p RGB pass in 19.1 us alone vs 20.3 for
// 36 x 30, +0.4% in the bench, despite 100 bytes of L1-resident spills)
#define ILS_COL2_SPECS(X)                                                                                    \
  X(5, 30, 36, 8, 2) X(0, 36, 30, 8, 2) X(1, 36, 30, 6, 3) X(2, 36, 30, 4, 4) X(3, 36, 30, 10, 1) X(4, 36, 30, 10, 2) \
      X(6, 36, 30, 16, 1) X(8, 48, 45, 8, 1) X(9, 45, 48, 8, 1) X(7, 48, 45, 4, 2) \
      X(10, 72, 60, 4, 1) X(11, 60, 72, 4, 1) X(12, 72, 60, 2, 2) X(14, 45, 48, 4, 2) X(15, 60, 72, 2, 2)

template <int N1, int N2, int CW, int MINB>
cudaError_t launch_col2_impl(const ColArgs<float>& a, int planes, cudaStream_t s);

#ifdef ILS_DEFINE_LAUNCHERS
template <int N1, int N2, int CW, int MINB>
cudaError_t launch_col2_impl(const ColArgs<float>& a, int planes, cudaStream_t s) {
  using S = Col2Shape<N1, N2, CW, MINB>;
  auto k = k_col2<N1, N2, CW, MINB>;
  cudaError_t e = smem_attr(reinterpret_cast<const void*>(k), S::SMEM);
  if (e != cudaSuccess) return e;
  const dim3 grid((a.Wc + CW - 1) / CW, planes);
  return launch_pdl(k, grid, S::NT, S::SMEM, s, a);
}
#endif

}  // namespace ils
