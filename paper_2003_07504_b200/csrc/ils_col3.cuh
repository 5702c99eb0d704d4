// Three-stage register-light column solve (sm_100a), H = N1 * N2 * N3.
//
// The column half of one ILS iteration (reference solver.py:127-130: fft2 of
// the right-hand side, / denom, ifft2) on a strip of CW spectrum columns,
// like k_col2 (ils_col2.cuh) but with the M = N2 N3 point inner transform
// split once more, so no thread ever holds more than max(N1, N2, N3) <= ~18
// values.  That keeps the kernel near 40-64 registers, i.e. 2-3x the
// resident warps of k_col2 (96 registers, 18 warps/SM), which was latency
// bound (ncu: 42% issue, long-scoreboard the top stall).  Index maps
// (forward, DIR = -1; the inverse retraces them with conjugate twiddles):
//
//   n = n23 + M n1,  n23 = n3 + N3 n2;   k = k1 + N1 k23,  k23 = k2 + N2 k3
//
//   stage A   thread (n23, c): rows n23 + M n1 straight from global memory,
//             DFT_N1 over n1, * w_H^(n23 k1)          -> Y[k1][n23]
//   stage B1  thread (k1, n3, c): Y[k1][n3 + N3 n2] over n2, DFT_N2,
//             * w_M^(n3 k2)                            -> Z[k1][k2][n3] (same slots)
//   stage B2  thread (k1, k2, c): Z[k1][k2][n3] over n3, DFT_N3 -> X[k1 + N1 (k2 + N2 k3)],
//             * 1/(H W denom), inverse DFT_N3 on the same registers, back in place
//   stage B1' inverse of B1 (conjugate twiddle first), stage A' inverse of A,
//             rows straight back to global memory (in place, or the slab
//             plan's reverse all-to-all blocks, as k_col2).
//
// Shared memory holds one strip: element (idx, c) at idx * CW + c with
// idx = k1 M + n23 (Y) / k1 M + k2 N3 + n3 (Z); B1 reads and writes the same
// slots per thread, so it needs no barrier between its load and store.  In
// every stage consecutive threads touch consecutive idx (stride-N3 in B2),
// i.e. whole 128-byte wavefronts.
#pragma once

#include "ils_kernels.cuh"

namespace ils {

template <int N1, int N2, int N3, int CW>
struct Col3Shape {
  static constexpr int M = N2 * N3;
  static constexpr int H = N1 * M;
  static constexpr int TA = M, TB1 = N1 * N3, TB2 = N1 * N2;
  static constexpr int TMAX = TA > TB1 ? (TA > TB2 ? TA : TB2) : (TB1 > TB2 ? TB1 : TB2);
  static constexpr int NT = (CW * TMAX + 31) / 32 * 32;
  static constexpr int TILE = (H * CW + 1) & ~1;  // complex elements (whole 16-byte pairs: the tables follow)
  // tile + w_H^m (m < H) + w_M^m (m < M) + wy (H floats)
  static constexpr size_t SMEM = (size_t)TILE * 8 + (size_t)H * 8 + (size_t)M * 8 + (size_t)H * 4;
};

template <int N1, int N2, int N3, int CW, int MINB>
__global__ void __launch_bounds__(Col3Shape<N1, N2, N3, CW>::NT, MINB) k_col3(const ColArgs<float> A) {
  using S = Col3Shape<N1, N2, N3, CW>;
  constexpr int H = S::H, M = S::M;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cx<float>* buf = reinterpret_cast<cx<float>*>(smem_raw);
  cx<float>* twH = buf + S::TILE;                // exp(-2 pi i m / H), m < H
  cx<float>* twM = twH + H;                      // exp(-2 pi i m / M), m < M
  float* swy = reinterpret_cast<float*>(twM + M);  // 2 - 2 cos(2 pi ky / H)
  const int t = threadIdx.x;
  const int c = t % CW, r = t / CW;  // r: the stage's work index
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * CW;
  const bool colok = c0 + c < A.Wc;
  cx<float>* Spl = A.S + (size_t)b * A.S_ps + c0 + c;

#ifndef ILS_PDL_LATE
  pdl_trigger();
#endif
  for (int m = t; m < H; m += S::NT) {  // constant tables: before the wait on the previous pass
    twH[m] = ldg_cx(A.tw2 + m);
    swy[m] = __ldg(A.wy + m);
  }
  for (int m = t; m < M; m += S::NT) twM[m] = ldg_cx(A.tw2 + (size_t)m * N1);  // w_M^m = w_H^(m N1)
  pdl_wait();

  // ---------------- stage A: strided rows -> DFT_N1 -> w_H^(n23 k1) -> Y[k1][n23]
  cx<float> v[N1];
  const bool actA = r < M;
  if (actA) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1)
      v[n1] = colok ? ldg_cx(Spl + (size_t)(r + M * n1) * A.S_rp) : cx<float>{0.f, 0.f};
  }
  __syncthreads();  // the twiddle tables
  if (actA) {
    dft<N1, -1>(v);
    cx<float>* d = buf + r * CW + c;
    d[0] = v[0];
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) d[k1 * M * CW] = cmul(v[k1], twH[r * k1]);
  }
  __syncthreads();

  // ---------------- stage B1: per (k1, n3): DFT_N2 over n2, * w_M^(n3 k2), in place
  const int k1b = r / N3, n3b = r - k1b * N3;
  const bool actB1 = r < S::TB1;
  if (actB1) {
    cx<float> w[N2];
    cx<float>* d = buf + (k1b * M + n3b) * CW + c;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) w[n2] = d[n2 * N3 * CW];
    dft<N2, -1>(w);
    d[0] = w[0];
#pragma unroll
    for (int k2 = 1; k2 < N2; ++k2) d[k2 * N3 * CW] = cmul(w[k2], twM[n3b * k2]);
  }
  __syncthreads();

  // ---------------- stage B2: per (k1, k2): DFT_N3 -> / denom -> inverse DFT_N3
  if (r < S::TB2) {
    const int k1 = r / N2, k2 = r - k1 * N2;
    cx<float> z[N3];
    cx<float>* d = buf + (k1 * M + k2 * N3) * CW + c;
#pragma unroll
    for (int n3 = 0; n3 < N3; ++n3) z[n3] = d[n3 * CW];
    dft<N3, -1>(z);
    // / denom (solver.py:100-102, 130) with the 1/(H W) of both inverses, the
    // expression k_col / k_col2 use (bit-identical scale); ky = k1 + N1 (k2 + N2 k3)
    const float cl2 = A.cl2_of(b);
    const float base = 1.f + cl2 * __ldg(A.wx + min(c0 + c, A.Wc - 1));
#pragma unroll
    for (int k3 = 0; k3 < N3; ++k3)
      z[k3] = scale(z[k3], fast_div(A.inv_hw, base + cl2 * swy[k1 + N1 * (k2 + N2 * k3)]));
    dft<N3, +1>(z);
#pragma unroll
    for (int n3 = 0; n3 < N3; ++n3) d[n3 * CW] = z[n3];
  }
  __syncthreads();

  // ---------------- stage B1': conj w_M^(n3 k2), inverse DFT_N2 over k2, in place
  if (actB1) {
    cx<float> w[N2];
    cx<float>* d = buf + (k1b * M + n3b) * CW + c;
    w[0] = d[0];
#pragma unroll
    for (int k2 = 1; k2 < N2; ++k2) w[k2] = cmulc(d[k2 * N3 * CW], twM[n3b * k2]);
    dft<N2, +1>(w);
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) d[n2 * N3 * CW] = w[n2];
  }
  __syncthreads();

#ifdef ILS_PDL_LATE
  pdl_trigger();
#endif
  // ---------------- stage A': conj w_H^(n23 k1), inverse DFT_N1 -> rows
  if (actA) {
    const cx<float>* d = buf + r * CW + c;
    v[0] = d[0];
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmulc(d[k1 * M * CW], twH[r * k1]);
    dft<N1, +1>(v);
    if (!colok) return;
    if (A.P == 0) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) Spl[(size_t)(r + M * n1) * A.S_rp] = v[n1];
      return;
    }
    // slab plan: row y to its owner p and, as the first / last row of p, to
    // p-1 / p+1 as their bottom / top halo (k_col2's fused scatter)
    cx<float>* dpl = A.dst + c0 + c;
    int p = 0;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int y = r + M * n1;
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
}

// (id, N1, N2, N3, CW, min CTAs per SM).  Opt-in (ILS_COL3_SPEC=id, or -2 for
// the first entry with N1 N2 N3 = H): on the B200 it measured no faster than
// k_col2 at 1080 rows (20.1 vs 19.9 us per 1080p RGB pass; 2.4x the resident
// warps but +25% instructions, 5 barriers and per-CTA table staging) and
// slower at 2160 / 4320 rows (123 vs 81 us, 580 vs 462 us).
#define ILS_COL3_SPECS(X)                                                                                      \
  X(7, 10, 12, 9, 4, 3) X(8, 10, 12, 9, 2, 6) X(0, 10, 12, 9, 4, 2) X(1, 12, 10, 9, 4, 2) X(2, 10, 12, 9, 2, 4)     \
      X(3, 9, 12, 10, 4, 2) X(9, 12, 15, 12, 2, 3) X(4, 12, 15, 12, 2, 2) X(10, 16, 15, 18, 2, 2) X(5, 15, 16, 18, 2, 1) \
      X(6, 16, 15, 18, 2, 1)

template <int N1, int N2, int N3, int CW, int MINB>
cudaError_t launch_col3_impl(const ColArgs<float>& a, int planes, cudaStream_t s);

#ifdef ILS_DEFINE_LAUNCHERS
template <int N1, int N2, int N3, int CW, int MINB>
cudaError_t launch_col3_impl(const ColArgs<float>& a, int planes, cudaStream_t s) {
  using S = Col3Shape<N1, N2, N3, CW>;
  auto k = k_col3<N1, N2, N3, CW, MINB>;
  cudaError_t e = smem_attr(reinterpret_cast<const void*>(k), S::SMEM);
  if (e != cudaSuccess) return e;
  const dim3 grid((a.Wc + CW - 1) / CW, planes);
  return launch_pdl(k, grid, S::NT, S::SMEM, s, a);
}
#endif

}  // namespace ils
