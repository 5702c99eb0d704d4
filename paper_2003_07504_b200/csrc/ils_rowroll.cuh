// Rolling-band row pass for wide rows (sm_100a): the first and the fused row
// pass (MODE_F0 / MODE_IT) of 3840- and 7680-wide planes (C4, C5).
//
// Same arithmetic as k_row (ils_kernels.cuh: c2r -> fused stencil -> f add ->
// r2c; reference smoother.py:162-169, penalty.py:117-126, solver.py:33-49,
// 127-129), different schedule.  k_row gives every CTA a band of b rows plus
// one halo row above and below, all resident at once; with 31-61 KB lines
// that is b = 5 and 7 inverse transforms per 5 rows (40% extra c2r work)
// at one or two CTAs per SM.  Here a CTA walks a long chunk of rows
// (~15-45) through a ring of NG + 1 line slots (NG = line groups per CTA):
//
//   step j:  A  c2r of rows j+1 .. j+NG  (the slots the previous step's
//               r2c lines left; their TMA loads were issued as soon as those
//               stores had read the slots)
//            B  stencil of rows j .. j+NG-1 (u_j from the previous step,
//               mu_y of the row above carried in a shared-memory row), rhs
//               written over the u rows no later row reads
//            C  r2c of the rhs rows (+ f on the first butterfly pass), TMA
//               store, then the next step's spectrum rows into the same slots
//
// so each row is inverse-transformed once (plus two per chunk), the loads of
// step j+1 overlap step j's r2c, and the smaller CTA footprint fits two CTAs
// per SM at either width with 128 registers (k_row: one CTA, 80 registers
// and 0.3-1.1 KB of spills per thread).  Rows wrap periodically within the plane.  The
// pixel arithmetic (aux, mul_rn / fma_rn, packed pairs) is k_row's, so the
// result is bit-identical to it.
#pragma once

#include "ils_kernels.cuh"

namespace ils {

// line groups per CTA of a compile-time row plan, and the register budget
template <class FS>
constexpr int kRollGroupsOf = kRowThreads / FS::G;
#ifndef ILS_ROLL_MINB  // (tuning: resident CTAs per SM the registers are budgeted for)
#define ILS_ROLL_MINB 2  // 128 registers: no spills at 3840 or 7680 (3 CTAs / 80 registers spill at 3840)
#endif
template <class FS>
constexpr int kRollBlocksOf = ILS_ROLL_MINB;

// PF = 1: a second set of NG slots, so the spectrum rows of step j+2 load
// while step j+1 runs (the rows of the next step are otherwise waited for
// right after their loads are issued)
template <class FS, int SMODE, int PF>
__global__ void __launch_bounds__(kRowThreads, kRollBlocksOf<FS>) k_row_roll(const RowArgs<float> A) {
  using T = float;
  constexpr int G = FS::G;
  constexpr int NG = kRollGroupsOf<FS>;
  constexpr int NS = (1 + PF) * NG + 1;
  constexpr int W = 2 * FS::n;
  constexpr int QW = W > kNarrowMaxW ? 8 : 4;
  constexpr int GMAX = (W / QW + kRowThreads - 1) / kRowThreads;
  constexpr bool WSMEM = FS::swz != 3;
  constexpr bool IT = SMODE == MODE_IT;
  static_assert(W % QW == 0 && NG >= 1, "rolling rows need whole stencil strips");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ unsigned long long bars[NS];
  using Grp = GroupT<G>;
  const int tid = threadIdx.x;
  const Grp g{tid / G, G, tid % G};
  const int b = blockIdx.y;
  const int H = A.H;
  const int r0 = blockIdx.x * A.band;
  const int r1 = min(r0 + A.band, H);
  const Lines<T, true> L{reinterpret_cast<cx<T>*>(smem_raw), A.LP};
  const PenaltyDev<T>& P = A.pen;
  const T lam2 = A.nlam > 0 ? A.lam2_tab[min(b, A.nlam - 1)] : P.lam2;
  const T* fpl = A.f + (size_t)b * A.f_ps;
  cx<T>* const swreal = WSMEM ? reinterpret_cast<cx<T>*>(smem_raw) + (size_t)NS * A.LP : const_cast<cx<T>*>(A.wreal);
  // mu_y of the row above, per column: carried from step to step in shared
  // memory (each thread reads and writes only its own strips), not registers
  // (16-byte aligned: float4 strips; the twiddle table is rounded up to whole pairs)
  T* smyup = reinterpret_cast<T*>(reinterpret_cast<cx<T>*>(smem_raw) + (size_t)NS * A.LP +
                                  (WSMEM ? ((A.N / 2 + 2) & ~1) : 0));
  __shared__ unsigned long long wbar;  // the packing twiddles: one bulk copy (whole pairs)
  TwCache<T, FS> twc;
  fill_twcache(twc, A.fft, g);
  if (tid < NS) mbar_init(&bars[tid], 1);
  if (WSMEM && tid == 0) mbar_init(&wbar, 1);
  mbar_fence_init();
  if (WSMEM && tid == 0) {
    const unsigned wb = (unsigned)(((A.N / 2 + 2) & ~1) * sizeof(cx<T>));
    mbar_expect_tx(&wbar, wb);
    bulk_g2s(swreal, A.wreal, wb, &wbar);
  }
  const unsigned spec_bytes = (unsigned)((A.Wc * sizeof(cx<T>) + 15) & ~size_t(15));
  pdl_trigger();
#ifdef ILS_ROLL_F_PREFETCH  // (tuning: the chunk's f rows into L2 up front -- at 3840 wide the
                            // frame does not fit L2 and the rows are read twice: +100 MB DRAM)
  if (IT)
    for (int y = r0 + tid; y < r1; y += kRowThreads)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(fpl + (size_t)y * A.f_rp),
                   "r"((unsigned)(W * sizeof(T)))
                   : "memory");
#endif
  __syncthreads();  // barriers initialised
  pdl_wait();
  if (WSMEM) mbar_wait(&wbar, 0);

  // (no lambdas here: a closure capturing the kernel's parameter block by
  // reference makes nvcc copy it to local memory and read every field, the
  // FFT plan included, with generic loads)
  const cx<T>* Sin_b = IT ? A.Sin + (size_t)b * A.S_ps : nullptr;
  const long long S_rp = A.S_rp, f_rp = A.f_rp;
  // slab plans (C5 over ranks): rows are not periodic (halo rows -1 and H are
  // present) and spectrum rows move as the all-to-all blocks' column segments
  const int nseg = A.sin_seg.n;
  unsigned seg_bytes = 0;
  for (int q = 0; q < nseg; ++q)
    seg_bytes += (unsigned)(((A.sin_seg.c0[q + 1] - A.sin_seg.c0[q] + 1) & ~1) * sizeof(cx<T>));
#define ROWY(y) (A.wrap ? wrapi((y), H) : (y))
  // one thread: TMA of row y (f for the first pass, the spectrum otherwise) into a slot
#define ILS_ROLL_ISSUE(slot, y)                                                                                  \
  do {                                                                                                           \
    if (IT && nseg > 0) { /* slab plan: the row's P column segments from the all-to-all blocks */               \
      mbar_expect_tx(&bars[slot], seg_bytes);                                                                    \
      for (int q_ = 0; q_ < nseg; ++q_)                                                                          \
        bulk_g2s(L.line(slot) + A.sin_seg.c0[q_], A.Sin + A.sin_seg.off[q_] + (long long)(y)*A.sin_seg.pitch[q_], \
                 (unsigned)(((A.sin_seg.c0[q_ + 1] - A.sin_seg.c0[q_] + 1) & ~1) * sizeof(cx<T>)), &bars[slot]); \
    } else if (IT) {                                                                                             \
      mbar_expect_tx(&bars[slot], spec_bytes);                                                                   \
      bulk_g2s_hint(L.line(slot), Sin_b + (long long)(y)*S_rp, spec_bytes, &bars[slot], l2_evict_first());      \
    } else {                                                                                                     \
      mbar_expect_tx(&bars[slot], (unsigned)(W * sizeof(T)));                                                    \
      bulk_g2s(L.line(slot), fpl + (long long)(y)*f_rp, (unsigned)(W * sizeof(T)), &bars[slot]);                 \
    }                                                                                                            \
  } while (0)
  unsigned phase = 0;  // bit s: parity of the next completion of bars[s] (uniform over the CTA)
  // the owning group waits for a slot's row and makes it u (c2r; the first pass loads f as-is)
#define ILS_ROLL_LAND(slot)                                                                                      \
  do {                                                                                                           \
    mbar_wait(&bars[slot], (phase >> (slot)) & 1u);                                                              \
    if (IT) {                                                                                                    \
      c2r_pre<T>(L.line(slot), FS::n, TwTab<T, WSMEM>{swreal}, g);                                                \
      fft_line<T, +1, FS>(L.line(slot), A.fft, g, NoPre{}, &twc);                                                \
    }                                                                                                            \
  } while (0)

  // ---------------- prologue: rows r0-1 and r0; mu_y of row r0-1
  if (tid == 0) {
    ILS_ROLL_ISSUE(0, ROWY(r0 - 1));
    ILS_ROLL_ISSUE(1 % NS, r0);
  }
  if (NG == 1) {
    if (g.id == 0) {
      ILS_ROLL_LAND(0);
      ILS_ROLL_LAND(1);
    }
  } else {
    if (g.id < 2) ILS_ROLL_LAND(g.id);
  }
  phase ^= 3u;
  __syncthreads();
#pragma unroll
  for (int gi = 0; gi < GMAX; ++gi) {
    const int gg = tid + gi * kRowThreads;
    if (gg * QW >= W) continue;
#pragma unroll
    for (int q = 0; q < QW; ++q) {
      const int x = gg * QW + q;
      smyup[x] = aux<false>(L.get(1, x) - L.get(0, x), P);
    }
  }
  __syncthreads();  // slot 0 (row r0-1) is free
  int p = 1 % NS;   // slot of u_j
  {  // the first step's rows (and with PF the second step's)
    const int ahead = min((1 + PF) * NG, r1 - r0);
    if (tid < ahead) ILS_ROLL_ISSUE((p + 1 + tid) % NS, ROWY(r0 + 1 + tid));
  }
  T chk = T(0);  // fma(x, 0, chk) turns NaN on any non-finite u of the chunk
  float2 chk2 = make_float2(0.f, 0.f);

  for (int j = r0; j < r1; j += NG) {
    const int ng = min(NG, r1 - j);
    // ---- A: u rows j+1 .. j+ng
    for (int i = g.id; i < ng; i += NG) ILS_ROLL_LAND((p + 1 + i) % NS);
    for (int i = 0; i < ng; ++i) phase ^= 1u << ((p + 1 + i) % NS);
    __syncthreads();

    // ---- B: stencil rows j .. j+ng-1 (k_row phase B, one row per slot pair)
    T rhs[NG][GMAX][QW];
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      if (i >= ng) break;  // block-uniform
      const int sc = (p + i) % NS, sd = (p + i + 1) % NS;
#pragma unroll
      for (int gi = 0; gi < GMAX; ++gi) {
        const int gg = tid + gi * kRowThreads;
        if (gg * QW >= W) continue;
        const int x0 = gg * QW;
        T uc[QW], ud[QW], myup[QW];
        L.template get_strip<QW>(sc, x0, uc);
        L.template get_strip<QW>(sd, x0, ud);
#pragma unroll
        for (int q = 0; q < QW; q += 4) {
          const float4 m4 = *reinterpret_cast<const float4*>(smyup + x0 + q);
          myup[q] = m4.x;
          myup[q + 1] = m4.y;
          myup[q + 2] = m4.z;
          myup[q + 3] = m4.w;
        }
        T mxp = aux<false>(uc[0] - L.get(sc, wrapi(x0 - 1, W)), P);
        const T uright = L.get(sc, wrapi(x0 + QW, W));
#if ILS_F32X2
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
          const float2 ay = __fadd2_rn(make_float2(myup[p2], myup[p2 + 1]), make_float2(-my[p2], -my[p2 + 1]));
          const float2 a = __fadd2_rn(make_float2(ax0, ax1), ay);
          const float2 l2 = make_float2(lam2, lam2);
          const float2 r = IT ? __fmul2_rn(l2, a) : __ffma2_rn(l2, a, make_float2(uc[p2], uc[p2 + 1]));
          rhs[i][gi][p2] = r.x;
          rhs[i][gi][p2 + 1] = r.y;
          chk2 = __ffma2_rn(make_float2(uc[p2], uc[p2 + 1]), make_float2(0.f, 0.f), chk2);
        }
#pragma unroll
        for (int q = 0; q < QW; q += 4)
          *reinterpret_cast<float4*>(smyup + x0 + q) = make_float4(my[q], my[q + 1], my[q + 2], my[q + 3]);
#else
#pragma unroll
        for (int q = 0; q < QW; ++q) {
          const T ur = q + 1 < QW ? uc[q + 1] : uright;
          const T mxq = aux<false>(ur - uc[q], P);
          const T myq = aux<false>(ud[q] - uc[q], P);
          const T a = (mxp - mxq) + (myup[q] - myq);
          rhs[i][gi][q] = IT ? mul_rn(lam2, a) : fma_rn(lam2, a, uc[q]);
          chk = fma_rn(uc[q], T(0), chk);
          smyup[x0 + q] = myq;
          mxp = mxq;
        }
#endif
      }
    }
    __syncthreads();  // every thread is past the u rows j .. j+ng-1
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      if (i >= ng) break;
#pragma unroll
      for (int gi = 0; gi < GMAX; ++gi) {
        const int gg = tid + gi * kRowThreads;
        if (gg * QW < W) L.template set_strip<QW>((p + i) % NS, gg * QW, rhs[i][gi]);
      }
    }
    __syncthreads();

    // ---- C: r2c of the rhs rows, TMA store, next step's rows into the freed slots
    // the step (1 + PF) ahead: its row jn + 1 + i goes into rhs slot (p + i)
    const int jn = j + (1 + PF) * NG, ngn = jn < r1 ? min(NG, r1 - jn) : 0;
    for (int i = g.id; i < ng; i += NG) {
      const int sl = (p + i) % NS;
      cx<T>* z = L.line(sl);
      if (IT) {
        const AddPair<T> pre{reinterpret_cast<const cx<T>*>(fpl + (size_t)(j + i) * A.f_rp)};
        fft_line<T, -1, FS>(z, A.fft, g, pre, &twc);
      } else {
        fft_line<T, -1, FS>(z, A.fft, g, NoPre{}, &twc);
      }
      r2c_post<T>(z, FS::n, TwTab<T, WSMEM>{swreal}, g);
      if (g.rank == 0) {
        if (A.sout_seg.n > 0) {  // slab plan: fused pack into the P all-to-all blocks
          const SegRows& so = A.sout_seg;
          for (int q = 0; q < so.n; ++q)
            bulk_s2g(A.Sout + so.off[q] + (long long)(j + i) * so.pitch[q], z + so.c0[q],
                     (unsigned)(((so.c0[q + 1] - so.c0[q] + 1) & ~1) * sizeof(cx<T>)));
        } else {
          bulk_s2g(A.Sout + (size_t)b * A.S_ps + (size_t)(j + i) * A.S_rp, z, spec_bytes);
        }
        if (i < ngn) {  // full steps: slot (p + i) hosts row jn + 1 + i
          bulk_wait_reads();
          ILS_ROLL_ISSUE(sl, ROWY(jn + 1 + i));
        }
#ifndef ILS_ROLL_NO_L2PF
        // one step further ahead, into L2 only (no shared memory to spare):
        // the row this slot's next load will fetch, and the f row the next
        // step's r2c adds -- the step's loads then come from L2, not DRAM
        // (3840 / 7680 wide: the planes do not fit L2)
#ifndef ILS_ROLL_L2PF_STEPS
#define ILS_ROLL_L2PF_STEPS 1
#endif
        const int y2 = jn + ILS_ROLL_L2PF_STEPS * NG + 1 + i;
        if (y2 <= r1) {
          if (IT && nseg == 0)
            prefetch_l2(Sin_b + (long long)ROWY(y2) * S_rp, spec_bytes);
          else if (!IT)
            prefetch_l2(fpl + (long long)ROWY(y2) * f_rp, (unsigned)(W * sizeof(T)));
        }
        if (IT && j + ILS_ROLL_L2PF_STEPS * NG + i < r1)
          prefetch_l2(fpl + (size_t)(j + ILS_ROLL_L2PF_STEPS * NG + i) * f_rp, (unsigned)(W * sizeof(T)));
#endif
      }
    }
    p = (p + ng) % NS;
  }
  chk = chk + (chk2.x + chk2.y);
  const bool bad = !finite_(chk);
  if (__syncthreads_or(bad) && tid == 0) atomicMin(A.status, IT ? A.iter : 0);
  bulk_wait_reads();
#undef ILS_ROLL_ISSUE
#undef ILS_ROLL_LAND
#undef ROWY
}

template <class FS>
cudaError_t launch_row_roll_impl(const RowArgs<float>& a, dim3 grid, size_t smem, int pf, cudaStream_t s);

#ifdef ILS_DEFINE_LAUNCHERS
template <class FS>
cudaError_t launch_row_roll_impl(const RowArgs<float>& a, dim3 grid, size_t smem, int pf, cudaStream_t s) {
  auto k = a.mode == MODE_IT ? (pf ? k_row_roll<FS, MODE_IT, 1> : k_row_roll<FS, MODE_IT, 0>)
                             : (pf ? k_row_roll<FS, MODE_F0, 1> : k_row_roll<FS, MODE_F0, 0>);
  cudaError_t e = smem_attr(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, kRowThreads, smem, s, a);
}
#endif

}  // namespace ils
