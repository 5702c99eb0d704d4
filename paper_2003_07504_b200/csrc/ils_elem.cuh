// Standalone field kernels of the drop-in API (sm_100a).
//
// Inside ils_smooth these steps never touch memory: the gradients, the
// auxiliary update and the adjoint are fused into the row pass's stencil
// (ils_kernels.cuh, phase B) and the energy into its trace reduction.  The
// reference also exports them as functions (pkg/src/ilsmooth/__init__.py:
// 44-61), so callers that use them directly get these kernels:
//
//   k_grad      grad_x / grad_y            solver.py:33-40
//   k_adjoint   adjoint_accumulate         solver.py:43-49
//   k_aux       aux_update                 penalty.py:117-126 (derivative 64-66, 93-96)
//   k_energy_*  energy                     smoother.py:93-101 (value 60-62, 88-91)
//
// The arithmetic follows numpy's evaluation order with explicitly rounded
// operations (no FMA contraction), so the fp64 gradients and adjoint are
// bit-identical to the reference and aux_update / energy differ only by the
// libm pow/exp ulps and the summation order.
#pragma once

#include "ils_kernels.cuh"

namespace ils {

__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float pow_(float a, float b) { return powf(a, b); }
__device__ __forceinline__ double pow_(double a, double b) { return pow(a, b); }
__device__ __forceinline__ float exp_(float a) { return expf(a); }
__device__ __forceinline__ double exp_(double a) { return exp(a); }

// The reference's penalty in its own formulas (double-precision parameters
// narrowed once to T).
template <typename T>
struct PenaltyRef {
  int kind;  // 0 Charbonnier, 1 Welsch
  T p, eps, e, ph;  // Charbonnier: p, eps, p/2 - 1, p/2
  T g2x2;           // Welsch: 2 gamma^2
  T c, lam;
  // derivative: p * x * (x*x + eps)**(p/2 - 1)  |  2.0 * x * exp(-x*x / (2 g^2))
  __device__ __forceinline__ T derivative(T x) const {
    if (kind == 0) return mul_rn(mul_rn(p, x), pow_(add_rn(mul_rn(x, x), eps), e));
    return mul_rn(mul_rn(T(2), x), exp_(div_rn(mul_rn(-x, x), g2x2)));
  }
  // value: (x*x + eps)**(p/2)  |  2 g^2 * (1.0 - exp(-x*x / (2 g^2)))
  __device__ __forceinline__ T value(T x) const {
    if (kind == 0) return pow_(add_rn(mul_rn(x, x), eps), ph);
    return mul_rn(g2x2, sub_rn(T(1), exp_(div_rn(mul_rn(-x, x), g2x2))));
  }
};

// blockIdx.y = plane; a grid-stride loop over the plane's pixels
template <typename T>
__global__ void k_grad(const T* __restrict__ u, T* __restrict__ gx, T* __restrict__ gy, int H, int W, long long ps) {
  const long long n = (long long)H * W;
  const T* up = u + blockIdx.y * ps;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i - (long long)r * W);
    const T v = up[i];
    // np.roll(u, -1, axis) - u
    if (gx) gx[blockIdx.y * ps + i] = sub_rn(up[(long long)r * W + (c + 1 == W ? 0 : c + 1)], v);
    if (gy) gy[blockIdx.y * ps + i] = sub_rn(up[(long long)(r + 1 == H ? 0 : r + 1) * W + c], v);
  }
}

// np.roll(mu_x, 1, axis=1) - mu_x + np.roll(mu_y, 1, axis=0) - mu_y, left to right
template <typename T>
__global__ void k_adjoint(const T* __restrict__ mx, const T* __restrict__ my, T* __restrict__ out, int H, int W,
                          long long ps) {
  const long long n = (long long)H * W;
  const T* xp = mx + blockIdx.y * ps;
  const T* yp = my + blockIdx.y * ps;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i - (long long)r * W);
    T a = sub_rn(xp[(long long)r * W + (c == 0 ? W - 1 : c - 1)], xp[i]);
    a = add_rn(a, yp[(long long)(r == 0 ? H - 1 : r - 1) * W + c]);
    out[blockIdx.y * ps + i] = sub_rn(a, yp[i]);
  }
}

// c * x - derivative(x)
template <typename T>
__global__ void k_aux(const T* __restrict__ x, T* __restrict__ out, long long n, PenaltyRef<T> P) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const T v = x[i];
    out[i] = sub_rn(mul_rn(P.c, v), P.derivative(v));
  }
}

// energy partials: per plane, kEnergyBlocks blocks each write (sum d^2,
// sum phi(gx), sum phi(gy)) in f64, fixed shuffle tree and warp order
constexpr int kEnergyBlocks = 256;
template <typename T>
__global__ void k_energy_part(const T* __restrict__ u, const T* __restrict__ f, int H, int W, long long ps,
                              PenaltyRef<T> P, double* __restrict__ part) {
  __shared__ double red[32];
  const long long n = (long long)H * W;
  const T* up = u + blockIdx.y * ps;
  const T* fp = f + blockIdx.y * ps;
  double sd = 0.0, sx = 0.0, sy = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i - (long long)r * W);
    const T v = up[i];
    const T d = sub_rn(v, fp[i]);
    sd += double(mul_rn(d, d));
    sx += double(P.value(sub_rn(up[(long long)r * W + (c + 1 == W ? 0 : c + 1)], v)));
    sy += double(P.value(sub_rn(up[(long long)(r + 1 == H ? 0 : r + 1) * W + c], v)));
  }
  double* o = part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 3;
  sd = block_sum(sd, red);
  sx = block_sum(sx, red);
  sy = block_sum(sy, red);
  if (threadIdx.x == 0) {
    o[0] = sd;
    o[1] = sx;
    o[2] = sy;
  }
}

// out[b] = sum d^2 + lam * (sum phi(gx) + sum phi(gy))   (smoother.py:97-101)
__global__ void k_energy_fin(const double* __restrict__ part, int nblk, double lam, double* __restrict__ out) {
  __shared__ double red[32];
  const double* p = part + (size_t)blockIdx.x * nblk * 3;
  double s[3];
  for (int k = 0; k < 3; ++k) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) v += p[3 * i + k];
    s[k] = block_sum(v, red);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + lam * (s[1] + s[2]);
}

// dtype conversion of the drop-in's host planes (float64 numpy planes <->
// the fp32 compute planes): round to nearest even, as numpy's astype
template <typename S, typename D>
__global__ void k_convert(const S* __restrict__ src, D* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = D(src[i]);
}

// SolverPlan.denom (solver.py:100-102): 1 + (c lam / 2) (wy[r] + wx[x]),
// w = 2 - 2 cos(2 pi k / n), in float64
__global__ void k_denom(double* __restrict__ out, int H, int W, double cl2) {
  const long long n = (long long)H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), x = (int)(i - (long long)r * W);
    const double wx = 2.0 - 2.0 * cospi(2.0 * x / W);
    const double wy = 2.0 - 2.0 * cospi(2.0 * r / H);
    out[i] = __dadd_rn(1.0, __dmul_rn(cl2, wy + wx));  // numpy's roundings, no contraction
  }
}

// fft2 of real data (SolverPlan.f_hat, solver.py:69-75) from its half
// spectrum: X[k1][k2] = half[k1][k2] for k2 <= W/2, else conj(half[-k1 mod H][W - k2])
__global__ void k_hermitian_full(const cx<double>* __restrict__ half, long long pitch, cx<double>* __restrict__ full,
                                 int H, int W) {
  const long long n = (long long)H * W;
  const int wc = W / 2 + 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int k1 = (int)(i / W), k2 = (int)(i - (long long)k1 * W);
    if (k2 < wc) {
      full[i] = half[(long long)k1 * pitch + k2];
    } else {
      const cx<double> v = half[(long long)(k1 == 0 ? 0 : H - k1) * pitch + (W - k2)];
      full[i] = cx<double>{v.x, -v.y};
    }
  }
}

// detail_enhance's boost (applications.py:90-92) on given planes: clip01(u + k (f - u))
template <typename T>
__global__ void k_detail_boost(const T* __restrict__ f, const T* __restrict__ u, T* __restrict__ out, long long n,
                               T k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = detail_epilogue(u[i], f[i], k);
}

// ------------------------------------------------------------ tone mapping (applications.py:111-183)
// log10 luminance (:143, :166) narrowed to the compute type, one copy per scale plane
template <typename T>
__global__ void k_tm_log(const double* __restrict__ lum, T* __restrict__ f, long long npx, int nplanes, double off) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npx; i += (long long)gridDim.x * blockDim.x) {
    const T v = T(log10(__dadd_rn(lum[i], off)));
    for (int s = 0; s < nplanes; ++s) f[(size_t)s * npx + i] = v;
  }
}

// min / max of the coarsest base (_compress_base, :111-118): per-block partials ...
template <typename T>
__global__ void k_tm_minmax(const T* __restrict__ base, long long npx, double* __restrict__ part) {
  __shared__ double smin[32], smax[32];
  double lo = INFINITY, hi = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npx; i += (long long)gridDim.x * blockDim.x) {
    const double v = double(base[i]);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = lo;
    smax[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, smin[w]);
      hi = fmax(hi, smax[w]);
    }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
  }
}
// ... and the scalars: sc[0] = max, sc[1] = spread = max - min, sc[2] = cf = target / spread
__global__ void k_tm_minmax_fin(const double* __restrict__ part, int nblk, double target, double* __restrict__ sc) {
  if (threadIdx.x != 0) return;
  double lo = INFINITY, hi = -INFINITY;
  for (int i = 0; i < nblk; ++i) {
    lo = fmin(lo, part[2 * i]);
    hi = fmax(hi, part[2 * i + 1]);
  }
  const double spread = hi - lo;
  sc[0] = hi;
  sc[1] = spread;
  sc[2] = target / spread;
}

// log_lum_out (:145-147 single, :175-180 multi, left to right as numpy) ->
// _recolor (:121-129): clip01((C / lum)**saturation * 10**log_lum_out), float64
template <typename T>
__global__ void k_tm_finish(const double* __restrict__ lum, const double* __restrict__ rgb, const T* __restrict__ bases,
                            int nscales, long long npx, double off, double w0, double w1, double w2, double sat,
                            const double* __restrict__ sc, double* __restrict__ out) {
  const double mx = sc[0], cf = sc[2];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npx; i += (long long)gridDim.x * blockDim.x) {
    const double l = lum[i];
    const double ll = log10(__dadd_rn(l, off));
    double lo;
    if (nscales == 1) {
      const double b = double(bases[i]);
      lo = __dadd_rn(__dmul_rn(__dsub_rn(b, mx), cf), __dsub_rn(ll, b));
    } else {
      const double b0 = double(bases[i]), b1 = double(bases[npx + i]), b2 = double(bases[2 * npx + i]);
      lo = __dmul_rn(__dsub_rn(b2, mx), cf);
      lo = __dadd_rn(lo, __dmul_rn(w2, __dsub_rn(b1, b2)));
      lo = __dadd_rn(lo, __dmul_rn(w1, __dsub_rn(b0, b1)));
      lo = __dadd_rn(lo, __dmul_rn(w0, __dsub_rn(ll, b0)));
    }
    const double lum_out = pow(10.0, lo);
    for (int c = 0; c < 3; ++c) {
      const double v = __dmul_rn(pow(__ddiv_rn(rgb[(size_t)c * npx + i], l), sat), lum_out);
      out[(size_t)c * npx + i] = fmin(fmax(v, 0.0), 1.0);
    }
  }
}

}  // namespace ils
