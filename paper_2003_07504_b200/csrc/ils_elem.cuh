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

}  // namespace ils
