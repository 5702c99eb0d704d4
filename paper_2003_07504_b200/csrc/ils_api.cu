// C ABI of the ILS hot path: plans, launch sequencing, host I/O pipeline.
//
// Reference interfaces replaced (see include/ils_b200.h for the per-function
// citations): make_plan/SolverPlan (solver.py:52-106), solve_ls
// (solver.py:109-134), smooth_plane/smooth_color (smoother.py:132-217).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <limits>
#include <string>
#include <vector>

#include "../../include/ils_b200.h"
#include "ils_kernels.cuh"
#include "ils_col2.cuh"
#include "ils_col3.cuh"
#include "ils_rowroll.cuh"
#include "ils_elem.cuh"

using namespace ils;

namespace {

thread_local std::string g_err;

ils_status fail(ils_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define ILS_CUDA(call)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) return fail(ILS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));     \
  } while (0)

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// ------------------------------------------------------------ radix planning
const int kUnrolled[] = {16, 15, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2};

// A group of G threads owns one n-point line; a radix-R pass gives each
// thread ceil((n/R)/G) butterflies, which must fit its KM = MAXE/R slots
// (generic primes: one butterfly per thread).
bool pass_fits(int R, long long n, int G, int maxe, bool unrolled = false) {
  const long long tasks = n / R;
  // generic primes beyond one butterfly per thread: fft_pass_bigprime, one
  // output per register slot (the device dispatch in fft_line_rt mirrors this)
  if (R > 16 && !unrolled && (R > kMaxGenericPrime || tasks > G)) return n <= (long long)maxe * G;
  const int km = (R <= 16 || unrolled) ? std::max(1, maxe / R) : 1;  // KmOf<R, ME> (ils_fft.cuh)
  return (tasks + G - 1) / G <= km;
}

struct FftHost {
  int n = 1;
  int G = 32;
  int swz = 0;  // 1: XOR-swizzled line layout
  std::vector<int> radix;
  std::vector<int> tw_off, gen_off;
  std::vector<double> tw;  // interleaved re/im
};

bool better(const std::vector<int>& a, const std::vector<int>& b) {
  if (b.empty()) return true;
  if (a.size() != b.size()) return a.size() < b.size();
  const int ma = *std::min_element(a.begin(), a.end()), mb = *std::min_element(b.begin(), b.end());
  if (ma != mb) return ma > mb;
  return a > b;
}

void dfs(int rem, int maxr, long long elems, int nthr, int maxe, std::vector<int>& cur, std::vector<int>& best,
         bool& found) {
  if (rem == 1) {
    if (!found || better(cur, best)) best = cur;
    found = true;
    return;
  }
  if (found && cur.size() + 1 > best.size()) return;
  // generic odd primes (17 and up) must stand alone, largest first (radices
  // are placed in non-increasing order)
  int big = 1;
  for (int d = 2, r = rem; d <= r; ++d) {
    if ((long long)d * d > r) d = r;
    while (r % d == 0) {
      r /= d;
      big = d;
    }
  }
  if (big >= 17) {
    if (big > maxr || !pass_fits(big, elems, nthr, maxe)) return;
    cur.push_back(big);
    dfs(rem / big, big, elems, nthr, maxe, cur, best, found);
    cur.pop_back();
    return;
  }
  for (int R : kUnrolled) {
    if (R > maxr || rem % R) continue;
    if (!pass_fits(R, elems, nthr, maxe)) continue;
    cur.push_back(R);
    dfs(rem / R, R, elems, nthr, maxe, cur, best, found);
    cur.pop_back();
  }
}

// fft_pass_bigprime holds MAXE outputs per thread of a group of <= 256: a
// line whose largest prime factor exceeds that cannot be planned
constexpr int kMaxBigPrimeLine = 16 * 256;
bool has_big_prime(int n, int dtype) {
  for (int p = 2; (long long)p * p <= n; ++p)
    while (n % p == 0) n /= p;
  return n > kMaxBigPrimeLine / (dtype == ILS_F32 ? 1 : 2);
}

struct SpecHost {
  int id, swz, G, me, n;
  std::vector<int> radix;
};
#define ILS_HOST_SPEC(ID, SWZ, GG, ME, N, ...) SpecHost{ID, SWZ, GG, ME, N, {__VA_ARGS__}},
const SpecHost kRowSpecs[] = {ILS_ROW_SPECS(ILS_HOST_SPEC)};
const SpecHost kColSpecs[] = {ILS_COL_SPECS(ILS_HOST_SPEC)};
#undef ILS_HOST_SPEC
struct Col2Host {
  int id, n1, n2, cw;
};
#define ILS_HOST_COL2(ID, N1, N2, CW, MINB) Col2Host{ID, N1, N2, CW},
const Col2Host kCol2Specs[] = {ILS_COL2_SPECS(ILS_HOST_COL2)};
#undef ILS_HOST_COL2
struct Col3Host {
  int id, n1, n2, n3, cw;
};
#define ILS_HOST_COL3(ID, N1, N2, N3, CW, MINB) Col3Host{ID, N1, N2, N3, CW},
const Col3Host kCol3Specs[] = {ILS_COL3_SPECS(ILS_HOST_COL3)};
#undef ILS_HOST_COL3

// Shared-memory wavefronts of one transform relative to the conflict-free
// ideal, for a line layout (identity or XOR swizzle), following exactly the
// index pattern of fft_pass.  E = complex elements per 128 B (16 fp32, 8 fp64);
// a warp's request is served in phases of E lanes.
double bank_cost(int n, const std::vector<int>& radix, int G, int kind, int E, int maxe) {
  const int sh = E == 16 ? 4 : 3;
  auto lay = [&](int e) {
    if (kind == 0) return e;
    const int s = kind == 1 ? (e >> sh) : (e >> sh) ^ (e >> (sh + 1));
    return e ^ (s & (E - 1));
  };
  auto wave = [&](const int* addr, const bool* act, int lanes, double& tot, double& ideal) {
    for (int p0 = 0; p0 < lanes; p0 += E) {
      int cnt[16] = {0};
      int seen[32];
      int ns = 0;
      bool any = false;
      for (int l = p0; l < p0 + E && l < lanes; ++l) {
        if (!act[l]) continue;
        any = true;
        bool dup = false;
        for (int q = 0; q < ns; ++q) dup = dup || seen[q] == addr[l];
        if (dup) continue;
        seen[ns++] = addr[l];
        cnt[addr[l] % E]++;
      }
      if (!any) continue;
      ideal += 1;
      tot += *std::max_element(cnt, cnt + E);
    }
  };
  double tot = 0, ideal = 0;
  int Ns = 1;
  const int np = (int)radix.size();
  for (int pi = 0; pi < np; ++pi) {
    const int R = radix[pi];
    // lines are identity-laid at both ends of the transform (ils_fft.cuh)
    auto lay_in = [&](int e) { return pi == 0 ? e : lay(e); };
    auto lay_out = [&](int e) { return pi == np - 1 ? e : lay(e); };
    const int nb = n / R, km = std::max(1, maxe / R);
    for (int k = 0; k < km; ++k)
      for (int w0 = 0; w0 < G; w0 += 32) {
        int ld[32], st[32];
        bool act[32];
        for (int r = 0; r < R; ++r) {
          for (int l = 0; l < 32; ++l) {
            const int j = w0 + l + k * G;
            act[l] = j < nb;
            ld[l] = lay_in(j + r * nb);
            st[l] = lay_out((j - j % Ns) * R + j % Ns + r * Ns);
          }
          wave(ld, act, 32, tot, ideal);
          wave(st, act, 32, tot, ideal);
        }
      }
    Ns *= R;
  }
  return ideal > 0 ? tot / ideal : 1.0;
}

// Radix plan + twiddles for an n-point line transform.  A compile-time spec
// (fp32 hot sizes) fixes radices, group size and layout; otherwise the plan
// with fewest passes at the smallest group size G (32..256) for which every
// pass fits, and the layout with fewer simulated bank conflicts.
bool make_fft(int n, int maxe, FftHost& out, const SpecHost* spec, int E, int maxG = 256) {
  out = FftHost{};
  out.n = n;
  if (spec) {
    for (int R : spec->radix)
      if (!pass_fits(R, n, spec->G, spec->me, true)) return false;
    out.radix = spec->radix;
    out.G = spec->G;
    out.swz = spec->swz;
  } else {
    bool ok = n <= 1;
    for (int G = 32; G <= maxG && !ok; G *= 2) {
      std::vector<int> cur, best;
      bool found = false;
      dfs(n, 1 << 30, n, G, maxe, cur, best, found);
      if (found) {
        out.radix = best;
        out.G = G;
        ok = true;
      }
    }
    if (!ok) return false;
    double best = 1e300;
    for (int kind = 0; kind < 3; ++kind) {
      const double c = bank_cost(n, out.radix, out.G, kind, E, maxe);
      if (c < best - 1e-9) {
        best = c;
        out.swz = kind;
      }
    }
  }
  if ((int)out.radix.size() > kMaxPass) return false;
  long long Ns = 1;
  for (int R : out.radix) {
    out.tw_off.push_back((int)(out.tw.size() / 2));
    if (R <= 16 || spec) {  // unrolled radices: w^m only, powers formed in registers
      for (long long m = 0; m < Ns; ++m) {
        const sc_t w = sincos2pi(-m, Ns * R);
        out.tw.push_back(w.c);
        out.tw.push_back(w.s);
      }
    } else {
      for (long long m = 0; m < Ns; ++m)
        for (int r = 1; r < R; ++r) {
          const sc_t w = sincos2pi(-(long long)r * m, Ns * R);
          out.tw.push_back(w.c);
          out.tw.push_back(w.s);
        }
    }
    out.gen_off.push_back((int)(out.tw.size() / 2));
    if (R > 16 && !spec)
      for (int q = 0; q < R; ++q) {
        const sc_t w = sincos2pi(-q, R);
        out.tw.push_back(w.c);
        out.tw.push_back(w.s);
      }
    Ns *= R;
  }
  return true;
}

}  // namespace

// ------------------------------------------------------------ plan
struct ils_plan {
  int B, H, W, N, Wc, Sp;
  bool packed;
  int dtype, device;
  ils_params prm;
  int band, row_threads, row_grid, LP;
  size_t row_smem;
  int fin_band = 0;     // rows per CTA of the final pass without trace (no halo)
  size_t fin_smem = 0;  // its shared memory
  int C, CS, col_threads, col_grid;
  bool col_wide = false;  // k_col<FftRtWide>: 512 threads, one group per line
  size_t col_smem;
  int row_spec = -1, col_spec = -1;  // compile-time FFT plan ids (-1: runtime plan)
  int col2 = -1;                     // two-stage column solve (ILS_COL2_SPECS id), -1: k_col
  int col3 = -1;                     // three-stage column solve (ILS_COL3_SPECS id), -1: none (takes precedence)
  int roll_rows = 0;                 // > 0: F0 / IT row passes by k_row_roll, chunks of this many rows
  size_t roll_smem = 0;
  int roll_pf = 0;                   // k_row_roll prefetch depth (one more set of line slots)
  int sms = 148;                     // SMs of the plan's device (waves model)
  FftHost rowf, colf;
  void* d_tables = nullptr;
  size_t off_rowtw, off_coltw, off_wreal, off_wx, off_wy, off_tw2, off_sink;  // byte offsets
  size_t spec_bytes;                                       // one half spectrum
  size_t off_fcopy;                                        // workspace: planar f of the 8-bit path
  size_t epart_elems;                                      // doubles for trace partials
  // slab decomposition (ils_slab_plan_create): this rank's rows / columns
  bool slab = false;
  int P = 1, rank = 0;
  int row0[kMaxSeg + 1] = {0}, col0[kMaxSeg + 1] = {0}, pitch[kMaxSeg] = {0};
  int Hl = 0, Wcl = 0;  // local rows, local spectrum columns
  // penalty-splitting baseline (ils_hqs_plan_create): beta_n = beta0 kappa^n
  double hqs_beta0 = 0, hqs_kappa = 0;
  uint64_t uid = 0;  // process-unique plan id (host-pipeline graph cache key)
};

namespace {

template <typename T>
size_t esz() {
  return sizeof(cx<T>);
}

template <size_t K>
int spec_me(const SpecHost (&tab)[K], int id) {
  for (const SpecHost& s : tab)
    if (s.id == id) return s.me;
  return 16;
}

template <size_t K>
const SpecHost* find_spec(const SpecHost (&tab)[K], int n) {
  if (env_int("ILS_NO_SPECS", 0)) return nullptr;
  for (const SpecHost& s : tab)
    if (s.n == n) return &s;
  return nullptr;
}

bool choose_row(ils_plan& p, int maxe, size_t elt) {
  const SpecHost* spec = (p.dtype == ILS_F32 && p.packed) ? find_spec(kRowSpecs, p.N) : nullptr;
  p.row_spec = spec ? spec->id : -1;
  if (!make_fft(p.N, maxe, p.rowf, spec, elt == 8 ? 16 : 8)) {
    if (!spec || !make_fft(p.N, maxe, p.rowf, nullptr, elt == 8 ? 16 : 8)) return false;
    p.row_spec = -1;
  }
  if (p.W > kWideMaxW || (p.W > kNarrowMaxW && !p.packed)) return false;  // stencil strip registers
  const int line = p.packed ? p.N + 1 : p.N;
  // a swizzled layout permutes inside whole 128-byte blocks: round up to them
  const int E = elt == 8 ? 16 : 8;
  // interior passes swizzle elements < n inside whole 128-byte blocks
  int LP = std::max(p.rowf.swz ? (p.N + E - 1) / E * E : 0, (line + 1) & ~1);
  if (p.rowf.swz == 3) LP = std::max(LP, (p.N + p.N / 32 + 1) & ~1);  // padded interior layout
  // packing twiddles staged in shared memory, except for kind-3 plans (L1)
#ifndef ILS_WREAL_SMEM
  const size_t wreal_bytes = (p.packed && p.rowf.swz != 3) ? (size_t)((p.N / 2 + 2) & ~1) * elt : 0;  // whole pairs
#else
  const size_t wreal_bytes = p.packed ? (size_t)((p.N / 2 + 2) & ~1) * elt : 0;
#endif
  // Band size: minimise (waves x per-CTA work).  A CTA of band b transforms
  // b+2 lines c2r and b lines r2c; k CTAs fit an SM while smem <= 228/k KB
  // and the register budget (kRowBlocksOf) allows them.
  const int force = env_int("ILS_ROW_BAND", 0);
  double best = 1e300;
  for (int band = 1; band <= std::min(p.H, kMaxBandLines - 2); ++band) {
    if (force && band != std::min(force, p.H)) continue;
    const size_t smem = (size_t)(band + 2) * LP * elt + wreal_bytes;
    if (smem > 227 * 1024) break;
    // resident CTAs/SM: register budget (kRowBlocksOf: 3 for <= 16 elements per
    // thread compile-time plans) and 228 KB of shared memory
#ifdef ILS_ROW_MINB
    const int reg_cap = ILS_ROW_MINB;
#else
    // (the cost model's resident-CTA cap: kRowBlocksOf, except that the
    // 1920-point plan keeps the 3-CTA model it was tuned with -- its band
    // choice, 5, measured best; shared memory holds it to one CTA anyway)
    const int reg_cap = p.row_spec >= 0 ? (p.N >= 3840 ? 1 : 3) : 2;
#endif
    const int per_sm = (int)std::min<size_t>(reg_cap, (228 * 1024) / (smem + 1024));
    const long ctas = (long)p.B * ((p.H + band - 1) / band);
    // issue-bound: time ~ the busiest SM's work (b+2 c2r, b r2c, b stencil rows)
    const double per_sm_ctas = (double)((ctas + p.sms - 1) / p.sms);
    const double cost = per_sm_ctas * (2.5 * band + 2.0) * (per_sm == 1 ? 1.5 : per_sm == 2 ? 1.0 : 0.9);
    if (cost < best * (1 - 1e-9)) {
      best = cost;
      p.band = band;
      p.row_smem = smem;
    }
  }
  if (best == 1e300) return false;
  // the final pass (no stencil, no halo rows) of the 3840 / 7680-wide plans:
  // registers budgeted for ILS_FIN_MINB CTAs per SM (kRowBlocksOfMode), so
  // pick its own row count per CTA that lets them share an SM
  p.fin_band = p.band + 2;
  p.fin_smem = p.row_smem;
  if (spec && p.row_spec >= 0 && spec->n >= 1920 && ILS_FIN_MINB > 1) {
    // cost ~ waves x (rows + 1) per CTA; among the rows counts within 8% of
    // the best, the smallest: a smaller CTA co-resides better with the other
    // lane's passes (4K, two lanes: 4 rows 1301 frames/s, 6 rows 1190)
    std::vector<double> cost(p.band + 3, 1e300);
    std::vector<size_t> smems(p.band + 3, 0);
    double fbest = 1e300;
    const int forced = env_int("ILS_FIN_BAND", 0);  // (tuning)
    for (int L = 1; L <= p.band + 2; ++L) {
      if (forced && L != std::min(forced, p.band + 2)) continue;
      const size_t sm = (size_t)L * LP * elt + wreal_bytes;
      const int per_sm = (int)std::min<size_t>(ILS_FIN_MINB, (228 * 1024) / (sm + 1024));
      if (per_sm < 1) break;
      const long slots = (long)p.sms * per_sm;
      const long ctas = (long)p.B * ((p.H + L - 1) / L);
      cost[L] = (double)((ctas + slots - 1) / slots) * (L + 1.0);
      smems[L] = sm;
      fbest = std::min(fbest, cost[L]);
    }
    for (int L = 1; L <= p.band + 2; ++L)
      if (cost[L] <= 1.08 * fbest) {
        p.fin_band = L;
        p.fin_smem = smems[L];
        break;
      }
  }
  p.row_threads = (spec && p.row_spec >= 0 && spec->n == 960) ? ILS_ROW_THREADS_960 : kRowThreads;
  p.LP = LP;
  p.row_grid = (p.H + p.band - 1) / p.band;
  // rolling-band first / fused passes for the wide compile-time plans: a ring
  // of (line groups + 1) slots per CTA, chunks sized for one wave of
  // resident CTAs (cost ~ waves x (rows + 2 prologue rows) per CTA)
  p.roll_rows = 0;
  if (spec && p.row_spec >= 0 && ILS_ROW_SPEC_ROLL(p.row_spec) && p.dtype == ILS_F32 && p.packed && p.W % 8 == 0 &&
      !env_int("ILS_NO_ROLL", 0)) {
    const int ng = kRowThreads / spec->G;
    const int minb = ILS_ROLL_MINB;  // kRollBlocksOf
    // slots + packing twiddles (whole pairs) + the mu_y row (ils_rowroll.cuh);
    // the prefetching ring (2 NG + 1 slots) when it still fits minb CTAs per SM
    auto roll_smem = [&](int pf) {
      return (size_t)((1 + pf) * ng + 1) * LP * elt + (size_t)((p.N / 2 + 2) & ~1) * elt + (size_t)p.W * sizeof(float);
    };
    // (prefetch depth 1 measured no faster at 3840 -- 178.7 vs 176.2 us per
    // 4K RGB fused pass -- and it halves the resident CTAs at 7680: opt-in)
    p.roll_pf = env_int("ILS_ROLL_PF", 0) > 0 && (228 * 1024) / (roll_smem(1) + 1024) >= (size_t)minb;
    const size_t smem = roll_smem(p.roll_pf);
    const int per_sm = (int)std::min<size_t>(minb, (228 * 1024) / (smem + 1024));
    if (per_sm >= 1) {
      const long slots = (long)p.sms * per_sm;
      double rbest = 1e300;
      const int forced = env_int("ILS_ROLL_ROWS", 0);
      for (int R = forced ? 1 : 2; R <= p.H; ++R) {
        if (forced && R != std::min(forced, p.H)) continue;
        const long ctas = (long)p.B * ((p.H + R - 1) / R);
        const double cost = (double)((ctas + slots - 1) / slots) * (R + 2);
        if (cost < rbest * (1 - 1e-9)) {
          rbest = cost;
          p.roll_rows = R;
        }
      }
      p.roll_smem = smem;
    }
  }
  return true;
}

bool choose_col(ils_plan& p, int maxe, size_t elt) {
  const SpecHost* spec = p.dtype == ILS_F32 ? find_spec(kColSpecs, p.H) : nullptr;
  p.col_spec = spec ? spec->id : -1;
  p.col_wide = false;
  if (!make_fft(p.H, maxe, p.colf, spec, elt == 8 ? 16 : 8)) {
    p.col_spec = -1;
    if (!make_fft(p.H, maxe, p.colf, nullptr, elt == 8 ? 16 : 8)) {
      // long columns: one 512-thread group per line (k_col<FftRtWide>)
      if (!make_fft(p.H, maxe, p.colf, nullptr, elt == 8 ? 16 : 8, 2 * kColThreads)) return false;
      p.col_wide = true;
    }
  }
  const int E = elt == 8 ? 16 : 8;  // complex elements per 128 B
  const int col_nt = p.col_wide ? 2 * kColThreads : kColThreads;
  const int ngroups = col_nt / p.colf.G;
  const int force = env_int("ILS_COL_COLS", 0);
  const int base = (p.H + E - 1) / E * E;
  double best = 1e300;
  for (int C = 1; C <= std::min(p.Wc, 32); ++C) {
    if (force && C != std::min(force, p.Wc)) continue;
    // line pitch: pick the offset whose transposing copy has fewest conflicts
    int bestCS = base;
    int bestw = 1 << 30;
    for (int o = 0; o < E; ++o) {
      const int CS = base + o;
      int tot = 0;
      for (int t0 = 0; t0 < 64; t0 += E) {
        int cnt[16] = {0};
        for (int t = t0; t < t0 + E; ++t) {
          const int y = t / C, c = t % C;
          const int e = c * CS + y;  // tile lines are identity-laid outside the FFT passes
          cnt[e % E]++;
        }
        tot += *std::max_element(cnt, cnt + E);
      }
      if (tot < bestw) {
        bestw = tot;
        bestCS = CS;
      }
    }
    const size_t smem = (size_t)C * bestCS * elt + (size_t)p.H * (elt / 2);  // tile + wy
    if (smem > 227 * 1024) break;
    // resident CTAs/SM: k_col is register-bounded to 3 (launch bounds), smem to 228 KB
    const int per_sm = (int)std::min<size_t>(p.col_wide ? 1 : kColMinBlocks, (228 * 1024) / (smem + 1024));
    const long strips = (p.Wc + C - 1) / C;
    const long ctas = (long)p.B * strips;
    // the pass is issue-bound: time ~ the busiest SM's column count
    const double per_sm_ctas = (double)((ctas + p.sms - 1) / p.sms);
    // 32-byte sectors a strip's row segment touches (rows are 32 B aligned)
    double sectors = 0;
    for (long s = 0; s < strips; ++s) {
      const long b0 = s * C * (long)elt, b1 = std::min<long>((s + 1) * C, p.Wc) * (long)elt;
      sectors += (double)((b1 + 31) / 32 - b0 / 32);
    }
    sectors /= strips;
    const double col_sectors = (double)elt / 32.0;  // one column's share at perfect coalescing
    const double cost = per_sm_ctas * (C + 0.25 * (sectors / col_sectors - C) + 0.5) * (per_sm == 1 ? 1.5 : 1.0);
    if (cost < best * (1 - 1e-6) || (cost < best * (1 + 1e-6) && C > p.C)) {
      best = cost;
      p.C = C;
      p.CS = bestCS;
      p.col_smem = smem;
    }
  }
  if (best == 1e300) return false;
  p.col_threads = col_nt;
  p.col_grid = (p.Wc + p.C - 1) / p.C;
  // the solve pass (COL_SOLVE) of fp32 plans whose height has a two-stage
  // kernel runs k_col2; the standalone transforms keep k_col
  p.col2 = -1;
  if (p.dtype == ILS_F32 && !env_int("ILS_NO_SPECS", 0) && !env_int("ILS_NO_COL2", 0))
    for (const Col2Host& c : kCol2Specs)
      if (c.n1 * c.n2 == p.H && p.col2 < 0) p.col2 = c.id;
  const int force2 = env_int("ILS_COL2_SPEC", -1);
  if (p.col2 >= 0 && force2 >= 0)
    for (const Col2Host& c : kCol2Specs)
      if (c.id == force2 && c.n1 * c.n2 == p.H) p.col2 = c.id;
  // the three-stage kernel is opt-in (ILS_COL3_SPEC=id, or -2 for the first
  // split of H): measured no faster than k_col2 at 1080 rows and slower at
  // 2160 / 4320, so k_col2 stays the default
  p.col3 = -1;
  const int force3 = env_int("ILS_COL3_SPEC", -1);
  if (p.dtype == ILS_F32 && !env_int("ILS_NO_SPECS", 0) && force3 != -1)
    for (const Col3Host& c : kCol3Specs)
      if (c.n1 * c.n2 * c.n3 == p.H && (force3 < 0 ? p.col3 < 0 : c.id == force3)) p.col3 = c.id;
  return true;
}

template <typename T>
void fill_fft_dev(FftDev<T>& d, const FftHost& h, const void* base, size_t off) {
  d.n = h.n;
  d.G = h.G;
  d.laykind = h.swz;
  d.npass = (int)h.radix.size();
  for (int i = 0; i < kMaxPass; ++i) {
    d.radix[i] = i < d.npass ? h.radix[i] : 1;
    d.tw_off[i] = i < d.npass ? h.tw_off[i] : 0;
    d.gen_off[i] = i < d.npass ? h.gen_off[i] : 0;
  }
  d.tw = reinterpret_cast<const cx<T>*>(static_cast<const char*>(base) + off);
}

template <typename T>
PenaltyDev<T> pen_dev(const ils_params& q) {
  PenaltyDev<T> P{};
  P.kind = q.kind;
  P.p = T(q.p);
  P.pe = T(q.p / 2.0 - 1.0);
  P.ph = T(q.p / 2.0);
  P.eps = T(q.eps);
  const double g2 = q.gamma * q.gamma;
  const double log2e = 1.4426950408889634;  // exp(x) = 2^(x log2 e)
  P.wk = q.kind == ILS_WELSCH ? T(-log2e / (2.0 * g2)) : T(0);
  P.eps0 = q.kind == ILS_CHARBONNIER ? T(q.eps) : T(0);
  P.E = q.kind == ILS_CHARBONNIER ? T(q.p / 2.0 - 1.0) : P.wk;
  P.coef = q.kind == ILS_CHARBONNIER ? T(-q.p) : T(-2.0);
  P.floor = -std::numeric_limits<T>::infinity();
  P.g2x2 = T(2.0 * g2);
  P.c = T(q.c);
  P.lam = T(q.lam);
  P.lam2 = T(q.lam / 2.0);
  return P;
}

// HQS iteration n (hqs.py:49-66): field step m = soft_threshold(grad u, alpha)
// with alpha = lam / (2 beta_n), then solve_ls with lam_n = 2 beta_n, c = 1,
// i.e. rhs = f + beta_n D^T m and denominator 1 + beta_n (wy + wx).  The soft
// threshold is the penalty form mu = x max(1 - alpha |x|^-1, 0).
double hqs_beta(const ils_plan* p, int n) { return p->hqs_beta0 * std::pow(p->hqs_kappa, n); }

template <typename T>
PenaltyDev<T> pen_soft(double alpha, double beta) {
  PenaltyDev<T> P{};
  P.kind = ILS_SOFT;
  P.eps0 = T(0);
  P.E = T(-0.5);
  P.coef = T(-alpha);
  P.c = T(1);
  P.floor = T(0);
  P.lam = T(2.0 * beta);
  P.lam2 = T(beta);
  return P;
}

template <typename T>
RowArgs<T> row_args(const ils_plan* p) {
  RowArgs<T> a{};
  a.wrap = 1;
  a.B = p->B;
  a.H = p->H;
  a.W = p->W;
  a.N = p->N;
  a.Wc = p->Wc;
  a.band = p->band;
  a.LP = p->LP;
  a.S_rp = p->Sp;
  a.S_ps = (long long)p->H * p->Sp;
  a.pen = pen_dev<T>(p->prm);
  fill_fft_dev<T>(a.fft, p->rowf, p->d_tables, p->off_rowtw);
  a.wreal = reinterpret_cast<const cx<T>*>(static_cast<const char*>(p->d_tables) + p->off_wreal);
  return a;
}

template <typename T>
ColArgs<T> col_args(const ils_plan* p, cx<T>* S, int mode) {
  ColArgs<T> a{};
  a.B = p->B;
  a.H = p->H;
  a.Wc = p->Wc;
  a.C = p->C;
  a.CS = p->CS;
  a.S = S;
  a.S_rp = p->Sp;
  a.S_ps = (long long)p->H * p->Sp;
  a.wx = reinterpret_cast<const T*>(static_cast<const char*>(p->d_tables) + p->off_wx);
  a.wy = reinterpret_cast<const T*>(static_cast<const char*>(p->d_tables) + p->off_wy);
  a.tw2 = reinterpret_cast<const cx<T>*>(static_cast<const char*>(p->d_tables) + p->off_tw2);
  a.cl2 = T(p->prm.c * p->prm.lam / 2.0);
  a.inv_hw = T(1.0 / ((double)p->H * (double)p->W));
  a.mode = mode;
  fill_fft_dev<T>(a.fft, p->colf, p->d_tables, p->off_coltw);
  return a;
}

template <typename T>
cudaError_t launch_row(const ils_plan* p, int mode, RowArgs<T> a, cudaStream_t s) {
  a.mode = mode;
  // the final pass without energy trace needs no halo rows: it fills the
  // band's 2 halo line slots with 2 more rows of its own (same shared memory,
  // one CTA transforms band + 2 lines in the same round of line groups)
  int gx = p->row_grid;
  size_t smem = p->row_smem;
  if (mode == MODE_FIN && a.epart == nullptr) {
    a.band = p->fin_band;
    gx = (p->H + a.band - 1) / a.band;
    smem = p->fin_smem;
  }
  const dim3 grid(gx, p->B);
  if constexpr (std::is_same<T, float>::value) {
    // rolling band: plain periodic planes, no trace / 8-bit ingest / soft threshold
    const bool roll = p->roll_rows > 0 && (mode == MODE_F0 || mode == MODE_IT) && a.wrap == 1 && a.sin_seg.n == 0 &&
                      a.sout_seg.n == 0 && a.epart == nullptr && a.f8 == nullptr && a.pen.kind != ILS_SOFT;
    if (roll) {
      a.band = p->roll_rows;
      const dim3 rgrid((p->H + p->roll_rows - 1) / p->roll_rows, p->B);
      switch (p->row_spec) {
#define ILS_CASE(ID, ...)                                                        \
  case ID:                                                                       \
    if constexpr (ILS_ROW_SPEC_ROLL(ID))                                         \
      return launch_row_roll_impl<RowSpec<ID>::type>(a, rgrid, p->roll_smem, p->roll_pf, s); \
    break;
        ILS_ROW_SPECS(ILS_CASE)
#undef ILS_CASE
        default:
          break;
      }
    }
    switch (p->row_spec) {
#define ILS_CASE(ID, ...) \
  case ID:                \
    return launch_row_impl<float, true, RowSpec<ID>::type, ILS_ROW_SPEC_WIDE(ID)>(a, grid, p->row_threads, smem, s);
      ILS_ROW_SPECS(ILS_CASE)
#undef ILS_CASE
      default:
        break;
    }
  }
  if (p->W > kNarrowMaxW) return launch_row_impl<T, true, FftRt, true>(a, grid, p->row_threads, smem, s);
  return p->packed ? launch_row_impl<T, true, FftRt>(a, grid, p->row_threads, smem, s)
                   : launch_row_impl<T, false, FftRt>(a, grid, p->row_threads, smem, s);
}

template <typename T>
cudaError_t launch_col2(const ils_plan* p, const ColArgs<T>& a, int planes, cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value) {
    switch (p->col2) {
#define ILS_CASE(ID, N1, N2, CW, MINB) \
  case ID:                             \
    return launch_col2_impl<N1, N2, CW, MINB>(a, planes, s);
      ILS_COL2_SPECS(ILS_CASE)
#undef ILS_CASE
      default:
        break;
    }
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_col3(const ils_plan* p, const ColArgs<T>& a, int planes, cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value) {
    switch (p->col3) {
#define ILS_CASE(ID, N1, N2, N3, CW, MINB) \
  case ID:                                 \
    return launch_col3_impl<N1, N2, N3, CW, MINB>(a, planes, s);
      ILS_COL3_SPECS(ILS_CASE)
#undef ILS_CASE
      default:
        break;
    }
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_col(const ils_plan* p, const ColArgs<T>& a, cudaStream_t s) {
  if (p->col3 >= 0 && a.mode == COL_SOLVE) return launch_col3<T>(p, a, p->B, s);
  if (p->col2 >= 0 && a.mode == COL_SOLVE) return launch_col2<T>(p, a, p->B, s);
  const dim3 grid(p->col_grid, p->B);
  if constexpr (std::is_same<T, float>::value) {
    switch (p->col_spec) {
#define ILS_CASE(ID, ...) \
  case ID:                \
    return launch_col_impl<float, ColSpec<ID>::type>(a, grid, p->col_threads, p->col_smem, s);
      ILS_COL_SPECS(ILS_CASE)
#undef ILS_CASE
      default:
        break;
    }
  }
  if (p->col_wide) return launch_col_impl<T, FftRtWide>(a, grid, p->col_threads, p->col_smem, s);
  return launch_col_impl<T, FftRt>(a, grid, p->col_threads, p->col_smem, s);
}

// f8 / u8 (8-bit interleaved frames, ch channels): F0 reads f8 and keeps a
// planar copy of f in the workspace for the later passes; FIN writes u8.
template <typename T>
ils_status smooth_t(const ils_plan* p, const T* f, T* u, int64_t ps, void* ws, cudaStream_t s, int32_t* status,
                    double* energies, const unsigned char* f8 = nullptr, unsigned char* u8 = nullptr, int ch = 1,
                    const ils_epilogue* epi = nullptr, const double* plane_lam = nullptr, int nlam = 0) {
  cx<T>* Sa = static_cast<cx<T>*>(ws);
  cx<T>* Sb = reinterpret_cast<cx<T>*>(static_cast<char*>(ws) + p->spec_bytes);
  double* ep = reinterpret_cast<double*>(static_cast<char*>(ws) + 2 * p->spec_bytes + 256);
  const size_t per_pass = (size_t)p->B * p->row_grid;
  ILS_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int32_t), s));
  RowArgs<T> a = row_args<T>(p);
  a.f = f;
  a.f_ps = ps;
  a.f_rp = p->W;
  a.u = u;
  a.u_ps = ps;
  a.u_rp = p->W;
  a.status = status;
  // per-plane lambda: the values the uniform plan would derive for that lambda
  // (pen_dev: lam / 2, col_args: c lam / 2), so a plane's result is bitwise
  // the one of a plan built for its own lambda
  T cl2_tab[kMaxPlaneLam] = {};
  if (nlam > 0) {
    if (nlam > kMaxPlaneLam || energies || p->prm.kind == ILS_SOFT) return fail(ILS_EINVAL, "bad per-plane lambda table");
    a.nlam = nlam;
    for (int k = 0; k < nlam; ++k) {
      a.lam2_tab[k] = T(plane_lam[k] / 2.0);
      cl2_tab[k] = T(p->prm.c * plane_lam[k] / 2.0);
    }
  }
  if (f8) {
    // 8-bit ingest: deinterleave + v/255 into the workspace's planar f, which
    // every row pass (F0 included) then reads as an ordinary fp32 plane
    a.ch = ch;
    a.fcopy = reinterpret_cast<T*>(static_cast<char*>(ws) + p->off_fcopy);
    a.f = a.fcopy;
    a.f_ps = (int64_t)p->H * p->W;
    // compile-time fp32 plans with 3-channel rows: the first row pass loads the
    // interleaved byte rows itself (TMA into the tail of each line slot) and
    // writes the planar f on the way; otherwise a separate deinterleave kernel
    const bool fuse = std::is_same<T, float>::value && p->row_spec >= 0 && p->packed && p->W % 128 == 0 &&
                      ch == 3 && (size_t)p->LP * sizeof(cx<T>) >= (size_t)p->W * (ch + 1) &&
                      reinterpret_cast<uintptr_t>(f8) % 16 == 0 &&
                      !env_int("ILS_NO_FUSED_INGEST", 0);
    if (fuse) {
      a.f8 = f8;
    } else {
      const int npx = p->H * p->W;
      const int frames = p->B / ch;
      const long long work = (ch == 3 && (npx & 3) == 0) ? npx / 4 : (long long)npx * ch;  // per frame
      const int bx =
          (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, (long long)p->sms * 8 / frames));
      k_u8_planar<T><<<dim3(bx, frames), 256, 0, s>>>(f8, a.fcopy, ch, npx);
      ILS_CUDA(cudaGetLastError());
    }
  }
  const int iters = p->prm.iters;
  cx<T>* cur = Sa;
  cx<T>* nxt = Sb;
  const bool hqs = p->prm.kind == ILS_SOFT;
  for (int n = 0; n < iters; ++n) {
    a.iter = n;
    a.Sin = n == 0 ? nullptr : cur;
    a.Sout = n == 0 ? cur : nxt;
    a.epart = energies ? ep + n * per_pass : nullptr;
    if (hqs) a.pen = pen_soft<T>(p->prm.lam / (2.0 * hqs_beta(p, n)), hqs_beta(p, n));
    ILS_CUDA(launch_row<T>(p, n == 0 ? MODE_F0 : MODE_IT, a, s));
    a.f8 = nullptr;
    if (n > 0) std::swap(cur, nxt);
    ColArgs<T> ca = col_args<T>(p, cur, COL_SOLVE);
    if (hqs) ca.cl2 = T(hqs_beta(p, n));
    if (nlam > 0) {
      ca.nlam = nlam;
      for (int k = 0; k < nlam; ++k) ca.cl2_tab[k] = cl2_tab[k];
    }
    ILS_CUDA(launch_col<T>(p, ca, s));
  }
  a.iter = iters;
  a.Sin = cur;
  a.Sout = nullptr;
  a.epart = energies ? ep + iters * per_pass : nullptr;
  a.u8 = u8;
  a.ch = ch;
  if (epi && epi->kind == ILS_EPI_DETAIL) {
    a.epi = 1;
    a.epi_k = T(epi->k);
    if (f8) a.f = a.fcopy;
  }
  ILS_CUDA(launch_row<T>(p, MODE_FIN, a, s));
  if (energies) {
    for (int n = 0; n <= iters; ++n) {
      k_energy_reduce<<<p->B, 256, 0, s>>>(ep + n * per_pass, p->row_grid, p->B, energies + (size_t)n * p->B);
    }
    ILS_CUDA(cudaGetLastError());
  }
  return ILS_OK;
}

template <typename T>
ils_status solve_t(const ils_plan* p, const T* f, const T* mx, const T* my, T* u, int64_t ps, void* ws,
                   cudaStream_t s, int32_t* status) {
  cx<T>* Sa = static_cast<cx<T>*>(ws);
  ILS_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int32_t), s));
  RowArgs<T> a = row_args<T>(p);
  a.f = f;
  a.mux = mx;
  a.muy = my;
  a.f_ps = ps;
  a.f_rp = p->W;
  a.u = u;
  a.u_ps = ps;
  a.u_rp = p->W;
  a.status = status;
  a.iter = 1;
  a.Sout = Sa;
  ILS_CUDA(launch_row<T>(p, MODE_MU, a, s));
  ILS_CUDA(launch_col<T>(p, col_args<T>(p, Sa, COL_SOLVE), s));
  a.Sin = Sa;
  a.Sout = nullptr;
  a.f = nullptr;
  ILS_CUDA(launch_row<T>(p, MODE_FIN, a, s));
  return ILS_OK;
}

ils_status plan_create_impl(ils_plan** out, int32_t batch, int32_t height, int32_t width, const ils_params* params,
                            int32_t dtype, int32_t device, double hqs_beta0, double hqs_kappa);

// Runs an entry point on the plan's device (restoring the caller's current
// device on exit), so a plan built for cuda:1 works whatever device the
// calling thread has selected.
struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) changed = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

// Plane buffers the row passes move as whole rows: packed plans load / store
// sample pairs as one complex element (2 * sizeof(T) alignment, even plane
// stride); compile-time fp32 plans move whole rows with TMA bulk copies
// (16-byte aligned rows: pointer and plane stride in bytes multiples of 16).
ils_status check_io(const ils_plan* p, const void* f, const void* u, int64_t ps) {
  if (!p->packed) return ILS_OK;
  const size_t es = p->dtype == ILS_F32 ? 4 : 8;
  const bool bulk = p->dtype == ILS_F32 && p->row_spec >= 0 && p->W % 8 == 0;
  const size_t al = bulk ? 16 : 2 * es;
  for (const void* q : {f, u})
    if (q && reinterpret_cast<uintptr_t>(q) % al)
      return fail(ILS_EINVAL, "plane buffer %p is not %zu-byte aligned (required for %dx%d planes)", q, al, p->H, p->W);
  if (((size_t)ps * es) % al)
    return fail(ILS_EINVAL, "plane_stride %lld elements is not a multiple of %zu bytes (required for %dx%d planes)",
                (long long)ps, al, p->H, p->W);
  return ILS_OK;
}


ils_status validate(const ils_params* q) {
  if (!q) return fail(ILS_EINVAL, "params is NULL");
  if (!(q->lam > 0.0 && std::isfinite(q->lam))) return fail(ILS_EINVAL, "lam must be finite and positive, got %g", q->lam);
  if (q->iters < 1) return fail(ILS_EINVAL, "iters must be an integer >= 1, got %d", q->iters);
  double c0;
  if (q->kind == ILS_CHARBONNIER) {
    if (!(q->p > 0.0 && q->p <= 1.0)) return fail(ILS_EINVAL, "p must be in (0,1]");
    if (!(q->eps > 0.0)) return fail(ILS_EINVAL, "eps must be positive, got %g", q->eps);
    c0 = q->p * std::pow(q->eps, q->p / 2.0 - 1.0);
  } else if (q->kind == ILS_WELSCH) {
    if (!(q->gamma > 0.0)) return fail(ILS_EINVAL, "gamma must be positive, got %g", q->gamma);
    c0 = 2.0;
  } else {
    return fail(ILS_EINVAL, "unknown penalty kind %d", q->kind);
  }
  if (!std::isfinite(q->c) || q->c < c0 * (1.0 - 1e-12))
    return fail(ILS_EINVAL, "c=%.17g is below the penalty's minimum curvature %.17g", q->c, c0);
  return ILS_OK;
}

}  // namespace

extern "C" {

int32_t ils_abi_version(void) { return ILS_ABI_VERSION; }
const char* ils_last_error(void) { return g_err.c_str(); }

ils_status ils_plan_create(ils_plan** out, int32_t batch, int32_t height, int32_t width, const ils_params* params,
                           int32_t dtype, int32_t device) {
  if (!out) return fail(ILS_EINVAL, "out is NULL");
  *out = nullptr;
  ils_status st = validate(params);
  if (st != ILS_OK) return st;
  return plan_create_impl(out, batch, height, width, params, dtype, device, 0.0, 0.0);
}

ils_status ils_hqs_plan_create(ils_plan** out, int32_t batch, int32_t height, int32_t width,
                               const ils_hqs_params* hp, int32_t dtype, int32_t device) {
  if (!out) return fail(ILS_EINVAL, "out is NULL");
  *out = nullptr;
  if (!hp) return fail(ILS_EINVAL, "params is NULL");
  // HqsParams.__post_init__ (hqs.py:33-43)
  if (!(hp->lam > 0.0 && std::isfinite(hp->lam))) return fail(ILS_EINVAL, "lam must be finite and positive, got %g", hp->lam);
  if (hp->beta0 != 0.0 && !(hp->beta0 > 0.0 && std::isfinite(hp->beta0)))
    return fail(ILS_EINVAL, "beta0 must be finite and positive, got %g", hp->beta0);
  if (!(hp->kappa > 1.0 && std::isfinite(hp->kappa))) return fail(ILS_EINVAL, "kappa must be finite and > 1, got %g", hp->kappa);
  if (hp->iters < 1) return fail(ILS_EINVAL, "iters must be an integer >= 1, got %d", hp->iters);
  ils_params q{};
  q.kind = ILS_SOFT;
  q.lam = hp->lam;
  q.c = 1.0;
  q.iters = hp->iters;
  const double beta0 = hp->beta0 == 0.0 ? 2.0 * hp->lam : hp->beta0;  // HqsParams.initial_beta (hqs.py:45-47)
  return plan_create_impl(out, batch, height, width, &q, dtype, device, beta0, hp->kappa);
}

}  // extern "C"

namespace {

ils_status plan_create_impl(ils_plan** out, int32_t batch, int32_t height, int32_t width, const ils_params* params,
                            int32_t dtype, int32_t device, double hqs_beta0, double hqs_kappa) {
  if (batch < 1) return fail(ILS_EINVAL, "batch must be >= 1, got %d", batch);
  if (height < 1 || width < 1) return fail(ILS_EINVAL, "invalid plan size %dx%d", height, width);
  if (dtype != ILS_F32 && dtype != ILS_F64) return fail(ILS_EINVAL, "unknown dtype %d", dtype);
  if (has_big_prime(height, dtype) || has_big_prime(width % 2 == 0 ? width / 2 : width, dtype))
    return fail(ILS_EUNSUPPORTED, "plane size %dx%d has a prime factor beyond the direct-DFT pass (%d)", height,
                width, kMaxBigPrimeLine / (dtype == ILS_F32 ? 1 : 2));
  ils_plan* p = new ils_plan();
  p->B = batch;
  p->H = height;
  p->W = width;
  p->packed = (width % 2 == 0);
  p->N = p->packed ? width / 2 : width;
  p->Wc = width / 2 + 1;
  p->Sp = (p->Wc + 3) & ~3;  // 32-byte aligned spectrum rows (fp32)
  p->dtype = dtype;
  p->device = device;
  p->prm = *params;
  p->hqs_beta0 = hqs_beta0;
  p->hqs_kappa = hqs_kappa;
  static std::atomic<uint64_t> next_uid{1};
  p->uid = next_uid++;
  const size_t elt = dtype == ILS_F32 ? sizeof(cx<float>) : sizeof(cx<double>);
  const int maxe = dtype == ILS_F32 ? 16 : 8;
  if (device >= 0) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0) p->sms = sms;
  }
  if (!choose_row(*p, maxe, elt) || !choose_col(*p, maxe, elt)) {
    delete p;
    return fail(ILS_EUNSUPPORTED, "no launch configuration fits plane size %dx%d", height, width);
  }
  // device tables: row twiddles, col twiddles, wreal, wx, wy (all in T)
  const size_t rs = dtype == ILS_F32 ? 4 : 8;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  p->off_rowtw = off;
  off = align(off + p->rowf.tw.size() * rs);
  p->off_coltw = off;
  off = align(off + p->colf.tw.size() * rs);
  p->off_wreal = off;
  const int nwr = p->N / 2 + 1;
  off = align(off + 2 * nwr * rs);
  p->off_wx = off;
  off = align(off + p->Wc * rs);
  p->off_wy = off;
  off = align(off + p->H * rs);
  p->off_tw2 = off;
  off = align(off + 2 * p->H * rs);
  p->off_sink = off;  // scratch status word for ils_irfft2
  off += 256;
  std::vector<double> host(off / 8 + 1, 0.0);
  std::vector<char> bytes(off, 0);
  auto put = [&](size_t o, const std::vector<double>& v) {
    if (dtype == ILS_F64) {
      memcpy(bytes.data() + o, v.data(), v.size() * 8);
    } else {
      std::vector<float> f(v.begin(), v.end());
      memcpy(bytes.data() + o, f.data(), f.size() * 4);
    }
  };
  put(p->off_rowtw, p->rowf.tw);
  put(p->off_coltw, p->colf.tw);
  std::vector<double> wr(2 * nwr), wx(p->Wc), wy(p->H);
  for (int k = 0; k < nwr; ++k) {
    const sc_t w = sincos2pi(-k, width);
    wr[2 * k] = w.c;
    wr[2 * k + 1] = w.s;
  }
  // w = 2 - 2 cos(2 pi k / n): solver.py:100-101
  for (int k = 0; k < p->Wc; ++k) wx[k] = 2.0 - 2.0 * sincos2pi(k, width).c;
  for (int k = 0; k < p->H; ++k) wy[k] = 2.0 - 2.0 * sincos2pi(k, height).c;
  put(p->off_wreal, wr);
  put(p->off_wx, wx);
  put(p->off_wy, wy);
  std::vector<double> tw2(2 * p->H);  // exp(-2 pi i m / H)
  for (int m = 0; m < p->H; ++m) {
    const sc_t w = sincos2pi(-m, height);
    tw2[2 * m] = w.c;
    tw2[2 * m + 1] = w.s;
  }
  put(p->off_tw2, tw2);
  p->spec_bytes = ((size_t)batch * height * p->Sp * elt + 255) & ~size_t(255);
  p->epart_elems = (size_t)(params->iters + 1) * batch * p->row_grid;
  p->off_fcopy = (2 * p->spec_bytes + 256 + p->epart_elems * sizeof(double) + 255) & ~size_t(255);
  if (device < 0) {  // host-only plan: planning/introspection, cannot run
    *out = p;
    return ILS_OK;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_tables, off);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_tables, bytes.data(), off, cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (p->d_tables) cudaFree(p->d_tables);
    delete p;
    return fail(ILS_ECUDA, "plan tables: %s", cudaGetErrorString(e));
  }
  *out = p;
  return ILS_OK;
}

}  // namespace

extern "C" {

void ils_plan_destroy(ils_plan* p) {
  if (!p) return;
  if (p->d_tables) cudaFree(p->d_tables);
  delete p;
}

ils_status ils_workspace_size(const ils_plan* p, size_t* bytes) {
  if (!p || !bytes) return fail(ILS_EINVAL, "NULL argument");
  // [Sa][Sb][status][trace partials][planar f of the 8-bit path]
  *bytes = p->off_fcopy + (size_t)p->B * p->H * p->W * (p->dtype == ILS_F32 ? 4 : 8);
  return ILS_OK;
}

ils_status ils_plan_get_info(const ils_plan* p, ils_plan_info* i) {
  if (!p || !i) return fail(ILS_EINVAL, "NULL argument");
  memset(i, 0, sizeof *i);
  i->batch = p->B;
  i->height = p->H;
  i->width = p->W;
  i->dtype = p->dtype;
  i->packed = p->packed;
  i->row_band = p->band;
  i->row_threads = p->row_threads;
  i->row_group = p->rowf.G;
  i->col_group = p->colf.G;
  i->row_spec = p->row_spec;
  i->col_spec = p->col_spec;
  i->row_swz = p->rowf.swz;
  i->col_swz = p->colf.swz;
  i->row_grid = p->row_grid;
  i->row_smem = (int32_t)p->row_smem;
  i->col_cols = p->C;
  i->col_threads = p->col_threads;
  i->col_grid = p->col_grid;
  i->col_smem = (int32_t)p->col_smem;
  i->row_passes = (int32_t)p->rowf.radix.size();
  i->col_passes = (int32_t)p->colf.radix.size();
  for (size_t k = 0; k < p->rowf.radix.size() && k < 16; ++k) i->row_radix[k] = p->rowf.radix[k];
  for (size_t k = 0; k < p->colf.radix.size() && k < 16; ++k) i->col_radix[k] = p->colf.radix[k];
  i->spec_pitch = p->Sp;
  i->launches_per_call = 2 * p->prm.iters + 1;
  i->col2_spec = p->col2;
  for (const Col2Host& c : kCol2Specs)
    if (c.id == p->col2) {
      i->col2_n1 = c.n1;
      i->col2_n2 = c.n2;
      i->col2_cols = c.cw;
    }
  i->row_roll_rows = p->roll_rows;
  i->col3_spec = p->col3;
  for (const Col3Host& c : kCol3Specs)
    if (c.id == p->col3) {
      i->col3_n1 = c.n1;
      i->col3_n2 = c.n2;
      i->col3_n3 = c.n3;
      i->col3_cols = c.cw;
    }
  return ILS_OK;
}

ils_status ils_smooth(const ils_plan* p, const void* f, void* u, int64_t ps, void* ws, void* stream, int32_t* status,
                      double* energies) {
  if (!p || !f || !u || !ws || !status) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (p->slab) return fail(ILS_EINVAL, "slab plans run through ils_slab_row_pass / ils_slab_col_pass");
  if (ps < (int64_t)p->H * p->W) return fail(ILS_EINVAL, "plane_stride %lld < H*W", (long long)ps);
  if (energies && p->prm.kind == ILS_SOFT) return fail(ILS_EINVAL, "the penalty-splitting baseline has no energy trace");
  if (ils_status st = check_io(p, f, u, ps)) return st;
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->dtype == ILS_F32)
    return smooth_t<float>(p, static_cast<const float*>(f), static_cast<float*>(u), ps, ws, s, status, energies);
  return smooth_t<double>(p, static_cast<const double*>(f), static_cast<double*>(u), ps, ws, s, status, energies);
}

ils_status ils_smooth_epilogue(const ils_plan* p, const void* f, void* u, int64_t ps, void* ws, void* stream,
                              int32_t* status, const ils_epilogue* epi) {
  if (!p || !f || !u || !ws || !status || !epi) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (p->slab) return fail(ILS_EINVAL, "slab plans run through ils_slab_row_pass / ils_slab_col_pass");
  if (ps < (int64_t)p->H * p->W) return fail(ILS_EINVAL, "plane_stride %lld < H*W", (long long)ps);
  if (epi->kind != ILS_EPI_NONE && epi->kind != ILS_EPI_DETAIL) return fail(ILS_EINVAL, "unknown epilogue %d", epi->kind);
  if (!(epi->k >= 0.0 && std::isfinite(epi->k)))  // DetailBoost.__post_init__ (applications.py:29-31)
    return fail(ILS_EINVAL, "boost k must be finite and >= 0, got %g", epi->k);
  if (ils_status st = check_io(p, f, u, ps)) return st;
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->dtype == ILS_F32)
    return smooth_t<float>(p, static_cast<const float*>(f), static_cast<float*>(u), ps, ws, s, status, nullptr,
                           nullptr, nullptr, 1, epi);
  return smooth_t<double>(p, static_cast<const double*>(f), static_cast<double*>(u), ps, ws, s, status, nullptr,
                          nullptr, nullptr, 1, epi);
}

ils_status ils_gaussian_blur(const void* x, void* y, void* tmp, int32_t batch, int32_t height, int32_t width,
                             int64_t ps, double sigma, int32_t dtype, void* stream) {
  if (!x || !y || !tmp) return fail(ILS_EINVAL, "NULL argument");
  if (batch < 1 || height < 1 || width < 1 || ps < (int64_t)height * width) return fail(ILS_EINVAL, "bad blur shape");
  if (dtype != ILS_F32 && dtype != ILS_F64) return fail(ILS_EINVAL, "unknown dtype %d", dtype);
  if (!(sigma >= 0.0 && std::isfinite(sigma))) return fail(ILS_EINVAL, "sigma must be finite and >= 0, got %g", sigma);
  const int r = sigma == 0.0 ? 0 : (int)std::ceil(3.0 * sigma);
  if (r > kMaxGaussRadius) return fail(ILS_EUNSUPPORTED, "sigma %g: blur radius %d > %d", sigma, r, kMaxGaussRadius);
  // kernel = exp(-x^2 / 2 sigma^2) / sum (applications.py:217-220), in double
  std::vector<double> w(r + 1, 1.0);
  double sum = 1.0;
  for (int j = 1; j <= r; ++j) {
    w[j] = std::exp(-(double)j * j / (2.0 * sigma * sigma));
    sum += 2.0 * w[j];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto run = [&](auto tag) -> ils_status {
    using T = decltype(tag);
    GaussW<T> g{};
    g.r = r;
    // numpy normalises the full (2r+1)-tap array: kernel /= kernel.sum(), summed left to right
    double tot = 0.0;
    for (int j = -r; j <= r; ++j) tot += w[std::abs(j)];
    (void)sum;
    for (int j = 0; j <= r; ++j) g.w[j] = T(w[j] / tot);
    const dim3 gc((width + 127) / 128, (height + 31) / 32, batch);
    k_gauss_cols<T><<<gc, 128, 0, s>>>(static_cast<const T*>(x), static_cast<T*>(tmp), height, width, ps, g);
    ILS_CUDA(cudaGetLastError());
    const size_t sm = (size_t)(width + 2 * r) * sizeof(T);
    if (sm > 48 * 1024) ILS_CUDA(cudaFuncSetAttribute(k_gauss_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_gauss_rows<T><<<dim3(height, batch), 256, sm, s>>>(static_cast<const T*>(tmp), static_cast<T*>(y), width, ps, g);
    ILS_CUDA(cudaGetLastError());
    return ILS_OK;
  };
  return dtype == ILS_F32 ? run(float{}) : run(double{});
}

ils_status ils_smooth_u8(const ils_plan* p, const uint8_t* f, uint8_t* u, int32_t channels, void* ws, void* stream,
                         int32_t* status) {
  if (!p || !f || !u || !ws || !status) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (p->slab) return fail(ILS_EINVAL, "slab plans run through ils_slab_row_pass / ils_slab_col_pass");
  if (channels < 1 || p->B % channels != 0)
    return fail(ILS_EINVAL, "plan batch %d is not a whole number of %d-channel frames", p->B, channels);
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t ps = (int64_t)p->H * p->W;
  if (p->dtype == ILS_F32)
    return smooth_t<float>(p, nullptr, nullptr, ps, ws, s, status, nullptr, f, u, channels);
  return smooth_t<double>(p, nullptr, nullptr, ps, ws, s, status, nullptr, f, u, channels);
}

ils_status ils_solve_ls(const ils_plan* p, const void* f, const void* mx, const void* my, void* u, int64_t ps,
                        void* ws, void* stream, int32_t* status) {
  if (!p || !f || !mx || !my || !u || !ws || !status) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (ps < (int64_t)p->H * p->W) return fail(ILS_EINVAL, "plane_stride %lld < H*W", (long long)ps);
  if (ils_status st = check_io(p, f, u, ps)) return st;
  if (ils_status st = check_io(p, mx, my, ps)) return st;
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->dtype == ILS_F32)
    return solve_t<float>(p, static_cast<const float*>(f), static_cast<const float*>(mx),
                          static_cast<const float*>(my), static_cast<float*>(u), ps, ws, s, status);
  return solve_t<double>(p, static_cast<const double*>(f), static_cast<const double*>(mx),
                         static_cast<const double*>(my), static_cast<double*>(u), ps, ws, s, status);
}

constexpr int kIoSlots = 4;  // host pipeline: batches in flight (2 per compute lane)

ils_status ils_host_io_size(const ils_plan* p, size_t* bytes) {
  if (!p || !bytes) return fail(ILS_EINVAL, "NULL argument");
  const size_t es = p->dtype == ILS_F32 ? 4 : 8;
  const size_t batch_bytes = ((size_t)p->B * p->H * p->W * es + 255) & ~size_t(255);
  size_t ws = 0;
  ils_workspace_size(p, &ws);
  // kIoSlots x (f, u) + status words + the second compute lane's workspace
  *bytes = 2 * kIoSlots * batch_bytes + 1024 + ws;
  return ILS_OK;
}

}  // extern "C"

namespace {

// Streams, events and the pinned status words of the host pipeline, created
// once per (thread, device) and reused by every call on that thread (creating
// them per call cost about a millisecond of pinned allocation and stream
// setup, serialised in front of every batch group).  Thread-local, so plans
// stay shareable across threads; intentionally never freed (process exit
// may run after the CUDA context is gone).
// Each I/O slot's batch (status reset, the passes) is captured once per
// (plan, buffers) into a CUDA graph and replayed on its lane: graph launches
// keep the passes' programmatic-dependent-launch edges inside one submission
// (ILS_HOST_GRAPHS=0: plain stream launches).
struct SlotGraphs {
  uint64_t uid = 0;
  int kind = -1, ch = 0;
  const void *io = nullptr, *ws = nullptr;
  cudaGraphExec_t ex[kIoSlots] = {};
};
constexpr int kGraphCache = 8;

struct HostRes {
  cudaStream_t h2d = nullptr, d2h = nullptr, lane1 = nullptr, cap = nullptr;
  cudaEvent_t ev_in[kIoSlots] = {}, ev_comp[kIoSlots] = {}, ev_out[kIoSlots] = {};
  int32_t* hstat = nullptr;
  int hcap = 0;
  SlotGraphs graphs[kGraphCache];
  int next_victim = 0;
};

cudaError_t host_res(int device, int nstat, HostRes** out) {
  static thread_local HostRes* cache[64] = {};
  if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
  HostRes*& R = cache[device];
  if (!R) {
    HostRes* n = new HostRes();
    cudaError_t e = cudaStreamCreateWithFlags(&n->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&n->d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&n->lane1, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&n->cap, cudaStreamNonBlocking);
    for (int i = 0; i < kIoSlots && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&n->ev_in[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&n->ev_comp[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&n->ev_out[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return e;  // partially built resources leak (error path only)
    R = n;
  }
  if (R->hcap < nstat) {
    if (R->hstat) cudaFreeHost(R->hstat);
    R->hstat = nullptr;
    R->hcap = 0;
    const int cap = std::max(nstat, 64);
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&R->hstat), sizeof(int32_t) * cap, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    R->hcap = cap;
  }
  *out = R;
  return cudaSuccess;
}

// Pipelined host path shared by ils_smooth_host / ils_smooth_host_u8: batch k
// runs on compute lane k & 1 (the caller's stream with the caller's
// workspace, or an internal stream with the second workspace carved from
// io_dev), so consecutive batches' kernels overlap each other and the
// host->device / device->host copies (kIoSlots I/O slots, so a lane's next
// batch never waits for its previous result's device->host copy).
// run(f_dev, u_dev, status_dev, ws, stream) enqueues one batch.
template <class Run>
ils_status host_pipeline(const ils_plan* p, const void* f_host, void* u_host, size_t in_bytes, size_t out_bytes,
                         int32_t nbatches, void* ws, void* io_dev, void* stream, int32_t* bad_iter, int kind, int ch,
                         Run run) {
  if (bad_iter) *bad_iter = -1;
  const size_t slot_in = (in_bytes + 255) & ~size_t(255), slot_out = (out_bytes + 255) & ~size_t(255);
  char* io = static_cast<char*>(io_dev);
  constexpr int NS = kIoSlots;
  char* fslot[NS];
  char* uslot[NS];
  int32_t* st[NS];
  for (int i = 0; i < NS; ++i) {
    fslot[i] = io + i * slot_in;
    uslot[i] = io + NS * slot_in + i * slot_out;
    st[i] = reinterpret_cast<int32_t*>(io + NS * (slot_in + slot_out) + 128 * i);
  }
  // the I/O slots are sized for the plan's dtype; the second workspace follows them
  const size_t es = p->dtype == ILS_F32 ? 4 : 8;
  const size_t full_slot = ((size_t)p->B * p->H * p->W * es + 255) & ~size_t(255);
  void* wsl[2] = {ws, io + 2 * NS * full_slot + 1024};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ils_status rc = ILS_OK;
#define ILS_TRY(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      rc = fail(ILS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));                     \
      return rc;                                                                         \
    }                                                                                    \
  } while (0)
  int dev = 0;
  ILS_TRY(cudaGetDevice(&dev));
  HostRes* R = nullptr;
  ILS_TRY(host_res(dev, nbatches, &R));
  cudaStream_t lane[2] = {s, R->lane1};
  cudaStream_t h2d = R->h2d, d2h = R->d2h;
  cudaEvent_t *ev_in = R->ev_in, *ev_comp = R->ev_comp, *ev_out = R->ev_out;
  int32_t* hstat = R->hstat;
  auto cleanup = [] {};
  // slot graphs for this (plan, path, buffers): look up, or capture once
  SlotGraphs* G = nullptr;
  if (env_int("ILS_HOST_GRAPHS", 1)) {
    for (SlotGraphs& g : R->graphs)
      if (g.uid == p->uid && g.kind == kind && g.ch == ch && g.io == io_dev && g.ws == ws) G = &g;
    if (!G) {
      G = &R->graphs[R->next_victim];
      R->next_victim = (R->next_victim + 1) % kGraphCache;
      for (cudaGraphExec_t& x : G->ex)
        if (x) {
          cudaGraphExecDestroy(x);
          x = nullptr;
        }
      G->uid = 0;
      for (int sl = 0; sl < NS; ++sl) {
        ILS_TRY(cudaStreamBeginCapture(R->cap, cudaStreamCaptureModeThreadLocal));
        const ils_status r = run(fslot[sl], uslot[sl], st[sl], wsl[sl & 1], R->cap);
        cudaGraph_t graph = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(R->cap, &graph);
        if (r != ILS_OK) {
          if (graph) cudaGraphDestroy(graph);
          return r;
        }
        if (ec != cudaSuccess) return fail(ILS_ECUDA, "host pipeline capture: %s", cudaGetErrorString(ec));
        const cudaError_t ei = cudaGraphInstantiate(&G->ex[sl], graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) return fail(ILS_ECUDA, "host pipeline graph: %s", cudaGetErrorString(ei));
      }
      G->uid = p->uid;
      G->kind = kind;
      G->ch = ch;
      G->io = io_dev;
      G->ws = ws;
    }
  }
  // the caller's stream may still be producing host-visible state: order h2d after it
  ILS_TRY(cudaEventRecord(ev_out[0], s));
  ILS_TRY(cudaStreamWaitEvent(h2d, ev_out[0], 0));
  ILS_TRY(cudaStreamWaitEvent(d2h, ev_out[0], 0));
  ILS_TRY(cudaStreamWaitEvent(lane[1], ev_out[0], 0));
  for (int k = 0; k < nbatches; ++k) {
    const int sl = k % NS, ln = k & 1;
    const char* fh = static_cast<const char*>(f_host) + (size_t)k * in_bytes;
    char* uh = static_cast<char*>(u_host) + (size_t)k * out_bytes;
    if (k >= NS) ILS_TRY(cudaStreamWaitEvent(h2d, ev_comp[sl], 0));  // f slot consumed by batch k-NS
    ILS_TRY(cudaMemcpyAsync(fslot[sl], fh, in_bytes, cudaMemcpyHostToDevice, h2d));
    ILS_TRY(cudaEventRecord(ev_in[sl], h2d));
    ILS_TRY(cudaStreamWaitEvent(lane[ln], ev_in[sl], 0));
    if (k >= NS) ILS_TRY(cudaStreamWaitEvent(lane[ln], ev_out[sl], 0));  // u slot drained by batch k-NS
    if (G) {
      ILS_TRY(cudaGraphLaunch(G->ex[sl], lane[ln]));  // = run(fslot[sl], uslot[sl], st[sl], wsl[ln], lane[ln])
    } else {
      ils_status r = run(fslot[sl], uslot[sl], st[sl], wsl[ln], lane[ln]);
      if (r != ILS_OK) {
        cleanup();
        return r;
      }
    }
    ILS_TRY(cudaEventRecord(ev_comp[sl], lane[ln]));
    ILS_TRY(cudaStreamWaitEvent(d2h, ev_comp[sl], 0));
    ILS_TRY(cudaMemcpyAsync(uh, uslot[sl], out_bytes, cudaMemcpyDeviceToHost, d2h));
    ILS_TRY(cudaMemcpyAsync(hstat + k, st[sl], sizeof(int32_t), cudaMemcpyDeviceToHost, d2h));
    ILS_TRY(cudaEventRecord(ev_out[sl], d2h));
  }
  ILS_TRY(cudaStreamSynchronize(d2h));
  ILS_TRY(cudaStreamSynchronize(lane[1]));
  ILS_TRY(cudaStreamSynchronize(s));
#undef ILS_TRY
  int worst = ILS_STATUS_CLEAN;
  for (int k = 0; k < nbatches; ++k) worst = std::min(worst, (int)hstat[k]);
  cleanup();
  if (worst != ILS_STATUS_CLEAN) {
    if (bad_iter) *bad_iter = worst;
    if (worst == 0) return fail(ILS_ENONFINITE_INPUT, "image plane contains non-finite values");
    return fail(ILS_ENONFINITE, "non-finite iterate at iteration %d", worst);
  }
  return ILS_OK;
}

}  // namespace

extern "C" {

ils_status ils_smooth_host(const ils_plan* p, const void* f_host, void* u_host, int64_t ps, int32_t nbatches,
                           void* ws, void* io_dev, void* stream, int32_t* bad_iter) {
  if (!p || !f_host || !u_host || !ws || !io_dev) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (nbatches < 1) return fail(ILS_EINVAL, "nbatches must be >= 1");
  if (ps != (int64_t)p->H * p->W) return fail(ILS_EINVAL, "host planes must be dense (plane_stride == H*W)");
  if (ils_status st = check_io(p, ws, io_dev, ps)) return st;
  DeviceGuard dg(p->device);
  const size_t bytes = (size_t)p->B * ps * (p->dtype == ILS_F32 ? 4 : 8);
  return host_pipeline(p, f_host, u_host, bytes, bytes, nbatches, ws, io_dev, stream, bad_iter, 0, 0,
                       [&](void* fd, void* ud, int32_t* st, void* w, cudaStream_t ls) {
                         return ils_smooth(p, fd, ud, ps, w, ls, st, nullptr);
                       });
}

ils_status ils_smooth_host_u8(const ils_plan* p, const uint8_t* f_host, uint8_t* u_host, int32_t channels,
                              int32_t nbatches, void* ws, void* io_dev, void* stream, int32_t* bad_iter) {
  if (!p || !f_host || !u_host || !ws || !io_dev) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (nbatches < 1) return fail(ILS_EINVAL, "nbatches must be >= 1");
  DeviceGuard dg(p->device);
  const size_t bytes = (size_t)p->B * p->H * p->W;
  return host_pipeline(p, f_host, u_host, bytes, bytes, nbatches, ws, io_dev, stream, bad_iter, 1, channels,
                       [&](void* fd, void* ud, int32_t* st, void* w, cudaStream_t ls) {
                         return ils_smooth_u8(p, static_cast<const uint8_t*>(fd), static_cast<uint8_t*>(ud), channels,
                                              w, ls, st);
                       });
}

ils_status ils_launch_pass(const ils_plan* p, int32_t pass, const void* f, void* u, int64_t ps, void* ws,
                           void* stream, int32_t* status) {
  if (!p || !ws || !status) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (pass < 0 || pass > 7 || pass == 4) return fail(ILS_EINVAL, "pass must be 0..3 or 5..7, got %d", pass);
  if (ils_status st = check_io(p, f, u, ps)) return st;
  DeviceGuard dg(p->device);
  const bool second = (pass & 4) != 0;
  pass &= 3;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto run = [&](auto tag) -> ils_status {
    using T = decltype(tag);
    cx<T>* Sa = static_cast<cx<T>*>(ws);
    cx<T>* Sb = reinterpret_cast<cx<T>*>(static_cast<char*>(ws) + p->spec_bytes);
    if (second) std::swap(Sa, Sb);
    if (pass == 1) {
      ILS_CUDA(launch_col<T>(p, col_args<T>(p, Sa, COL_SOLVE), s));
      return ILS_OK;
    }
    RowArgs<T> a = row_args<T>(p);
    a.f = static_cast<const T*>(f);
    a.f_ps = ps;
    a.f_rp = p->W;
    a.u = static_cast<T*>(u);
    a.u_ps = ps;
    a.u_rp = p->W;
    a.status = status;
    a.iter = pass == 3 ? p->prm.iters : 1;
    a.Sin = Sa;
    a.Sout = pass == 0 ? Sa : Sb;
    const int mode = pass == 0 ? MODE_F0 : (pass == 2 ? MODE_IT : MODE_FIN);
    ILS_CUDA(launch_row<T>(p, mode, a, s));
    return ILS_OK;
  };
  return p->dtype == ILS_F32 ? run(float{}) : run(double{});
}

ils_status ils_rfft2(const ils_plan* p, const void* x, int64_t ps, void* spec, int64_t pitch, void* stream) {
  if (!p || !x || !spec) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (pitch < p->Wc) return fail(ILS_EINVAL, "spec_pitch %lld < width/2+1", (long long)pitch);
  if (ils_status st = check_io(p, x, nullptr, ps)) return st;
  if (pitch % 2 || reinterpret_cast<uintptr_t>(spec) % 16) return fail(ILS_EINVAL, "spectrum rows must be 16-byte aligned (even spec_pitch)");
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto run = [&](auto tag) -> ils_status {
    using T = decltype(tag);
    RowArgs<T> a = row_args<T>(p);
    a.f = static_cast<const T*>(x);
    a.f_ps = ps;
    a.f_rp = p->W;
    a.Sout = static_cast<cx<T>*>(spec);
    a.S_rp = (int)pitch;
    a.S_ps = (long long)p->H * pitch;
    ILS_CUDA(launch_row<T>(p, MODE_R2C, a, s));
    ColArgs<T> c = col_args<T>(p, static_cast<cx<T>*>(spec), COL_FWD);
    c.S_rp = (int)pitch;
    c.S_ps = (long long)p->H * pitch;
    ILS_CUDA(launch_col<T>(p, c, s));
    return ILS_OK;
  };
  return p->dtype == ILS_F32 ? run(float{}) : run(double{});
}

ils_status ils_irfft2(const ils_plan* p, void* spec, int64_t pitch, void* x, int64_t ps, void* stream) {
  if (!p || !x || !spec) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (pitch < p->Wc) return fail(ILS_EINVAL, "spec_pitch %lld < width/2+1", (long long)pitch);
  if (ils_status st = check_io(p, nullptr, x, ps)) return st;
  if (pitch % 2 || reinterpret_cast<uintptr_t>(spec) % 16) return fail(ILS_EINVAL, "spectrum rows must be 16-byte aligned (even spec_pitch)");
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto run = [&](auto tag) -> ils_status {
    using T = decltype(tag);
    ColArgs<T> c = col_args<T>(p, static_cast<cx<T>*>(spec), COL_INV);
    c.S_rp = (int)pitch;
    c.S_ps = (long long)p->H * pitch;
    ILS_CUDA(launch_col<T>(p, c, s));
    RowArgs<T> a = row_args<T>(p);
    a.Sin = static_cast<const cx<T>*>(spec);
    a.S_rp = (int)pitch;
    a.S_ps = (long long)p->H * pitch;
    a.u = static_cast<T*>(x);
    a.u_ps = ps;
    a.u_rp = p->W;
    a.iter = 1;
    a.status = reinterpret_cast<int*>(static_cast<char*>(p->d_tables) + p->off_sink);
    ILS_CUDA(launch_row<T>(p, MODE_FIN, a, s));
    return ILS_OK;
  };
  return p->dtype == ILS_F32 ? run(float{}) : run(double{});
}

ils_status ils_rgb_yuv(void* planes, int32_t dtype, int64_t ps, int64_t npx, int32_t frames, int32_t inverse,
                       void* stream) {
  if (!planes || frames < 1 || npx < 1 || ps < npx) return fail(ILS_EINVAL, "bad rgb_yuv arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long n = npx * frames;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  if (dtype == ILS_F32)
    k_rgb_yuv<float><<<blocks, 256, 0, s>>>(static_cast<float*>(planes), ps, npx, frames, inverse);
  else
    k_rgb_yuv<double><<<blocks, 256, 0, s>>>(static_cast<double*>(planes), ps, npx, frames, inverse);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

// ------------------------------------------------------------ standalone field kernels (drop-in API)
}  // extern "C"

namespace {
template <typename T>
PenaltyRef<T> pen_ref(const ils_params& q) {
  PenaltyRef<T> P{};
  P.kind = q.kind;
  P.p = T(q.p);
  P.eps = T(q.eps);
  P.e = T(q.p / 2.0 - 1.0);
  P.ph = T(q.p / 2.0);
  P.g2x2 = T(2.0 * (q.gamma * q.gamma));
  P.c = T(q.c);
  P.lam = T(q.lam);
  return P;
}

int elem_blocks(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8)); }

ils_status check_planes(int32_t batch, int32_t height, int32_t width, int64_t ps, int32_t dtype) {
  if (batch < 1 || height < 1 || width < 1) return fail(ILS_EINVAL, "invalid plane size %dx%d x %d", height, width, batch);
  if (ps < (int64_t)height * width) return fail(ILS_EINVAL, "plane_stride %lld < H*W", (long long)ps);
  if (dtype != ILS_F32 && dtype != ILS_F64) return fail(ILS_EINVAL, "unknown dtype %d", dtype);
  return ILS_OK;
}
}  // namespace

extern "C" {

ils_status ils_grad(const void* u, void* gx, void* gy, int32_t batch, int32_t height, int32_t width, int64_t ps,
                    int32_t dtype, void* stream) {
  if (!u || (!gx && !gy)) return fail(ILS_EINVAL, "NULL argument");
  ils_status st = check_planes(batch, height, width, ps, dtype);
  if (st != ILS_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const dim3 grid(elem_blocks((long long)height * width), batch);
  if (dtype == ILS_F32)
    k_grad<float><<<grid, 256, 0, s>>>(static_cast<const float*>(u), static_cast<float*>(gx), static_cast<float*>(gy),
                                       height, width, ps);
  else
    k_grad<double><<<grid, 256, 0, s>>>(static_cast<const double*>(u), static_cast<double*>(gx),
                                        static_cast<double*>(gy), height, width, ps);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

ils_status ils_adjoint_accumulate(const void* mx, const void* my, void* out, int32_t batch, int32_t height,
                                  int32_t width, int64_t ps, int32_t dtype, void* stream) {
  if (!mx || !my || !out) return fail(ILS_EINVAL, "NULL argument");
  ils_status st = check_planes(batch, height, width, ps, dtype);
  if (st != ILS_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const dim3 grid(elem_blocks((long long)height * width), batch);
  if (dtype == ILS_F32)
    k_adjoint<float><<<grid, 256, 0, s>>>(static_cast<const float*>(mx), static_cast<const float*>(my),
                                          static_cast<float*>(out), height, width, ps);
  else
    k_adjoint<double><<<grid, 256, 0, s>>>(static_cast<const double*>(mx), static_cast<const double*>(my),
                                           static_cast<double*>(out), height, width, ps);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

ils_status ils_aux_update(const ils_params* q, const void* x, void* out, int64_t n, int32_t dtype, void* stream) {
  if (!x || !out) return fail(ILS_EINVAL, "NULL argument");
  ils_status st = validate(q);  // includes _check_curvature (penalty.py:108-114)
  if (st != ILS_OK) return st;
  if (n < 0 || (dtype != ILS_F32 && dtype != ILS_F64)) return fail(ILS_EINVAL, "bad aux_update arguments");
  if (n == 0) return ILS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == ILS_F32)
    k_aux<float><<<elem_blocks(n), 256, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(out), n,
                                                pen_ref<float>(*q));
  else
    k_aux<double><<<elem_blocks(n), 256, 0, s>>>(static_cast<const double*>(x), static_cast<double*>(out), n,
                                                 pen_ref<double>(*q));
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

ils_status ils_energy(const ils_params* q, const void* u, const void* f, int32_t batch, int32_t height, int32_t width,
                      int64_t ps, int32_t dtype, double* out, void* scratch, void* stream) {
  if (!u || !f || !out || !scratch || !q) return fail(ILS_EINVAL, "NULL argument");
  if (!std::isfinite(q->lam)) return fail(ILS_EINVAL, "lam must be finite, got %g", q->lam);
  ils_params v = *q;  // energy needs the penalty only: lam / c / iters are not constrained here
  v.lam = 1.0;
  v.c = 1e300;
  v.iters = 1;
  ils_status st = validate(&v);
  if (st != ILS_OK) return st;
  st = check_planes(batch, height, width, ps, dtype);
  if (st != ILS_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(scratch);
  const dim3 grid(kEnergyBlocks, batch);
  if (dtype == ILS_F32)
    k_energy_part<float><<<grid, 256, 0, s>>>(static_cast<const float*>(u), static_cast<const float*>(f), height,
                                              width, ps, pen_ref<float>(*q), part);
  else
    k_energy_part<double><<<grid, 256, 0, s>>>(static_cast<const double*>(u), static_cast<const double*>(f), height,
                                               width, ps, pen_ref<double>(*q), part);
  ILS_CUDA(cudaGetLastError());
  k_energy_fin<<<batch, 256, 0, s>>>(part, kEnergyBlocks, q->lam, out);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

// ------------------------------------------------------------ tone mapping (applications.py:132-183)
}  // extern "C"

namespace {
size_t tm_layout(const ils_plan* p, size_t* off_f, size_t* off_u, size_t* off_part) {
  size_t ws = 0;
  ils_workspace_size(p, &ws);
  const size_t es = p->dtype == ILS_F32 ? 4 : 8;
  const size_t planes = ((size_t)p->B * p->H * p->W * es + 255) & ~size_t(255);
  *off_f = (ws + 255) & ~size_t(255);
  *off_u = *off_f + planes;
  *off_part = *off_u + planes;
  return *off_part + 2 * 256 * sizeof(double);
}
}  // namespace

extern "C" {

ils_status ils_tonemap_workspace_size(const ils_plan* p, size_t* bytes) {
  if (!p || !bytes) return fail(ILS_EINVAL, "NULL argument");
  size_t a, b, c;
  *bytes = tm_layout(p, &a, &b, &c);
  return ILS_OK;
}

ils_status ils_tonemap(const ils_plan* p, const double* lum, const double* rgb, double* out,
                       const ils_tonemap_params* tp, void* ws, void* stream, int32_t* status, double* sc) {
  if (!p || !lum || !rgb || !out || !tp || !ws || !status || !sc) return fail(ILS_EINVAL, "NULL argument");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (p->slab || p->prm.kind == ILS_SOFT) return fail(ILS_EINVAL, "tone mapping needs an ILS plan");
  if (tp->nscales != 1 && tp->nscales != 3) return fail(ILS_EINVAL, "nscales must be 1 or 3, got %d", tp->nscales);
  if (p->B != tp->nscales) return fail(ILS_EINVAL, "plan batch %d != nscales %d", p->B, tp->nscales);
  // TonemapParams.__post_init__ (applications.py:53-77)
  if (!(tp->target_range > 0.0 && std::isfinite(tp->target_range)))
    return fail(ILS_EINVAL, "target_range must be finite and positive, got %g", tp->target_range);
  if (!(tp->saturation > 0.0 && tp->saturation <= 1.0)) return fail(ILS_EINVAL, "saturation must be in (0,1], got %g", tp->saturation);
  if (!(tp->log_offset > 0.0 && std::isfinite(tp->log_offset)))
    return fail(ILS_EINVAL, "log_offset must be finite and positive, got %g", tp->log_offset);
  for (int k = 0; k < tp->nscales; ++k)
    if (!(tp->lam[k] > 0.0 && std::isfinite(tp->lam[k]))) return fail(ILS_EINVAL, "lambdas must be finite and positive");
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  size_t off_f, off_u, off_part;
  tm_layout(p, &off_f, &off_u, &off_part);
  char* w = static_cast<char*>(ws);
  double* part = reinterpret_cast<double*>(w + off_part);
  const long long npx = (long long)p->H * p->W;
  const int blocks = elem_blocks(npx);
  const int mblocks = std::min(256, blocks);
  auto run = [&](auto tag) -> ils_status {
    using T = decltype(tag);
    T* f = reinterpret_cast<T*>(w + off_f);
    T* u = reinterpret_cast<T*>(w + off_u);
    k_tm_log<T><<<blocks, 256, 0, s>>>(lum, f, npx, p->B, tp->log_offset);
    ILS_CUDA(cudaGetLastError());
    // all scales in one launch sequence, each plane with its own lambda
    ils_status st = smooth_t<T>(p, f, u, npx, ws, s, status, nullptr, nullptr, nullptr, 1, nullptr, tp->lam,
                                tp->nscales);
    if (st != ILS_OK) return st;
    k_tm_minmax<T><<<mblocks, 256, 0, s>>>(u + (size_t)(p->B - 1) * npx, npx, part);
    k_tm_minmax_fin<<<1, 32, 0, s>>>(part, mblocks, tp->target_range, sc);
    k_tm_finish<T><<<blocks, 256, 0, s>>>(lum, rgb, u, p->B, npx, tp->log_offset, tp->weights[0], tp->weights[1],
                                          tp->weights[2], tp->saturation, sc, out);
    ILS_CUDA(cudaGetLastError());
    return ILS_OK;
  };
  return p->dtype == ILS_F32 ? run(float{}) : run(double{});
}

ils_status ils_detail_boost(const void* f, const void* u, void* out, int64_t n, double k, int32_t dtype, void* stream) {
  if (!f || !u || !out || n < 0) return fail(ILS_EINVAL, "bad detail_boost arguments");
  if (!(k >= 0.0 && std::isfinite(k))) return fail(ILS_EINVAL, "boost k must be finite and >= 0, got %g", k);
  if (dtype != ILS_F32 && dtype != ILS_F64) return fail(ILS_EINVAL, "unknown dtype %d", dtype);
  if (n == 0) return ILS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == ILS_F32)
    k_detail_boost<float><<<elem_blocks(n), 256, 0, s>>>(static_cast<const float*>(f), static_cast<const float*>(u),
                                                        static_cast<float*>(out), n, float(k));
  else
    k_detail_boost<double><<<elem_blocks(n), 256, 0, s>>>(static_cast<const double*>(f),
                                                         static_cast<const double*>(u), static_cast<double*>(out), n, k);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

ils_status ils_convert(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n, void* stream) {
  if (!src || !dst || n < 0) return fail(ILS_EINVAL, "bad convert arguments");
  if ((src_dtype != ILS_F32 && src_dtype != ILS_F64) || (dst_dtype != ILS_F32 && dst_dtype != ILS_F64))
    return fail(ILS_EINVAL, "unknown dtype");
  if (n == 0) return ILS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = elem_blocks(n);
  if (src_dtype == ILS_F64 && dst_dtype == ILS_F32)
    k_convert<double, float><<<blocks, 256, 0, s>>>(static_cast<const double*>(src), static_cast<float*>(dst), n);
  else if (src_dtype == ILS_F32 && dst_dtype == ILS_F64)
    k_convert<float, double><<<blocks, 256, 0, s>>>(static_cast<const float*>(src), static_cast<double*>(dst), n);
  else if (src_dtype == ILS_F32)
    k_convert<float, float><<<blocks, 256, 0, s>>>(static_cast<const float*>(src), static_cast<float*>(dst), n);
  else
    k_convert<double, double><<<blocks, 256, 0, s>>>(static_cast<const double*>(src), static_cast<double*>(dst), n);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

ils_status ils_denominator(double* out, int32_t height, int32_t width, double lam, double c, void* stream) {
  if (!out || height < 1 || width < 1) return fail(ILS_EINVAL, "bad denominator arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_denom<<<elem_blocks((long long)height * width), 256, 0, s>>>(out, height, width, c * lam / 2.0);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

ils_status ils_hermitian_full(const void* half, int64_t pitch, void* full, int32_t height, int32_t width,
                              void* stream) {
  if (!half || !full || height < 1 || width < 1 || pitch < width / 2 + 1) return fail(ILS_EINVAL, "bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_hermitian_full<<<elem_blocks((long long)height * width), 256, 0, s>>>(
      static_cast<const cx<double>*>(half), pitch, static_cast<cx<double>*>(full), height, width);
  ILS_CUDA(cudaGetLastError());
  return ILS_OK;
}

// ------------------------------------------------------------ slab decomposition (C5)
ils_status ils_slab_plan_create(ils_plan** out, int32_t height, int32_t width, const ils_params* params,
                                int32_t dtype, int32_t device, int32_t nranks, int32_t rank) {
  if (!out) return fail(ILS_EINVAL, "out is NULL");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxSeg) return fail(ILS_EINVAL, "nranks must be in [1, %d], got %d", kMaxSeg, nranks);
  if (rank < 0 || rank >= nranks) return fail(ILS_EINVAL, "rank %d outside [0, %d)", rank, nranks);
  if (width % 2) return fail(ILS_EUNSUPPORTED, "slab plans need an even width, got %d", width);
  if (height < nranks) return fail(ILS_EINVAL, "height %d < nranks %d", height, nranks);
  const int Wc = width / 2 + 1;
  if (Wc < 2 * nranks + 1) return fail(ILS_EINVAL, "width %d too small for %d ranks", width, nranks);
  ils_plan* p = nullptr;
  // a host-only plan of the global shape for the FFT plans and tables, then
  // the launch geometry re-planned for this rank's rows and columns
  ils_status st = ils_plan_create(&p, 1, height, width, params, dtype, -1);
  if (st != ILS_OK) return st;
  p->slab = true;
  p->P = nranks;
  p->rank = rank;
  for (int q = 0; q <= nranks; ++q) {
    p->row0[q] = (int)((long long)q * height / nranks);
    // even column offsets (16-byte aligned segments), balanced to within 2
    p->col0[q] = q == nranks ? Wc : (int)(((long long)q * Wc / nranks) & ~1LL);
  }
  for (int q = 0; q < nranks; ++q) p->pitch[q] = (p->col0[q + 1] - p->col0[q] + 1) & ~1;
  p->Hl = p->row0[rank + 1] - p->row0[rank];
  p->Wcl = p->col0[rank + 1] - p->col0[rank];
  if (device >= 0) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0) p->sms = sms;
  }
  const size_t elt = dtype == ILS_F32 ? sizeof(cx<float>) : sizeof(cx<double>);
  const int maxe = dtype == ILS_F32 ? 16 : 8;
  const int H = p->H, Wcg = p->Wc;
  p->H = p->Hl;  // row geometry over the local rows
  bool ok = choose_row(*p, maxe, elt);
  p->H = H;
  p->Wc = p->Wcl;  // column geometry over the local columns
  ok = ok && choose_col(*p, maxe, elt);
  p->Wc = Wcg;
  if (!ok) {
    ils_plan_destroy(p);
    return fail(ILS_EUNSUPPORTED, "no slab launch configuration for %dx%d on %d ranks", height, width, nranks);
  }
  p->device = device;
  if (device >= 0) {  // device tables (same content as the host-only plan's)
    const int rs = dtype == ILS_F32 ? 4 : 8;
    (void)rs;
    ils_plan* full = nullptr;
    st = ils_plan_create(&full, 1, height, width, params, dtype, device);
    if (st != ILS_OK) {
      ils_plan_destroy(p);
      return st;
    }
    p->d_tables = full->d_tables;  // take ownership of the uploaded tables
    p->off_rowtw = full->off_rowtw;
    p->off_coltw = full->off_coltw;
    p->off_wreal = full->off_wreal;
    p->off_wx = full->off_wx;
    p->off_wy = full->off_wy;
    p->off_tw2 = full->off_tw2;
    p->off_sink = full->off_sink;
    full->d_tables = nullptr;
    ils_plan_destroy(full);
  }
  *out = p;
  return ILS_OK;
}

ils_status ils_slab_get_layout(const ils_plan* p, int32_t* row0, int32_t* col0, int32_t* pitch, int64_t* counts) {
  if (!p || !p->slab) return fail(ILS_EINVAL, "not a slab plan");
  const int P = p->P, me = p->rank;
  for (int q = 0; q <= P; ++q) {
    if (row0) row0[q] = p->row0[q];
    if (col0) col0[q] = p->col0[q];
  }
  for (int q = 0; q < P; ++q) {
    if (pitch) pitch[q] = p->pitch[q];
    if (counts) {  // complex elements: fwd send/recv, rev send/recv, per peer q
      const int Hq = p->row0[q + 1] - p->row0[q];
      counts[0 * kMaxSeg + q] = (int64_t)p->Hl * p->pitch[q];
      counts[1 * kMaxSeg + q] = (int64_t)Hq * p->pitch[me];
      counts[2 * kMaxSeg + q] = (int64_t)(Hq + 2) * p->pitch[me];
      counts[3 * kMaxSeg + q] = (int64_t)(p->Hl + 2) * p->pitch[q];
    }
  }
  return ILS_OK;
}

}  // extern "C"

namespace {
template <typename T>
ils_status slab_row_t(const ils_plan* p, int mode, const T* f_ext, const cx<T>* recv, cx<T>* send, T* u, int iter,
                      cudaStream_t s, int32_t* status) {
  RowArgs<T> a = row_args<T>(p);
  a.H = p->Hl;
  a.wrap = 0;
  a.f = f_ext ? f_ext + p->W : nullptr;  // row -1 is the top halo row
  a.f_ps = (long long)(p->Hl + 2) * p->W;
  a.f_rp = p->W;
  a.u = u;
  a.u_ps = (long long)p->Hl * p->W;
  a.u_rp = p->W;
  a.status = status;
  a.iter = iter;
  a.Sin = recv;
  a.Sout = send;
  a.S_ps = 0;
  long long in_off = 0, out_off = 0;
  a.sin_seg.n = a.sout_seg.n = p->P;
  for (int q = 0; q <= p->P; ++q) a.sin_seg.c0[q] = a.sout_seg.c0[q] = p->col0[q];
  for (int q = 0; q < p->P; ++q) {
    a.sin_seg.pitch[q] = a.sout_seg.pitch[q] = p->pitch[q];
    a.sin_seg.off[q] = in_off + p->pitch[q];  // block row 1 = local row 0
    a.sout_seg.off[q] = out_off;
    in_off += (long long)(p->Hl + 2) * p->pitch[q];
    out_off += (long long)p->Hl * p->pitch[q];
  }
  a.mode = mode;
  const dim3 grid(p->row_grid, 1);
  cudaError_t e;
  if constexpr (std::is_same<T, float>::value) {
    // the rolling-band first / fused passes on the slab's rows (as launch_row;
    // chunk rows for the slab height, one plane per launch)
    if (p->roll_smem > 0 && (mode == MODE_F0 || mode == MODE_IT) && a.pen.kind != ILS_SOFT &&
        !env_int("ILS_NO_ROLL", 0)) {
      const long slots = (long)p->sms * std::min<long>(ILS_ROLL_MINB, (228 * 1024) / (p->roll_smem + 1024));
      int R = 0;
      double best = 1e300;
      for (int r = 2; r <= p->Hl; ++r) {
        const double cost = (double)(((p->Hl + r - 1) / r + slots - 1) / slots) * (r + 2);
        if (cost < best * (1 - 1e-9)) {
          best = cost;
          R = r;
        }
      }
      if (const int forced = env_int("ILS_ROLL_ROWS", 0)) R = std::min(forced, p->Hl);
      if (R > 0) {
        a.band = R;
        const dim3 rgrid((p->Hl + R - 1) / R, 1);
        switch (p->row_spec) {
#define ILS_CASE(ID, ...)                                                                               \
  case ID:                                                                                              \
    if constexpr (ILS_ROW_SPEC_ROLL(ID)) {                                                              \
      e = launch_row_roll_impl<RowSpec<ID>::type>(a, rgrid, p->roll_smem, p->roll_pf, s);              \
      if (e != cudaSuccess) return fail(ILS_ECUDA, "slab row pass: %s", cudaGetErrorString(e));        \
      return ILS_OK;                                                                                    \
    }                                                                                                   \
    break;
          ILS_ROW_SPECS(ILS_CASE)
#undef ILS_CASE
          default:
            break;
        }
        a.band = p->band;
      }
    }
    // the final pass (no halo rows): its own rows per CTA, as launch_row
    dim3 g2 = grid;
    size_t smem = p->row_smem;
    if (mode == MODE_FIN) {
      a.band = p->fin_band;
      g2 = dim3((p->Hl + a.band - 1) / a.band, 1);
      smem = p->fin_smem;
    }
    switch (p->row_spec) {
#define ILS_CASE(ID, ...)                                                                                      \
  case ID:                                                                                                     \
    e = launch_row_impl<float, true, RowSpec<ID>::type, ILS_ROW_SPEC_WIDE(ID)>(a, g2, p->row_threads, smem, s); \
    if (e != cudaSuccess) return fail(ILS_ECUDA, "slab row pass: %s", cudaGetErrorString(e));                 \
    return ILS_OK;
      ILS_ROW_SPECS(ILS_CASE)
#undef ILS_CASE
      default:
        break;
    }
  }
  e = p->W > kNarrowMaxW ? launch_row_impl<T, true, FftRt, true>(a, grid, p->row_threads, p->row_smem, s)
                         : launch_row_impl<T, true, FftRt>(a, grid, p->row_threads, p->row_smem, s);
  if (e != cudaSuccess) return fail(ILS_ECUDA, "slab row pass: %s", cudaGetErrorString(e));
  return ILS_OK;
}

template <typename T>
ils_status slab_col_t(const ils_plan* p, cx<T>* recv, cx<T>* send, cudaStream_t s) {
  ColArgs<T> c = col_args<T>(p, recv, COL_SOLVE);
  const int me = p->rank;
  c.Wc = p->Wcl;
  c.S_rp = p->pitch[me];
  c.S_ps = 0;
  c.wx += p->col0[me];
  c.P = p->P;
  long long off = 0;
  for (int q = 0; q <= p->P; ++q) c.r0[q] = p->row0[q];
  for (int q = 0; q < p->P; ++q) {
    c.dst_off[q] = off;
    off += (long long)(p->row0[q + 1] - p->row0[q] + 2) * p->pitch[me];
  }
  c.dst = send;
  const dim3 grid(p->col_grid, 1);
  cudaError_t e;
  if (p->col3 >= 0) {
    e = launch_col3<T>(p, c, 1, s);
    if (e != cudaSuccess) return fail(ILS_ECUDA, "slab col pass: %s", cudaGetErrorString(e));
    return ILS_OK;
  }
  if (p->col2 >= 0) {
    e = launch_col2<T>(p, c, 1, s);
    if (e != cudaSuccess) return fail(ILS_ECUDA, "slab col pass: %s", cudaGetErrorString(e));
    return ILS_OK;
  }
  if constexpr (std::is_same<T, float>::value) {
    switch (p->col_spec) {
#define ILS_CASE(ID, ...)                                                                    \
  case ID:                                                                                   \
    e = launch_col_impl<float, ColSpec<ID>::type>(c, grid, p->col_threads, p->col_smem, s);  \
    if (e != cudaSuccess) return fail(ILS_ECUDA, "slab col pass: %s", cudaGetErrorString(e)); \
    return ILS_OK;
      ILS_COL_SPECS(ILS_CASE)
#undef ILS_CASE
      default:
        break;
    }
  }
  e = p->col_wide ? launch_col_impl<T, FftRtWide>(c, grid, p->col_threads, p->col_smem, s)
                  : launch_col_impl<T, FftRt>(c, grid, p->col_threads, p->col_smem, s);
  if (e != cudaSuccess) return fail(ILS_ECUDA, "slab col pass: %s", cudaGetErrorString(e));
  return ILS_OK;
}
}  // namespace

extern "C" {

ils_status ils_slab_row_pass(const ils_plan* p, int32_t mode, const void* f_ext, const void* recv, void* send,
                             void* u, int32_t iter, void* stream, int32_t* status) {
  if (!p || !p->slab) return fail(ILS_EINVAL, "not a slab plan");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (mode != MODE_F0 && mode != MODE_IT && mode != MODE_FIN) return fail(ILS_EINVAL, "mode must be 0, 1 or 3");
  if (!status || (mode != MODE_FIN && !send) || (mode != MODE_F0 && !recv) || (mode == MODE_FIN && !u) || !f_ext)
    return fail(ILS_EINVAL, "NULL argument");
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->dtype == ILS_F32)
    return slab_row_t<float>(p, mode, static_cast<const float*>(f_ext), static_cast<const cx<float>*>(recv),
                             static_cast<cx<float>*>(send), static_cast<float*>(u), iter, s, status);
  return slab_row_t<double>(p, mode, static_cast<const double*>(f_ext), static_cast<const cx<double>*>(recv),
                            static_cast<cx<double>*>(send), static_cast<double*>(u), iter, s, status);
}

ils_status ils_slab_col_pass(const ils_plan* p, void* recv, void* send, void* stream) {
  if (!p || !p->slab) return fail(ILS_EINVAL, "not a slab plan");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (!recv || !send) return fail(ILS_EINVAL, "NULL argument");
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->dtype == ILS_F32)
    return slab_col_t<float>(p, static_cast<cx<float>*>(recv), static_cast<cx<float>*>(send), s);
  return slab_col_t<double>(p, static_cast<cx<double>*>(recv), static_cast<cx<double>*>(send), s);
}

}  // extern "C"

// ------------------------------------------------------------ C5 over NCCL in one call
// The slab smooth of dist.SlabSmoother as a C entry point: the row / column
// slab passes above with the two transposes as NCCL grouped send/recv on the
// caller's stream.  NCCL is bound at run time (dlopen of libnccl.so.2, or
// ILS_NCCL_LIB), so the library has no link-time NCCL dependency and a
// process that never calls these functions never loads it.
#include <dlfcn.h>

namespace {

struct NcclApi {
  bool loaded = false;
  std::string error;
  int (*get_unique_id)(ils_nccl_id*) = nullptr;
  int (*comm_init_rank)(void**, int, ils_nccl_id, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*error_string)(int) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* path = getenv("ILS_NCCL_LIB");
    void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.error = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<int (*)(ils_nccl_id*)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<int (*)(void**, int, ils_nccl_id, int)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<int (*)(void*)>(sym("ncclCommDestroy"));
    api.send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclSend"));
    api.recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclRecv"));
    api.group_start = reinterpret_cast<int (*)()>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<int (*)()>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<const char* (*)(int)>(sym("ncclGetErrorString"));
    api.loaded = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.send && api.recv &&
                 api.group_start && api.group_end;
    if (!api.loaded) api.error = "NCCL library lacks the point-to-point API";
  });
  return api;
}

constexpr int kNcclUint8 = 1;  // ncclUint8: blocks move as bytes

ils_status nccl_fail(const char* what, int r) {
  const NcclApi& n = nccl();
  return fail(ILS_ECUDA, "%s: NCCL error %d (%s)", what, r, n.error_string ? n.error_string(r) : "?");
}

// block sizes in bytes per peer for the four all-to-all buffers (ils_slab_get_layout)
struct DistLayout {
  size_t bytes[4][kMaxSeg];
  size_t off[4][kMaxSeg];
  size_t total[4];
};

DistLayout dist_layout(const ils_plan* p) {
  DistLayout d{};
  int64_t counts[4 * kMaxSeg];
  ils_slab_get_layout(p, nullptr, nullptr, nullptr, counts);
  const size_t elt = p->dtype == ILS_F32 ? sizeof(cx<float>) : sizeof(cx<double>);
  for (int k = 0; k < 4; ++k) {
    size_t o = 0;
    for (int q = 0; q < p->P; ++q) {
      d.bytes[k][q] = (size_t)counts[k * kMaxSeg + q] * elt;
      d.off[k][q] = o;
      o += d.bytes[k][q];
    }
    d.total[k] = (o + 255) & ~size_t(255);
  }
  return d;
}

ils_status dist_a2a(const ils_plan* p, const DistLayout& d, int sk, int rk, const char* send, char* recv, void* comm,
                    cudaStream_t s) {
  const NcclApi& n = nccl();
  int r = n.group_start();
  if (r) return nccl_fail("ncclGroupStart", r);
  for (int q = 0; q < p->P; ++q) {
    if (d.bytes[sk][q] && (r = n.send(send + d.off[sk][q], d.bytes[sk][q], kNcclUint8, q, comm, s))) break;
    if (d.bytes[rk][q] && (r = n.recv(recv + d.off[rk][q], d.bytes[rk][q], kNcclUint8, q, comm, s))) break;
  }
  const int r2 = n.group_end();
  if (r) return nccl_fail("ncclSend/ncclRecv", r);
  if (r2) return nccl_fail("ncclGroupEnd", r2);
  return ILS_OK;
}

}  // namespace

extern "C" {

ils_status ils_nccl_get_unique_id(ils_nccl_id* id) {
  if (!id) return fail(ILS_EINVAL, "NULL argument");
  const NcclApi& n = nccl();
  if (!n.loaded) return fail(ILS_ECUDA, "%s", n.error.c_str());
  const int r = n.get_unique_id(id);
  return r ? nccl_fail("ncclGetUniqueId", r) : ILS_OK;
}

ils_status ils_nccl_comm_create(void** comm, int32_t nranks, const ils_nccl_id* id, int32_t rank, int32_t device) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(ILS_EINVAL, "bad communicator arguments");
  const NcclApi& n = nccl();
  if (!n.loaded) return fail(ILS_ECUDA, "%s", n.error.c_str());
  DeviceGuard dg(device);
  const int r = n.comm_init_rank(comm, nranks, *id, rank);
  return r ? nccl_fail("ncclCommInitRank", r) : ILS_OK;
}

ils_status ils_nccl_comm_destroy(void* comm) {
  if (!comm) return ILS_OK;
  const NcclApi& n = nccl();
  if (!n.loaded) return fail(ILS_ECUDA, "%s", n.error.c_str());
  const int r = n.comm_destroy(comm);
  return r ? nccl_fail("ncclCommDestroy", r) : ILS_OK;
}

ils_status ils_dist_workspace_size(const ils_plan* p, size_t* bytes) {
  if (!p || !p->slab || !bytes) return fail(ILS_EINVAL, "not a slab plan");
  const DistLayout d = dist_layout(p);
  *bytes = d.total[0] + d.total[1] + d.total[2] + d.total[3];
  return ILS_OK;
}

ils_status ils_smooth_dist(const ils_plan* p, const void* f_ext, void* u, int32_t planes, int64_t f_ext_stride,
                           int64_t u_stride, void* ws, void* comm, void* stream, int32_t* status) {
  if (!p || !p->slab) return fail(ILS_EINVAL, "not a slab plan");
  if (!p->d_tables) return fail(ILS_EINVAL, "plan was created host-only (device < 0)");
  if (!f_ext || !u || !ws || !comm || !status || planes < 1) return fail(ILS_EINVAL, "NULL argument");
  if (f_ext_stride < (int64_t)(p->Hl + 2) * p->W || u_stride < (int64_t)p->Hl * p->W)
    return fail(ILS_EINVAL, "plane strides smaller than the rank's rows");
  const NcclApi& n = nccl();
  if (!n.loaded) return fail(ILS_ECUDA, "%s", n.error.c_str());
  DeviceGuard dg(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const DistLayout d = dist_layout(p);
  char* fwd_send = static_cast<char*>(ws);
  char* fwd_recv = fwd_send + d.total[0];
  char* rev_send = fwd_recv + d.total[1];
  char* rev_recv = rev_send + d.total[2];
  ILS_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int32_t), s));
  const int iters = p->prm.iters;
  const size_t es = p->dtype == ILS_F32 ? 4 : 8;
  for (int c = 0; c < planes; ++c) {  // dist.SlabSmoother.smooth, one plane after the other
    const char* fe = static_cast<const char*>(f_ext) + (size_t)c * f_ext_stride * es;
    char* uc = static_cast<char*>(u) + (size_t)c * u_stride * es;
    ils_status st = ils_slab_row_pass(p, MODE_F0, fe, nullptr, fwd_send, nullptr, 0, stream, status);
    for (int it = 0; it < iters && st == ILS_OK; ++it) {
      st = dist_a2a(p, d, 0, 1, fwd_send, fwd_recv, comm, s);
      if (st == ILS_OK) st = ils_slab_col_pass(p, fwd_recv, rev_send, stream);
      if (st == ILS_OK) st = dist_a2a(p, d, 2, 3, rev_send, rev_recv, comm, s);
      if (st == ILS_OK && it + 1 < iters) st = ils_slab_row_pass(p, MODE_IT, fe, rev_recv, fwd_send, nullptr, it + 1, stream, status);
    }
    if (st == ILS_OK) st = ils_slab_row_pass(p, MODE_FIN, fe, rev_recv, nullptr, uc, iters, stream, status);
    if (st != ILS_OK) return st;
  }
  return ILS_OK;
}

}  // extern "C"
