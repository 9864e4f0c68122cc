// Log-domain Sinkhorn baseline on the GPU.
//
// Restates the reference's sinkhorn_solve (sinkhorn.py:58-130):
//   phi_i = eps log f_i - eps LSE_j((psi_j - C_ij)/eps)      (rows with f_i > 0)
//   psi_j = eps log g_j - eps LSE_i((phi_i - C_ij)/eps)      (columns with g_j > 0)
// until the l1 marginal violation of X = exp((phi+psi-C)/eps) is <= tol.
// Zero-mass rows/columns are excluded exactly as the reference's masks do.
//
// One iteration = two streaming passes over C (16 B per entry), each an
// online max-rescaled log-sum-exp with a fixed reduction order:
//   R: one warp per row (coalesced 128-bit loads along the row)     -> phi
//   C: TM x 512 tiles, per-(tile, column) partials (max, sum), then a
//      fixed-order combine over the row tiles                        -> psi
// The row violation of iterate t falls out of the row pass of t+1 by the LSE
// identity rows(X_t)_i = exp(phi_t,i/eps + LSE_i(psi_t)); the column
// violation from the combine.  The final plan is materialised once and its
// violation recomputed from explicit row/column sums (the reported value).
#include <math.h>

#include "solver_internal.h"

namespace pdot {
namespace {

constexpr int kSkThreads = 256;

struct Lse {
  double m, s;  // running max and sum of exp(x - m)
};

__device__ __forceinline__ void lse_add(Lse& a, double x) {
  if (x == -INFINITY) return;
  if (x > a.m) {
    a.s = a.s * exp(a.m - x) + 1.0;
    a.m = x;
  } else {
    a.s += exp(x - a.m);
  }
}

__device__ __forceinline__ Lse lse_merge(Lse a, Lse b) {
  if (b.m == -INFINITY) return a;
  if (a.m == -INFINITY) return b;
  if (a.m >= b.m) return Lse{a.m, a.s + b.s * exp(b.m - a.m)};
  return Lse{b.m, b.s + a.s * exp(a.m - b.m)};
}

__device__ __forceinline__ double lse_value(Lse a) { return a.m + log(a.s); }

struct SkArgs {
  const double* C;
  int64_t ldc, m, n, ldx, TM, T;
  const double* f;
  const double* g;
  double eps, inv_eps;
  const double* phi_old;  // phi_t (row violation of iterate t)
  double* phi_new;        // phi_{t+1}
  const double* psi;      // psi_t for the row pass / psi_{t+1} output for the combine
  double* psi_out;
  double* part_m;         // [T][ldx]
  double* part_s;
  double* rowfeas;        // per row-block |rows(X_t) - f| partials
  double* colfeas;        // per column-block |cols(X_{t+1}) - g| partials
  int32_t* flags;         // [0] done, [1] non-finite, [2] iterations, [3] reason
};

// R: warp per row.  Writes phi_{t+1} and the row-violation partials of X_t.
__global__ void __launch_bounds__(kSkThreads) sk_row_kernel(SkArgs a) {
  if (a.flags[0]) return;
  __shared__ double red[kSkThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double feas = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * (kSkThreads / 32) + warp; i < a.m; i += (int64_t)gridDim.x * (kSkThreads / 32)) {
    const double fi = a.f[i];
    if (!(fi > 0.0)) {  // excluded row (sinkhorn.py:80-83): zero row of the plan
      if (lane == 0) a.phi_new[i] = 0.0;
      continue;
    }
    Lse acc{-INFINITY, 0.0};
    const double* Ci = a.C + i * a.ldc;
    for (int64_t j = 2 * lane; j < a.n; j += 64) {
      const double2 c = __ldcs(reinterpret_cast<const double2*>(Ci + j));
      const double2 ps = __ldg(reinterpret_cast<const double2*>(a.psi + j));
      const double2 gj = __ldg(reinterpret_cast<const double2*>(a.g + j));
      lse_add(acc, gj.x > 0.0 ? (ps.x - c.x) * a.inv_eps : -INFINITY);
      if (j + 1 < a.n) lse_add(acc, gj.y > 0.0 ? (ps.y - c.y) * a.inv_eps : -INFINITY);
    }
#pragma unroll
    for (int msk = 16; msk >= 1; msk >>= 1) {
      Lse o;
      o.m = __shfl_xor_sync(0xffffffffu, acc.m, msk);
      o.s = __shfl_xor_sync(0xffffffffu, acc.s, msk);
      acc = (lane & msk) ? lse_merge(o, acc) : lse_merge(acc, o);  // same order on both lanes
    }
    if (lane == 0) {
      const double L = lse_value(acc);
      a.phi_new[i] = a.eps * log(fi) - a.eps * L;          // sinkhorn.py:51
      const double r = exp(a.phi_old[i] * a.inv_eps + L);  // rows(X_t)_i
      feas += fabs(r - fi);
    }
  }
  if (lane == 0) red[warp] = feas;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kSkThreads / 32; ++w) s += red[w];
    a.rowfeas[blockIdx.x] = s;
  }
}

// C: per-(row tile, column) LSE partials of (phi_i - C_ij)/eps over the tile's rows.
__global__ void __launch_bounds__(kSkThreads) sk_col_kernel(SkArgs a) {
  if (a.flags[0]) return;
  const int64_t j = ((int64_t)blockIdx.x * kSkThreads + threadIdx.x) * 2;
  const int64_t t = blockIdx.y;
  const int64_t i0 = t * a.TM, i1 = imin64(a.m, i0 + a.TM);
  if (j >= a.n) return;
  Lse c0{-INFINITY, 0.0}, c1{-INFINITY, 0.0};
  for (int64_t i = i0; i < i1; ++i) {
    const double fi = __ldg(a.f + i);
    if (!(fi > 0.0)) continue;
    const double ph = __ldg(a.phi_new + i);
    const double2 c = __ldcs(reinterpret_cast<const double2*>(a.C + i * a.ldc + j));
    lse_add(c0, (ph - c.x) * a.inv_eps);
    lse_add(c1, (ph - c.y) * a.inv_eps);
  }
  *reinterpret_cast<double2*>(a.part_m + t * a.ldx + j) = make_double2(c0.m, c1.m);
  *reinterpret_cast<double2*>(a.part_s + t * a.ldx + j) = make_double2(c0.s, c1.s);
}

// combine the tile partials in row-tile order -> psi_{t+1}, column violation of X_{t+1}
__global__ void __launch_bounds__(kSkThreads) sk_colfin_kernel(SkArgs a) {
  if (a.flags[0]) return;
  __shared__ double red[kSkThreads / 32];
  const int64_t j = (int64_t)blockIdx.x * kSkThreads + threadIdx.x;
  double feas = 0.0;
  int bad = 0;
  if (j < a.n) {
    const double gj = a.g[j];
    if (gj > 0.0) {
      Lse acc{-INFINITY, 0.0};
      for (int64_t t = 0; t < a.T; ++t) acc = lse_merge(acc, Lse{a.part_m[t * a.ldx + j], a.part_s[t * a.ldx + j]});
      const double L = lse_value(acc);
      const double ps = a.eps * log(gj) - a.eps * L;  // sinkhorn.py:55
      a.psi_out[j] = ps;
      feas = fabs(exp(ps * a.inv_eps + L) - gj);
      bad = !isfinite(ps);
    } else {
      a.psi_out[j] = 0.0;
    }
  }
  for (int msk = 16; msk >= 1; msk >>= 1) {
    feas += __shfl_xor_sync(0xffffffffu, feas, msk);
    bad |= __shfl_xor_sync(0xffffffffu, bad, msk);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = feas;
  if (lane == 0 && bad) atomicOr(&a.flags[1], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kSkThreads / 32; ++w) s += red[w];
    a.colfeas[blockIdx.x] = s;
  }
}

// controller between R and C: feasibility of iterate t, loop-top limits.
__global__ void sk_ctl_kernel(SkArgs a, int nrb, int ncb, double tol, int64_t max_iters, double* colfeas_saved,
                              double* feas_out, int64_t* iters, uint64_t deadline_ns) {
  if (a.flags[0] || threadIdx.x != 0) return;
  const int64_t t = *iters;
  double rf = 0.0;
  for (int b = 0; b < nrb; ++b) rf += a.rowfeas[b];
  bool non_finite = a.flags[1] != 0;
  if (t >= 1) {
    const double feas = rf + *colfeas_saved;  // rows then columns, sinkhorn.py:111-113
    *feas_out = feas;
    if (non_finite) {  // sinkhorn.py:107-108 (an overflowing plan alone is just "not converged")
      a.flags[1] = 1;
      a.flags[0] = 1;
      return;
    }
    if (feas <= tol) {
      a.flags[0] = 1;
      a.flags[3] = 1;  // tolerance
      return;
    }
  }
  if (t >= max_iters) {
    a.flags[0] = 1;
    a.flags[3] = 2;  // iteration_limit
    return;
  }
  if (deadline_ns != 0 && globaltimer_ns() > deadline_ns) {
    a.flags[0] = 1;
    a.flags[3] = 3;  // time_limit
    return;
  }
  *iters = t + 1;
  a.flags[2] = (int32_t)(t + 1);
}

__global__ void sk_colsum_save(SkArgs a, int ncb, double* colfeas_saved) {
  if (a.flags[0] || threadIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < ncb; ++b) s += a.colfeas[b];
  *colfeas_saved = s;
}

// materialise X = exp((phi + psi - C)/eps) on the unmasked block, zeros elsewhere
__global__ void sk_plan_kernel(const double* C, int64_t ldc, int64_t m, int64_t n, const double* f,
                               const double* g, const double* phi, const double* psi, double eps, double* X,
                               int64_t ldx) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    double v = 0.0;
    if (f[i] > 0.0 && g[j] > 0.0) v = exp((phi[i] + psi[j] - C[i * ldc + j]) / eps);  // sinkhorn.py:46-47
    X[i * ldx + j] = v;
  }
}

}  // namespace
}  // namespace pdot

using namespace pdot;

extern "C" int pdot_sinkhorn_solve(pdot_solver* h, const pdot_sinkhorn_config* cfg, double elapsed_before_s,
                                   pdot_result* res) {
  if (!h || !cfg) return set_error(PDOT_EINVAL, "null argument");
  if (!h->problem_set || !h->host.C) return set_error(PDOT_ESTATE, "sinkhorn needs an explicit cost matrix");
  if (h->nranks != 1) return set_error(PDOT_EINVAL, "sinkhorn runs on a single GPU");
  if (!(cfg->penalty > 0)) return set_error(PDOT_EINVAL, "penalty must be positive");
  if (!(cfg->tol > 0) || cfg->max_iters < 1 || !(cfg->time_limit_s > 0))
    return set_error(PDOT_EINVAL, "tol, max_iters and time_limit_s must be positive");
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  const auto wall0 = std::chrono::steady_clock::now();
  const Ctl& c = h->host;
  cudaStream_t s = h->stream;
  // buffers: phi/psi ping-pong in slots 4 and 5, plan + final potentials in slot 0
  SkArgs a{};
  a.C = c.C;
  a.ldc = c.ldc;
  a.m = h->m;
  a.n = h->n;
  a.ldx = h->ldx;
  a.TM = h->TM;
  a.T = h->T;
  a.f = c.f;
  a.g = c.g;
  a.eps = cfg->penalty;
  a.inv_eps = 1.0 / cfg->penalty;
  a.part_m = c.colpart;
  a.part_s = c.colpart + h->T * h->ldx;
  a.rowfeas = c.rowblk;
  a.colfeas = c.colblk;
  double* phi[2] = {c.slot[4].p, c.slot[5].p};
  double* psi[2] = {c.slot[4].q, c.slot[5].q};
  double* scal = c.vec_a;  // [0] saved column violation, [1] feasibility, [2..3] iteration counter
  int32_t* flags = reinterpret_cast<int32_t*>(c.vec_b);
  int64_t* iters = reinterpret_cast<int64_t*>(scal + 2);
  a.flags = flags;
  const int nrb = (int)std::min<int64_t>((h->m + 7) / 8, 148 * 8);
  const int ncb = (int)((h->n + kSkThreads - 1) / kSkThreads);
  const dim3 cgrid((unsigned)((h->n + 2 * kSkThreads - 1) / (2 * kSkThreads)), (unsigned)h->T);
  cudaError_t e;
#define SKCK(x)                                                   \
  do {                                                            \
    if ((e = (x)) != cudaSuccess) return cuda_error(e, #x, __LINE__); \
  } while (0)
  SKCK(cudaMemsetAsync(phi[0], 0, h->m * sizeof(double), s));
  SKCK(cudaMemsetAsync(psi[0], 0, h->n * sizeof(double), s));
  SKCK(cudaMemsetAsync(flags, 0, 4 * sizeof(int32_t), s));
  SKCK(cudaMemsetAsync(scal, 0, 4 * sizeof(double), s));
  // time limit: checked by the host between batches (the reference checks at
  // the loop top, sinkhorn.py:97-99); an exhausted budget stops before iterating
  const double remaining = cfg->time_limit_s - elapsed_before_s;
  const uint64_t deadline = 0;
  static const int32_t stop_now[4] = {1, 0, 0, 3};
  if (remaining <= 0) SKCK(cudaMemcpyAsync(flags, stop_now, sizeof(stop_now), cudaMemcpyHostToDevice, s));
  // one "step" = R(t+1), ctl(t), C(t+1), combine(t+1), save column violation
  const int batch = cfg->poll_iters > 0 ? cfg->poll_iters : 16;
  int64_t launched = 0;
  int32_t hflags[4] = {0, 0, 0, 0};
  for (;;) {
    for (int b = 0; b < batch; ++b, ++launched) {
      const int cur = (int)(launched & 1), nxt = cur ^ 1;
      a.phi_old = phi[cur];
      a.phi_new = phi[nxt];
      a.psi = psi[cur];
      a.psi_out = psi[nxt];
      sk_row_kernel<<<nrb, kSkThreads, 0, s>>>(a);
      sk_ctl_kernel<<<1, 32, 0, s>>>(a, nrb, ncb, cfg->tol, cfg->max_iters, scal, scal + 1, iters, deadline);
      sk_col_kernel<<<cgrid, kSkThreads, 0, s>>>(a);
      sk_colfin_kernel<<<ncb, kSkThreads, 0, s>>>(a);
      sk_colsum_save<<<1, 32, 0, s>>>(a, ncb, scal);
      h->launches += 5;
    }
    SKCK(cudaGetLastError());
    SKCK(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s));
    SKCK(cudaStreamSynchronize(s));
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    if (hflags[0]) break;
    if (el + elapsed_before_s > cfg->time_limit_s) {
      SKCK(cudaMemcpyAsync(flags, stop_now, sizeof(int32_t), cudaMemcpyHostToDevice, s));
      SKCK(cudaStreamSynchronize(s));
      hflags[3] = 3;
      break;
    }
  }
  int64_t t = 0;
  SKCK(cudaMemcpyAsync(&t, iters, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SKCK(cudaStreamSynchronize(s));
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  if (hflags[1]) {
    if (prev >= 0) cudaSetDevice(prev);
    return set_error(PDOT_ENONFINITE, "numerical failure: non-finite potential");
  }
  // the potentials of iterate t live in buffer (t & 1)... the step that produced
  // iterate t wrote into buffer ((t-1)&1)^1 = t&1 (phi/psi after t updates)
  const int fin = (int)(t & 1);
  SKCK(cudaMemcpyAsync(c.slot[0].p, phi[fin], h->m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SKCK(cudaMemcpyAsync(c.slot[0].q, psi[fin], h->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  sk_plan_kernel<<<148 * 16, 256, 0, s>>>(c.C, c.ldc, h->m, h->n, c.f, c.g, phi[fin], psi[fin], cfg->penalty,
                                          c.slot[0].X, h->ldx);
  h->launches += 1;
  // slot 0 now holds the Sinkhorn plan and potentials; slots 4/5 the potential
  // buffers: refresh their screening metadata for later PDHG passes
  pdot::launch_slot_meta(c, 0, true, s);
  pdot::launch_slot_meta(c, 4, false, s);
  pdot::launch_slot_meta(c, 5, false, s);
  SKCK(cudaGetLastError());
  SKCK(cudaStreamSynchronize(s));
#undef SKCK
  if (res) {
    memset(res, 0, sizeof(*res));
    res->reason = hflags[3];
    res->final_slot = 0;
    res->iterations = t;
    res->elapsed_s = wall + elapsed_before_s;
  }
  if (prev >= 0) cudaSetDevice(prev);
  return PDOT_OK;
}
