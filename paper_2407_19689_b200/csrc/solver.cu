// Host runtime and C ABI of libpdot.so (include/pdot.h).
//
// One handle = one m x n problem shape on one GPU: it owns the NSLOT primal-dual
// slots, the reduction partials, the device control block, a host-mapped status
// mirror and trace ring, and one CUDA graph of `L` (stream pass, finalize pass)
// pairs.  pdot_solve() replays that graph until the device controller reports
// done; the host only polls the mapped status between graph launches (two
// batches in flight), so no iteration waits on the host.
#include <cuda_runtime.h>
#include <math.h>

#include <cmath>
#include <stdio.h>
#include <string.h>

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for Nsight Systems / ncu --nvtx

#include "../../include/pdot.h"
#include "pdot_internal.cuh"

using pdot::Ctl;

#include "solver_internal.h"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %s (%s) at solver.cu:%d in %s", cudaGetErrorName(e),
           cudaGetErrorString(e), line, what);
  return set_err(PDOT_ECUDA, buf);
}

}  // namespace
namespace pdot {
int set_error(int code, const std::string& msg) { return set_err(code, msg); }
int cuda_error(cudaError_t e, const char* what, int line) { return cuda_fail(e, what, line); }
}  // namespace pdot
namespace {

#define CK(x)                                                  \
  do {                                                         \
    cudaError_t e_ = (x);                                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x, __LINE__); \
  } while (0)

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

__global__ void stamp_deadline_kernel(Ctl* c, uint64_t remaining_ns) {
  c->deadline_ns = pdot::globaltimer_ns() + remaining_ns;
}

__global__ void set_int_kernel(int32_t* p, int32_t v) { *p = v; }

__global__ void apply_at_kernel(const double* __restrict__ p, const double* __restrict__ q, int64_t m,
                                int64_t n, double* __restrict__ out, int64_t ldo) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    out[i * ldo + j] = p[i] + q[j];  // operator.py:43
  }
}

__global__ void gen_cost_kernel(double* __restrict__ C, int64_t row0, int64_t m, int64_t n, int64_t ldc,
                                int kind, int64_t a0, int64_t a1, int64_t a2, int64_t a3) {
  const int64_t total = m * ldc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t il = e / ldc, j = e - il * ldc;
    const int64_t i = row0 + il;
    int64_t v = 0;
    if (j < n) {
      if (kind == PDOT_COST_SQEUCLID_GRID || kind == PDOT_COST_L1_GRID) {
        const int64_t r = a0;
        const int64_t di = i / r - j / r, dj = i % r - j % r;
        v = (kind == PDOT_COST_SQEUCLID_GRID) ? di * di + dj * dj : (di < 0 ? -di : di) + (dj < 0 ? -dj : dj);
      } else {
        const int64_t sc = a1, tc = a3;
        const int64_t ai = 2 * (i / sc), bi = 2 * (i % sc);
        const int64_t cj = j / tc, dj = j % tc;
        const int64_t x = ai - cj, y = bi - dj;
        v = (x < 0 ? -x : x) + (y < 0 ? -y : y);
      }
    }
    C[e] = (double)v;
  }
}

// deterministic sum of squares: per-block fixed tree, then one block in order
__global__ void sumsq_partial_kernel(const double* __restrict__ C, int64_t m, int64_t n, int64_t ldc,
                                     double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    const double v = C[i * ldc + j];
    acc = __fma_rn(v, v, acc);
  }
  for (int msk = 16; msk >= 1; msk >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, msk);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void sum_final_kernel(const double* __restrict__ part, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    *out = sqrt(s);
  }
}

int check_ld(int64_t ld, int64_t n, const char* what) {
  if (ld < n || (ld & 1)) {
    return set_err(PDOT_EINVAL, std::string(what) + ": leading dimension must be >= n and even");
  }
  return PDOT_OK;
}

int upload_ctl(pdot_solver* h) {
  CK(cudaMemcpyAsync(h->dev, &h->host, sizeof(Ctl), cudaMemcpyHostToDevice, h->stream));
  return PDOT_OK;
}

int download_ctl(pdot_solver* h) {
  CK(cudaMemcpyAsync(&h->host, h->dev, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PDOT_OK;
}

// one (stream, finalize) pass with an explicit op, outside any graph
int launch_pass(pdot_solver* h, int op);

int run_pass(pdot_solver* h, int op) {
  if (h->virtual_shards) return set_err(PDOT_ESTATE, "virtual shards are stepped with pdot_shard_pass");
  if (int rc = launch_pass(h, op)) return rc;
  CK(cudaGetLastError());
  return PDOT_OK;
}

void unit_ctl(pdot_solver* h) {
  Ctl& c = h->host;
  c.unit = 1;
  c.unit_avg = 0;
  c.done = 0;
  c.status = nullptr;
  c.ring = nullptr;
  c.kkt_write_viol = 0;
  c.viol_out = nullptr;
}

int copy_matrix(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t m, int64_t n,
                cudaStream_t s) {
  CK(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double), n * sizeof(double), m,
                       cudaMemcpyDefault, s));
  return PDOT_OK;
}

int copy_vec(double* dst, const double* src, int64_t n, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, s));
  return PDOT_OK;
}

// ---------------------------------------------------------------------------
// NCCL (torch's libnccl.so.2, loaded at run time only for multi-GPU handles)
// ---------------------------------------------------------------------------
struct NcclId {
  char internal[128];
};
struct NcclApi {
  bool ok = false;
  int (*get_unique_id)(NcclId*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclId, int) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(int) = nullptr;
};
constexpr int kNcclFloat64 = 8;  // ncclDouble

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* lib = nullptr;
  for (const char* nm : names) {
    lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (lib) break;
  }
  if (!lib) return api;
  api.get_unique_id = (int (*)(NcclId*))dlsym(lib, "ncclGetUniqueId");
  api.comm_init_rank = (int (*)(void**, int, NcclId, int))dlsym(lib, "ncclCommInitRank");
  api.all_gather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(lib, "ncclAllGather");
  api.comm_destroy = (int (*)(void*))dlsym(lib, "ncclCommDestroy");
  api.error_string = (const char* (*)(int))dlsym(lib, "ncclGetErrorString");
  api.ok = api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy && api.error_string;
  return api;
}

int nccl_fail(int r, const char* what) {
  std::string msg = std::string("NCCL error in ") + what + ": ";
  msg += nccl().error_string ? nccl().error_string(r) : "unknown";
  return set_err(PDOT_ENCCL, msg);
}

// Group-aligned row range of one shard (all ranks share the global tiling).
int shard_geometry(int64_t m_total, int64_t TM, int nranks, int rank, int64_t* Tg, int64_t* GS, int* g0,
                   int* g1, int64_t* row0, int64_t* row1) {
  const int64_t T = (m_total + TM - 1) / TM;
  if (nranks != 1 && nranks != 2 && nranks != 4 && nranks != 8)
    return set_err(PDOT_EINVAL, "row sharding supports 1, 2, 4 or 8 shards");
  if (rank < 0 || rank >= nranks) return set_err(PDOT_EINVAL, "rank out of range");
  if (nranks > 1 && T % pdot::kGroups != 0)
    return set_err(PDOT_EINVAL, "row sharding needs the number of 128-row tiles to be a multiple of 8");
  const int64_t gs = (T + pdot::kGroups - 1) / pdot::kGroups;
  const int per = pdot::kGroups / nranks;
  *Tg = T;
  *GS = gs;
  *g0 = rank * per;
  *g1 = (rank + 1) * per;
  const int64_t t0 = std::min<int64_t>((int64_t)*g0 * gs, T), t1 = std::min<int64_t>((int64_t)*g1 * gs, T);
  *row0 = std::min(t0 * TM, m_total);
  *row1 = std::min(t1 * TM, m_total);
  return PDOT_OK;
}

bool split_mode(const pdot_solver* h) { return h->nranks > 1 || h->force_split; }

// all-gather of the per-group partials (in place: every rank owns a contiguous chunk)
int exchange(pdot_solver* h) {
  if (h->virtual_shards) return PDOT_OK;  // the host copies between handles
  if (h->host.p2p) return PDOT_OK;        // the finalize kernels exchanged over peer memory
  if (!h->nccl_comm) return set_err(PDOT_ESTATE, "sharded handle without a communicator");
  const int per = pdot::kGroups / h->nranks;
  const size_t count = (size_t)per * h->gstride;
  double* send = h->gbuf + (size_t)h->rank * count;
  const int r = nccl().all_gather(send, h->gbuf, count, kNcclFloat64, h->nccl_comm, h->stream);
  if (r != 0) return nccl_fail(r, "ncclAllGather");
  return PDOT_OK;
}

// one pass: K1, then K2 (single GPU) or K2a -> exchange -> K2b (row shards)
// K1 of a pass: the dense TMA walker, or K0 screen + K1 sparse walker
int launch_k1(pdot_solver* h, int op) {
  if (h->host.screen) {
    pdot::launch_screened_pass(h->dev, h->host, op, h->stream);
    return (op < 0 || pdot::unit_pass(h->host, op)) ? 3 : 1;
  }
  // (dense walker below)
  pdot::launch_stream_pass(h->dev, h->host, op, h->stream);
  return 1;
}

// PDOT_DEBUG_SYNC=1: synchronise after K1 and K2 of every non-graph pass and
// name the failing one (debugging aid; never set in measurements)
int debug_sync(pdot_solver* h, const char* what) {
  static const bool on = getenv("PDOT_DEBUG_SYNC") && atoi(getenv("PDOT_DEBUG_SYNC")) != 0;
  if (!on) return PDOT_OK;
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(h->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return PDOT_OK;
  const cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(e, what, __LINE__);
  return PDOT_OK;
}

int launch_pass(pdot_solver* h, int op) {
  h->launches += launch_k1(h, op);
  if (int rc = debug_sync(h, "K1 of a pass")) return rc;
  if (!split_mode(h)) {
    pdot::launch_finalize_pass(h->dev, h->host, op, pdot::FIN_FUSED, h->stream);
    if (int rc = debug_sync(h, "K2 of a pass")) return rc;
    h->launches += 1;
  } else {
    pdot::launch_finalize_pass(h->dev, h->host, op, pdot::FIN_A, h->stream);
    if (int rc = exchange(h)) return rc;
    pdot::launch_finalize_pass(h->dev, h->host, op, pdot::FIN_B, h->stream);
    h->launches += 2;
  }
  return PDOT_OK;
}

// kernels per pass (graph replays count launches without re-launching)
int launches_per_pass(const pdot_solver* h) { return (h->host.screen ? 3 : 1) + (split_mode(h) ? 2 : 1); }

// screening metadata of one slot after its matrix / duals were written outside
// the STEP kernels: occupancy scanned from the data (or cleared for a zero
// matrix) and the dual bounds recomputed
void slot_meta(pdot_solver* h, int slot, bool X_written, bool X_zero) {
  const Ctl& c = h->host;
  uint32_t* occ = c.occ + (int64_t)slot * c.nbands * c.nstrips;
  if (X_zero) cudaMemsetAsync(occ, 0, (size_t)c.nbands * c.nstrips * sizeof(uint32_t), h->stream);
  pdot::launch_slot_meta(c, slot, X_written && !X_zero, h->stream);
}

// the slot matrix holds arbitrary data: every cell may be nonzero
void occ_invalidate(pdot_solver* h, int slot) {
  const Ctl& c = h->host;
  cudaMemsetAsync(c.occ + (int64_t)slot * c.nbands * c.nstrips, 0x01,
                  (size_t)c.nbands * c.nstrips * sizeof(uint32_t), h->stream);
  pdot::launch_tocc_fill(c, slot, 1, h->stream);
}

// Slack certificates start over with every solve (and resume): no records
// (NaN), zero drift.  PDOT_SREC=0 turns them off.
int srec_reset(pdot_solver* h) {
  Ctl& c = h->host;
  static const int env_on = getenv("PDOT_SREC") ? atoi(getenv("PDOT_SREC")) : 1;
  c.sr_on = c.screen && c.srec && env_on;
  if (!c.sr_on) return PDOT_OK;
  CK(cudaMemsetAsync(c.srec, 0xff, (size_t)c.nbands * c.ncells * sizeof(double), h->stream));
  CK(cudaMemsetAsync(c.sdp, 0, (size_t)c.nbands * sizeof(double), h->stream));
  CK(cudaMemsetAsync(c.sdq, 0, (size_t)c.ncells * sizeof(double), h->stream));
  return PDOT_OK;
}

// (re)build min C for the bound problem when screening is on
int screen_setup(pdot_solver* h) {
  Ctl& c = h->host;
  c.screen = 0;
  if (!h->screen_on || !h->problem_set) return PDOT_OK;
  pdot::launch_minc_build(c, h->minc_buf, h->stream);
  CK(cudaGetLastError());
  c.minc = h->minc_buf;
  c.screen = 1;
  return PDOT_OK;
}

// Device -> pageable host copy of an m x n matrix through the pinned double
// buffer: chunk k+1 is DMA'd while host threads copy chunk k out (page faults of
// fresh destination pages are taken in parallel too).
int d2h_matrix_bounced(pdot_solver* h, double* dst, int64_t ldd, const double* src, int64_t lds, int64_t m,
                       int64_t n) {
  const int64_t row_bytes = n * (int64_t)sizeof(double);
  if ((int64_t)h->bounce_bytes < row_bytes) return copy_matrix(dst, ldd, src, lds, m, n, h->stream);
  const int64_t rows_per = (int64_t)h->bounce_bytes / row_bytes;
  const int64_t nchunks = (m + rows_per - 1) / rows_per;
  const unsigned nthreads = 8;
  auto copy_out = [&](int64_t k) {
    const int64_t r0 = k * rows_per, rows = std::min(rows_per, m - r0);
    const char* b = reinterpret_cast<const char*>(h->bounce[k & 1]);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nthreads; ++t) {
      const int64_t a = rows * t / nthreads, e = rows * (t + 1) / nthreads;
      pool.emplace_back([=]() {
        for (int64_t r = a; r < e; ++r)
          memcpy(dst + (r0 + r) * ldd, b + r * row_bytes, (size_t)row_bytes);
      });
    }
    for (auto& th : pool) th.join();
  };
  for (int64_t k = 0; k < nchunks; ++k) {
    const int64_t r0 = k * rows_per, rows = std::min(rows_per, m - r0);
    CK(cudaMemcpy2DAsync(h->bounce[k & 1], (size_t)row_bytes, src + r0 * lds, (size_t)lds * sizeof(double),
                         (size_t)row_bytes, (size_t)rows, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaEventRecord(h->bounce_ev[k & 1], h->stream));
    if (k > 0) copy_out(k - 1);  // overlaps with the DMA of chunk k
    CK(cudaEventSynchronize(h->bounce_ev[k & 1]));
  }
  if (nchunks > 0) copy_out(nchunks - 1);
  return PDOT_OK;
}

bool is_pageable_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

void drain_ring(pdot_solver* h) {
  const int64_t head = h->status_h->ring_head;
  for (int64_t t = h->ring_tail; t < head; ++t) {
    const pdot::Event& e = h->ring_h[t & (pdot::kRingCap - 1)];
    pdot_event o;
    o.type = e.type;
    o.ia = e.ia;
    o.x = e.x;
    o.y = e.y;
    o.z = e.z;
    h->events.push_back(o);
  }
  h->ring_tail = head;
}

int build_graph(pdot_solver* h, int L) {
  if (h->graph && h->graph_L == L) return PDOT_OK;
  if (h->graph) {
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int rc = PDOT_OK;
  const int64_t before = h->launches;
  for (int i = 0; i < L && rc == PDOT_OK; ++i) rc = launch_pass(h, -1);
  h->launches = before;
  CK(cudaStreamEndCapture(h->stream, &g));
  if (rc) return rc;
  CK(cudaGraphInstantiate(&h->graph, g, 0));
  cudaGraphDestroy(g);
  h->graph_L = L;
  return PDOT_OK;
}

int auto_batch(const pdot_solver* h) {
  // aim for ~10 ms of work per graph launch (dense walker), 4..64 passes; a
  // screened pass costs about a twentieth of a dense one on sparse plans, so
  // poll every ~2 ms there (the controller may finish mid-batch: the rest of
  // the batch's kernels then exit at once)
  const double est_us = (h->host.screen ? 2.0 : 40.0) * (double)h->m * (double)h->n / 6.0e6 + 8.0;
  int L = (int)((h->host.screen ? 2000.0 : 10000.0) / est_us);
  if (L < 4) L = 4;
  if (L > 64) L = 64;
  return L;
}

// A restart paused for a host-evaluated primal weight (pdot_config.host_omega):
// omega = exp(theta log(dpq / dX) + (1 - theta) log(omega)) with the host's libm,
// the functions the reference's math.exp / math.log call (pdhg.py:185), same
// operation order, no contraction; then the device applies the restart.
int host_omega_resume(pdot_solver* h) {
  CK(cudaStreamSynchronize(h->stream));
  if (int rc = download_ctl(h)) return rc;
  const Ctl& c = h->host;
  const double omega = std::exp(c.theta * std::log(c.om_dpq / c.om_dX) + (1.0 - c.theta) * std::log(c.omega));
  pdot::launch_resume_restart(h->dev, omega, h->stream);
  h->launches += 1;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
  return download_ctl(h);
}

// NVTX range for the lifetime of a scope (no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// replay the graph until the controller reports done
int drive(pdot_solver* h, int L) {
  NvtxRange nv("pdot: solve loop (graph replays)");
  int rc = build_graph(h, L);
  if (rc) return rc;
  int64_t i = 0;
  for (;;) {
    CK(cudaGraphLaunch(h->graph, h->stream));
    h->launches += launches_per_pass(h) * L;
    CK(cudaEventRecord(h->ev[i & 1], h->stream));
    if (i > 0) {
      CK(cudaEventSynchronize(h->ev[(i - 1) & 1]));
      drain_ring(h);
      if (h->status_h->done) {
        if (!h->status_h->pause) break;
        // the batch in flight exits at once (done); resume after the host's omega
        if (int rc2 = host_omega_resume(h)) return rc2;
        i = 0;
        continue;
      }
    }
    ++i;
  }
  CK(cudaEventRecord(h->t1, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  drain_ring(h);
  return PDOT_OK;
}

int result_from_ctl(pdot_solver* h, pdot_result* res, double wall_s) {
  int rc = download_ctl(h);
  if (rc) return rc;
  const Ctl& c = h->host;
  h->saved = c;
  h->has_saved = true;
  if (res) {
    res->reason = c.reason;
    res->final_slot = c.sFinal;
    res->iterations = c.total;
    res->restarts = c.outer;
    res->passes = c.passes;
    res->rejected = c.rejected;
    res->final_relative_kkt = c.final_rel;
    res->eta = c.eta;
    res->omega = c.omega;
    res->scale_R = c.scale_R;
    res->elapsed_s = wall_s;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->t0, h->t1);
    res->device_s = ms * 1e-3;
  }
  if (c.error == pdot::E_NONFINITE)
    return set_err(PDOT_ENONFINITE, "numerical failure: non-finite iterate");
  if (c.error == pdot::E_LINESEARCH)
    return set_err(PDOT_ELINESEARCH, "step-size line search failed to find an admissible eta");
  if (c.error == pdot::E_EXCHANGE)
    return set_err(PDOT_ENCCL, "peer-memory exchange timed out (a rank stopped participating)");
  return PDOT_OK;
}

}  // namespace

extern "C" {

const char* pdot_last_error(void) { return g_err.c_str(); }

int pdot_version(void) { return 1; }

// Rows per streaming tile: 128 (measured best from 4096^2 up), halved for
// small plans until the grid has at least one tile per SM (1024^2: TM = 16,
// 5x faster than 128).  Depends on the GLOBAL shape only, so every shard of a
// row-sharded run uses the same tiling and reduction tree.
static int64_t row_tile(int64_t m_total, int64_t n) {
  int64_t TM = 128;
  const int64_t U = (n + pdot::kTileN - 1) / pdot::kTileN;
  while (TM > 16 && ((m_total + TM - 1) / TM) * U < 148) TM /= 2;
  if (const char* e = getenv("PDOT_TM")) TM = atoll(e);
  if (TM != 8 && TM != 16 && TM != 32 && TM != 64 && TM != 128 && TM != 256) TM = 128;
  return TM;
}

int pdot_shard_rows(int64_t m_total, int64_t n, int nranks, int rank, int64_t* row0, int64_t* row1) {
  if (m_total < 1 || n < 1) return set_err(PDOT_EINVAL, "plan dimensions must be positive");
  int64_t Tg, GS, r0, r1;
  int g0, g1;
  if (int rc = shard_geometry(m_total, row_tile(m_total, n), nranks, rank, &Tg, &GS, &g0, &g1, &r0, &r1)) return rc;
  if (row0) *row0 = r0;
  if (row1) *row1 = r1;
  return PDOT_OK;
}

int pdot_create(int64_t m, int64_t n, int device, pdot_solver** out) {
  return pdot_create_shard(m, n, 1, 0, device, out);
}

int pdot_create_shard(int64_t m_total, int64_t n, int nranks, int rank, int device, pdot_solver** out) {
  if (!out) return set_err(PDOT_EINVAL, "null output handle");
  *out = nullptr;
  if (m_total < 1 || n < 1) return set_err(PDOT_EINVAL, "plan dimensions must be positive");
  const int64_t TM = row_tile(m_total, n);
  int64_t Tg, GS, row0, row1;
  int g0, g1;
  if (int rc = shard_geometry(m_total, TM, nranks, rank, &Tg, &GS, &g0, &g1, &row0, &row1)) return rc;
  const int64_t m = row1 - row0;
  if (m < 1) return set_err(PDOT_EINVAL, "empty row shard");
  DeviceGuard dg(device);
  CK(cudaSetDevice(device));
  pdot_solver* h = new pdot_solver();
  h->device = device;
  h->m = m;
  h->n = n;
  h->ldx = round_up(n, 2);
  h->TM = TM;
  h->T = (m + TM - 1) / TM;
  h->nranks = nranks;
  h->rank = rank;
  h->m_total = m_total;
  h->row0 = row0;
  h->gstride = round_up(4 * h->ldx + pdot::kMaxRowScal, 2);
  h->U = (n + pdot::kTileN - 1) / pdot::kTileN;
  h->CB = (n + 127) / 128;  // finalize column blocks (kColsPerBlock)

  const int64_t mat = m * h->ldx;
  const int64_t per_slot = mat + round_up(m, 2) + h->ldx;
  size_t bytes_slots = (size_t)per_slot * pdot::kNSlot * sizeof(double);
  // work: colpart T*4*ldx, rowpart U*4*m, tilescal T*U*kMaxNS, rowblk T*16, colblk CB*8,
  //       rows_out 4*m, cols_out 4*ldx, vec_a 2*m, vec_b 2*ldx, scratch 64
  const int64_t w_colpart = h->T * 4 * h->ldx;
  const int64_t w_rowpart = h->U * 4 * round_up(m, 2);
  const int64_t w_tiles = h->T * h->U * pdot::kMaxNS;
  const int64_t w_rowblk = h->T * pdot::kMaxRowScal;
  const int64_t w_colblk = 2 * h->CB * pdot::kMaxColScal;  // one per 64-column half
  const int64_t w_rows = 4 * round_up(m, 2), w_cols = 4 * h->ldx;
  const int64_t w_va = 2 * round_up(m, 2), w_vb = 2 * h->ldx;
  const int64_t w_gbuf = pdot::kGroups * h->gstride;
  const int64_t w_total = w_colpart + w_rowpart + w_tiles + w_rowblk + w_colblk + w_rows + w_cols + w_va +
                          w_vb + w_gbuf + 4096;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaMalloc(&h->dev, sizeof(Ctl))) != cudaSuccess ||
      (e = cudaMalloc(&h->slot_mem, bytes_slots)) != cudaSuccess ||
      (e = cudaMalloc(&h->work, (size_t)w_total * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&h->counter, sizeof(unsigned) * 4)) != cudaSuccess ||
      (e = cudaHostAlloc(&h->status_h, sizeof(pdot::Status), cudaHostAllocMapped)) != cudaSuccess ||
      (e = cudaHostAlloc(&h->ring_h, sizeof(pdot::Event) * pdot::kRingCap, cudaHostAllocMapped)) !=
          cudaSuccess ||
      (e = cudaHostGetDevicePointer(&h->status_d, h->status_h, 0)) != cudaSuccess ||
      (e = cudaHostGetDevicePointer(&h->ring_d, h->ring_h, 0)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev[0], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev[1], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreate(&h->t0)) != cudaSuccess || (e = cudaEventCreate(&h->t1)) != cudaSuccess) {
    int rc = cuda_fail(e, "pdot_create allocation", __LINE__);
    pdot_destroy(h);
    return rc;
  }
  memset((void*)h->status_h, 0, sizeof(pdot::Status));
  if ((size_t)m * n * sizeof(double) >= ((size_t)64 << 20)) {  // plans of >= 64 MB
    h->bounce_bytes = (size_t)64 << 20;
    for (int i = 0; i < 2; ++i) {
      if ((e = cudaHostAlloc(&h->bounce[i], h->bounce_bytes, cudaHostAllocDefault)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&h->bounce_ev[i], cudaEventDisableTiming)) != cudaSuccess) {
        int rc = cuda_fail(e, "pdot_create bounce buffers", __LINE__);
        pdot_destroy(h);
        return rc;
      }
    }
  }
  {  // block-screening metadata (screen.cu): a few MB even at 16384^2
    const int64_t nbands = (m + pdot::kBand - 1) / pdot::kBand;
    const int64_t ncells = (n + pdot::kCell - 1) / pdot::kCell;
    const int64_t nstrips = (n + pdot::kStrip - 1) / pdot::kStrip;
    const int64_t nbt = TM / pdot::kBand;
    const int64_t tiles = h->T * h->U;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 255) & ~(size_t)255;
      return o;
    };
    const size_t o_minc = take(nbands * ncells * sizeof(double));
    const size_t o_occ = take(pdot::kNSlot * nbands * nstrips * sizeof(uint32_t));
    const size_t o_pmax = take(pdot::kNSlot * nbands * sizeof(double));
    const size_t o_qmax = take(pdot::kNSlot * ncells * sizeof(double));
    const int64_t nunits = nbands * nstrips;
    const int64_t ncp = h->U * 32;  // cells per band, padded to whole tiles
    const int64_t mpad = round_up(m, 2);
    (void)nunits;
    const size_t o_uflag = take(nbands * ncp + pdot::kListPad);
    const size_t o_ulist = take((nbands * ncp + pdot::kListPad) * sizeof(uint32_t));
    const size_t o_ucount = take(sizeof(unsigned));
    const size_t o_bcr = take(nbands * h->U * sizeof(uint32_t));
    const size_t o_bct = take(h->T * ncp * sizeof(uint32_t));
    const size_t o_tflag = take(h->T * h->U);
    const size_t o_tlist = take(h->T * h->U * sizeof(int32_t));
    const size_t o_tcount = take(sizeof(unsigned));
    const size_t o_stat = take(pdot::ST_COUNT * sizeof(unsigned long long));
    const size_t o_tocc = take(pdot::kNSlot * tiles);
    const size_t o_tminc = take(tiles * sizeof(double));
    const size_t o_srec = take(nbands * ncells * sizeof(double));
    const size_t o_sdp = take(nbands * sizeof(double));
    const size_t o_sdq = take(ncells * sizeof(double));
    // cell partials of screened passes (written sparsely, read back only where
    // the bit maps say so: never zeroed)
    const size_t o_ccol = take(nbands * pdot::kMaxNQ * h->ldx * sizeof(double));
    const size_t o_crow = take(ncp * pdot::kMaxNQ * mpad * sizeof(double));
    const size_t o_cscal = take(nbands * ncp * pdot::kMaxNS * sizeof(double));
    char* base = nullptr;
    // only the metadata needs zeroing; the unit partials are written before they are read
    if ((e = cudaMalloc(&base, off)) != cudaSuccess || (e = cudaMemsetAsync(base, 0, o_ccol, h->stream)) != cudaSuccess) {
      int rc = cuda_fail(e, "pdot_create screening metadata", __LINE__);
      pdot_destroy(h);
      return rc;
    }
    h->screen_mem = base;
    h->minc_buf = reinterpret_cast<double*>(base + o_minc);
    Ctl& c = h->host;
    c.nbt = (int32_t)nbt;
    c.nbands = nbands;
    c.ncells = ncells;
    c.nstrips = nstrips;
    c.occ = reinterpret_cast<uint32_t*>(base + o_occ);
    c.pmax = reinterpret_cast<double*>(base + o_pmax);
    c.qmax = reinterpret_cast<double*>(base + o_qmax);
    c.uflag = reinterpret_cast<uint8_t*>(base + o_uflag);
    c.ulist = reinterpret_cast<uint32_t*>(base + o_ulist);
    c.ucount = reinterpret_cast<unsigned*>(base + o_ucount);
    c.sstat = reinterpret_cast<unsigned long long*>(base + o_stat);
    c.bcr = reinterpret_cast<uint32_t*>(base + o_bcr);
    c.bct = reinterpret_cast<uint32_t*>(base + o_bct);
    c.tileflag = reinterpret_cast<uint8_t*>(base + o_tflag);
    c.tlist = reinterpret_cast<int32_t*>(base + o_tlist);
    c.tcount = reinterpret_cast<unsigned*>(base + o_tcount);
    c.tocc = reinterpret_cast<uint8_t*>(base + o_tocc);
    c.tminc = reinterpret_cast<const double*>(base + o_tminc);
    c.srec = reinterpret_cast<double*>(base + o_srec);
    c.sdp = reinterpret_cast<double*>(base + o_sdp);
    c.sdq = reinterpret_cast<double*>(base + o_sdq);
    c.ccol = reinterpret_cast<double*>(base + o_ccol);
    c.crow = reinterpret_cast<double*>(base + o_crow);
    c.cscal = reinterpret_cast<double*>(base + o_cscal);
    c.ncp = ncp;
    c.mpad = mpad;
    // a cell-list entry is one 32-bit word, (band << cbits) | cell: cbits grows with
    // the row of cells (n > 65536 needs more than 12 bits), the band takes the rest
    int cbits = 12;
    while (((int64_t)1 << cbits) < ncp) ++cbits;
    c.cbits = cbits;
    h->screen_ok = cbits < 32 && nbands <= ((int64_t)1 << (32 - cbits));
    // PDOT_SCREEN=0/1 forces the walker; by default the screened pass is used
    // from 2^22 plan entries up (below that the plan is L2-resident and the
    // single dense launch per pass wins, e.g. 1024^2)
    if (getenv("PDOT_K2_TRACE") && atoi(getenv("PDOT_K2_TRACE")) != 0) {
      unsigned long long* kd = nullptr;
      if (cudaMalloc(&kd, (size_t)((h->CB + h->T) * 4 + 32) * sizeof(unsigned long long)) == cudaSuccess) {
        c.kdbg = kd;
        c.ktl = kd + (h->CB + h->T) * 4;
        unsigned long long init[16];
        for (int k = 0; k < 16; ++k) init[k] = (k < 8 && (k & 1) == 0) ? ~0ull : 0ull;
        cudaMemcpy(c.ktl, init, sizeof(init), cudaMemcpyHostToDevice);
      }
    }
    const char* env = getenv("PDOT_SCREEN");
    h->screen_on = h->screen_ok && (env ? atoi(env) != 0 : (double)m_total * (double)n >= (double)(1 << 22));
  }
  if (nranks > 1) {  // peer-memory exchange buffer (separate allocation: shareable by CUDA IPC)
    h->xbuf_bytes = (size_t)(2 * pdot::kGroups * h->gstride) * sizeof(double) +
                    (2 * pdot::kMaxRanks + 1) * sizeof(unsigned long long);
    if ((e = cudaMalloc(&h->xbuf, h->xbuf_bytes)) != cudaSuccess ||
        (e = cudaMemsetAsync(h->xbuf, 0, h->xbuf_bytes, h->stream)) != cudaSuccess) {
      int rc = cuda_fail(e, "pdot_create exchange buffer", __LINE__);
      pdot_destroy(h);
      return rc;
    }
  }
  if ((e = cudaMemsetAsync(h->slot_mem, 0, bytes_slots, h->stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(h->work, 0, (size_t)w_total * sizeof(double), h->stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(h->counter, 0, sizeof(unsigned) * 4, h->stream)) != cudaSuccess) {
    int rc = cuda_fail(e, "pdot_create memset", __LINE__);
    pdot_destroy(h);
    return rc;
  }
  Ctl& c = h->host;  // value-initialised with the handle; the screening fields are already set
  c.m = m;
  c.n = n;
  c.ldx = h->ldx;
  c.ldc = h->ldx;
  c.T = h->T;
  c.U = h->U;
  c.TM = TM;
  c.CB = h->CB;
  c.ncolblk = (n + 63) / 64;
  for (int s = 0; s < pdot::kNSlot; ++s) {
    double* base = h->slot_mem + (size_t)s * per_slot;
    c.slot[s].X = base;
    c.slot[s].p = base + mat;
    c.slot[s].q = base + mat + round_up(m, 2);
  }
  double* w = h->work;
  c.colpart = w; w += w_colpart;
  c.rowpart = w; w += w_rowpart;
  c.tilescal = w; w += w_tiles;
  c.rowblk = w; w += w_rowblk;
  c.colblk = w; w += w_colblk;
  c.rows_out = w; w += w_rows;
  c.cols_out = w; w += w_cols;
  c.vec_a = w; w += w_va;
  c.vec_b = w; w += w_vb;
  c.gbuf = w; w += w_gbuf;
  h->gbuf = c.gbuf;
  c.gstride = h->gstride;
  c.m_total = m_total;
  c.row0 = row0;
  c.Tg = Tg;
  c.t0 = row0 / TM;
  c.GS = GS;
  c.g0 = g0;
  c.g1 = g1;
  c.nranks = nranks;
  c.rank = rank;
  c.counter = h->counter;
  c.status = h->status_d;
  c.ring = h->ring_d;
  c.op = pdot::OP_NONE;
  c.done = 1;
  c.sX = 0;
  c.sA = c.sZ = c.sB = 0;
  if (upload_ctl(h) != PDOT_OK || cudaStreamSynchronize(h->stream) != cudaSuccess) {
    int rc = set_err(PDOT_ECUDA, "pdot_create: control block upload failed");
    pdot_destroy(h);
    return rc;
  }
  // kernel attributes (per device), outside any capture
  pdot::prepare_stream_kernel();
  pdot::prepare_sparse_kernel();
  pdot::launch_stream_pass(h->dev, h->host, pdot::OP_NONE, h->stream);
  if ((e = cudaStreamSynchronize(h->stream)) != cudaSuccess) {
    int rc = cuda_fail(e, "pdot_create warmup", __LINE__);
    pdot_destroy(h);
    return rc;
  }
  *out = h;
  return PDOT_OK;
}

int pdot_destroy(pdot_solver* h) {
  if (!h) return PDOT_OK;
  DeviceGuard dg(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->nccl_comm && nccl().ok) nccl().comm_destroy(h->nccl_comm);
  for (int r = 0; r < pdot::kMaxRanks; ++r)
    if (h->ipc_opened[r]) cudaIpcCloseMemHandle(h->ipc_opened[r]);
  if (h->xbuf) cudaFree(h->xbuf);
  if (h->dev) cudaFree(h->dev);
  if (h->slot_mem) cudaFree(h->slot_mem);
  if (h->work) cudaFree(h->work);
  if (h->screen_mem) cudaFree(h->screen_mem);
  if (h->d2h_count) cudaFree(h->d2h_count);
  if (h->counter) cudaFree(h->counter);
  if (h->status_h) cudaFreeHost(h->status_h);
  for (int i = 0; i < 2; ++i) {
    if (h->bounce[i]) cudaFreeHost(h->bounce[i]);
    if (h->bounce_ev[i]) cudaEventDestroy(h->bounce_ev[i]);
  }
  if (h->ring_h) cudaFreeHost(h->ring_h);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->t0) cudaEventDestroy(h->t0);
  if (h->t1) cudaEventDestroy(h->t1);
  if (h->ph0) cudaEventDestroy(h->ph0);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return PDOT_OK;
}

int pdot_geometry(const pdot_solver* h, int64_t* ldx, int64_t* row_tile, int64_t* n_row_tiles,
                  int64_t* n_col_tiles) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  if (ldx) *ldx = h->ldx;
  if (row_tile) *row_tile = h->TM;
  if (n_row_tiles) *n_row_tiles = h->T;
  if (n_col_tiles) *n_col_tiles = h->U;
  return PDOT_OK;
}

int pdot_set_problem(pdot_solver* h, const double* C_dev, int64_t ldc, const double* f_dev,
                     const double* g_dev, double cost_fro_norm, double marginal_norm) {
  if (!h || !C_dev || !f_dev || !g_dev) return set_err(PDOT_EINVAL, "null argument");
  if (int rc = check_ld(ldc, h->n, "C")) return rc;
  if (((uintptr_t)C_dev & 15) != 0) return set_err(PDOT_EINVAL, "C must be 16-byte aligned");
  if (h->graph && h->host.ldc != ldc) {  // K1 takes ldc as a captured kernel parameter
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  h->host.C = C_dev;
  h->host.ldc = ldc;
  h->host.cost_kind = pdot::COST_EXPLICIT;
  h->host.f = f_dev;
  h->host.g = g_dev;
  h->host.cost_fro = cost_fro_norm;
  h->host.marg_norm = marginal_norm;
  h->problem_set = true;
  DeviceGuard dg(h->device);
  return screen_setup(h);
}

int pdot_set_problem_implicit(pdot_solver* h, int kind, const int64_t* a, const double* f_dev,
                              const double* g_dev, double cost_fro_norm, double marginal_norm) {
  if (!h || !a || !f_dev || !g_dev) return set_err(PDOT_EINVAL, "null argument");
  const int64_t m_total = h->m_total, n = h->n;
  if (kind == PDOT_COST_SQEUCLID_GRID || kind == PDOT_COST_L1_GRID) {
    if (a[0] != a[1] || a[0] * a[1] != n || m_total != n) return set_err(PDOT_EINVAL, "grid cost needs m = n = r*r");
  } else if (kind == PDOT_COST_L1_RECT) {
    if (a[0] * a[1] != m_total || a[2] * a[3] != n) return set_err(PDOT_EINVAL, "rect cost shape mismatch");
  } else {
    return set_err(PDOT_EINVAL, "unknown cost kind");
  }
  if (h->graph && h->host.ldc != h->ldx) {  // K1 takes ldc as a captured kernel parameter
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  h->host.C = nullptr;
  h->host.ldc = h->ldx;
  h->host.cost_kind = kind == PDOT_COST_SQEUCLID_GRID ? pdot::COST_SQEUCLID
                      : kind == PDOT_COST_L1_GRID     ? pdot::COST_L1GRID
                                                      : pdot::COST_L1RECT;
  for (int i = 0; i < 4; ++i) h->host.cost_a[i] = a[i];
  h->host.f = f_dev;
  h->host.g = g_dev;
  h->host.cost_fro = cost_fro_norm;
  h->host.marg_norm = marginal_norm;
  h->problem_set = true;
  DeviceGuard dg(h->device);
  return screen_setup(h);
}

int pdot_set_slot(pdot_solver* h, int slot, const double* X_any, int64_t ldX, const double* p_any,
                  const double* q_any) {
  if (!h || slot < 0 || slot >= pdot::kNSlot) return set_err(PDOT_EINVAL, "bad handle or slot");
  DeviceGuard dg(h->device);
  const pdot::Slot& s = h->host.slot[slot];
  if (X_any) {
    if (ldX < h->n) return set_err(PDOT_EINVAL, "X: leading dimension must be >= n");
    if (int rc = copy_matrix(s.X, h->ldx, X_any, ldX, h->m, h->n, h->stream)) return rc;
  } else {
    CK(cudaMemsetAsync(s.X, 0, (size_t)h->m * h->ldx * sizeof(double), h->stream));
  }
  if (p_any) {
    if (int rc = copy_vec(s.p, p_any, h->m, h->stream)) return rc;
  } else {
    CK(cudaMemsetAsync(s.p, 0, h->m * sizeof(double), h->stream));
  }
  if (q_any) {
    if (int rc = copy_vec(s.q, q_any, h->n, h->stream)) return rc;
  } else {
    CK(cudaMemsetAsync(s.q, 0, h->n * sizeof(double), h->stream));
  }
  slot_meta(h, slot, true, X_any == nullptr);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
  return PDOT_OK;
}

int pdot_get_slot(pdot_solver* h, int slot, double* X_any, int64_t ldX, double* p_any, double* q_any) {
  if (!h || slot < 0 || slot >= pdot::kNSlot) return set_err(PDOT_EINVAL, "bad handle or slot");
  DeviceGuard dg(h->device);
  const pdot::Slot& s = h->host.slot[slot];
  if (X_any) {
    if (ldX < h->n) return set_err(PDOT_EINVAL, "X: leading dimension must be >= n");
    if (h->bounce[0] && is_pageable_host(X_any)) {
      if (int rc = d2h_matrix_bounced(h, X_any, ldX, s.X, h->ldx, h->m, h->n)) return rc;
    } else if (int rc = copy_matrix(X_any, ldX, s.X, h->ldx, h->m, h->n, h->stream)) {
      return rc;
    }
  }
  if (p_any)
    if (int rc = copy_vec(p_any, s.p, h->m, h->stream)) return rc;
  if (q_any)
    if (int rc = copy_vec(q_any, s.q, h->n, h->stream)) return rc;
  CK(cudaStreamSynchronize(h->stream));
  return PDOT_OK;
}

// Sparse device -> host copy of a slot (screened handles): only the cells whose
// occupancy byte is set are moved; every other cell is +0.0 in device memory
// (the screening invariant), so X_host must come zero-filled (np.zeros).  The
// occupied cells are gathered into device staging, DMA'd through the pinned
// double buffer and scattered by host threads while the next chunk moves.
int pdot_get_slot_sparse(pdot_solver* h, int slot, double* X_host, int64_t ldX, double* p_any, double* q_any,
                         int64_t* cells_out) {
  NvtxRange nv("pdot: sparse device->host plan copy");
  if (!h || slot < 0 || slot >= pdot::kNSlot || !X_host) return set_err(PDOT_EINVAL, "bad argument");
  if (ldX < h->n) return set_err(PDOT_EINVAL, "X: leading dimension must be >= n");
  if (!h->host.screen) return set_err(PDOT_ESTATE, "sparse copy needs a screened handle (occupancy maintained)");
  DeviceGuard dg(h->device);
  const Ctl& c = h->host;
  if (!h->d2h_count) CK(cudaMalloc(&h->d2h_count, sizeof(unsigned)));
  const unsigned cnt = pdot::launch_occ_list(c, slot, c.ulist, h->d2h_count, h->stream);
  CK(cudaGetLastError());
  if (cells_out) *cells_out = cnt;
  constexpr int64_t kCellVals = pdot::kBand * pdot::kCell;  // 128 doubles per cell
  if (cnt > 0) {
    // chunk = what fits one pinned bounce buffer and the device staging area (the
    // per-pass cell partial buffer, idle between solves)
    if (!h->bounce[0]) {
      // the same 64 MB the dense path allocates for big plans: a later dense
      // get_slot on this handle reuses the buffer (d2h_matrix_bounced)
      const size_t want = (size_t)64 << 20;
      for (int i = 0; i < 2; ++i) {
        CK(cudaHostAlloc(&h->bounce[i], want, cudaHostAllocDefault));
        CK(cudaEventCreateWithFlags(&h->bounce_ev[i], cudaEventDisableTiming));
      }
      h->bounce_bytes = want;
    }
    const int64_t stage_cells = (c.nbands * pdot::kMaxNQ * c.ldx) / kCellVals;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>((int64_t)(h->bounce_bytes / (kCellVals * 8)), stage_cells));
    const int64_t nchunks = ((int64_t)cnt + chunk - 1) / chunk;
    std::vector<uint32_t> list(cnt);
    CK(cudaMemcpyAsync(list.data(), c.ulist, cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
    auto scatter = [&](int64_t k) {
      const int64_t k0 = k * chunk, k1 = std::min<int64_t>((int64_t)cnt, k0 + chunk);
      const double* b = h->bounce[k & 1];
      // visit the chunk's cells in row order and give each host thread a
      // contiguous row range: first touches of the zero-filled destination then
      // fault pages in without threads contending for the same page tables
      std::vector<int64_t> order((size_t)(k1 - k0));
      for (int64_t t = k0; t < k1; ++t) order[t - k0] = t;
      std::sort(order.begin(), order.end(), [&](int64_t a, int64_t e) { return list[a] < list[e]; });
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      const unsigned nthreads = (k1 - k0) > 2048 ? std::min(hw, 32u) : 1;
      auto work = [&, b, k0](int64_t a, int64_t e) {
        for (int64_t u = a; u < e; ++u) {
          const int64_t t = order[u];
          const uint32_t entry = list[t];
          const int64_t i0 = pdot::entry_band(entry, c.cbits) * pdot::kBand;
          const int64_t j0 = pdot::entry_cell(entry, c.cbits) * pdot::kCell;
          const int64_t rows = std::min<int64_t>(pdot::kBand, h->m - i0), cols = std::min<int64_t>(pdot::kCell, h->n - j0);
          const double* src = b + (t - k0) * kCellVals;
          for (int64_t r = 0; r < rows; ++r)
            memcpy(X_host + (i0 + r) * ldX + j0, src + r * pdot::kCell, (size_t)cols * sizeof(double));
        }
      };
      if (nthreads == 1) {
        work(0, (int64_t)order.size());
        return;
      }
      std::vector<std::thread> pool;
      const int64_t nn = (int64_t)order.size();
      for (unsigned t = 0; t < nthreads; ++t) pool.emplace_back(work, nn * t / nthreads, nn * (t + 1) / nthreads);
      for (auto& th : pool) th.join();
    };
    for (int64_t k = 0; k < nchunks; ++k) {
      const int64_t k0 = k * chunk, k1 = std::min<int64_t>((int64_t)cnt, k0 + chunk);
      pdot::launch_cell_gather(c, slot, c.ulist, k0, k1, c.ccol, h->stream);
      CK(cudaMemcpyAsync(h->bounce[k & 1], c.ccol, (size_t)(k1 - k0) * kCellVals * sizeof(double),
                         cudaMemcpyDeviceToHost, h->stream));
      CK(cudaEventRecord(h->bounce_ev[k & 1], h->stream));
      if (k == 0) CK(cudaStreamSynchronize(h->stream));  // the list is on the host now
      if (k > 0) scatter(k - 1);  // overlaps with the DMA of chunk k
      CK(cudaEventSynchronize(h->bounce_ev[k & 1]));
    }
    scatter(nchunks - 1);
  }
  if (p_any)
    if (int rc = copy_vec(p_any, c.slot[slot].p, h->m, h->stream)) return rc;
  if (q_any)
    if (int rc = copy_vec(q_any, c.slot[slot].q, h->n, h->stream)) return rc;
  CK(cudaStreamSynchronize(h->stream));
  return PDOT_OK;
}

int pdot_slot_ptrs(pdot_solver* h, int slot, double** X, double** p, double** q) {
  if (!h || slot < 0 || slot >= pdot::kNSlot) return set_err(PDOT_EINVAL, "bad handle or slot");
  if (X) *X = h->host.slot[slot].X;
  if (p) *p = h->host.slot[slot].p;
  if (q) *q = h->host.slot[slot].q;
  return PDOT_OK;
}

int pdot_begin(pdot_solver* h, const pdot_config* cfg, double elapsed_before_s) {
  NvtxRange nv("pdot: begin (start KKT setup)");
  if (!h || !cfg) return set_err(PDOT_EINVAL, "null argument");
  if (!h->problem_set) return set_err(PDOT_ESTATE, "pdot_set_problem was not called");
  // pdhg.py:61-75
  if (!(cfg->tol > 0) || !(cfg->time_limit_s > 0) || cfg->max_iters < 1)
    return set_err(PDOT_EINVAL, "tol, time_limit_s and max_iters must be positive");
  if (!(cfg->beta > 0.0 && cfg->beta < 1.0)) return set_err(PDOT_EINVAL, "beta must lie in (0, 1)");
  if (!(0.0 < cfg->beta_sufficient && cfg->beta_sufficient < cfg->beta_necessary && cfg->beta_necessary < 1.0))
    return set_err(PDOT_EINVAL, "need 0 < beta_sufficient < beta_necessary < 1");
  if (cfg->kkt_stride < 1) return set_err(PDOT_EINVAL, "kkt_stride must be >= 1");
  if (!(cfg->omega0 > 0)) return set_err(PDOT_EINVAL, "step parameters must be positive");
  DeviceGuard dg(h->device);
  h->wall0 = std::chrono::steady_clock::now();
  h->elapsed_before = elapsed_before_s;
  h->poll_L = cfg->poll_passes > 0 ? cfg->poll_passes : auto_batch(h);
  Ctl& c = h->host;
  c.unit = 0;
  c.unit_avg = 0;
  c.tol = cfg->tol;
  c.beta = cfg->beta;
  c.beta_suff = cfg->beta_sufficient;
  c.beta_nec = cfg->beta_necessary;
  c.beta_art = cfg->beta_artificial;
  c.theta = cfg->theta;
  c.eps_zero = cfg->eps_zero;
  c.max_iters = cfg->max_iters;
  c.kkt_stride = cfg->kkt_stride;
  c.adaptive = cfg->adaptive;
  c.relative = cfg->relative;
  c.trace_level = cfg->trace_level;
  c.host_omega = cfg->host_omega;
  c.omega_wait = 0;
  c.eta = cfg->eta0 > 0 ? cfg->eta0 : 1.0 / (2.0 * sqrt((double)(h->m_total + h->n)));  // pdhg.py:225-227
  c.omega = cfg->omega0;
  c.tau = c.sigma = c.kd = c.rkd = c.kd_dual = c.rkd_dual = 0.0;
  c.sAsrc = 0;
  c.lagA = 0;
  c.avg_written = 0;
  c.avg_slot = 0;
  c.total = c.inner = c.outer = c.passes = c.halvings = c.rejected = 0;
  c.pending = 0;
  c.sX = c.sA = c.sZ = c.sB = c.sFinal = 0;
  c.sXn = 1;
  c.sAn = 2;
  c.op = pdot::OP_KKT;
  c.done = 0;
  c.reason = c.error = 0;
  c.ring_head = 0;
  c.status = h->status_d;
  c.ring = h->ring_d;
  c.kkt_write_viol = 0;
  c.viol_out = nullptr;
  const double remaining = cfg->time_limit_s - elapsed_before_s;
  c.stop_request = remaining <= 0.0 ? 1 : 0;
  c.deadline_ns = 0;
  memset((void*)h->status_h, 0, sizeof(pdot::Status));
  h->ring_tail = 0;
  h->events.clear();
  if (int rc = srec_reset(h)) return rc;
  if (int rc = upload_ctl(h)) return rc;
  if (c.sstat)  // the pass-gap statistics start over: no gap across the host's work between solves
    CK(cudaMemsetAsync(c.sstat + pdot::ST_K2_END, 0, sizeof(unsigned long long), h->stream));
  if (remaining > 0.0 && remaining < 1e9) {
    stamp_deadline_kernel<<<1, 1, 0, h->stream>>>(h->dev, (uint64_t)(remaining * 1e9));
    h->launches += 1;
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(h->t0, h->stream));
  return PDOT_OK;
}

int pdot_advance(pdot_solver* h, int64_t max_passes, pdot_progress* prog) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  if (h->virtual_shards) return set_err(PDOT_ESTATE, "virtual shards are stepped with pdot_shard_pass");
  DeviceGuard dg(h->device);
  if (max_passes < 0) {
    if (int rc = drive(h, h->poll_L)) return rc;
  } else {
    for (int64_t i = 0; i < max_passes; ++i) {
      if (int rc = run_pass(h, -1)) return rc;
      if (h->host.host_omega) {  // a pass may have paused for a host-evaluated omega
        CK(cudaStreamSynchronize(h->stream));
        if (h->status_h->pause)
          if (int rc = host_omega_resume(h)) return rc;
      }
    }
    CK(cudaEventRecord(h->t1, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    drain_ring(h);
  }
  if (prog) {
    if (int rc = download_ctl(h)) return rc;
    const Ctl& c = h->host;
    prog->done = c.done;
    prog->roles[0] = c.sX;
    prog->roles[1] = c.sA;
    prog->roles[2] = c.sZ;
    prog->roles[3] = c.sB;
    prog->op = c.op;
    prog->iterations = c.total;
    prog->restarts = c.outer;
    prog->passes = c.passes;
    prog->avg_written = c.avg_written;
    prog->avg_slot = c.avg_slot;
  }
  return PDOT_OK;
}

int pdot_finish(pdot_solver* h, pdot_result* res) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  DeviceGuard dg(h->device);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - h->wall0).count();
  return result_from_ctl(h, res, wall + h->elapsed_before);
}

int pdot_solve(pdot_solver* h, const pdot_config* cfg, double elapsed_before_s, pdot_result* res) {
  if (int rc = pdot_begin(h, cfg, elapsed_before_s)) return rc;
  if (int rc = pdot_advance(h, -1, nullptr)) return rc;
  return pdot_finish(h, res);
}

int pdot_resume(pdot_solver* h, int64_t max_iters, pdot_result* res) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  DeviceGuard dg(h->device);
  if (!h->has_saved) return set_err(PDOT_ESTATE, "pdot_resume: no finished solve on this handle");
  h->host = h->saved;
  Ctl& c = h->host;
  if (c.unit || c.error || c.reason == pdot::R_TOL || c.reason == pdot::R_NONE)
    return set_err(PDOT_ESTATE, "pdot_resume: no limited run to resume");
  c.max_iters = max_iters;
  c.done = 0;
  c.reason = 0;
  c.op = pdot::OP_STEP;  // re-run the trial that the limit discarded
  c.deadline_ns = 0;
  c.stop_request = 0;
  memset((void*)h->status_h, 0, sizeof(pdot::Status));
  h->status_h->ring_head = c.ring_head;
  if (int rc = srec_reset(h)) return rc;
  if (int rc = upload_ctl(h)) return rc;
  CK(cudaEventRecord(h->t0, h->stream));
  const auto wall0 = std::chrono::steady_clock::now();
  if (int rc = drive(h, h->poll_L)) return rc;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  return result_from_ctl(h, res, wall);
}

int64_t pdot_get_events(pdot_solver* h, pdot_event* out, int64_t cap) {
  if (!h) return 0;
  const int64_t k = std::min<int64_t>(cap, (int64_t)h->events.size());
  if (out && k > 0) memcpy(out, h->events.data(), k * sizeof(pdot_event));
  h->events.erase(h->events.begin(), h->events.begin() + k);
  return k;
}

int pdot_round(pdot_solver* h, int slot, double* Xf_any, int64_t ldX, double* out3) {
  NvtxRange nv("pdot: rounding");
  if (!h || slot < 0 || slot >= pdot::kNSlot) return set_err(PDOT_EINVAL, "bad handle or slot");
  if (!h->problem_set) return set_err(PDOT_ESTATE, "pdot_set_problem was not called");
  DeviceGuard dg(h->device);
  Ctl& c = h->host;
  unit_ctl(h);
  c.sX = slot;
  const int scratch = (slot + 1) % pdot::kNSlot;
  c.viol_out = Xf_any ? c.slot[scratch].X : nullptr;
  c.round_stage = 0;
  c.op = pdot::OP_ROUND;
  if (int rc = upload_ctl(h)) return rc;
  for (int stage = 0; stage < 4; ++stage) {
    set_int_kernel<<<1, 1, 0, h->stream>>>(&h->dev->round_stage, stage);
    h->launches += 1;
    if (int rc = run_pass(h, pdot::OP_ROUND)) return rc;
  }
  double outv[24];
  CK(cudaMemcpyAsync(outv, h->dev->out, sizeof(outv), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (out3) {
    out3[0] = outv[pdot::OUT_ROUND_OBJ];
    out3[1] = outv[pdot::OUT_ROUND_DUAL];
    out3[2] = outv[pdot::OUT_ROUND_L1VIOL];
  }
  if (Xf_any) {
    occ_invalidate(h, scratch);  // X_feas now lives in the scratch slot
    if (ldX < h->n) return set_err(PDOT_EINVAL, "X_feas: leading dimension must be >= n");
    if (int rc = copy_matrix(Xf_any, ldX, c.slot[scratch].X, h->ldx, h->m, h->n, h->stream)) return rc;
    CK(cudaStreamSynchronize(h->stream));
  }
  return PDOT_OK;
}

int pdot_unit_step(pdot_solver* h, double tau, double sigma, double k) {
  if (!h || !h->problem_set) return set_err(PDOT_ESTATE, "problem not set");
  DeviceGuard dg(h->device);
  Ctl& c = h->host;
  unit_ctl(h);
  const bool avg = k > 0;
  c.unit_avg = avg ? 1 : 0;
  // with k: average matrix in slot 2 -> slot 3 (from the input iterate), average
  // duals in slot 3 updated in place from the trial duals (the loop's lazy/eager split)
  c.sX = 0; c.sXn = 1;
  c.sAsrc = avg ? 2 : 0; c.sA = avg ? 3 : 0; c.sAn = avg ? 3 : 2;
  c.tau = tau; c.sigma = sigma;
  c.kd = avg ? k : 1.0; c.rkd = 1.0 / c.kd;
  c.kd_dual = c.kd; c.rkd_dual = c.rkd;
  c.op = pdot::OP_STEP;
  if (int rc = upload_ctl(h)) return rc;
  if (int rc = run_pass(h, pdot::OP_STEP)) return rc;
  CK(cudaStreamSynchronize(h->stream));
  return PDOT_OK;
}

int pdot_unit_bound(pdot_solver* h, double omega, double eps_zero, double* out5) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  DeviceGuard dg(h->device);
  Ctl& c = h->host;
  unit_ctl(h);
  c.sX = 0; c.sXn = 1;
  c.omega = omega; c.eps_zero = eps_zero;
  c.op = pdot::OP_DIFF;
  if (int rc = upload_ctl(h)) return rc;
  if (int rc = run_pass(h, pdot::OP_DIFF)) return rc;
  double o[5];
  CK(cudaMemcpyAsync(o, &h->dev->out[0], 5 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (out5) memcpy(out5, o, sizeof(o));
  return PDOT_OK;
}

static int unit_kkt_impl(pdot_solver* h, bool with_cost, double scale_R, double* viol_any, int64_t ldV,
                         double* rows_any, double* cols_any, double* out10) {
  DeviceGuard dg(h->device);
  Ctl& c = h->host;
  unit_ctl(h);
  const double* Csave = c.C;
  const int32_t kind_save = c.cost_kind;
  if (!with_cost) {
    c.C = nullptr;
    c.cost_kind = pdot::COST_EXPLICIT;
  }
  c.sX = 0;
  c.scale_R = scale_R;
  c.kkt_write_viol = (viol_any && with_cost) ? 1 : 0;
  c.viol_out = c.kkt_write_viol ? c.slot[1].X : nullptr;
  c.op = pdot::OP_KKT;
  int rc = upload_ctl(h);
  c.C = Csave;
  c.cost_kind = kind_save;
  if (rc) return rc;
  if ((rc = run_pass(h, pdot::OP_KKT))) return rc;
  if (c.kkt_write_viol) occ_invalidate(h, 1);  // the violation matrix lives in slot 1
  double o[10];
  CK(cudaMemcpyAsync(o, &h->dev->out[0], 10 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  if (rows_any && (rc = copy_vec(rows_any, c.rows_out, h->m, h->stream))) return rc;
  if (cols_any && (rc = copy_vec(cols_any, c.cols_out, h->n, h->stream))) return rc;
  if (c.kkt_write_viol && (rc = copy_matrix(viol_any, ldV, c.slot[1].X, h->ldx, h->m, h->n, h->stream)))
    return rc;
  CK(cudaStreamSynchronize(h->stream));
  if (out10) memcpy(out10, o, sizeof(o));
  return PDOT_OK;
}

int pdot_unit_kkt(pdot_solver* h, double scale_R, double* viol_any, int64_t ldV, double* rows_any,
                  double* cols_any, double* out10) {
  if (!h || !h->problem_set) return set_err(PDOT_ESTATE, "problem not set");
  if (!(scale_R > 0)) return set_err(PDOT_EINVAL, "scale_R must be positive");
  if (viol_any && ldV < h->n) return set_err(PDOT_EINVAL, "viol: leading dimension must be >= n");
  return unit_kkt_impl(h, true, scale_R, viol_any, ldV, rows_any, cols_any, out10);
}

int pdot_unit_apply_A(pdot_solver* h, double* rows_any, double* cols_any) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  return unit_kkt_impl(h, false, 1.0, nullptr, 0, rows_any, cols_any, nullptr);
}

int pdot_apply_At(const double* p_dev, const double* q_dev, int64_t m, int64_t n, double* out_dev,
                  int64_t ldo) {
  if (!p_dev || !q_dev || !out_dev || m < 1 || n < 1 || ldo < n) return set_err(PDOT_EINVAL, "bad argument");
  const int64_t total = m * n;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 32);
  apply_at_kernel<<<blocks, threads>>>(p_dev, q_dev, m, n, out_dev, ldo);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return PDOT_OK;
}

int pdot_gen_cost(double* C_dev, int64_t m, int64_t n, int64_t ldc, int kind, const int64_t* a) {
  if (!a) return set_err(PDOT_EINVAL, "bad argument");
  const int64_t m_total = (kind == PDOT_COST_L1_RECT) ? a[0] * a[1] : a[0] * a[1];
  if (m != m_total) return set_err(PDOT_EINVAL, "cost shape mismatch");
  return pdot_gen_cost_rows(C_dev, 0, m, n, ldc, kind, a);
}

int pdot_gen_cost_rows(double* C_dev, int64_t row0, int64_t rows, int64_t n, int64_t ldc, int kind,
                       const int64_t* a) {
  if (!C_dev || !a || rows < 1 || n < 1 || ldc < n || row0 < 0) return set_err(PDOT_EINVAL, "bad argument");
  if (kind == PDOT_COST_SQEUCLID_GRID || kind == PDOT_COST_L1_GRID) {
    if (a[0] != a[1] || a[0] * a[1] != n || row0 + rows > n) return set_err(PDOT_EINVAL, "grid cost needs m = n = r*r");
  } else if (kind == PDOT_COST_L1_RECT) {
    if (row0 + rows > a[0] * a[1] || a[2] * a[3] != n) return set_err(PDOT_EINVAL, "rect cost shape mismatch");
  } else {
    return set_err(PDOT_EINVAL, "unknown cost kind");
  }
  gen_cost_kernel<<<148 * 16, 256>>>(C_dev, row0, rows, n, ldc, kind, a[0], a[1], a[2], a[3]);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return PDOT_OK;
}

int pdot_fro_norm(const double* C_dev, int64_t m, int64_t n, int64_t ldc, double* out) {
  if (!C_dev || !out || m < 1 || n < 1 || ldc < n) return set_err(PDOT_EINVAL, "bad argument");
  const int nb = 148 * 8;
  double* part = nullptr;
  CK(cudaMalloc(&part, (nb + 1) * sizeof(double)));
  sumsq_partial_kernel<<<nb, 256>>>(C_dev, m, n, ldc, part);
  sum_final_kernel<<<1, 32>>>(part, nb, part + nb);
  cudaError_t e = cudaMemcpy(out, part + nb, sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(part);
  if (e != cudaSuccess) return cuda_fail(e, "pdot_fro_norm", __LINE__);
  return PDOT_OK;
}

int pdot_time_stream_kernel(pdot_solver* h, int iters, double* ms_per_launch) {
  if (!h || iters < 1 || !h->problem_set) return set_err(PDOT_EINVAL, "bad argument");
  DeviceGuard dg(h->device);
  Ctl& c = h->host;
  c.unit = 0;
  c.done = 0;
  c.status = nullptr;
  c.ring = nullptr;
  // a full (lagged-average) STEP pass: X, previous average, outputs all distinct
  c.sX = 0; c.sAsrc = 1; c.sA = 3; c.sXn = 2; c.sAn = 4; c.lagA = 1;
  c.tau = 1e-3; c.sigma = 1e-3; c.kd = 3.0; c.rkd = 1.0 / 3.0; c.kd_dual = 4.0; c.rkd_dual = 0.25;
  c.op = pdot::OP_STEP;
  if (int rc = upload_ctl(h)) return rc;
  // always the dense TMA walker: this is the 40 B/entry roofline probe
  for (int i = 0; i < 2; ++i) pdot::launch_stream_pass(h->dev, h->host, pdot::OP_STEP, h->stream);
  CK(cudaEventRecord(h->t0, h->stream));
  for (int i = 0; i < iters; ++i) pdot::launch_stream_pass(h->dev, h->host, pdot::OP_STEP, h->stream);
  CK(cudaEventRecord(h->t1, h->stream));
  h->launches += iters + 2;
  for (int s = 0; s < pdot::kNSlot; ++s) occ_invalidate(h, s);  // the dense walker kept no occupancy
  CK(cudaEventSynchronize(h->t1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->t0, h->t1));
  if (ms_per_launch) *ms_per_launch = ms / iters;
  c.status = h->status_d;
  c.ring = h->ring_d;
  c.done = 1;
  c.op = pdot::OP_NONE;
  return upload_ctl(h);
}

int64_t pdot_kernel_launches(const pdot_solver* h) { return h ? h->launches : 0; }

int pdot_nccl_unique_id(void* out128) {
  if (!out128) return set_err(PDOT_EINVAL, "null output");
  if (!nccl().ok) return set_err(PDOT_ENCCL, "libnccl.so.2 could not be loaded");
  NcclId id;
  const int r = nccl().get_unique_id(&id);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, id.internal, sizeof(id.internal));
  return PDOT_OK;
}

int pdot_comm_init(pdot_solver* h, const void* id128) {
  if (!h || !id128) return set_err(PDOT_EINVAL, "null argument");
  if (h->nranks == 1) {
    // a 1-rank communicator: only useful to exercise the split pass sequence
    // (K2a -> ncclAllGather -> K2b) on one GPU; PDOT_FORCE_SPLIT=1 enables it
    const char* e = getenv("PDOT_FORCE_SPLIT");
    if (!e || atoi(e) == 0) return PDOT_OK;
    h->force_split = true;
  }
  if (!nccl().ok) return set_err(PDOT_ENCCL, "libnccl.so.2 could not be loaded");
  DeviceGuard dg(h->device);
  NcclId id;
  memcpy(id.internal, id128, sizeof(id.internal));
  void* comm = nullptr;
  const int r = nccl().comm_init_rank(&comm, h->nranks, id, h->rank);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  h->nccl_comm = comm;
  h->virtual_shards = false;
  if (h->graph) {
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  return PDOT_OK;
}

int pdot_shard_info(const pdot_solver* h, int64_t* m_total, int64_t* row0, int32_t* nranks, int32_t* rank) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  if (m_total) *m_total = h->m_total;
  if (row0) *row0 = h->row0;
  if (nranks) *nranks = h->nranks;
  if (rank) *rank = h->rank;
  return PDOT_OK;
}

int pdot_set_virtual(pdot_solver* h, int on) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  if (h->nranks == 1) return set_err(PDOT_EINVAL, "virtual exchange needs a sharded handle");
  h->virtual_shards = on != 0;
  return PDOT_OK;
}

int pdot_shard_pass(pdot_solver* h, int phase, pdot_progress* prog) {
  if (!h || h->nranks == 1) return set_err(PDOT_EINVAL, "pdot_shard_pass needs a sharded handle");
  DeviceGuard dg(h->device);
  if (!h->ph0) CK(cudaEventCreate(&h->ph0));
  CK(cudaEventRecord(h->ph0, h->stream));
  if (phase == 0) {
    h->launches += launch_k1(h, -1);
    pdot::launch_finalize_pass(h->dev, h->host, -1, pdot::FIN_A, h->stream);
    h->launches += 1;
  } else {
    pdot::launch_finalize_pass(h->dev, h->host, -1, pdot::FIN_B, h->stream);
    h->launches += 1;
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(h->t1, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaEventElapsedTime(&h->phase_ms[phase ? 1 : 0], h->ph0, h->t1));
  drain_ring(h);
  if (prog) {
    if (int rc = download_ctl(h)) return rc;
    const Ctl& c = h->host;
    prog->done = c.done;
    prog->roles[0] = c.sX;
    prog->roles[1] = c.sA;
    prog->roles[2] = c.sZ;
    prog->roles[3] = c.sB;
    prog->op = c.op;
    prog->iterations = c.total;
    prog->restarts = c.outer;
    prog->passes = c.passes;
    prog->avg_written = c.avg_written;
    prog->avg_slot = c.avg_slot;
  }
  return PDOT_OK;
}

// Device time (CUDA events) of the last pdot_shard_pass call of each phase:
// phase 0 = this shard's K0 / K1 / K1b / K2a, phase 1 = its K2b (combine +
// controller).  Per-shard latency model of a row-sharded pass.
int pdot_shard_pass_ms(const pdot_solver* h, double* ms2) {
  if (!h || !ms2) return set_err(PDOT_EINVAL, "null argument");
  ms2[0] = h->phase_ms[0];
  ms2[1] = h->phase_ms[1];
  return PDOT_OK;
}

int pdot_exchange_local(pdot_solver** hs, int count) {
  if (!hs || count < 1) return set_err(PDOT_EINVAL, "bad argument");
  for (int i = 0; i < count; ++i)
    if (!hs[i] || hs[i]->nranks != count || hs[i]->rank != i || hs[i]->device != hs[0]->device)
      return set_err(PDOT_EINVAL, "pdot_exchange_local: handles must be ranks 0..count-1 on one device");
  DeviceGuard dg(hs[0]->device);
  CK(cudaDeviceSynchronize());
  const int per = pdot::kGroups / count;
  for (int src = 0; src < count; ++src) {
    const size_t chunk = (size_t)per * hs[src]->gstride;
    for (int dst = 0; dst < count; ++dst) {
      if (dst == src) continue;
      CK(cudaMemcpy(hs[dst]->gbuf + (size_t)src * chunk, hs[src]->gbuf + (size_t)src * chunk,
                    chunk * sizeof(double), cudaMemcpyDeviceToDevice));
    }
  }
  CK(cudaDeviceSynchronize());
  return PDOT_OK;
}

int pdot_time_finalize(pdot_solver* h, int iters, double* ms_per_launch) {
  if (!h || iters < 1 || !h->problem_set) return set_err(PDOT_EINVAL, "bad argument");
  DeviceGuard dg(h->device);
  Ctl& c = h->host;
  unit_ctl(h);
  c.sX = 0; c.sA = 1; c.sXn = 2; c.sAn = 3; c.sAsrc = 4;
  c.unit_avg = 1;
  c.tau = 1e-3; c.sigma = 1e-3; c.kd = 3.0; c.rkd = 1.0 / 3.0; c.kd_dual = 4.0; c.rkd_dual = 0.25;
  c.op = pdot::OP_STEP;
  if (int rc = upload_ctl(h)) return rc;
  launch_k1(h, pdot::OP_STEP);
  for (int i = 0; i < 2; ++i) pdot::launch_finalize_pass(h->dev, h->host, pdot::OP_STEP, pdot::FIN_FUSED, h->stream);
  CK(cudaEventRecord(h->t0, h->stream));
  for (int i = 0; i < iters; ++i) pdot::launch_finalize_pass(h->dev, h->host, pdot::OP_STEP, pdot::FIN_FUSED, h->stream);
  CK(cudaEventRecord(h->t1, h->stream));
  h->launches += iters + 3;
  CK(cudaEventSynchronize(h->t1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->t0, h->t1));
  if (ms_per_launch) *ms_per_launch = ms / iters;
  return PDOT_OK;
}

int pdot_ipc_handle(pdot_solver* h, void* out64) {
  if (!h || !out64) return set_err(PDOT_EINVAL, "null argument");
  if (!h->xbuf) return set_err(PDOT_EINVAL, "peer-memory exchange needs a sharded handle");
  DeviceGuard dg(h->device);
  cudaIpcMemHandle_t ih;
  CK(cudaIpcGetMemHandle(&ih, h->xbuf));
  memcpy(out64, &ih, sizeof(ih));
  return PDOT_OK;
}

int pdot_p2p_open(pdot_solver* h, const void* handles64, int count) {
  if (!h || !handles64 || count != h->nranks) return set_err(PDOT_EINVAL, "need one IPC handle per rank");
  DeviceGuard dg(h->device);
  const char* base = static_cast<const char*>(handles64);
  for (int r = 0; r < count; ++r) {
    if (r == h->rank) {
      h->host.xpeer[r] = h->xbuf;
      continue;
    }
    cudaIpcMemHandle_t ih;
    memcpy(&ih, base + (size_t)r * sizeof(ih), sizeof(ih));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_opened[r] = p;
    h->host.xpeer[r] = static_cast<double*>(p);
  }
  h->host.p2p = 1;
  h->host.xerror = 0;
  if (h->graph) {
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  return upload_ctl(h);
}

int pdot_p2p_link_local(pdot_solver** hs, int count) {
  if (!hs || count < 2) return set_err(PDOT_EINVAL, "bad argument");
  for (int i = 0; i < count; ++i)
    if (!hs[i] || hs[i]->nranks != count || hs[i]->rank != i || !hs[i]->xbuf || hs[i]->device != hs[0]->device)
      return set_err(PDOT_EINVAL, "pdot_p2p_link_local: handles must be ranks 0..count-1 on one device");
  for (int i = 0; i < count; ++i) {
    for (int r = 0; r < count; ++r) hs[i]->host.xpeer[r] = hs[r]->xbuf;
    hs[i]->host.p2p = 1;
    hs[i]->host.xerror = 0;
    DeviceGuard dg(hs[i]->device);
    if (int rc = upload_ctl(hs[i])) return rc;
  }
  return PDOT_OK;
}

// Peer-memory exchange protocol under genuinely concurrent ranks (test hook):
// the linked handles' control blocks drive pdot::p2p_protocol_kernel, one block
// per rank in a single cooperative launch.  out3r[3 r + {0,1,2}] = rank r's
// value mismatches, longest wait (ns) and exchange-timeout flag.  Each
// handle's exchange counter advances by `rounds`, as after that many passes.
int pdot_p2p_selftest(pdot_solver** hs, int count, int rounds, double delay_us, unsigned long long* out3r) {
  if (!hs || count < 2 || count > pdot::kMaxRanks || rounds < 1 || !out3r) return set_err(PDOT_EINVAL, "bad argument");
  for (int i = 0; i < count; ++i)
    if (!hs[i] || !hs[i]->host.p2p || hs[i]->nranks != count || hs[i]->rank != i || hs[i]->device != hs[0]->device)
      return set_err(PDOT_EINVAL, "pdot_p2p_selftest: needs ranks 0..count-1 linked on one device");
  DeviceGuard dg(hs[0]->device);
  std::vector<Ctl> ctls(count);
  for (int i = 0; i < count; ++i) ctls[i] = hs[i]->host;
  Ctl* ctl_dev = nullptr;
  unsigned long long* out_dev = nullptr;
  CK(cudaMalloc(&ctl_dev, count * sizeof(Ctl)));
  CK(cudaMalloc(&out_dev, 3 * count * sizeof(unsigned long long)));
  cudaStream_t s = hs[0]->stream;
  for (int i = 0; i < count; ++i) CK(cudaStreamSynchronize(hs[i]->stream));
  CK(cudaMemcpyAsync(ctl_dev, ctls.data(), count * sizeof(Ctl), cudaMemcpyHostToDevice, s));
  const cudaError_t le = (cudaError_t)pdot::launch_p2p_protocol_test(ctl_dev, count, rounds,
                                                                     (unsigned long long)(delay_us * 1e3), out_dev, s);
  if (le != cudaSuccess) {
    cudaFree(ctl_dev);
    cudaFree(out_dev);
    return cuda_fail(le, "cooperative launch", __LINE__);
  }
  CK(cudaMemcpyAsync(out3r, out_dev, 3 * count * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(ctl_dev);
  cudaFree(out_dev);
  return PDOT_OK;
}

// Host -> device copy of an m x n matrix into a device buffer (leading
// dimension ldd).  Page-locked sources go by one direct DMA.  Pageable sources
// (a plain numpy array, the reference's own input type) are staged through two
// 64 MB pinned buffers: host threads copy chunk k+1 into one while the DMA of
// chunk k drains the other, instead of the driver's single-threaded staging.
int pdot_h2d_matrix(double* dst_dev, int64_t ldd, const double* src, int64_t lds, int64_t m, int64_t n,
                    int device) {
  NvtxRange nv("pdot: host->device cost matrix");
  if (!dst_dev || !src || m < 0 || n < 0 || ldd < n || lds < n) return set_err(PDOT_EINVAL, "bad argument");
  if (m == 0 || n == 0) return PDOT_OK;
  DeviceGuard dg(device);
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static cudaStream_t st = nullptr;
  static double* pin[2] = {nullptr, nullptr};
  static cudaEvent_t ev[2] = {nullptr, nullptr};
  static int st_device = -1;
  constexpr size_t kChunk = (size_t)64 << 20;
  if (st_device != device) {  // (re)create the staging resources on this device
    if (st) {
      for (int i = 0; i < 2; ++i) {
        cudaFreeHost(pin[i]);
        cudaEventDestroy(ev[i]);
      }
      cudaStreamDestroy(st);
      st = nullptr;
    }
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaHostAlloc(&pin[i], kChunk, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    st_device = device;
  }
  if (!is_pageable_host(src)) {
    CK(cudaMemcpy2DAsync(dst_dev, ldd * sizeof(double), src, lds * sizeof(double), n * sizeof(double), m,
                         cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return PDOT_OK;
  }
  const int64_t row_bytes = n * (int64_t)sizeof(double);
  if ((int64_t)kChunk < row_bytes) {  // rows wider than a staging buffer: the driver's path
    CK(cudaMemcpy2DAsync(dst_dev, ldd * sizeof(double), src, lds * sizeof(double), n * sizeof(double), m,
                         cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return PDOT_OK;
  }
  const int64_t rows_per = (int64_t)kChunk / row_bytes;
  const int64_t nchunks = (m + rows_per - 1) / rows_per;
  const unsigned nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (int64_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    const int64_t r0 = k * rows_per, rows = std::min(rows_per, m - r0);
    if (k >= 2) CK(cudaEventSynchronize(ev[b]));  // the DMA that last read this buffer is done
    char* dstb = reinterpret_cast<char*>(pin[b]);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nthreads; ++t) {
      const int64_t a = rows * t / nthreads, e = rows * (t + 1) / nthreads;
      pool.emplace_back([=]() {
        for (int64_t r = a; r < e; ++r) memcpy(dstb + r * row_bytes, src + (r0 + r) * lds, (size_t)row_bytes);
      });
    }
    for (auto& th : pool) th.join();
    CK(cudaMemcpy2DAsync(dst_dev + r0 * ldd, ldd * sizeof(double), pin[b], (size_t)row_bytes, (size_t)row_bytes,
                         (size_t)rows, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(ev[b], st));
  }
  CK(cudaStreamSynchronize(st));
  return PDOT_OK;
}

// debugging aid (PDOT_K2_TRACE=1): per-block K2 timestamps {entry, work done,
// ticket, 0} of the last screened STEP pass; returns the block count
int pdot_debug_k2(pdot_solver* h, unsigned long long* out, int64_t cap) {
  if (!h || !h->host.kdbg) return 0;
  DeviceGuard dg(h->device);
  const int64_t nb = h->CB + h->T;
  const int64_t k = std::min<int64_t>(cap, nb * 4 + 32);
  if (cudaMemcpy(out, h->host.kdbg, k * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return (int)nb;
}

int pdot_set_screening(pdot_solver* h, int on) {
  if (!h) return set_err(PDOT_EINVAL, "null handle");
  DeviceGuard dg(h->device);
  const bool was = h->host.screen != 0;
  if (on && !h->screen_ok)
    return set_err(PDOT_EINVAL, "block screening needs (bands x cells) of the plan to fit a 32-bit cell list entry");
  h->screen_on = on != 0;
  if (int rc = screen_setup(h)) return rc;
  if (h->host.screen && !was) {
    // the dense walker kept no occupancy: rescan every slot (memory is the truth)
    for (int s = 0; s < pdot::kNSlot; ++s) slot_meta(h, s, true, false);
  }
  if (h->graph) {  // the pass topology changed
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
  return PDOT_OK;
}

int pdot_screen_stats(pdot_solver* h, int reset, unsigned long long* out12) {
  if (!h || !out12) return set_err(PDOT_EINVAL, "null argument");
  unsigned long long* out8 = out12;
  DeviceGuard dg(h->device);
  unsigned long long st[pdot::ST_COUNT];
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(st, h->host.sstat, sizeof(st), cudaMemcpyDeviceToHost));
  out8[0] = st[pdot::ST_PASSES];
  out8[1] = st[pdot::ST_CELLS];
  out8[2] = st[pdot::ST_TILES];
  out8[3] = st[pdot::ST_BYTES];
  out8[4] = st[pdot::ST_META];
  out8[5] = st[pdot::ST_K1_NS];
  out8[6] = (unsigned long long)h->host.screen;
  out8[7] = (unsigned long long)(h->host.nbands * h->host.ncells);
  out12[8] = st[pdot::ST_K2_MAIN];
  out12[9] = st[pdot::ST_K2_CTL];
  out12[10] = st[pdot::ST_T0K0];
  out12[11] = st[pdot::ST_T1K0];
  out12[12] = st[pdot::ST_DONE0];
  out12[13] = st[pdot::ST_GAP_K2K0];
  out12[14] = st[pdot::ST_K0K1];
  out12[15] = st[pdot::ST_K1K2];
  out12[16] = st[pdot::ST_GAP_LAUNCH];
  if (reset) {
    CK(cudaMemset(h->host.sstat + pdot::ST_K0_START, 0, 8 * sizeof(unsigned long long)));
    CK(cudaMemset(h->host.sstat, 0, 7 * sizeof(unsigned long long)));
    CK(cudaMemset(h->host.sstat + pdot::ST_K2_MAIN, 0, 2 * sizeof(unsigned long long)));
    CK(cudaMemset(h->host.sstat + pdot::ST_T0K0, 0, 3 * sizeof(unsigned long long)));
  }
  return PDOT_OK;
}

}  // extern "C"
