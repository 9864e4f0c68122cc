// The pdot_solver handle (shared by the C-ABI translation units).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <string>
#include <vector>

#include "../../include/pdot.h"
#include "pdot_internal.cuh"

using pdot::Ctl;

struct pdot_solver {
  int device = 0;
  int64_t m = 0, n = 0, ldx = 0, TM = 0, T = 0, U = 0, CB = 0;
  cudaStream_t stream = nullptr;
  Ctl host{};
  Ctl* dev = nullptr;
  double* slot_mem = nullptr;
  double* work = nullptr;
  unsigned* counter = nullptr;
  pdot::Status* status_h = nullptr;
  pdot::Status* status_d = nullptr;
  pdot::Event* ring_h = nullptr;
  pdot::Event* ring_d = nullptr;
  int64_t ring_tail = 0;
  std::vector<pdot_event> events;
  cudaGraphExec_t graph = nullptr;
  int graph_L = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaEvent_t ph0 = nullptr;              // start of the last pdot_shard_pass call (per-phase timing)
  float phase_ms[2] = {0.f, 0.f};         // device time of the last pdot_shard_pass call of each phase
  int64_t launches = 0;
  bool problem_set = false;
  std::chrono::steady_clock::time_point wall0;
  double elapsed_before = 0.0;
  int poll_L = 8;
  Ctl saved{};          // control block of the last solve (unit calls reuse the device block)
  bool has_saved = false;
  // ---- row sharding ----
  int nranks = 1, rank = 0;
  int64_t m_total = 0, row0 = 0;
  double* gbuf = nullptr;
  int64_t gstride = 0;
  void* nccl_comm = nullptr;  // ncclComm_t when nranks > 1 and a communicator was attached
  bool virtual_shards = false;  // exchange driven by the host (single-GPU emulation)
  bool force_split = false;     // 1-rank communicator exercising the multi-GPU pass sequence
  // pinned double buffer for device->pageable-host copies of large matrices
  // (allocated at handle creation for large plans): DMA at pinned speed
  // overlapped with a multi-threaded copy-out
  double* xbuf = nullptr;       // peer-memory exchange buffer (sharded handles)
  size_t xbuf_bytes = 0;
  void* ipc_opened[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double* bounce[2] = {nullptr, nullptr};
  // block screening (screen.cu): metadata allocation, min C of the bound problem
  char* screen_mem = nullptr;
  double* minc_buf = nullptr;
  unsigned* d2h_count = nullptr;  // counter of the sparse device->host copy
  bool screen_ok = true;        // the plan geometry fits the 32-bit cell list (solver.cu, pdot_create)
  bool screen_on = true;        // screened passes (default from 2^22 entries; PDOT_SCREEN / pdot_set_screening)
  size_t bounce_bytes = 0;
  cudaEvent_t bounce_ev[2] = {nullptr, nullptr};
};


namespace pdot {
// error helpers shared with sinkhorn.cu (defined in solver.cu)
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what, int line);
}  // namespace pdot
