// Internal definitions shared by the PDOT CUDA translation units.
//
// Layout: every m x n matrix is row-major fp64 with an even
// leading dimension, so a thread can own an aligned column pair and move it with
// one 128-bit load/store.  A "slot" is one primal-dual point (X, p, q); the
// solver keeps NSLOT slots and moves ROLES (current, average, anchor, best, the
// two outputs of the in-flight pass) between them instead of copying matrices.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pdot {

constexpr int kWarps = 8;                 // warps per streaming CTA
constexpr int kThreads = kWarps * 32;     // 256 worker threads
constexpr int kBlockThreads = kThreads + 32;  // + one producer warp (TMA walker)
constexpr int kTileN = kWarps * 64;       // 512 columns per tile (each lane: 2 columns)
constexpr int kMaxNQ = 4;                 // row/col quantities per pass (STEP: e, d, X+, A')
constexpr int kMaxNS = 8;                 // per-tile scalar partials
constexpr int kGroups = 8;                // row-tile groups of the hierarchical reduction
constexpr int kNSlot = 7;
constexpr int kRedThreads = 256;          // finalize-kernel block size
constexpr int kMaxRowScal = 16;           // per-row-tile scalar partials (finalize)
constexpr int kMaxColScal = 8;            // per-column-block scalar partials (finalize)
constexpr int kRingCap = 1 << 16;         // trace/event ring entries (host mapped)
constexpr int kListPad = 1 << 14;         // extra cell-list entries: K1 reads every warp's first two
                                          // entries before it knows the list length (<= 1024 SMs)

// Block screening of the STEP pass (screen.cu).  The plan is cut
// into cells of kBand rows x kCell columns; a warp strip is kStrip = 4 cells.
// A cell is SKIPPABLE in a pass when X and the lagged average are zero there
// and neither dual pair violates it: RN(max p + max q) <= min C over the cell
// (same for the averaged duals).  Then every output and every reduction term
// of the cell is exactly +0, so skipping it leaves all results bit-identical.
constexpr int kBand = 8;
constexpr int kCell = 16;
constexpr int kStrip = 64;
constexpr int kCellsPerStrip = kStrip / kCell;  // 4: one byte each in a 32-bit word
// per-cell flags of a K0 unit word (one byte per cell)
enum UnitFlag : uint32_t { U_ACT = 1, U_LDX = 2, U_LDA = 4, U_ZX = 8, U_ZA = 16 };
// screening statistics (uint64 counters, accumulated over a solve)
enum ScreenStat : int {
  ST_PASSES = 0,    // screened STEP passes
  ST_CELLS = 1,     // active cells processed by K1
  ST_TILES = 2,     // cells visited by K1 (active or stale-zeroing)
  ST_BYTES = 3,     // bytes K1 moved (cell loads/stores + tile partials)
  ST_META = 4,      // bytes K0 read/wrote (screen metadata)
  ST_K1_NS = 5,     // summed K1 durations (%globaltimer, first CTA start -> last CTA end)
  ST_K0_NS = 6,     // summed K0 durations
  ST_T0 = 7,        // scratch: start / end stamps / done-CTA counters of the running pass
  ST_T1 = 8,
  ST_DONE1 = 9,
  ST_T0K0 = 10,
  ST_T1K0 = 11,
  ST_DONE0 = 12,
  ST_K2_T0 = 13,    // K2 of screened STEP passes: start stamp (block 0),
  ST_K2_MAIN = 14,  // summed time from start to the last block's ticket,
  ST_K2_CTL = 15,   // summed time of the controller tail (last block)
  ST_K0_START = 16, // scratch: K0 start (block 0) of the running screened STEP pass
  ST_K1_END = 17,   // scratch: K1 end (last CTA) of the running pass
  ST_K2_END = 18,   // scratch: end of the last K2 (controller write-back done)
  ST_GAP_K2K0 = 19, // summed: previous K2 end -> K0 start (launch gap between passes)
  ST_K0K1 = 20,     // summed: K0 start -> K1 start (K0 + one launch gap)
  ST_K1K2 = 21,     // summed: K1 end -> K2 start (K1b + two launch gaps)
  ST_K0_ENTRY = 22, // scratch: K0 block 0's first instruction (before it reads the control block)
  ST_GAP_LAUNCH = 23,  // summed: previous K2 end -> K0 entry (the part of the gap before K0 runs)
  ST_COUNT = 24,
};

enum Op : int {
  OP_STEP = 0,   // trial step + running average + dual-violation of the input iterate
  OP_DIST = 1,   // ||cand - anchor||^2 at an adaptive restart
  OP_KKT = 2,    // KKT blocks of one slot (start of solve / unit kkt_error / apply_A)
  OP_DIFF = 3,   // rows/cols/norm of (slot b - slot a)   (unit stepsize_bound)
  OP_ROUND = 4,  // one of the rounding passes (stage in ctl->round_stage)
  OP_NONE = 5,
};

// Ctl::out[] layout.  Unit KKT: [0..9] = gap, composite, relative, pobj, dobj,
// primal_sq, dual_sq, |X|^2, |p|^2, |q|^2.  Unit bound: [0..4] = bound, |dX|^2,
// |dp|^2, |dq|^2, coupling.  Rounding stages use the named slots below.
enum OutSlot : int {
  OUT_ROUND_L1VIOL = 19,  // l1 marginal violation of X_feas       (stage 3)
  OUT_ROUND_TOTAL = 20,   // total row deficit sum(err_r)           (stage 2)
  OUT_ROUND_CORRECT = 21, // 1 if the rank-one correction applies   (stage 2)
  OUT_ROUND_OBJ = 22,     // <C, X_feas>                            (stage 3)
  OUT_ROUND_DUAL = 23,    // f.p + g.q of the rounded slot          (stage 3)
};

enum Reason : int { R_NONE = 0, R_TOL = 1, R_ITER = 2, R_TIME = 3 };
enum Err : int { E_OK = 0, E_NONFINITE = 1, E_LINESEARCH = 2, E_EXCHANGE = 3 };
constexpr int kMaxRanks = 8;

enum EvType : int { EV_START = 1, EV_ACCEPT = 2, EV_CAND = 3, EV_RESTART = 4, EV_REJECT = 5 };

struct Event {
  int32_t type;
  int32_t ia;      // restart length (EV_RESTART)
  double x, y, z;  // ACCEPT: eta, bound ; CAND: cand_kkt, kkt_cur, kkt_avg (ia: current won) ;
                   // RESTART: kkt, omega ; START: kkt ; REJECT: eta, bound
};

// Host-mapped status mirror: written by the controller every pass, read by the
// host poll loop without any copy or synchronisation.
struct Status {
  volatile int32_t done;
  volatile int32_t reason;
  volatile int32_t error;
  volatile int32_t final_slot;
  volatile int64_t total;
  volatile int64_t outer;
  volatile int64_t passes;
  volatile int64_t ring_head;
  volatile int32_t pause;   // the controller waits for the host (host-evaluated omega)
  int32_t pad_;
};

struct Slot {
  double* X;
  double* p;
  double* q;
};

// Device control block.  Written only by the controller thread (last block of
// the finalize kernel) and read by every kernel of the next pass.
struct Ctl {
  // ---- problem / config (set once) ----
  int64_t m, n, ldc, ldx;
  int64_t T, U;            // row tiles (local), column tiles
  int64_t TM;              // rows per tile
  int64_t CB;              // finalize column blocks (kColsPerBlock = 128 columns each)
  int64_t ncolblk;         // column-side scalar partials: one per 64 columns
  // ---- row sharding; single GPU: m_total = m, Tg = T, t0 = 0, groups 0..8 ----
  int64_t m_total, row0;   // global rows, first local row
  int64_t Tg, t0, GS;      // global row tiles, first local tile, tiles per reduction group
  int32_t g0, g1;          // local reduction groups [g0, g1)
  int32_t nranks, rank;
  double* gbuf;            // [kGroups][gstride]: per-group column sums (4 x ldx) + 16 scalars
  int64_t gstride;
  // peer-memory exchange (p2p = 1): every rank's exchange buffer, mapped into this
  // rank's address space: [2 parities][kGroups][gstride] doubles, [2][kMaxRanks]
  // uint64 sequence flags, then this rank's own exchange counter (device-only:
  // host uploads of this block never reset it).  K2a stores its groups into all
  // ranks' buffers and publishes counter+1; K2b acquires every rank's flag,
  // combines locally and advances the counter.
  double* xpeer[8];
  int32_t p2p, xerror;
  double cost_fro, marg_norm;
  double tol, beta, beta_suff, beta_nec, beta_art, theta, eps_zero;
  int64_t max_iters, kkt_stride;
  int32_t adaptive, relative, unit, trace_level;
  int32_t unit_avg;        // unit STEP call that also updates a running average
  uint64_t deadline_ns;    // %globaltimer deadline (0 = none)
  int32_t stop_request;    // host may set to force a time-limit stop
  int32_t host_omega;      // adaptive restarts pause for a host-evaluated omega (pdot_config.host_omega)
  int32_t omega_wait;      // paused: om_dX / om_dpq hold the restart distances
  double om_dX, om_dpq;
  // ---- step state ----
  double eta, omega, tau, sigma;
  double kd, rkd;            // lazy matrix average: k of the iterate being averaged, RN(1/k)
  double kd_dual, rkd_dual;  // eager dual average: k of the trial iterate
  // ---- counters ----
  int64_t total, inner, outer, passes, halvings, rejected;
  // ---- KKT bookkeeping ----
  double epoch_kkt, prev_cand, best_kkt, best_rel, scale_R;
  int32_t pending;          // KKT of the current iterate awaits this pass's dual violation
  double pend_psq_cur, pend_pobj_cur, pend_dobj_cur;
  double pend_dobj_avg;
  double cand_kkt, cand_rel;   // candidate that triggered the pending restart
  double final_rel;
  // ---- roles ----
  int32_t sX, sA, sZ, sB, sXn, sAn, sCand, sFinal;
  // Lazy running average: after an accepted step the average slot sA holds the
  // new dual average (p, q) but its matrix is written by the NEXT pass from the
  // accepted iterate and the previous average matrix in slot sAsrc (lagA = 1).
  // A rejected trial's re-run then streams only C and X (24 instead of 40 B/entry).
  int32_t sAsrc, lagA;
  int32_t avg_written, avg_slot;  // this pass wrote the average matrix into avg_slot (trace)
  int32_t op, done, reason, error;
  int32_t round_stage;
  int32_t kkt_write_viol;   // unit kkt_error: also write the dual-violation matrix
  // ---- unit-call outputs (indices: OutSlot) ----
  double out[24];
  // ---- ring ----
  int64_t ring_head;
  // ---- pointers ----
  const double* C;
  const double* f;
  const double* g;
  // implicit (matrix-free) cost: C == nullptr and cost_kind > 0 -> C_ij generated
  // from grid coordinates in registers (exact integers, identical to the explicit C)
  int32_t cost_kind;       // 0 explicit, 1 sq-Euclidean grid, 2 L1 grid, 3 L1 rectangular
  int64_t cost_a[4];
  Slot slot[kNSlot];
  double* colpart;    // [T][NQ][ldx]
  double* rowpart;    // [U][NQ][m]
  double* tilescal;   // [T][U][kMaxNS]
  double* rowblk;     // [T][kMaxRowScal]
  double* colblk;     // [CB][kMaxColScal]
  double* rows_out;   // [NQ][m] full row sums of the last unit pass (finalize writes; STEP
  double* cols_out;   // [NQ][ldx] ... column sums      passes skip them: nothing reads them)
  double* vec_a;      // scratch m (rounding row scale / error)
  double* vec_b;      // scratch n (rounding col scale / error)
  double* viol_out;   // unit kkt: dual-violation matrix (ldx) or null
  // ---- block screening (screen.cu; screen != 0: STEP / DIST / start-KKT passes run
  //      K0 screen + K1 unit walker, and K2 reduces per-unit partials) ----
  int32_t screen, nbt;       // nbt = bands per tile = TM / kBand
  int64_t nbands, ncells, nstrips, mpad;
  const double* minc;        // [nbands][ncells]  min C over each cell (-inf if any entry is not finite)
  uint32_t* occ;             // [kNSlot][nbands][nstrips] per-cell "X has a nonzero bit pattern" bytes
  double* pmax;              // [kNSlot][nbands]  NaN-propagating max of p over each band
  double* qmax;              // [kNSlot][ncells]  ... of q over each cell (-inf for cells past n)
  uint8_t* uflag;            // [nbands*ncp] K0 -> K1 flag byte of each listed cell (parallel to ulist)
  uint32_t* ulist;           // cells K1 visits this pass: (band << cbits) | cell
  unsigned int* ucount;      // length of ulist (K0 appends, K2 resets)
  int64_t ncp;               // cells per row of cells, padded to whole tiles (U * 32)
  int32_t cbits, cbits_pad_;  // cell-index bits of a ulist entry: smallest >= 12 with 2^cbits >= ncp
                              // (pdot_create rejects screening when nbands does not fit the rest)
  uint32_t* bcr;             // [nbands][U]  bit k: cell k of column tile u wrote partials this pass
  uint32_t* bct;             // [T][ncp]     bit b: band b of row tile t of this cell wrote partials
  uint8_t* tileflag;         // [T][U] the tile's partials are valid (0: screened out, all +0)
  int32_t* tlist;            // [T*U] tiles with active cells this pass (K1b assembles them)
  uint8_t* tocc;             // [kNSlot][T*U] the tile may hold a nonzero (OR of its cells' occ bytes, a superset)
  const double* tminc;       // [T*U] min C over the tile's cells (-inf if any entry is not finite)
  unsigned int* tcount;      // length of tlist (K0 appends, K2 resets)
  double* ccol;              // [nbands][kMaxNQ][ldx]  cell column partials (band partial of the tree)
  double* crow;              // [ncp][kMaxNQ][mpad]   cell row partials (8-lane butterfly per row)
  double* cscal;             // [nbands][ncp][kMaxNS] cell scalars
  // Slack certificates (STEP passes of a solve): K1 records for every cell it
  // computes a lower bound on min_ij (C_ij - p_i - q_j) over both dual pairs,
  // shifted by the band / cell drift counters at that pass; K2 adds each pass's
  // largest dual change per band / cell to the counters (rounded up).  K0 drops
  // a cell with no mass whose record still exceeds the drift since it was
  // written, so p_i + q_j <= C_ij holds there exactly as the coarse bound would
  // show.  A restart keeps them: both new pairs are the candidate's, one of the
  // two pairs the records bound.
  double* srec;              // [nbands][ncells] record (NaN / -inf: none)
  double* sdp;               // [nbands] cumulative band drift of p / p-average
  double* sdq;               // [ncells] cumulative cell drift of q / q-average
  int32_t sr_on, sr_pad_;
  unsigned long long* sstat; // [ST_COUNT]
  unsigned long long* kdbg;  // PDOT_K2_TRACE=1: per-block K2 timestamps of the last screened STEP pass
  unsigned long long* ktl;   // PDOT_K2_TRACE=1: pass timeline {K0, K1, K1b, K2} x {first start, last end}
  unsigned int* counter;   // last-block-done counter for the finalize kernel
  Status* status;          // host mapped
  Event* ring;             // host mapped, kRingCap entries
};
static_assert(sizeof(Ctl) % 8 == 0, "the controller copies Ctl as 8-byte words");

// cell-list entries: band in the high bits, cell index in the low cbits
__host__ __device__ __forceinline__ uint32_t cell_entry(int64_t band, int64_t cell, int cbits) {
  return (uint32_t)(((uint64_t)band << cbits) | (uint64_t)cell);
}
__host__ __device__ __forceinline__ int64_t entry_band(uint32_t e, int cbits) { return (int64_t)(e >> cbits); }
__host__ __device__ __forceinline__ int64_t entry_cell(uint32_t e, int cbits) {
  return (int64_t)(e & ((1u << cbits) - 1u));
}

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream2(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Transposed butterfly over groups of W consecutive lanes, masks ASCENDING
// (1, 2, ..., W/2): V independent per-lane values (V a power of two <= W) are
// summed across the group with one shuffle per value per halving step.  The
// first log2(V) steps route the values (transposition), the rest is a plain
// butterfly on one value.  Afterwards lane L holds the group total of value
// transpose_owner_index<V>(L); lanes with (L % W) < V hold distinct indices
// (transpose_is_writer).  Ascending masks make the 32-lane tree the
// composition of 8-lane (16-column cell) trees: ((c0 + c1) + (c2 + c3)).
template <int V, int W = 32>
__device__ __forceinline__ void warp_transpose_sum(double (&v)[V]) {
  const int lane = threadIdx.x & 31;
  int mask = 1;
#pragma unroll
  for (int w = V / 2; w >= 1; w /= 2) {
    const bool upper = (lane & mask) != 0;
#pragma unroll
    for (int t = 0; t < w; ++t) {
      const double send = upper ? v[t] : v[t + w];
      const double keep = upper ? v[t + w] : v[t];
      v[t] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
    }
    mask <<= 1;
  }
#pragma unroll
  for (; mask < W; mask <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], mask);
}

template <int V>
__device__ __forceinline__ constexpr int log2_pow2() {
  return (V >= 32) ? 5 : (V >= 16) ? 4 : (V >= 8) ? 3 : (V >= 4) ? 2 : (V >= 2) ? 1 : 0;
}

// value index held by `lane` after warp_transpose_sum<V, W>: step k (mask 2^k)
// kept the half selected by lane bit k, i.e. index bit (log2 V - 1 - k)
template <int V>
__device__ __forceinline__ int transpose_owner_index(int lane) {
  constexpr int lg = log2_pow2<V>();
  int idx = 0;
#pragma unroll
  for (int k = 0; k < lg; ++k) idx |= ((lane >> k) & 1) << (lg - 1 - k);
  return idx;
}

// one writer per value index in every group of W lanes
template <int V, int W = 32>
__device__ __forceinline__ bool transpose_is_writer(int lane) {
  return ((lane & (W - 1)) >> log2_pow2<V>()) == 0;
}

// Transposed butterfly with an explicit mask order M[0..NM): the first log2(V)
// masks route values (lane bit of mask k selects index bit log2(V)-1-k), the
// rest add the remaining value.  Every sum is the xor-pairing tree of the masks
// in order, the same tree a plain butterfly over those masks builds.
template <int V, int NM>
__device__ __forceinline__ void tsum(double (&v)[V], const int (&M)[NM]) {
#pragma unroll
  for (int k = 0, w = V / 2; k < NM; ++k) {
    const int mask = M[k];
    if (w >= 1) {
      const bool upper = (threadIdx.x & mask) != 0;
#pragma unroll
      for (int t = 0; t < V / 2; ++t) {
        if (t < w) {
          const double send = upper ? v[t] : v[t + w];
          const double keep = upper ? v[t + w] : v[t];
          v[t] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
        }
      }
      w /= 2;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], mask);
    }
  }
}
// first value index held by this lane after tsum<V> (it holds indices idx .. idx + V/2^steps - 1)
template <int V, int NM>
__device__ __forceinline__ int tsum_index(const int (&M)[NM]) {
  constexpr int lg = log2_pow2<V>();
  int idx = 0;
#pragma unroll
  for (int k = 0; k < NM && k < lg; ++k) idx |= ((threadIdx.x & M[k]) ? 1 : 0) << (lg - 1 - k);
  return idx;
}

// xor butterfly of one value over groups of W lanes, masks ascending
template <int W = 32>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
  for (int msk = 1; msk < W; msk <<= 1) x += __shfl_xor_sync(0xffffffffu, x, msk);
  return x;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ double sqr_acc(double acc, double x) { return __fma_rn(x, x, acc); }
__device__ __forceinline__ double mul_acc(double acc, double x, double y) { return __fma_rn(x, y, acc); }

// max that propagates NaN (screening bounds: a NaN dual must keep its cells active)
__device__ __forceinline__ double max_nan(double a, double b) { return (a > b || a != a) ? a : b; }
// an upper bound on |a - b| (rounded up; NaN if either is NaN)
__device__ __forceinline__ double absdiff_ru(double a, double b) { return max_nan(__dsub_ru(a, b), __dsub_ru(b, a)); }

// numpy np.maximum(x, 0.0) for a scalar: NaN propagates, -0.0 stays -0.0
__device__ __forceinline__ double relu_np(double x) { return x < 0.0 ? 0.0 : x; }

// x / k, correctly rounded (bit-identical to IEEE division), for a positive
// integer-valued k with rk = RN(1/k).  Markstein: q0 = RN(x*rk) is faithful,
// r = x - k*q0 is exact under FMA, and RN(q0 + r*rk) = RN(x/k) whenever no
// intermediate underflows; |x| < 2^-900 (never seen on the path) takes the
// library division.  Replaces a ~70-instruction IEEE division per element.
__device__ __forceinline__ double div_by_count(double x, double k, double rk) {
  if (fabs(x) < 0x1p-900 && x != 0.0) return __ddiv_rn(x, k);
  const double q0 = __dmul_rn(x, rk);
  const double r = __fma_rn(-q0, k, x);
  return __fma_rn(r, rk, q0);
}

// C_ij of the generated cost families from row/column coordinates (pdot_gen_cost).
enum CostKind : int { COST_EXPLICIT = 0, COST_SQEUCLID = 1, COST_L1GRID = 2, COST_L1RECT = 3 };

struct CostGen {
  int kind;
  int64_t a0, a1, a2, a3;
  int64_t row0;  // global index of local row 0 (row shards)
  __device__ __forceinline__ double2 row_coord(int64_t i_local) const {
    const int64_t i = row0 + i_local;
    if (kind == COST_L1RECT) return make_double2((double)(2 * (i / a1)), (double)(2 * (i % a1)));
    return make_double2((double)(i / a0), (double)(i % a0));
  }
  __device__ __forceinline__ double2 col_coord(int64_t j) const {
    if (kind == COST_L1RECT) return make_double2((double)(j / a3), (double)(j % a3));
    return make_double2((double)(j / a0), (double)(j % a0));
  }
  // row coordinates advance incrementally row by row (no division in the loop)
  __device__ __forceinline__ void next_row(double2& r) const {
    const double step = (kind == COST_L1RECT) ? 2.0 : 1.0;
    const double wrap = (kind == COST_L1RECT) ? (double)(2 * a1) : (double)a0;
    r.y += step;
    if (r.y == wrap) {
      r.y = 0.0;
      r.x += step;
    }
  }
  __device__ __forceinline__ double cost(double2 r, double2 cc) const {
    const double da = r.x - cc.x, db = r.y - cc.y;  // exact (small integers)
    if (kind == COST_SQEUCLID) return da * da + db * db;
    return fabs(da) + fabs(db);
  }
};

// Copy the control block into shared memory (one round trip for all of its
// fields, instead of a chain of dependent global loads at kernel entry); every
// thread of the block must call it.  The kernels only write through the
// pointers it holds, never its fields.
__device__ __forceinline__ void ctl_to_shared(const Ctl* __restrict__ g, Ctl* s) {
  constexpr int kW = (int)(sizeof(Ctl) / sizeof(unsigned long long));
  const unsigned long long* gw = reinterpret_cast<const unsigned long long*>(g);
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(s);
  for (int i = threadIdx.x; i < kW; i += blockDim.x) sw[i] = __ldcg(gw + i);
  __syncthreads();
}

// Programmatic dependent launch (pdl_edge): a kernel lets its stream successor
// be scheduled early (launch_dependents), and a kernel that may have been
// launched early waits here for its predecessor's completion and memory before
// reading anything (a no-op for a plain launch)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// debugging aid (PDOT_K2_TRACE=1): kernel k of a screened STEP pass records
// its first block start / last block end in the pass timeline
__device__ __forceinline__ void tl_start(unsigned long long* tl, int k) {
  if (tl && threadIdx.x == 0) atomicMin(tl + 2 * k, (unsigned long long)globaltimer_ns());
}
__device__ __forceinline__ void tl_end(unsigned long long* tl, int k) {
  if (tl && threadIdx.x == 0) atomicMax(tl + 2 * k + 1, (unsigned long long)globaltimer_ns());
}

// ---------------------------------------------------------------------------
// host-side launchers (defined in the .cu files)
// ---------------------------------------------------------------------------
void launch_stream_pass(const Ctl* ctl_dev, const Ctl& ctl_host, int force_op, cudaStream_t s);
enum FinMode : int { FIN_FUSED = 0, FIN_A = 1, FIN_B = 2 };
void launch_finalize_pass(Ctl* ctl_dev, const Ctl& ctl_host, int force_op, int mode, cudaStream_t s);
// resume a restart paused for a host-evaluated primal weight
void launch_resume_restart(Ctl* ctl_dev, double omega, cudaStream_t s);
// peer-exchange protocol self-test: nranks emulated ranks in one cooperative launch
int launch_p2p_protocol_test(Ctl* ctls_dev, int nranks, int rounds, unsigned long long delay_ns,
                             unsigned long long* out_dev, cudaStream_t s);
size_t stream_smem_bytes(int64_t TM);
void prepare_stream_kernel();
// block-screened pass (screen.cu): K0 screen + K1 unit walker, or the generic
// walker over all tiles for the unit calls that the screen does not cover
void launch_screened_pass(const Ctl* ctl_dev, const Ctl& ctl_host, int force_op, cudaStream_t s);
void prepare_sparse_kernel();
// whether a pass kernel is launched as a programmatic dependent of its predecessor
bool pdl_edge(const char* name);
// a pass whose partials are per-unit (screened) rather than per-tile
__host__ __device__ __forceinline__ bool unit_pass(const Ctl& c, int op) {
  return c.screen && (op == OP_STEP || (!c.unit && (op == OP_DIST || op == OP_KKT)));
}
// screening metadata: min C per cell, per-slot occupancy and dual bounds
void launch_minc_build(const Ctl& ctl_host, double* minc, cudaStream_t s);
void launch_slot_meta(const Ctl& ctl_host, int slot, bool scan_occ, cudaStream_t s);
void launch_tocc_fill(const Ctl& ctl_host, int slot, int value, cudaStream_t s);
// sparse device->host copy of a slot matrix: occupied cells -> list, list -> staging (8 x 16 each)
unsigned launch_occ_list(const Ctl& ctl_host, int slot, uint32_t* list, unsigned* count_dev, cudaStream_t s);
void launch_cell_gather(const Ctl& ctl_host, int slot, const uint32_t* list, int64_t k0, int64_t k1, double* out,
                        cudaStream_t s);

}  // namespace pdot
