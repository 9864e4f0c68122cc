// Block-screened STEP pass (K0 screen + K1 sparse walker) and its metadata.
//
// Restarted PDHG on OT keeps the plan extremely sparse: at 16384^2 about 4 of
// 16384 entries per row are nonzero, and only entries near the transport
// support violate the duals.  An entry (i, j) contributes exactly +0 to every
// output and every reduction of a STEP pass when
//     X_ij == 0,  A_ij == 0 (lagged average input),
//     p_i + q_j <= C_ij  and  pbar_i + qbar_j <= C_ij
// (then X+ = max(0, 0 - tau (C - p - q)) = 0, e = d = A' = 0 and both dual
// violations are 0; see pass_ops.cuh StepOp::elem).  Screening works on cells
// of kBand x kCell = 8 x 16 entries:
//     RN(max_band p + max_cell q) <= min_cell C   =>   p_i + q_j <= C_ij
// because rounding is monotone.  Skipped cells add +0 to sums that started at
// +0, so every partial, and hence every result, is bit-identical to the dense
// TMA walker (stream.cu); tests/test_gpu_screen.py checks exactly that.
// The same condition is also certified, for cells the bound above keeps, by a
// slack record: K1 stores a rounded-down lower bound on the cell's exact
// min (C_ij - p_i - q_j) over both dual pairs, shifted by per-band / per-cell
// drift counters that K2 raises by each pass's largest dual change (rounded
// up); K0 drops the cell while the record still exceeds the drift since
// (pdot_internal.cuh, Ctl::srec; tests/test_gpu_slack_cert.py and
// tests/test_slack_cert_soundness.py).
//
// Invariant: slot memory always holds the dense values.  occ[slot] marks cells
// whose bits may be nonzero (a superset); a cell with occ = 0 is all +0.0 in
// memory.  K1 therefore writes zeros into an output cell that it does not
// compute only when that cell's old occ bit says it may hold stale data.
//
//   K0 screen_kernel  (persistent, one warp per tile): a tile-level screen
//       (tile min C, tile maxima of the duals, tile occupancy), then for the
//       remaining tiles the per-cell screen: flag bytes, the list of cells K1
//       visits (each with its flag byte), the bit maps K1b reads the cell
//       partials by, the tile flag and the list of tiles with active cells.
//   K1 unit_kernel    (persistent, one warp per listed cell): cp.async stages
//       the next cell's C / X / A / duals while the current one runs the same
//       StepOp::elem as the dense walker; stores X+ / A' where nonzero (or
//       stale), updates cell and tile occupancy, writes the cell partials.
//   K1b tile_kernel   (CTA per listed tile and part): reassembles the tile partials of
//       the canonical tree from the cell partials.
//   Non-STEP unit calls (KKT of a unit call, DIFF, ROUND) take generic_kernel
//   over all tiles.
// K2 (finalize.cu) skips tiles whose flag is 0: their partials are +0.
#include <stdio.h>
#include <limits.h>
#include <stdlib.h>

#include <string>

#include "pass_ops.cuh"

#ifdef PDOT_DEVICE_CHECKS
#define DCHECK(cond, tag, a, b)                                                                     \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("DCHECK %s failed at %s:%d (%lld, %lld) block %d thread %d\n", tag, __FILE__, __LINE__, \
             (long long)(a), (long long)(b), blockIdx.x, threadIdx.x);                              \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define DCHECK(cond, tag, a, b) \
  do {                          \
  } while (0)
#endif

namespace pdot {
namespace {

constexpr int kSparseCtasPerSm = 2;

__device__ __forceinline__ bool nz2(double2 v) {
  return (__double_as_longlong(v.x) | __double_as_longlong(v.y)) != 0;
}

__device__ __forceinline__ bool step_with_avg(const Ctl& c) { return c.unit ? c.unit_avg != 0 : c.lagA != 0; }

// ---------------------------------------------------------------------------
// K0: screening, one warp per tile (TM x 512: nbt bands x 32 cells).
//   Tile level first: with no occupied cell in any slot the pass reads or
//   writes, and RN(max p + max q) <= min C over the whole tile (current and
//   averaged duals), every cell is inactive: flag 0, nothing listed.
//   Otherwise per cell, lane = (band quarter bq, strip s) over nbt / 4 rounds:
//   STEP: a cell is active when X or the lagged average has a nonzero there,
//         or a dual pair may violate it; stale output cells are flagged ZX/ZA.
//   DIST: active where the candidate or the anchor has a nonzero.
//   KKT:  active where X has a nonzero or the duals may violate.
// Outputs: flag words, the list of cells K1 visits (active or stale), and the
// bit maps K2 reads the cell partials by: bcr (per band and column tile) and
// bct (per row tile and cell).
// ---------------------------------------------------------------------------
// K1's fixed geometry (set once per handle) travels as a KERNEL PARAMETER: its
// fields sit in the constant bank and feed instructions directly, instead of
// being reloaded from the control block in global memory for every cell (the
// 128-register budget does not keep them all live).  KGeo exposes the same
// member names as Ctl, so the cell functions are templates over the context
// type; the per-pass output slots come from the control block (dyn).  ldc is
// fixed while the problem is bound: pdot_set_problem drops the captured graph
// when it changes.
struct KGeo {
  int64_t m, n, ldx, ldc, mpad, nbands, nstrips, ncells, ncp, T, U;
  int64_t occ_stride, tiles;  // nbands * nstrips, T * U
  int32_t nbt, cbits, nbt_log2, pad_;
  uint32_t* occ;
  uint8_t* tocc;
  double* ccol;
  double* crow;
  double* cscal;
  uint32_t* ulist;
  uint8_t* uflag;
  unsigned int* ucount;
  // K1b (tile_kernel): the bit maps, tile list and per-tile partials it writes
  int64_t TM;
  uint32_t* bcr;
  uint32_t* bct;
  int32_t* tlist;
  unsigned int* tcount;
  double* colpart;
  double* rowpart;
  double* tilescal;
  // slack certificates (STEP cells of a solve when the control block's sr_on)
  double* srec;
  const double* sdp;
  const double* sdq;
  // K0 (screen_kernel): the bounds it reads and the flags it writes
  const double* qmax;
  const double* pmax;
  const double* minc;
  const double* tminc;
  uint8_t* tileflag;
};
// PDOT_K0_PROF (measurement builds only): phase times of the cell-by-cell tiles,
// summed over a solve, printed by K0 at pass 600
#ifdef PDOT_K0_PROF
__device__ unsigned long long g_k0prof[8];
#endif
constexpr int kScreenWarps = 8;
constexpr int kScreenCtasPerSm = 2;  // 128 registers; 3 or 4 per SM spill and run slower (C3 11.4k -> 11.3k / 10.7k iter/s)

__global__ void __launch_bounds__(32 * kScreenWarps, kScreenCtasPerSm) screen_kernel(const Ctl* __restrict__ ctlp, int force_op,
                                                                                     unsigned long long* sstat0,
                                                                                     const KGeo g) {
  if (sstat0 && blockIdx.x == 0 && threadIdx.x == 0) sstat0[ST_K0_ENTRY] = globaltimer_ns();
  __shared__ Ctl ctl_s;  // the control block, one round trip for all fields
  ctl_to_shared(ctlp, &ctl_s);
  const Ctl& c = ctl_s;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  unsigned long long* tl = op == OP_STEP ? c.ktl : nullptr;
  tl_start(tl, 0);
  if (op == OP_STEP && !c.unit && c.sstat && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer_ns(), k2e = c.sstat[ST_K2_END];
    c.sstat[ST_K0_START] = t0;
    if (k2e != 0 && t0 > k2e) {
      c.sstat[ST_GAP_K2K0] += t0 - k2e;
      const unsigned long long ke = c.sstat[ST_K0_ENTRY];
      if (ke > k2e) c.sstat[ST_GAP_LAUNCH] += ke - k2e;
    }
    c.sstat[ST_K2_END] = 0;  // only a STEP pass right after a STEP pass counts a gap
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tiles = g.tiles;
#ifdef PDOT_K0_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0 && c.passes == 600 && op == OP_STEP) {
    const double n = (double)g_k0prof[0];
    printf("K0PROF cell-by-cell tiles %.0f per pass; per tile (ns): tile start->flags decided %.0f, ->chunks done %.0f, "
           "->list slots %.0f, ->end %.0f; kernel entry->first tile %.0f\n",
           n / 600.0, g_k0prof[1] / n, g_k0prof[2] / n, g_k0prof[3] / n, g_k0prof[4] / n, g_k0prof[5] / (double)g_k0prof[6]);
  }
  const unsigned long long tk_entry = globaltimer_ns();
  bool first_tile = true;
#endif
  // the pass's slots and switches, once (registers: the loop's global stores
  // would otherwise force reloads of the shared control block)
  const bool with_avg = op == OP_STEP && step_with_avg(c);
  const int sx = op == OP_DIST ? c.sCand : c.sX;
  const int sa = op == OP_DIST ? c.sZ : c.sAsrc;
  const int sA = c.sA, sXn = c.sXn;
  const bool use_rec = op == OP_STEP && !c.unit && c.sr_on;
  // a non-finite step (tau) would turn 0 * inf into NaN: screen nothing
  const bool open = op == OP_STEP && !isfinite(c.tau);
  unsigned long long* const sstat = c.sstat;
  // persistent: one wave of CTAs, each warp walks tiles warp, warp + nw, ...
  for (int64_t tile = (int64_t)blockIdx.x * kScreenWarps + warp; tile < tiles;
       tile += (int64_t)gridDim.x * kScreenWarps) {
    // 32-bit division: tile indices fit (T * U < 2^31), and the 64-bit one is a subroutine call
    const int64_t tt = (uint32_t)tile / (uint32_t)g.U, tu = tile - tt * g.U;
#ifdef PDOT_K0_PROF
    const unsigned long long tp0 = globaltimer_ns();
    if (first_tile && lane == 0 && op == OP_STEP) {
      atomicAdd(&g_k0prof[5], tp0 - tk_entry);
      atomicAdd(&g_k0prof[6], 1ull);
    }
    first_tile = false;
#endif
    const bool bound = op != OP_DIST, bound_avg = op == OP_STEP;
    // ---- tile level: 32 cell maxima of q, nbt band maxima of p, min C, occupancy
    const int64_t tcell = tu * 32 + lane;
    const bool okc = bound && tcell < g.ncells;
    const double Qc = okc ? __ldcg(g.qmax + sx * g.ncells + tcell) : -INFINITY;
    const double Qac = (okc && bound_avg) ? __ldcg(g.qmax + sA * g.ncells + tcell) : -INFINITY;
    // slack certificates (STEP passes of a solve): the cells' drift counters
    const double dQc = (okc && use_rec) ? __ldcg(g.sdq + tcell) : 0.0;
    // lane bl < nbt (<= 32): band bl's maxima of p (current, average) and drift counter
    const int64_t lbnd = tt * g.nbt + lane;
    const bool okb = bound && lane < g.nbt && lbnd < g.nbands;
    const double Pl = okb ? __ldcg(g.pmax + sx * g.nbands + lbnd) : -INFINITY;
    const double Pal = (okb && bound_avg) ? __ldcg(g.pmax + sA * g.nbands + lbnd) : -INFINITY;
    const double dPl = (okb && use_rec) ? __ldcg(g.sdp + lbnd) : 0.0;
    uint32_t occ_any = 0;
    double mc = INFINITY;
    if (lane == 0) {
      occ_any = __ldcg(g.tocc + sx * tiles + tile);
      if (op == OP_DIST || with_avg) occ_any |= __ldcg(g.tocc + sa * tiles + tile);
      if (op == OP_STEP) occ_any |= __ldcg(g.tocc + sXn * tiles + tile);
      if (with_avg) occ_any |= __ldcg(g.tocc + sA * tiles + tile);
      if (bound) mc = __ldcg(g.tminc + tile);
    }
    double Q = Qc, Qa = Qac;
#pragma unroll
    for (int msk = 1; msk < 32; msk <<= 1) {
      Q = max_nan(Q, __shfl_xor_sync(0xffffffffu, Q, msk));
      Qa = max_nan(Qa, __shfl_xor_sync(0xffffffffu, Qa, msk));
    }
    // RN(max p + max q) <= min C, tested band by band with a vote (rounding is
    // monotone: the same decision); !(a <= b) keeps NaN bounds active
    const double mcb = __shfl_sync(0xffffffffu, mc, 0);
    const bool bad = okb && (!(Pl + Q <= mcb) || (bound_avg && !(Pal + Qa <= mcb)));
    const bool full = __shfl_sync(0xffffffffu, occ_any ? 1 : 0, 0) || open || __any_sync(0xffffffffu, bad);
    if (!full) {
      if (lane == 0) g.tileflag[tile] = 0;
    } else {
#ifdef PDOT_K0_PROF
      const unsigned long long tp1 = globaltimer_ns();
#endif
      if (lane == 0) {
        // the output slots' tile summaries are rebuilt by K1 from the cells it writes
        if (op == OP_STEP) g.tocc[sXn * tiles + tile] = 0;
        if (with_avg) g.tocc[sA * tiles + tile] = 0;
        // metadata traffic of a per-cell screen: per (band, strip) min C and the
        // cell maxima of q (current, average), 4 occupancy words, the flag word
        if (op == OP_STEP && sstat)
          atomicAdd(&sstat[ST_META], (unsigned long long)g.nbt * kWarps * (kCellsPerStrip * 8 * 3 + 4 * 4 + 4));
      }
      // ---- per cell: lane (bq, s) covers bands bq, bq + 4, ... of strip s
      const int s = lane & 7, bq = lane >> 3;
      const int64_t strip = tu * kWarps + s;
      const bool vstrip = strip < g.nstrips;
      const int64_t sstride = g.occ_stride;
      // this lane's 4 cells' q bounds and drift counters: the tile-level loads,
      // through shared memory (read where used, so they hold no registers)
      __shared__ double qsh[kScreenWarps][6][32];
      double(&qw)[6][32] = qsh[warp];
      __syncwarp();  // the previous tile's reads are done
      qw[0][lane] = Qc;
      qw[1][lane] = Qac;
      qw[2][lane] = dQc;
      qw[3][lane] = Pl;  // ... and the bands' (lane = band of the tile)
      qw[4][lane] = Pal;
      qw[5][lane] = dPl;
      __syncwarp();
      uint32_t listed_all = 0;   // 4 bits per round
      uint32_t tb[kCellsPerStrip] = {0u, 0u, 0u, 0u};  // bct bits (band of the tile) of this lane's cells
      bool any_act = false;
      const int nrounds = (g.nbt + 3) >> 2;
      // rounds in chunks of kChunk: every load of a chunk is issued before its
      // flags are computed and stored (one memory round trip per chunk)
#ifndef PDOT_K0_CHUNK
#define PDOT_K0_CHUNK 2
#endif
      constexpr int kChunk = PDOT_K0_CHUNK, kMaxRounds = 8;  // nbt <= 32
      uint32_t words[kMaxRounds];  // flag words of the rounds (static indices: unrolled)
#pragma unroll
      for (int r0 = 0; r0 < kMaxRounds; r0 += kChunk) {
        if (r0 >= nrounds) break;
        uint32_t ox[kChunk], oa[kChunk], zx[kChunk], za[kChunk];
        double mck[kChunk][kCellsPerStrip], rk[kChunk][kCellsPerStrip];
        bool valid[kChunk];
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
          const int bl = (r0 + u) * 4 + bq;
          const int64_t band = tt * g.nbt + bl;
          valid[u] = r0 + u < nrounds && bl < g.nbt && band < g.nbands && vstrip;
          const int64_t ow = band * g.nstrips + strip;
          ox[u] = valid[u] ? __ldcg(g.occ + sx * sstride + ow) : 0u;
          oa[u] = (valid[u] && (op == OP_DIST || with_avg)) ? __ldcg(g.occ + sa * sstride + ow) : 0u;
          zx[u] = (valid[u] && op == OP_STEP) ? __ldcg(g.occ + sXn * sstride + ow) : 0u;
          za[u] = (valid[u] && with_avg) ? __ldcg(g.occ + sA * sstride + ow) : 0u;
#pragma unroll
          for (int k = 0; k < kCellsPerStrip; ++k) {
            const int64_t cell = strip * kCellsPerStrip + k;
            mck[u][k] = (valid[u] && bound && cell < g.ncells) ? __ldcg(g.minc + band * g.ncells + cell) : 0.0;
            rk[u][k] = (valid[u] && use_rec && cell < g.ncells) ? __ldcg(g.srec + band * g.ncells + cell) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
          const int rd = r0 + u;
          const int bl = rd * 4 + bq;
          const int64_t band = tt * g.nbt + bl;
          uint32_t word = 0;
          if (valid[u]) {
#pragma unroll
            for (int k = 0; k < kCellsPerStrip; ++k) {
              const int64_t cell = strip * kCellsPerStrip + k;
              if (cell >= g.ncells) break;
              const uint32_t bx = (ox[u] >> (8 * k)) & 0xffu, ba = (oa[u] >> (8 * k)) & 0xffu;
              const uint32_t bzx = (zx[u] >> (8 * k)) & 0xffu, bza = (za[u] >> (8 * k)) & 0xffu;
              // a cell the coarse bound keeps is dropped when its slack record, less the
              // drift since (all rounded down), is still positive: then p_i + q_j <= C_ij
              // for both pairs (no certificate for a cell with a non-finite cost)
              const int kc = s * kCellsPerStrip + k;
              const bool coarse = (bound && !(qw[3][bl] + qw[0][kc] <= mck[u][k])) ||
                                  (bound_avg && !(qw[4][bl] + qw[1][kc] <= mck[u][k]));
              const bool cert = use_rec && mck[u][k] != -INFINITY &&
                                __dsub_rd(__dsub_rd(rk[u][k], qw[5][bl]), qw[2][kc]) > 0.0;
              const bool act = bx || ba || open || (coarse && !cert);
              const uint32_t f = (act ? U_ACT : 0u) | (bx ? U_LDX : 0u) | (ba ? U_LDA : 0u) |
                                 (bzx ? U_ZX : 0u) | (bza ? U_ZA : 0u);
              word |= f << (8 * k);
            }
          }
          words[rd] = word;
          uint32_t listed = 0, actb = 0;
#pragma unroll
          for (int k = 0; k < kCellsPerStrip; ++k) {
            const uint32_t f = (word >> (8 * k)) & 0xffu;
            listed |= (f != 0u) << k;
            actb |= ((f & U_ACT) != 0u) << k;
            tb[k] |= ((f & U_ACT) != 0u ? 1u : 0u) << (bl & 31);
          }
          any_act |= actb != 0u;
          if (rd < 8) listed_all |= listed << (4 * rd);
          // bcr[band][tu]: bit 4 s + k = cell k of strip s (the 8 lanes of one band)
          uint32_t rbits = actb << (4 * s);
#pragma unroll
          for (int msk = 1; msk < 8; msk <<= 1) rbits |= __shfl_xor_sync(0xffffffffu, rbits, msk);
          if (s == 0 && rd < nrounds && bl < g.nbt && band < g.nbands) g.bcr[band * g.U + tu] = rbits;
        }
      }
      // warp-aggregated append of the listed cells: one atomic per tile
#ifdef PDOT_K0_PROF
      const unsigned long long tp2 = globaltimer_ns();
#endif
      const int cnt = __popc(listed_all);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      // both list appends in flight together: the tile list (lane 0) and the cells (lane 31)
      const bool any = __any_sync(0xffffffffu, any_act);
      unsigned tslot = 0;
      if (lane == 0 && any) tslot = atomicAdd(g.tcount, 1u);
      unsigned base = 0;
      if (lane == 31 && tot) base = atomicAdd(g.ucount, (unsigned)tot);
      base = __shfl_sync(0xffffffffu, base, 31);
#ifdef PDOT_K0_PROF
      const unsigned long long tp3 = globaltimer_ns();
#endif
      unsigned pos = base + (unsigned)(incl - cnt);
#pragma unroll
      for (int rd = 0; rd < kMaxRounds; ++rd) {
        if (rd >= nrounds) break;
        const uint32_t l4 = (listed_all >> (4 * rd)) & 0xfu;
        const int64_t band = tt * g.nbt + rd * 4 + bq;
#pragma unroll
        for (int k = 0; k < kCellsPerStrip; ++k)
          if ((l4 >> k) & 1u) {
            g.ulist[pos] = cell_entry(band, strip * kCellsPerStrip + k, g.cbits);
            g.uflag[pos] = (uint8_t)((words[rd] >> (8 * k)) & 0xffu);  // the cell's flags travel with it
            ++pos;
          }
      }
      // bct[tt][cell]: bit bl = band bl of the tile (OR over the 4 band quarters)
#pragma unroll
      for (int k = 0; k < kCellsPerStrip; ++k) {
        tb[k] |= __shfl_xor_sync(0xffffffffu, tb[k], 8);
        tb[k] |= __shfl_xor_sync(0xffffffffu, tb[k], 16);
      }
      if (bq == 0) {
#pragma unroll
        for (int k = 0; k < kCellsPerStrip; ++k) g.bct[tt * g.ncp + tu * 32 + s * kCellsPerStrip + k] = tb[k];
      }
      // the tile's partials are assembled by K1b, or are all +0 (flag 0)
      if (lane == 0) {
        g.tileflag[tile] = any ? 1 : 0;
        if (any) g.tlist[tslot] = (int32_t)tile;
      }
#ifdef PDOT_K0_PROF
      if (lane == 0 && op == OP_STEP) {
        const unsigned long long tp4 = globaltimer_ns();
        atomicAdd(&g_k0prof[0], 1ull);
        atomicAdd(&g_k0prof[1], tp1 - tp0);
        atomicAdd(&g_k0prof[2], tp2 - tp0);
        atomicAdd(&g_k0prof[3], tp3 - tp0);
        atomicAdd(&g_k0prof[4], tp4 - tp0);
      }
#endif
    }
  }
  if (tl) {
    __syncthreads();
    tl_end(tl, 0);
  }
}

// ---------------------------------------------------------------------------
// K1: one warp per listed cell (8 rows x 16 columns).  Lane = (row group rg =
// lane / 8 holding rows 2 rg and 2 rg + 1, column pair cp = lane % 8), so all
// 32 lanes carry elements.  The partials follow the canonical tree of
// pass_ops.cuh: column band partial ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) via
// pair sums and masks 8, 16; row values via the 8-lane butterfly; scalars as
// the lane-sequential row chain (passed from row group to row group) and the
// 8-lane butterfly.
// ---------------------------------------------------------------------------
struct CellGeo {
  int64_t band, cell, strip, i0, j;
  int rows, k, rg, cp;
  bool v0, v1;
};

template <class Cx>
__device__ __forceinline__ CellGeo cell_geo(const Cx& c, uint32_t entry) {
  const int lane = threadIdx.x & 31;
  CellGeo g;
  g.band = entry_band(entry, c.cbits);
  g.cell = entry_cell(entry, c.cbits);
  DCHECK(g.band < c.nbands, "band", g.band, c.nbands);
  DCHECK(g.cell < c.ncells, "cell", g.cell, c.ncells);
  g.strip = g.cell >> 2;
  g.k = (int)(g.cell & 3);
  g.i0 = g.band * kBand;
  g.rows = (int)imin64(kBand, c.m - g.i0);
  g.cp = lane & 7;
  g.rg = lane >> 3;
  g.j = g.cell * kCell + g.cp * 2;
  g.v0 = g.j < c.n;
  g.v1 = g.j + 1 < c.n;
  return g;
}

// Partial writes shared by every cell op.  o[rr][q][e]: the lane's outputs for
// row 2 rg + rr, column e; sacc: the lane's stage scalar partials (its two
// rows, element order).  The three reductions follow the canonical tree of
// pass_ops.cuh and run through a per-warp shared-memory transpose (each lane
// writes its values, then reads the ones it reduces):
//   columns: in-lane pair sum, then (rg0 + rg1) + (rg2 + rg3);
//   rows:    in-lane column-pair sum, then ((c0+c1)+(c2+c3))+((c4+c5)+(c6+c7));
//   scalars: (rg0 + rg1) + (rg2 + rg3) per column pair, then the column-pair
//            tree (its last two levels as shuffles over lane bits 0, 1).
// Strides 36 / 33 keep the 64-bit reads at two wavefronts (conflict-free).
constexpr int kColD = 36, kRowD = 33, kScalD = 33;
constexpr int kRedWarpDoubles = 8 * kColD;

// the calling warp's transpose buffer (one buffer per kernel for every op)
__device__ __forceinline__ double* warp_red_buf() {
  __shared__ double red_buf[kWarps * kRedWarpDoubles];
  return red_buf + (threadIdx.x >> 5) * kRedWarpDoubles;
}

template <int NQ, int NS, class Cx>
__device__ __forceinline__ void cell_flush(const Cx& c, const CellGeo& g, const double (&o)[2][NQ][2],
                                          const double (&sacc)[NS]) {
  static_assert(2 * NQ <= 8 && NS <= 8, "per-warp transpose buffer");
  const int lane = threadIdx.x & 31;
  double* S = warp_red_buf();
  // ---- column band partials
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int e = 0; e < 2; ++e) S[(2 * q + e) * kColD + lane] = o[0][q][e] + o[1][q][e];
  __syncwarp();
  if (NQ == 4) {  // lane (q, column pair cp)
    const int q = lane >> 3, cp = lane & 7;
    double a[4][2];
#pragma unroll
    for (int rg = 0; rg < 4; ++rg)
#pragma unroll
      for (int e = 0; e < 2; ++e) a[rg][e] = S[(2 * q + e) * kColD + rg * 8 + cp];
    const int64_t j = g.cell * kCell + cp * 2;
    if (j < c.n)
      *reinterpret_cast<double2*>(c.ccol + (g.band * kMaxNQ + q) * c.ldx + j) =
          make_double2((a[0][0] + a[1][0]) + (a[2][0] + a[3][0]), (a[0][1] + a[1][1]) + (a[2][1] + a[3][1]));
  } else if (lane < 16) {  // NQ == 1: lane (e, cp)
    const int e = lane >> 3, cp = lane & 7;
    double a[4];
#pragma unroll
    for (int rg = 0; rg < 4; ++rg) a[rg] = S[e * kColD + rg * 8 + cp];
    const int64_t j = g.cell * kCell + cp * 2;
    if (j < c.n) c.ccol[g.band * kMaxNQ * c.ldx + j + e] = (a[0] + a[1]) + (a[2] + a[3]);
  }
  __syncwarp();
  // ---- row values
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int q = 0; q < NQ; ++q) S[(rr * NQ + q) * kRowD + lane] = o[rr][q][0] + o[rr][q][1];
  __syncwarp();
  if (lane < 8 * NQ) {  // lane (q, row r)
    const int q = lane >> 3, r = lane & 7;
    const double* src = S + ((r & 1) * NQ + q) * kRowD + (r >> 1) * 8;
    double b[8];
#pragma unroll
    for (int cp = 0; cp < 8; ++cp) b[cp] = src[cp];
    const double v = ((b[0] + b[1]) + (b[2] + b[3])) + ((b[4] + b[5]) + (b[6] + b[7]));
    DCHECK(g.cell < c.ncp && (r >= g.rows || g.i0 + r < c.mpad), "crow", g.cell, g.i0 + r);
    if (r < g.rows) c.crow[(g.cell * kMaxNQ + q) * c.mpad + g.i0 + r] = v;
  }
  __syncwarp();
  // ---- scalars: lane (s, cq) reduces column pairs 2 cq, 2 cq + 1
#pragma unroll
  for (int s = 0; s < NS; ++s) S[s * kScalD + lane] = sacc[s];
  __syncwarp();
  {
    const int s = lane >> 2, cq = lane & 3;
    double t = 0.0;
    if (s < NS) {
      double d[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int rg = 0; rg < 4; ++rg) d[h][rg] = S[s * kScalD + rg * 8 + 2 * cq + h];
      t = ((d[0][0] + d[0][1]) + (d[0][2] + d[0][3])) + ((d[1][0] + d[1][1]) + (d[1][2] + d[1][3]));
    }
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    if (s < NS && cq == 0) c.cscal[(g.band * c.ncp + g.cell) * kMaxNS + s] = t;
  }
  __syncwarp();
}

// ---- STEP cells, software-pipelined: the warp copies the next cell's inputs
// (its C / X / A row segments and the dual values) into a shared-memory stage
// with cp.async while it computes the current cell, so the load latency
// overlaps compute.  Every lane reads back only what it copied itself, so a
// lane's own cp.async.wait_group is the only synchronisation needed.  Stage
// layout: field-major, lane-contiguous (conflict-free 16- and 8-byte reads).
// Stage layout: C, X, A as 16-byte fields (both rows of each lane), then the
// cell's duals ONCE (p, pa of its 8 rows; q, qa of its 16 columns), each copied
// by one lane and read back by the lanes that need it (16-byte broadcasts).
constexpr int kStMat = 32 * 16;                    // one 16-byte field of the warp
constexpr int kStP = 6 * kStMat;                   // p[8], then pa[8], q[16], qa[16]
constexpr int kStPa = kStP + 8 * 8;
constexpr int kStQ = kStPa + 8 * 8;
constexpr int kStQa = kStQ + 16 * 8;
constexpr int kStD = kStQa + 16 * 8;               // the band's and the cell's drift counters
constexpr int kStageBytes = kStD + 16;             // 3.4 KB per warp and stage
constexpr int kStages = 3;                         // copies run two cells ahead
constexpr size_t kUnitDynSmem = (size_t)kWarps * kStages * kStageBytes;

// The C / X / A row segments K1 stages are read once per pass: L2 evict-first,
// so that they do not push the pass's partials and the screening metadata out of
// L2 (C3: K2 to its last ticket 10.5 -> 9.5 us, controller reduce 2.5 -> 2.2 us;
// +4-5 % iterations/s, profiles/r02_evict_first_ab.json)
// (the policy is made once per kernel: a plain asm, so the compiler hoists it)
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool on, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst), "l"(src),
               "r"(on ? 16 : 0), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool on) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(on ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// issue the copies of one cell's inputs (zero-filled where not needed).  Lane
// L copies its C / X / A row pairs, p[L] (L < 8) or pa[L - 8] (8 <= L < 16), and
// q[L] (L < 16) or qa[L - 16] (L >= 16).
template <bool IMPLICIT, bool AVG, class Cx>
__device__ __forceinline__ void cell_issue(const StepOp& op, const Cx& c, uint32_t entry, uint32_t f,
                                           unsigned char* stage, bool sr) {
  const int lane = threadIdx.x & 31;
  const CellGeo g = cell_geo(c, entry);
  const bool act = (f & U_ACT) != 0;
  const bool ldx = act && (f & U_LDX);
  const bool lda = AVG && act && (f & U_LDA);
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(stage);
  const uint32_t f16 = base + lane * 16;
  const uint64_t pol = l2_evict_first();
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * g.rg + rr;
    const bool ok = act && r < g.rows && g.v0;
    const int64_t i = ok ? g.i0 + r : 0;
    const int64_t jj = ok ? g.j : 0;
    if (!IMPLICIT) cp_async16(f16 + (0 + rr) * kStMat, op.C + i * c.ldc + jj, ok, pol);
    cp_async16(f16 + (2 + rr) * kStMat, op.X + i * c.ldx + jj, ok && ldx, pol);
    cp_async16(f16 + (4 + rr) * kStMat, (AVG ? op.A : op.X) + i * c.ldx + jj, ok && lda, pol);
  }
  if (lane < 16) {  // p / pa of row lane & 7
    const int r = lane & 7;
    const bool ok = act && r < g.rows;
    const double* src = (lane < 8 ? op.p : op.pa) + (ok ? g.i0 + r : 0);
    cp_async8(base + kStP + lane * 8, src, ok);
  }
  {  // q / qa of column lane & 15 of the cell
    const int64_t jc = g.cell * kCell + (lane & 15);
    const bool ok = act && jc < c.n;
    const double* src = (lane < 16 ? op.q : op.qa) + (ok ? jc : 0);
    cp_async8(base + kStQ + lane * 8, src, ok);
  }
  if (sr && lane < 2) {  // slack certificates: the drift counters the cell's record is shifted by
    const bool ok = act;
    const double* src = lane == 0 ? c.sdp + (ok ? g.band : 0) : c.sdq + (ok ? g.cell : 0);
    cp_async8(base + kStD + lane * 8, src, ok);
  }
}

template <bool IMPLICIT, bool AVG, class Cx>
__device__ __forceinline__ void cell_step(const StepOp& op, const Cx& c, const Ctl& dyn, const CostGen& gen,
                                          uint32_t entry, uint32_t f,
                                          const unsigned char* stage, unsigned& bytes,
                                          unsigned long long& cells, bool sr) {
  constexpr int NQ = StepOp::NQ, NS = StepOp::NS;
  const int lane = threadIdx.x & 31;
  const CellGeo g = cell_geo(c, entry);
  const bool act = (f & U_ACT) != 0;  // cell-uniform
  const bool ldx = act && (f & U_LDX);
  const bool lda = AVG && act && (f & U_LDA);
  const bool zx = (f & U_ZX) != 0;
  const bool za = AVG && (f & U_ZA) != 0;
  if (lane == 0 && act) cells += 1;
  const double2* s16 = reinterpret_cast<const double2*>(stage) + lane;
  // the lane's two rows of p / pa and its column pair of q / qa (broadcast reads)
  const double2 p2 = *reinterpret_cast<const double2*>(stage + kStP + 16 * g.rg);
  const double2 pa2 = *reinterpret_cast<const double2*>(stage + kStPa + 16 * g.rg);
  double2 cc[2], xx[2], aa[2];
  const double pr[2] = {p2.x, p2.y}, par[2] = {pa2.x, pa2.y};
  bool okr[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * g.rg + rr;
    okr[rr] = act && r < g.rows && g.v0;
    cc[rr] = IMPLICIT ? make_double2(0.0, 0.0) : s16[(0 + rr) * 32];
    xx[rr] = s16[(2 + rr) * 32];
    aa[rr] = s16[(4 + rr) * 32];
    if (okr[rr]) bytes += (IMPLICIT ? 0 : 16) + (ldx ? 16 : 0) + (lda ? 16 : 0);
  }
  const double2 q2 = *reinterpret_cast<const double2*>(stage + kStQ + 16 * g.cp);
  const double2 qa2 = *reinterpret_cast<const double2*>(stage + kStQa + 16 * g.cp);
  const double qv[2] = {q2.x, q2.y}, qav[2] = {qa2.x, qa2.y};
  if (IMPLICIT && act) {
    const double2 c0 = gen.col_coord(g.j), c1 = gen.col_coord(g.j + 1);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const double2 rc = gen.row_coord(g.i0 + 2 * g.rg + rr);
      if (okr[rr]) cc[rr] = make_double2(gen.cost(rc, c0), gen.cost(rc, c1));
    }
  }
  double o[2][NQ][2];
  double sacc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
  bool nzx = false, nza = false;
  double smin = INFINITY;  // slack certificate: min over the lane's entries, rounded down
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * g.rg + rr;
    const bool inrow = r < g.rows && g.v0;
    const int64_t i = g.i0 + r;
    double o0[NQ], o1[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
    if (okr[rr]) {  // StepOp::elem in the dense walkers' element order
      op.template elem<AVG>(cc[rr].x, xx[rr].x, aa[rr].x, pr[rr], qv[0], par[rr], qav[0], o0, sacc);
      if (g.v1) op.template elem<AVG>(cc[rr].y, xx[rr].y, aa[rr].y, pr[rr], qv[1], par[rr], qav[1], o1, sacc);
      if (sr) {
        // C - (p + q) and C - (pa + qa), each a lower bound of the exact value
        smin = fmin(smin, fmin(__dsub_rd(cc[rr].x, __dadd_ru(pr[rr], qv[0])),
                               __dsub_rd(cc[rr].x, __dadd_ru(par[rr], qav[0]))));
        if (g.v1)
          smin = fmin(smin, fmin(__dsub_rd(cc[rr].y, __dadd_ru(pr[rr], qv[1])),
                                 __dsub_rd(cc[rr].y, __dadd_ru(par[rr], qav[1]))));
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      o[rr][q][0] = o0[q];
      o[rr][q][1] = o1[q];
    }
    const double2 xo = make_double2(o0[2], o1[2]);
    const bool nzr = nz2(xo);
    nzx |= nzr;
    if (inrow && (okr[rr] ? (zx || nzr) : zx)) {
      st_stream2(op.Xn + i * c.ldx + g.j, xo);
      bytes += 16;
    }
    if (AVG) {
      const double2 ao = make_double2(o0[3], o1[3]);
      const bool nar = nz2(ao);
      nza |= nar;
      if (inrow && (okr[rr] ? (za || nar) : za)) {
        st_stream2(op.An + i * c.ldx + g.j, ao);
        bytes += 16;
      }
    }
  }
  // occupancy bytes of the cell in the two output slots
  const bool anyx = __any_sync(0xffffffffu, nzx), anya = __any_sync(0xffffffffu, nza);
  if (lane == 0) {
    const int sXn = dyn.sXn, sA = dyn.sA;
    uint8_t* ox = reinterpret_cast<uint8_t*>(c.occ + sXn * c.occ_stride + g.band * c.nstrips + g.strip);
    ox[g.k] = anyx ? 1 : 0;
    const int64_t tile = (g.band >> c.nbt_log2) * c.U + g.strip / kWarps;  // nbt: a power of two
    if (anyx) c.tocc[sXn * c.tiles + tile] = 1;
    if (AVG) {
      uint8_t* oa = reinterpret_cast<uint8_t*>(c.occ + sA * c.occ_stride + g.band * c.nstrips + g.strip);
      oa[g.k] = anya ? 1 : 0;
      if (anya) c.tocc[sA * c.tiles + tile] = 1;
    }
  }
  if (act) {
    cell_flush<NQ, NS>(c, g, o, sacc);
    if (lane == 0) bytes += (unsigned)(NQ * kCell + NQ * kBand + NS) * 8 * 2;
    if (sr) {  // the cell's record: shifted by the drift counters (rounded down)
      // warp minimum in one REDUX: the high word of a positive double orders like
      // the double and, with the low word cleared, rounds it down; a slack <= 0
      // (or NaN) in any lane means no certificate
      const int key = smin > 0.0 ? __double2hiint(smin) : INT_MIN;
      const int kmin = __reduce_min_sync(0xffffffffu, key);
      if (lane == 0) {
        const double2 dd = *reinterpret_cast<const double2*>(stage + kStD);
        const double rec = kmin > 0 ? __dadd_rd(__dadd_rd(__hiloint2double(kmin, 0), dd.x), dd.y) : -INFINITY;
        c.srec[g.band * c.ncells + g.cell] = rec;
      }
    }
  }
}

// The list length and a warp's first two list entries, read at kernel entry
// (independent of the control block; the list has kListPad spare entries, so
// values past the length are read but not used)
struct ListHead {
  uint32_t e_cur, f_cur, e_nx, f_nx, e_n2, f_n2;
  unsigned ncells;
};
template <class Cx>
__device__ __forceinline__ ListHead list_head(const Cx& c, unsigned k0, unsigned nw) {
  ListHead h;
  h.e_cur = __ldcg(c.ulist + k0);
  h.f_cur = __ldcg(c.uflag + k0);
  h.e_nx = __ldcg(c.ulist + k0 + nw);
  h.f_nx = __ldcg(c.uflag + k0 + nw);
  h.e_n2 = __ldcg(c.ulist + k0 + 2 * nw);
  h.f_n2 = __ldcg(c.uflag + k0 + 2 * nw);
  h.ncells = __ldcg(c.ucount);
  return h;
}

// PDOT_K1_PROF (measurement builds only): per-warp K1 phase times, summed over
// a solve and printed by the last CTA of pass 600
#ifdef PDOT_K1_PROF
__device__ unsigned long long g_k1prof[16];
#endif

// the warp's STEP cells k = k0, k0 + nw, ...: copies of cell k + nw in flight
// while cell k is computed
template <bool IMPLICIT, bool AVG, class Cx>
__device__ __forceinline__ void step_cells(const StepOp& o, const Cx& c, const Ctl& dyn, const CostGen& gen, unsigned k0,
                                           unsigned nw, const ListHead& lh, unsigned char* stages,
                                           unsigned long long& bytes, unsigned long long& cells,
                                           unsigned long long tp_entry) {
  // the warp's cells k0, k0 + nw, ...: cell i's copies are issued two cells
  // ahead (stage i % 3) and its list entry three cells ahead
  uint32_t e0 = lh.e_cur, f0 = lh.f_cur, e1 = lh.e_nx, f1 = lh.f_nx, e2 = lh.e_n2, f2 = lh.f_n2;
  const unsigned ncells = lh.ncells;
  if (k0 >= ncells) return;
#ifdef PDOT_K1_PROF
  const unsigned long long tp_list = globaltimer_ns();
  unsigned long long tp_first = 0, np = 0;
#endif
  unsigned bytes32 = 0;  // this warp-lane's bytes (32-bit: a few hundred per cell)
  const bool sr = dyn.sr_on && !dyn.unit;  // slack certificates of this pass's cells
  cell_issue<IMPLICIT, AVG>(o, c, e0, f0, stages, sr);
  cp_async_commit();
  if (k0 + nw < ncells) cell_issue<IMPLICIT, AVG>(o, c, e1, f1, stages + kStageBytes, sr);
  cp_async_commit();
  int st = 0;
  for (unsigned k = k0; k < ncells; k += nw) {
    uint32_t e3 = 0, f3 = 0;
    if (k + 3 * nw < ncells) {
      e3 = __ldcg(c.ulist + k + 3 * nw);
      f3 = __ldcg(c.uflag + k + 3 * nw);
    }
    const int st2 = st == 0 ? 2 : st - 1;  // (st + 2) % 3
    if (k + 2 * nw < ncells) cell_issue<IMPLICIT, AVG>(o, c, e2, f2, stages + st2 * kStageBytes, sr);
    cp_async_commit();
    cp_async_wait<2>();  // this cell's copies have landed
#ifdef PDOT_K1_PROF
    if (tp_first == 0) tp_first = globaltimer_ns();
    ++np;
#endif
    cell_step<IMPLICIT, AVG>(o, c, dyn, gen, e0, f0, stages + st * kStageBytes, bytes32, cells, sr);
    e0 = e1; f0 = f1;
    e1 = e2; f1 = f2;
    e2 = e3; f2 = f3;
    st = st == 2 ? 0 : st + 1;
  }
  cp_async_wait<0>();
  bytes += bytes32;
#ifdef PDOT_K1_PROF
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long t_end = globaltimer_ns();
    atomicAdd(&g_k1prof[0], tp_list - tp_entry);   // entry -> list length known
    atomicAdd(&g_k1prof[1], tp_first - tp_entry);  // entry -> first cell's copies landed
    atomicAdd(&g_k1prof[2], t_end - tp_first);     // cells
    atomicAdd(&g_k1prof[3], np);
    atomicAdd(&g_k1prof[4], 1ull);
    atomicMax(&g_k1prof[5], t_end - tp_entry);
    atomicAdd(&g_k1prof[6], t_end - tp_entry);
  }
#endif
}

// restart distance (DIST) and the start KKT through the screen (NQ = 1), with
// the dense walkers' per-row compute()
template <class Op>
__device__ __forceinline__ void cell_one(const Op& op, const Ctl& c, uint32_t entry, uint32_t f, unsigned long long& bytes,
                                         unsigned long long& cells) {
  constexpr int NQ = Op::NQ, NS = Op::NS;
  const int lane = threadIdx.x & 31;
  const CellGeo cg = cell_geo(c, entry);
  if (!(f & U_ACT)) return;  // cell-uniform
  if (lane == 0) cells += 1;
  Geo g;  // the fields the ops read
  g.m = c.m; g.n = c.n; g.ldc = c.ldc; g.ldx = c.ldx; g.TM = c.TM;
  g.tu = 0; g.tt = 0; g.i0 = cg.i0; g.rows = cg.rows; g.j = cg.j;
  g.v0 = cg.v0;
  g.v1 = cg.v1;
  g.gen.kind = c.C ? 0 : c.cost_kind;
  g.gen.a0 = c.cost_a[0]; g.gen.a1 = c.cost_a[1]; g.gen.a2 = c.cost_a[2]; g.gen.a3 = c.cost_a[3];
  g.gen.row0 = c.row0;
  typename Op::Col cl;
  op.load_col(cl, g);
  typename Op::Frag fr[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * cg.rg + rr;
    if (r < cg.rows && cg.v0) {
      op.load(fr[rr], g, cg.i0 + r);
      bytes += 32;
    }
  }
  double o[2][NQ][2];
  double sacc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * cg.rg + rr;
    double o0[NQ], o1[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
    if (r < cg.rows && cg.v0) op.compute(fr[rr], g, cg.i0 + r, cl, o0, o1, sacc);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      o[rr][q][0] = o0[q];
      o[rr][q][1] = o1[q];
    }
  }
  cell_flush<NQ, NS>(c, cg, o, sacc);
}

__global__ void __launch_bounds__(kThreads, kSparseCtasPerSm) unit_kernel(const Ctl* __restrict__ ctlp, int force_op,
                                                                          const KGeo geo) {
#ifdef PDOT_K1_PROF
  const unsigned long long tp_entry = globaltimer_ns();
#else
  const unsigned long long tp_entry = 0;
#endif
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  // the list head and the control block travel together (one round trip); the
  // control block is read from shared memory from then on, so values the
  // register budget cannot keep live are re-read from there, not from HBM
  const ListHead lh = list_head(geo, gw, nw);
  __shared__ Ctl ctl_s;
  ctl_to_shared(ctlp, &ctl_s);
  const Ctl& c = ctl_s;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  __shared__ unsigned long long red[2][kWarps];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer_ns();
    c.sstat[ST_T0] = t0;
    if (op == OP_STEP && !c.unit) {
      const unsigned long long k0s = c.sstat[ST_K0_START];
      if (k0s != 0 && t0 > k0s) c.sstat[ST_K0K1] += t0 - k0s;
    }
  }
  unsigned long long* tl = op == OP_STEP ? c.ktl : nullptr;
  tl_start(tl, 1);
  const unsigned ncells = lh.ncells;
  unsigned long long bytes = 0, cells = 0;
  if (op == OP_STEP) {
    const StepOp o = make_step_op(c);
    CostGen gen;
    gen.kind = c.C ? 0 : c.cost_kind;
    gen.a0 = c.cost_a[0]; gen.a1 = c.cost_a[1]; gen.a2 = c.cost_a[2]; gen.a3 = c.cost_a[3];
    gen.row0 = c.row0;
    extern __shared__ __align__(16) unsigned char unit_dyn[];
    unsigned char* stages = unit_dyn + warp * kStages * kStageBytes;
    if (o.C) {
      if (o.with_avg) step_cells<false, true>(o, geo, c, gen, gw, nw, lh, stages, bytes, cells, tp_entry);
      else step_cells<false, false>(o, geo, c, gen, gw, nw, lh, stages, bytes, cells, tp_entry);
    } else {
      if (o.with_avg) step_cells<true, true>(o, geo, c, gen, gw, nw, lh, stages, bytes, cells, tp_entry);
      else step_cells<true, false>(o, geo, c, gen, gw, nw, lh, stages, bytes, cells, tp_entry);
    }
  } else if (op == OP_DIST) {
    DiffOp o;
    o.Xa = c.slot[c.sZ].X; o.Xb = c.slot[c.sCand].X;
    for (unsigned k = gw; k < ncells; k += nw) cell_one(o, c, __ldcg(c.ulist + k), __ldcg(c.uflag + k), bytes, cells);
  } else {
    KktOp o;
    const Slot& sx = c.slot[c.sX];
    o.C = c.C; o.X = sx.X; o.p = sx.p; o.q = sx.q; o.viol = nullptr;
    for (unsigned k = gw; k < ncells; k += nw) cell_one(o, c, __ldcg(c.ulist + k), __ldcg(c.uflag + k), bytes, cells);
  }
  // statistics: fire-and-forget reductions per CTA (no fence, no done counter:
  // the last CTA is not waited for); K2's controller turns the latest end stamp
  // into the pass's K1 time
#pragma unroll
  for (int msk = 16; msk >= 1; msk >>= 1) {
    bytes += __shfl_xor_sync(0xffffffffu, bytes, msk);
    cells += __shfl_xor_sync(0xffffffffu, cells, msk);
  }
  if (lane == 0) {
    red[0][warp] = bytes;
    red[1][warp] = cells;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tb = 0, tc = 0;
    for (int i = 0; i < kWarps; ++i) {
      tb += red[0][i];
      tc += red[1][i];
    }
    atomicAdd(&c.sstat[ST_BYTES], tb);
    atomicAdd(&c.sstat[ST_CELLS], tc);
    if (op == OP_STEP) atomicMax(&c.sstat[ST_K1_END], (unsigned long long)globaltimer_ns());
#ifdef PDOT_K1_PROF
    if (blockIdx.x == 0 && c.passes == 600) {
      const double w = (double)g_k1prof[4];
      printf("K1PROF per warp (ns): entry->list %.0f, entry->first cell %.0f, cells %.0f (%.2f cells, %.0f per cell), "
             "entry->end mean %.0f max %llu\n",
             g_k1prof[0] / w, g_k1prof[1] / w, g_k1prof[2] / w, g_k1prof[3] / w, (double)g_k1prof[2] / g_k1prof[3],
             g_k1prof[6] / w, g_k1prof[5]);
    }
#endif
  }
  tl_end(tl, 1);
}

// ---------------------------------------------------------------------------
// K1b: assembles the per-tile partials of the canonical tree (the same layout
// the dense walkers write: colpart / rowpart / tilescal) from the cell
// partials, for every tile with an active cell.  One CTA per listed tile and
// part (part < 0: all three in one CTA):
//   columns: thread = column pair, band-ordered sum of its cell column;
//   rows:    thread = row, strip-ordered sum of the strip values
//            ((c0 + c1) + (c2 + c3)) of the row segment's active cells;
//   scalars: thread (strip, scalar), band-ordered sum of strip-band values,
//            then the strips in order.
// ---------------------------------------------------------------------------
template <int NQ, int NS, class Cx>
__device__ __forceinline__ void assemble_tile(const Cx& c, int64_t tu, int64_t tt, double* sm, int part) {
  const int th = threadIdx.x;
  const int64_t b0 = tt * c.nbt;
  if (part < 0 || part == 0) {  // columns
    const int64_t j = tu * kTileN + th * 2;
    if (j < c.n) {
      uint32_t m = __ldg(c.bct + tt * c.ncp + j / kCell);
      double2 acc[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] = make_double2(0.0, 0.0);
      while (m) {
        int bb[4];
        int cnt = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bb[e] = 0;
          if (m) {
            bb[e] = __ffs(m) - 1;
            m &= m - 1;
            cnt = e + 1;
          }
        }
        double2 v[4][NQ];
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            v[e][q] = e < cnt ? __ldg(reinterpret_cast<const double2*>(c.ccol + ((b0 + bb[e]) * kMaxNQ + q) * c.ldx + j))
                              : make_double2(0.0, 0.0);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < cnt)
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              acc[q].x += v[e][q].x;
              acc[q].y += v[e][q].y;
            }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) *reinterpret_cast<double2*>(c.colpart + (tt * NQ + q) * c.ldx + j) = acc[q];
    }
  }
  if (part < 0 || part == 1) {  // rows: thread (row, quantity pair); active strips in order, two per round trip
    constexpr int QP = NQ >= 2 ? 2 : 1;
    constexpr int NSL = NQ / QP;
    const int per = (int)blockDim.x / NSL;
    const int qs = th / per;
    for (int r = th - qs * per; r < c.TM; r += per) {
      const int64_t i = tt * c.TM + r;
      if (i >= c.m) break;
      uint32_t word = __ldg(c.bcr + (i / kBand) * c.U + tu);
      const double* rb = c.crow + (tu * 32 * kMaxNQ + qs * QP) * c.mpad + i;  // cell (tu, 0), q = qs * QP
      const int64_t cstride = (int64_t)kMaxNQ * c.mpad;                       // next cell
      double acc[QP];
#pragma unroll
      for (int q = 0; q < QP; ++q) acc[q] = 0.0;
      while (word) {
        const int w0 = (__ffs(word) - 1) >> 2;
        const unsigned nib0 = (word >> (4 * w0)) & 0xfu;
        word &= ~(0xfu << (4 * w0));
        int w1 = 0;
        unsigned nib1 = 0u;
        if (word) {
          w1 = (__ffs(word) - 1) >> 2;
          nib1 = (word >> (4 * w1)) & 0xfu;
          word &= ~(0xfu << (4 * w1));
        }
        const double* p0 = rb + (int64_t)(4 * w0) * cstride;
        const double* p1 = rb + (int64_t)(4 * w1) * cstride;
        double v0[4][QP], v1[4][QP];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int q = 0; q < QP; ++q) {
            v0[x][q] = ((nib0 >> x) & 1u) ? __ldg(p0 + x * cstride + q * c.mpad) : 0.0;
            v1[x][q] = ((nib1 >> x) & 1u) ? __ldg(p1 + x * cstride + q * c.mpad) : 0.0;
          }
#pragma unroll
        for (int q = 0; q < QP; ++q) acc[q] += (v0[0][q] + v0[1][q]) + (v0[2][q] + v0[3][q]);
        if (nib1) {
#pragma unroll
          for (int q = 0; q < QP; ++q) acc[q] += (v1[0][q] + v1[1][q]) + (v1[2][q] + v1[3][q]);
        }
      }
#pragma unroll
      for (int q = 0; q < QP; ++q) c.rowpart[(tu * NQ + qs * QP + q) * c.m + i] = acc[q];
    }
  }
  if (part < 0 || part == 2) {  // scalars: thread (strip w, band bl) forms its strip-band values (one round
     // trip for all of them), then the band-ordered and strip-ordered sums run
     // on shared memory
    const int nb = (int)imin64(c.nbt, c.nbands - b0);
    const int w = th & 7, bl = th >> 3;
    if (bl < nb) {
      const unsigned nib = (__ldg(c.bcr + (b0 + bl) * c.U + tu) >> (4 * w)) & 0xfu;
      const double* base = c.cscal + ((b0 + bl) * c.ncp + tu * 32 + 4 * w) * kMaxNS;
      double v[4][NS];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int s = 0; s < NS; ++s) v[x][s] = ((nib >> x) & 1u) ? __ldg(base + x * kMaxNS + s) : 0.0;
#pragma unroll
      for (int s = 0; s < NS; ++s) sm[(bl * 8 + w) * 8 + s] = (v[0][s] + v[1][s]) + (v[2][s] + v[3][s]);
    }
    __syncthreads();
    double ws = 0.0;
    if (th < 64) {  // thread (w, s): band-ordered sum
      const int ww = th >> 3, s = th & 7;
      if (s < NS)
        for (int k = 0; k < nb; ++k) ws += sm[(k * 8 + ww) * 8 + s];
    }
    __syncthreads();
    if (th < 64) sm[th] = ws;
    __syncthreads();
    if (th < NS) {
      double acc = sm[th];
#pragma unroll
      for (int x = 1; x < kWarps; ++x) acc += sm[x * 8 + th];
      c.tilescal[(tt * c.U + tu) * kMaxNS + th] = acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads, 4) tile_kernel(const Ctl* __restrict__ ctlp, int force_op,
                                                            const KGeo c) {
  __shared__ double sm[32 * 8 * 8];  // [band][strip][scalar] strip-band values
  pdl_trigger();  // K2 may be scheduled as K1b's CTAs retire (its controller block starts its dry run)
  const Ctl& dyn = *ctlp;
  if (dyn.done || !dyn.screen) return;
  const int op = force_op >= 0 ? force_op : dyn.op;
  if (!unit_pass(dyn, op)) return;
  // the first item's tile is read before the list length is known (the grid
  // has at most 3 T U blocks, so blockIdx.x / 3 is inside the list buffer)
  int32_t tile_nx = __ldcg(c.tlist + blockIdx.x / 3u);
  const unsigned ntiles = __ldcg(c.tcount);
  const unsigned nitems = ntiles * 3u;
  unsigned long long* tl = op == OP_STEP ? dyn.ktl : nullptr;
  tl_start(tl, 2);
  // work item k = (listed tile k / 3, part k % 3): the column, row and scalar
  // sums of one tile run in three CTAs side by side
  for (unsigned k = blockIdx.x; k < nitems; k += gridDim.x) {
    const int32_t tile = tile_nx;
    if (k + gridDim.x < nitems) tile_nx = __ldcg(c.tlist + (k + gridDim.x) / 3u);
    const int part = (int)(k % 3u);
    const int64_t tt = (uint32_t)tile / (uint32_t)c.U, tu = tile - tt * c.U;  // 32-bit division
    if (op == OP_STEP) assemble_tile<4, 6>(c, tu, tt, sm, part);
    else if (op == OP_DIST) assemble_tile<1, 1>(c, tu, tt, sm, part);
    else assemble_tile<1, 3>(c, tu, tt, sm, part);
  }
  tl_end(tl, 2);
}

// the unit calls the screen does not cover (KKT of a unit call, DIFF, ROUND):
// the generic walker over every tile, per-tile partials
// A tile whose plan entries are all +0.0 in the slot being rounded: the
// row / column sums of the rounding stages 0-2 (rs_i * X, (rs_i * X) * cs_j)
// are exact +0 there, so its partials are written as the zeros the walker
// would produce, without reading the 512 KB of X.  (Stage 3 adds the rank-one
// correction err_r err_c^T / total, which is dense, and reads C: never skipped.)
__device__ __forceinline__ void zero_round_tile(const Ctl& c, int64_t tu, int64_t tt) {
  const int64_t i0 = tt * c.TM, rows = imin64(c.TM, c.m - i0);
  const int64_t col0 = tu * kTileN, cols = imin64(kTileN, c.n - col0);
  for (int64_t j = 2 * threadIdx.x; j < cols; j += 2 * blockDim.x)
    *reinterpret_cast<double2*>(c.colpart + tt * c.ldx + col0 + j) = make_double2(0.0, 0.0);
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) c.rowpart[tu * c.m + i0 + r] = 0.0;
  if (threadIdx.x == 0) {
    c.tilescal[(tt * c.U + tu) * kMaxNS] = 0.0;
    if (c.tileflag) c.tileflag[tt * c.U + tu] = 1;
  }
}

__global__ void __launch_bounds__(kThreads, 1) generic_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const Ctl& c = *ctlp;
  if (c.done) return;
  const int op = force_op >= 0 ? force_op : c.op;
  // rounding stages 0-2 on a screened handle: tiles without occupied cells are +0
  const bool skip_empty = op == OP_ROUND && c.round_stage <= 2 && c.screen && c.tocc != nullptr;
  const int64_t tiles = c.T * c.U;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    if (skip_empty && __ldcg(c.tocc + (int64_t)c.sX * tiles + t) == 0) {
      zero_round_tile(c, t % c.U, t / c.U);
    } else {
      generic_tile(op, c, smem, t % c.U, t / c.U);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// metadata kernels
// ---------------------------------------------------------------------------
// min C over each 8 x 16 cell; -inf when the cell holds a non-finite cost
// (0 * inf would be NaN in <C, X+>, so such cells are never skipped)
__global__ void minc_kernel(const double* __restrict__ C, int64_t ldc, CostGen gen, int64_t m, int64_t n,
                            int64_t nbands, int64_t ncells, double* __restrict__ out) {
  const int64_t total = nbands * ncells;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t band = e / ncells, cell = e - band * ncells;
    const int64_t i0 = band * kBand, j0 = cell * kCell;
    const int64_t i1 = imin64(i0 + kBand, m), j1 = imin64(j0 + kCell, n);
    double mn = INFINITY;
    bool bad = false;
    for (int64_t i = i0; i < i1; ++i) {
      const double2 rc = gen.kind > 0 ? gen.row_coord(i) : make_double2(0.0, 0.0);
      for (int64_t j = j0; j < j1; ++j) {
        const double v = C ? C[i * ldc + j] : gen.cost(rc, gen.col_coord(j));
        if (!isfinite(v)) bad = true;
        mn = fmin(mn, v);
      }
    }
    out[e] = bad ? -INFINITY : mn;
  }
}

// min C over each tile (from the cell minima; -inf propagates)
struct TileMeta {  // the geometry the tile metadata kernels need (kernel argument)
  int64_t nbt, nbands, nstrips, ncells, T, U;
  const double* minc;
  const uint32_t* occ;
  uint8_t* tocc;
};

__host__ TileMeta tile_meta(const Ctl& h) {
  return TileMeta{h.nbt, h.nbands, h.nstrips, h.ncells, h.T, h.U, h.minc, h.occ, h.tocc};
}

__global__ void tile_minc_kernel(const TileMeta c, double* __restrict__ tminc) {
  __shared__ double wmin[8];
  const int64_t tu = blockIdx.x, tt = blockIdx.y;
  const int s = threadIdx.x & 7, bl = threadIdx.x >> 3, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t band = tt * c.nbt + bl, strip = tu * kWarps + s;
  double mn = INFINITY;
  if (bl < c.nbt && band < c.nbands && strip < c.nstrips)
    for (int k = 0; k < kCellsPerStrip; ++k) {
      const int64_t cell = strip * kCellsPerStrip + k;
      if (cell < c.ncells) mn = fmin(mn, c.minc[band * c.ncells + cell]);
    }
#pragma unroll
  for (int msk = 1; msk < 32; msk <<= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, msk));
  if (lane == 0) wmin[warp] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mn = fmin(mn, wmin[w]);
    tminc[tt * c.U + tu] = mn;
  }
}

// tile summaries of one slot's occupancy bytes
__global__ void tocc_kernel(const TileMeta c, int slot) {
  const int64_t tu = blockIdx.x, tt = blockIdx.y;
  const int s = threadIdx.x & 7, bl = threadIdx.x >> 3;
  const int64_t band = tt * c.nbt + bl, strip = tu * kWarps + s;
  uint32_t w = 0;
  if (bl < c.nbt && band < c.nbands && strip < c.nstrips)
    w = c.occ[(int64_t)slot * c.nbands * c.nstrips + band * c.nstrips + strip];
  const int any = __syncthreads_or(w != 0u);
  if (threadIdx.x == 0) c.tocc[(int64_t)slot * c.T * c.U + tt * c.U + tu] = any ? 1 : 0;
}

// occupancy bytes of one slot matrix: cell flag = any nonzero bit pattern
__global__ void occ_scan_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, int64_t n, int64_t nbands,
                                int64_t ncells, uint8_t* __restrict__ occ_bytes, int64_t nstrips) {
  const int64_t total = nbands * nstrips * kCellsPerStrip;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t band = e / (nstrips * kCellsPerStrip), cell = e - band * nstrips * kCellsPerStrip;
    uint8_t f = 0;
    if (cell < ncells) {
      const int64_t i0 = band * kBand, j0 = cell * kCell;
      const int64_t i1 = imin64(i0 + kBand, m), j1 = imin64(j0 + kCell, n);
      for (int64_t i = i0; i < i1 && !f; ++i)
        for (int64_t j = j0; j < j1; ++j)
          if (__double_as_longlong(X[i * ldx + j]) != 0) {
            f = 1;
            break;
          }
    }
    occ_bytes[e] = f;  // word (band, strip) byte k = cell 4 strip + k (little endian)
  }
}

// NaN-propagating band maxima of p and cell maxima of q of one slot
__global__ void bounds_kernel(const double* __restrict__ p, const double* __restrict__ q, int64_t m, int64_t n,
                              int64_t nbands, int64_t ncells, double* __restrict__ pmax, double* __restrict__ qmax) {
  const int64_t total = nbands + ncells;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double mx = -INFINITY;
    if (e < nbands) {
      for (int64_t i = e * kBand; i < imin64((e + 1) * kBand, m); ++i) mx = max_nan(mx, p[i]);
      pmax[e] = mx;
    } else {
      const int64_t cell = e - nbands;
      for (int64_t j = cell * kCell; j < imin64((cell + 1) * kCell, n); ++j) mx = max_nan(mx, q[j]);
      qmax[cell] = mx;
    }
  }
}

// sparse device -> host copy of a slot matrix (pdot_get_slot with screening
// on): list the cells whose occupancy byte is set (the rest is +0.0 in memory),
// then gather them, 8 rows x 16 columns each, into a staging buffer
__global__ void occ_list_kernel(const uint8_t* __restrict__ occ_bytes, int64_t nbands, int64_t ncells,
                                int64_t nstrips, int cbits, uint32_t* __restrict__ list, unsigned* __restrict__ count) {
  const int64_t total = nbands * nstrips * kCellsPerStrip;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t band = e / (nstrips * kCellsPerStrip), cell = e - band * nstrips * kCellsPerStrip;
    const bool on = cell < ncells && occ_bytes[e] != 0;
    const unsigned bal = __ballot_sync(__activemask(), on);
    if (!on) continue;
    // one atomic per warp
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(bal) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned)__popc(bal));
    base = __shfl_sync(bal, base, leader);
    list[base + __popc(bal & ((1u << lane) - 1u))] = cell_entry(band, cell, cbits);
  }
}

__global__ void cell_gather_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, int64_t n, int cbits,
                                   const uint32_t* __restrict__ list, int64_t k0, int64_t k1,
                                   double* __restrict__ out) {
  // one warp per cell: lane = (row rg, column pair cp) as in the cell kernel
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = k0 + w; k < k1; k += nw) {
    const uint32_t entry = list[k];
    const int64_t band = entry_band(entry, cbits), cell = entry_cell(entry, cbits);
    const int cp = lane & 7, rg = lane >> 3;
    const int64_t j = cell * kCell + cp * 2;
    double* o = out + (k - k0) * (kBand * kCell);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int r = 2 * rg + rr;
      const int64_t i = band * kBand + r;
      double2 v = make_double2(0.0, 0.0);
      if (i < m && j < n) v = *reinterpret_cast<const double2*>(X + i * ldx + j);
      *reinterpret_cast<double2*>(o + r * kCell + cp * 2) = v;
    }
  }
}

}  // namespace

unsigned launch_occ_list(const Ctl& h, int slot, uint32_t* list, unsigned* count_dev, cudaStream_t s) {
  cudaMemsetAsync(count_dev, 0, sizeof(unsigned), s);
  const uint8_t* ob = reinterpret_cast<const uint8_t*>(h.occ + (int64_t)slot * h.nbands * h.nstrips);
  occ_list_kernel<<<148 * 8, 256, 0, s>>>(ob, h.nbands, h.ncells, h.nstrips, h.cbits, list, count_dev);
  unsigned cnt = 0;
  cudaMemcpyAsync(&cnt, count_dev, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return cnt;
}

void launch_cell_gather(const Ctl& h, int slot, const uint32_t* list, int64_t k0, int64_t k1, double* out,
                        cudaStream_t s) {
  const int64_t warps = k1 - k0;
  const unsigned blocks = (unsigned)imin64((warps * 32 + 255) / 256, 148 * 16);
  if (blocks > 0) cell_gather_kernel<<<blocks, 256, 0, s>>>(h.slot[slot].X, h.ldx, h.m, h.n, h.cbits, list, k0, k1, out);
}

void prepare_sparse_kernel() {
  cudaFuncSetAttribute(generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUnitDynSmem);
}

static size_t generic_smem_bytes(int64_t TM) {
  return (size_t)TM * kMaxNQ * kWarps * sizeof(double) + kWarps * 8 * sizeof(double);
}

// K2 is launched as a programmatic dependent of K1b (its controller block's
// instruction-cache dry run overlaps K1b's tail: C3 +1.8 % iterations/s,
// profiles/r02_pdl_edges_ab.json); PDOT_PDL_K2=0 launches it plainly.  PDL on the
// K0 -> K1 and K1 -> K1b edges measured slower and is not used.
bool pdl_edge(const char* name) {
  static const bool k2 = [] {
    const char* e = getenv("PDOT_PDL_K2");
    return e == nullptr || atoi(e) != 0;
  }();
  return std::string(name) == "k2" && k2;
}

void launch_screened_pass(const Ctl* ctl_dev, const Ctl& h, int force_op, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // graph passes (force_op < 0) are STEP / DIST / start-KKT; unit calls choose on the host
  if (force_op < 0 || unit_pass(h, force_op)) {
    unsigned g0 = (unsigned)imin64((h.T * h.U + kScreenWarps - 1) / kScreenWarps, (int64_t)sms * kScreenCtasPerSm);
    // test hook: PDOT_K0_BLOCKS caps K0's grid (read per launch), so that small
    // problems run the persistent tile walk with many tiles per warp
    if (const char* e = getenv("PDOT_K0_BLOCKS")) g0 = (unsigned)imin64(g0, imax64(1, atoi(e)));
    const KGeo geo{h.m, h.n, h.ldx, h.ldc, h.mpad, h.nbands, h.nstrips, h.ncells, h.ncp, h.T, h.U,
                   h.nbands * h.nstrips, h.T * h.U, h.nbt, h.cbits, __builtin_ctz((unsigned)h.nbt), 0,
                   h.occ, h.tocc, h.ccol, h.crow, h.cscal, h.ulist, h.uflag, h.ucount,
                   h.TM, h.bcr, h.bct, h.tlist, h.tcount, h.colpart, h.rowpart, h.tilescal,
                   h.srec, h.sdp, h.sdq, h.qmax, h.pmax, h.minc, h.tminc, h.tileflag};
    screen_kernel<<<g0, 32 * kScreenWarps, 0, s>>>(ctl_dev, force_op, h.sstat, geo);  // warp per tile, persistent
    if (getenv("PDOT_DEBUG_SYNC")) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) fprintf(stderr, "screen_kernel failed: %s\n", cudaGetErrorString(e));
    }
    // every warp reads list entries gw, gw + nw and gw + 2 nw up front: 3 nw <= kListPad
    const unsigned g1 = (unsigned)imin64((int64_t)sms * kSparseCtasPerSm, kListPad / (3 * kWarps));

    unit_kernel<<<g1, kThreads, kUnitDynSmem, s>>>(ctl_dev, force_op, geo);
    tile_kernel<<<(unsigned)imin64(h.T * h.U * 3, (int64_t)sms * 4), kThreads, 0, s>>>(ctl_dev, force_op, geo);
  } else {
    const unsigned grid = (unsigned)imin64(h.T * h.U, (int64_t)sms * 2);
    generic_kernel<<<grid, kThreads, generic_smem_bytes(h.TM), s>>>(ctl_dev, force_op);
  }
}

static dim3 tile_grid(const Ctl& h) { return dim3((unsigned)h.U, (unsigned)h.T); }
static unsigned tile_threads(const Ctl& h) { return (unsigned)(kWarps * h.nbt < 32 ? 32 : kWarps * h.nbt); }

void launch_minc_build(const Ctl& h, double* minc, cudaStream_t s) {
  CostGen gen;
  gen.kind = h.C ? 0 : h.cost_kind;
  gen.a0 = h.cost_a[0]; gen.a1 = h.cost_a[1]; gen.a2 = h.cost_a[2]; gen.a3 = h.cost_a[3];
  gen.row0 = h.row0;
  minc_kernel<<<148 * 8, 256, 0, s>>>(h.C, h.ldc, gen, h.m, h.n, h.nbands, h.ncells, minc);
  TileMeta tm = tile_meta(h);
  tm.minc = minc;
  tile_minc_kernel<<<tile_grid(h), tile_threads(h), 0, s>>>(tm, const_cast<double*>(h.tminc));
}

void launch_tocc_fill(const Ctl& h, int slot, int value, cudaStream_t s) {
  const int64_t tiles = h.T * h.U;
  if (value >= 0) cudaMemsetAsync(h.tocc + slot * tiles, value, (size_t)tiles, s);
  else tocc_kernel<<<tile_grid(h), tile_threads(h), 0, s>>>(tile_meta(h), slot);
}

void launch_slot_meta(const Ctl& h, int slot, bool scan_occ, cudaStream_t s) {
  const Slot& sl = h.slot[slot];
  if (scan_occ) {
    uint8_t* ob = reinterpret_cast<uint8_t*>(h.occ + (int64_t)slot * h.nbands * h.nstrips);
    occ_scan_kernel<<<148 * 8, 256, 0, s>>>(sl.X, h.ldx, h.m, h.n, h.nbands, h.ncells, ob, h.nstrips);
  }
  bounds_kernel<<<64, 256, 0, s>>>(sl.p, sl.q, h.m, h.n, h.nbands, h.ncells, h.pmax + (int64_t)slot * h.nbands,
                                   h.qmax + (int64_t)slot * h.ncells);
  launch_tocc_fill(h, slot, -1, s);  // the tile summaries follow the occupancy bytes
}

}  // namespace pdot
