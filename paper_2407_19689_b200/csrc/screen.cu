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
//
// Invariant: slot memory always holds the dense values.  occ[slot] marks cells
// whose bits may be nonzero (a superset); a cell with occ = 0 is all +0.0 in
// memory.  K1 therefore writes zeros into an output cell that it does not
// compute only when that cell's old occ bit says it may hold stale data.
//
//   K0 screen_kernel  (one CTA per tile, one thread per (band, strip)):
//       reads min C, dual bounds and occupancy; writes one unit word per
//       (band, strip) (a flag byte per cell), the tile flag, and appends the
//       tile to the visit list when any cell needs work.
//   K1 sparse_kernel  (persistent, 8 warps per CTA, one warp per strip):
//       walks the listed tiles; per band it loads C / X / A only for active
//       cells, runs the same StepOp::elem as the dense walker, stores X+ / A'
//       where nonzero (or stale), updates occupancy and flushes the tile's
//       partials exactly like the dense walker.  Non-STEP ops (start KKT,
//       restart distance, unit calls, rounding) take the generic walker over
//       all tiles.
// K2 (finalize.cu) skips tiles whose flag is 0: their partials are +0.
#include <stdio.h>
#include <stdlib.h>

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
// K0: screening.  One CTA per tile, thread (band, strip) of the tile.
//   STEP: a cell is active when X or the lagged average has a nonzero there,
//         or a dual pair may violate it; stale output cells are flagged ZX/ZA.
//   DIST: active where the candidate or the anchor has a nonzero.
//   KKT:  active where X has a nonzero or the duals may violate.
// Outputs: flag words, the list of cells K1 visits (active or stale), and the
// bit maps K2 reads the cell partials by: bcr (per band and column tile) and
// bct (per row tile and cell).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) screen_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  __shared__ uint32_t tilebits[32];  // per cell of the tile: bit bl = band bl active
  __shared__ unsigned warp_base[8];  // cell-list offsets of the CTA's warps
  unsigned long long* tl = op == OP_STEP ? c.ktl : nullptr;
  tl_start(tl, 0);
  const int64_t tu = blockIdx.x, tt = blockIdx.y;
  const int s = threadIdx.x & 7, bl = threadIdx.x >> 3;  // strip in tile, band in tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 32) tilebits[threadIdx.x] = 0u;
  const bool with_avg = op == OP_STEP && step_with_avg(c);
  const int64_t band = tt * c.nbt + bl;
  const int64_t strip = tu * kWarps + s;
  const bool inband = bl < c.nbt && band < c.nbands;
  const bool valid = inband && strip < c.nstrips;
  uint32_t word = 0;
  if (valid) {
    const int64_t sstride = c.nbands * c.nstrips;
    const int64_t ow = band * c.nstrips + strip;
    // every load of the unit is issued up front (one memory round trip)
    const int sx = op == OP_DIST ? c.sCand : c.sX;
    const uint32_t ox = __ldcg(c.occ + sx * sstride + ow);
    const uint32_t oa = (op == OP_DIST || with_avg) ? __ldcg(c.occ + (op == OP_DIST ? c.sZ : c.sAsrc) * sstride + ow) : 0u;
    const uint32_t zx = op == OP_STEP ? __ldcg(c.occ + c.sXn * sstride + ow) : 0u;
    const uint32_t za = with_avg ? __ldcg(c.occ + c.sA * sstride + ow) : 0u;
    const bool bound = op != OP_DIST;
    const bool bound_avg = op == OP_STEP;
    const double P = bound ? __ldcg(c.pmax + c.sX * c.nbands + band) : 0.0;
    const double Pa = bound_avg ? __ldcg(c.pmax + c.sA * c.nbands + band) : 0.0;
    double mc[kCellsPerStrip], Q[kCellsPerStrip], Qa[kCellsPerStrip];
#pragma unroll
    for (int k = 0; k < kCellsPerStrip; ++k) {
      const int64_t cell = strip * kCellsPerStrip + k;
      const bool ok = bound && cell < c.ncells;
      mc[k] = ok ? __ldcg(c.minc + band * c.ncells + cell) : 0.0;
      Q[k] = ok ? __ldcg(c.qmax + c.sX * c.ncells + cell) : 0.0;
      Qa[k] = (ok && bound_avg) ? __ldcg(c.qmax + c.sA * c.ncells + cell) : 0.0;
    }
    // a non-finite step (tau) would turn 0 * inf into NaN: screen nothing
    const bool open = op == OP_STEP && !isfinite(c.tau);
#pragma unroll
    for (int k = 0; k < kCellsPerStrip; ++k) {
      const int64_t cell = strip * kCellsPerStrip + k;
      if (cell >= c.ncells) break;
      const uint32_t bx = (ox >> (8 * k)) & 0xffu, ba = (oa >> (8 * k)) & 0xffu;
      const uint32_t bzx = (zx >> (8 * k)) & 0xffu, bza = (za >> (8 * k)) & 0xffu;
      // !(a <= b) keeps NaN bounds active
      const bool act = bx || ba || open || (bound && !(P + Q[k] <= mc[k])) ||
                       (bound_avg && !(Pa + Qa[k] <= mc[k]));
      const uint32_t f = (act ? U_ACT : 0u) | (bx ? U_LDX : 0u) | (ba ? U_LDA : 0u) | (bzx ? U_ZX : 0u) |
                         (bza ? U_ZA : 0u);
      word |= f << (8 * k);
    }
    c.unitw[ow] = word;
  }
  // per-cell bits of this thread's strip: listed (any flag) and active (partials)
  uint32_t listed = 0, actb = 0;
#pragma unroll
  for (int k = 0; k < kCellsPerStrip; ++k) {
    const uint32_t f = (word >> (8 * k)) & 0xffu;
    listed |= (f != 0u) << k;
    actb |= ((f & U_ACT) != 0u) << k;
  }
  // CTA-aggregated append of the listed cells: warp scan, one atomic per CTA
  const int cnt = __popc(listed);
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_base[warp] = (unsigned)incl;
  // bcr[band][tu]: bit 4 s + k = cell k of strip s (8 lanes of one band)
  uint32_t rbits = actb << (4 * s);
#pragma unroll
  for (int msk = 1; msk < 8; msk <<= 1) rbits |= __shfl_xor_sync(0xffffffffu, rbits, msk);
  if (s == 0 && inband) c.bcr[band * c.U + tu] = rbits;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    unsigned tot = 0;
    for (int w = 0; w < nw; ++w) {
      const unsigned t = warp_base[w];
      warp_base[w] = tot;
      tot += t;
    }
    const unsigned base = tot ? atomicAdd(c.ucount, tot) : 0u;
    for (int w = 0; w < nw; ++w) warp_base[w] += base;
  }
  // bct[tt][cell]: bit bl = band bl of the tile
#pragma unroll
  for (int k = 0; k < kCellsPerStrip; ++k)
    if ((actb >> k) & 1u) atomicOr(&tilebits[s * kCellsPerStrip + k], 1u << bl);
  const int any = __syncthreads_or(actb != 0u);
  unsigned pos = warp_base[warp] + (unsigned)(incl - cnt);
#pragma unroll
  for (int k = 0; k < kCellsPerStrip; ++k)
    if ((listed >> k) & 1u) c.ulist[pos++] = (uint32_t)((band << 12) | (strip * kCellsPerStrip + k));
  if (threadIdx.x < 32) c.bct[tt * c.ncp + tu * 32 + threadIdx.x] = tilebits[threadIdx.x];
  // the tile's partials are assembled by K1b, or are all +0 (flag 0)
  if (threadIdx.x == 0) {
    c.tileflag[tt * c.U + tu] = any ? 1 : 0;
    if (any) c.tlist[atomicAdd(c.tcount, 1u)] = (int32_t)(tt * c.U + tu);
  }
  tl_end(tl, 0);
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

__device__ __forceinline__ CellGeo cell_geo(const Ctl& c, uint32_t entry) {
  const int lane = threadIdx.x & 31;
  CellGeo g;
  g.band = entry >> 12;
  g.cell = entry & 0xfffu;
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
// row 2 rg + rr, column e; sacc: the lane's stage scalar partials (its two rows,
// element order), so the band partial is (s0 + s1) + (s2 + s3) over the row
// groups (masks 8, 16) and the cell value the 8-lane butterfly on top.
// Partial writes shared by every cell op.  o[rr][q][e]: the lane's outputs for
// row 2 rg + rr, column e; sacc: the lane's stage scalar partials (its two rows,
// element order), so the band partial is (s0 + s1) + (s2 + s3) over the row
// groups (masks 8, 16) and the cell value the 8-lane butterfly on top.
// Partial writes shared by every cell op.  o[rr][q][e]: the lane's outputs for
// row 2 rg + rr, column e; sacc: the lane's stage scalar partials (its two rows,
// element order), so the band partial is (s0 + s1) + (s2 + s3) over the row
// groups (masks 8, 16) and the cell value the 8-lane butterfly on top.  All
// three reductions use transposed butterflies (a few shuffles per value).
template <int NQ, int NS>
__device__ __forceinline__ void cell_flush(const Ctl& c, const CellGeo& g, const double (&o)[2][NQ][2],
                                          const double (&sacc)[NS]) {
  // column band partial: pair sum of the lane's two rows, then masks 8, 16;
  // afterwards lane (rg, cp) holds (x, y) of quantity q(rg) for its column pair
  {
    constexpr int V = 2 * NQ;
    double v[V];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      v[2 * q] = o[0][q][0] + o[1][q][0];
      v[2 * q + 1] = o[0][q][1] + o[1][q][1];
    }
    constexpr int M[2] = {8, 16};
    tsum<V, 2>(v, M);
    const int idx = tsum_index<V, 2>(M);
    if (g.v0) {
      if (NQ == 4) {
        *reinterpret_cast<double2*>(c.ccol + (g.band * kMaxNQ + idx / 2) * c.ldx + g.j) = make_double2(v[0], v[1]);
      } else if (g.rg < 2) {  // NQ == 1: rg 0 holds x, rg 1 holds y
        c.ccol[g.band * kMaxNQ * c.ldx + g.j + idx] = v[0];
      }
    }
  }
  // row values: 8-lane transposed butterfly over the column pairs
  {
    constexpr int V = 2 * NQ;
    double rv[V];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int q = 0; q < NQ; ++q) rv[rr * NQ + q] = o[rr][q][0] + o[rr][q][1];
    warp_transpose_sum<V, 8>(rv);
    if (transpose_is_writer<V, 8>(threadIdx.x & 31)) {
      const int idx = transpose_owner_index<V>(g.cp);
      const int r = 2 * g.rg + idx / NQ, q = idx % NQ;
      DCHECK(g.cell < c.ncp && (r >= g.rows || g.i0 + r < c.mpad), "crow", g.cell, g.i0 + r);
      if (r < g.rows) c.crow[(g.cell * kMaxNQ + q) * c.mpad + g.i0 + r] = rv[0];
    }
  }
  // scalars: stage partials pairwise over the row groups (masks 8, 16), then
  // the column pairs (masks 1, 2, 4)
  {
    constexpr int V = NS <= 1 ? 1 : NS <= 2 ? 2 : NS <= 4 ? 4 : 8;
    double v[V];
#pragma unroll
    for (int s = 0; s < V; ++s) v[s] = s < NS ? sacc[s] : 0.0;
    constexpr int M[5] = {8, 16, 1, 2, 4};
    tsum<V, 5>(v, M);
    const int idx = tsum_index<V, 5>(M);
    // every lane holds the total of index idx; the lanes with cp bits above the
    // routing steps clear write it
    constexpr int lg = log2_pow2<V>();
    const int routed = lg >= 3 ? 1 : 0;  // mask 1 (cp bit 0) routed for V = 8
    if (idx < NS && (g.cp >> routed) == 0)
      c.cscal[(g.band * c.ncp + g.cell) * kMaxNS + idx] = v[0];
  }
}

template <bool IMPLICIT, bool AVG>
__device__ __forceinline__ void cell_step(const StepOp& op, const Ctl& c, const CostGen& gen, uint32_t entry,
                                          unsigned long long& bytes, unsigned long long& cells) {
  constexpr int NQ = StepOp::NQ, NS = StepOp::NS;
  const int lane = threadIdx.x & 31;
  const CellGeo g = cell_geo(c, entry);
  const uint32_t f = (__ldcg(c.unitw + g.band * c.nstrips + g.strip) >> (8 * g.k)) & 0xffu;
  const bool act = (f & U_ACT) != 0;  // cell-uniform
  const bool ldx = act && (f & U_LDX);
  const bool lda = AVG && act && (f & U_LDA);
  const bool zx = (f & U_ZX) != 0;
  const bool za = AVG && (f & U_ZA) != 0;
  if (lane == 0 && act) cells += 1;
  const double2 zero2 = make_double2(0.0, 0.0);
  double2 cc[2], xx[2], aa[2];
  double pr[2], par[2];
  bool okr[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * g.rg + rr;
    okr[rr] = act && r < g.rows && g.v0;
    const int64_t i = g.i0 + r;
    if (IMPLICIT) {
      cc[rr] = zero2;
    } else {
      cc[rr] = okr[rr] ? ld_stream2(op.C + i * c.ldc + g.j) : zero2;
    }
    xx[rr] = (okr[rr] && ldx) ? ld_stream2(op.X + i * c.ldx + g.j) : zero2;
    aa[rr] = (okr[rr] && lda) ? ld_stream2(op.A + i * c.ldx + g.j) : zero2;
    pr[rr] = okr[rr] ? __ldg(op.p + i) : 0.0;
    par[rr] = okr[rr] ? __ldg(op.pa + i) : 0.0;
    if (okr[rr]) bytes += (IMPLICIT ? 0 : 16) + (ldx ? 16 : 0) + (lda ? 16 : 0);
  }
  double qv[2] = {0.0, 0.0}, qav[2] = {0.0, 0.0};
  if (act && g.v0) {
    qv[0] = op.q[g.j]; qav[0] = op.qa[g.j];
    if (g.v1) { qv[1] = op.q[g.j + 1]; qav[1] = op.qa[g.j + 1]; }
  }
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
    const int64_t sstride = c.nbands * c.nstrips;
    uint8_t* ox = reinterpret_cast<uint8_t*>(c.occ + c.sXn * sstride + g.band * c.nstrips + g.strip);
    ox[g.k] = anyx ? 1 : 0;
    if (AVG) {
      uint8_t* oa = reinterpret_cast<uint8_t*>(c.occ + c.sA * sstride + g.band * c.nstrips + g.strip);
      oa[g.k] = anya ? 1 : 0;
    }
  }
  if (act) {
    cell_flush<NQ, NS>(c, g, o, sacc);
    if (lane == 0) bytes += (unsigned long long)(NQ * kCell + NQ * kBand + NS) * 8 * 2;
  }
}

// restart distance (DIST) and the start KKT through the screen (NQ = 1), with
// the dense walkers' per-row compute()
template <class Op>
__device__ __forceinline__ void cell_one(const Op& op, const Ctl& c, uint32_t entry, unsigned long long& bytes,
                                         unsigned long long& cells) {
  constexpr int NQ = Op::NQ, NS = Op::NS;
  const int lane = threadIdx.x & 31;
  const CellGeo cg = cell_geo(c, entry);
  const uint32_t f = (__ldcg(c.unitw + cg.band * c.nstrips + cg.strip) >> (8 * cg.k)) & 0xffu;
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

__global__ void __launch_bounds__(kThreads, kSparseCtasPerSm) unit_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  __shared__ unsigned long long red[2][kWarps];
  if (blockIdx.x == 0 && threadIdx.x == 0) c.sstat[ST_T0] = globaltimer_ns();
  unsigned long long* tl = op == OP_STEP ? c.ktl : nullptr;
  tl_start(tl, 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned ncells = __ldcg(c.ucount);
  const unsigned gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  unsigned long long bytes = 0, cells = 0;
  if (op == OP_STEP) {
    const StepOp o = make_step_op(c);
    CostGen gen;
    gen.kind = c.C ? 0 : c.cost_kind;
    gen.a0 = c.cost_a[0]; gen.a1 = c.cost_a[1]; gen.a2 = c.cost_a[2]; gen.a3 = c.cost_a[3];
    gen.row0 = c.row0;
    for (unsigned k = gw; k < ncells; k += nw) {
      const uint32_t entry = __ldcg(c.ulist + k);
      if (o.C) {
        if (o.with_avg) cell_step<false, true>(o, c, gen, entry, bytes, cells);
        else cell_step<false, false>(o, c, gen, entry, bytes, cells);
      } else {
        if (o.with_avg) cell_step<true, true>(o, c, gen, entry, bytes, cells);
        else cell_step<true, false>(o, c, gen, entry, bytes, cells);
      }
    }
  } else if (op == OP_DIST) {
    DiffOp o;
    o.Xa = c.slot[c.sZ].X; o.Xb = c.slot[c.sCand].X;
    for (unsigned k = gw; k < ncells; k += nw) cell_one(o, c, __ldcg(c.ulist + k), bytes, cells);
  } else {
    KktOp o;
    const Slot& sx = c.slot[c.sX];
    o.C = c.C; o.X = sx.X; o.p = sx.p; o.q = sx.q; o.viol = nullptr;
    for (unsigned k = gw; k < ncells; k += nw) cell_one(o, c, __ldcg(c.ulist + k), bytes, cells);
  }
  // statistics: one atomic per CTA, then the last CTA stamps the end time
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
    __threadfence();
    const unsigned long long done = atomicAdd(&c.sstat[ST_DONE1], 1ull);
    if (done == gridDim.x - 1) {
      const unsigned long long t1 = globaltimer_ns();
      if (op == OP_STEP) {
        c.sstat[ST_K1_NS] += t1 - __ldcg(&c.sstat[ST_T0]);
        c.sstat[ST_TILES] += ncells;
        c.sstat[ST_PASSES] += 1;
        // K0 metadata traffic of this pass: min C + 4 occupancy words + flag word per (band, strip)
        c.sstat[ST_META] += (unsigned long long)c.nbands * c.nstrips * (kCellsPerStrip * 8 + 4 * 4 + 4);
      }
      c.sstat[ST_DONE1] = 0;
    }
  }
  tl_end(tl, 1);
}

// ---------------------------------------------------------------------------
// K1b: assembles the per-tile partials of the canonical tree (the same layout
// the dense walkers write: colpart / rowpart / tilescal) from the cell
// partials, for every tile with an active cell.  One CTA per listed tile:
//   columns: thread = column pair, band-ordered sum of its cell column;
//   rows:    thread = row, strip-ordered sum of the strip values
//            ((c0 + c1) + (c2 + c3)) of the row segment's active cells;
//   scalars: thread (strip, scalar), band-ordered sum of strip-band values,
//            then the strips in order.
// ---------------------------------------------------------------------------
template <int NQ, int NS>
__device__ __forceinline__ void assemble_tile(const Ctl& c, int64_t tu, int64_t tt, double* sm) {
  const int th = threadIdx.x;
  const int64_t b0 = tt * c.nbt;
  {  // columns
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
  for (int r = th; r < c.TM; r += blockDim.x) {  // rows
    const int64_t i = tt * c.TM + r;
    if (i >= c.m) break;
    uint32_t word = __ldg(c.bcr + (i / kBand) * c.U + tu);
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    while (word) {
      const int w = (__ffs(word) - 1) >> 2;  // next active strip, in order
      const unsigned nib = (word >> (4 * w)) & 0xfu;
      word &= ~(0xfu << (4 * w));
      const int64_t cb = tu * 32 + 4 * w;
      double v[4][NQ];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          v[x][q] = ((nib >> x) & 1u) ? __ldg(c.crow + ((cb + x) * kMaxNQ + q) * c.mpad + i) : 0.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] += (v[0][q] + v[1][q]) + (v[2][q] + v[3][q]);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) c.rowpart[(tu * NQ + q) * c.m + i] = acc[q];
  }
  {  // scalars: thread (strip w, band bl) forms its strip-band values (one round
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

__global__ void __launch_bounds__(kThreads) tile_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  __shared__ double sm[32 * 8 * 8];  // [band][strip][scalar] strip-band values
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  const unsigned ntiles = __ldcg(c.tcount);
  unsigned long long* tl = op == OP_STEP ? c.ktl : nullptr;
  tl_start(tl, 2);
  for (unsigned k = blockIdx.x; k < ntiles; k += gridDim.x) {
    const int32_t tile = __ldcg(c.tlist + k);
    const int64_t tu = tile % c.U, tt = tile / c.U;
    if (op == OP_STEP) assemble_tile<4, 6>(c, tu, tt, sm);
    else if (op == OP_DIST) assemble_tile<1, 1>(c, tu, tt, sm);
    else assemble_tile<1, 3>(c, tu, tt, sm);
  }
  tl_end(tl, 2);
}

// the unit calls the screen does not cover (KKT of a unit call, DIFF, ROUND):
// the generic walker over every tile, per-tile partials
__global__ void __launch_bounds__(kThreads, 1) generic_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const Ctl& c = *ctlp;
  if (c.done) return;
  const int op = force_op >= 0 ? force_op : c.op;
  for (int64_t t = blockIdx.x; t < c.T * c.U; t += gridDim.x) {
    generic_tile(op, c, smem, t % c.U, t / c.U);
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
                                int64_t nstrips, uint32_t* __restrict__ list, unsigned* __restrict__ count) {
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
    list[base + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)((band << 12) | cell);
  }
}

__global__ void cell_gather_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, int64_t n,
                                   const uint32_t* __restrict__ list, int64_t k0, int64_t k1,
                                   double* __restrict__ out) {
  // one warp per cell: lane = (row rg, column pair cp) as in the cell kernel
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = k0 + w; k < k1; k += nw) {
    const uint32_t entry = list[k];
    const int64_t band = entry >> 12, cell = entry & 0xfffu;
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
  occ_list_kernel<<<148 * 8, 256, 0, s>>>(ob, h.nbands, h.ncells, h.nstrips, list, count_dev);
  unsigned cnt = 0;
  cudaMemcpyAsync(&cnt, count_dev, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return cnt;
}

void launch_cell_gather(const Ctl& h, int slot, const uint32_t* list, int64_t k0, int64_t k1, double* out,
                        cudaStream_t s) {
  const int64_t warps = k1 - k0;
  const unsigned blocks = (unsigned)imin64((warps * 32 + 255) / 256, 148 * 16);
  if (blocks > 0) cell_gather_kernel<<<blocks, 256, 0, s>>>(h.slot[slot].X, h.ldx, h.m, h.n, list, k0, k1, out);
}

void prepare_sparse_kernel() {
  cudaFuncSetAttribute(generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
}

static size_t generic_smem_bytes(int64_t TM) {
  return (size_t)TM * kMaxNQ * kWarps * sizeof(double) + kWarps * 8 * sizeof(double);
}

void launch_screened_pass(const Ctl* ctl_dev, const Ctl& h, int force_op, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // graph passes (force_op < 0) are STEP / DIST / start-KKT; unit calls choose on the host
  if (force_op < 0 || unit_pass(h, force_op)) {
    dim3 g0((unsigned)h.U, (unsigned)h.T);
    // thread (band, strip) of the tile; at least one full warp (the append and
    // the bit maps use warp shuffles)
    const unsigned threads = (unsigned)(kWarps * h.nbt < 32 ? 32 : kWarps * h.nbt);
    screen_kernel<<<g0, threads, 0, s>>>(ctl_dev, force_op);
    if (getenv("PDOT_DEBUG_SYNC")) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) fprintf(stderr, "screen_kernel failed: %s\n", cudaGetErrorString(e));
    }
    unit_kernel<<<(unsigned)(sms * kSparseCtasPerSm), kThreads, 0, s>>>(ctl_dev, force_op);
    tile_kernel<<<(unsigned)imin64(h.T * h.U, (int64_t)sms * 4), kThreads, 0, s>>>(ctl_dev, force_op);
  } else {
    const unsigned grid = (unsigned)imin64(h.T * h.U, (int64_t)sms * 2);
    generic_kernel<<<grid, kThreads, generic_smem_bytes(h.TM), s>>>(ctl_dev, force_op);
  }
}

void launch_minc_build(const Ctl& h, double* minc, cudaStream_t s) {
  CostGen gen;
  gen.kind = h.C ? 0 : h.cost_kind;
  gen.a0 = h.cost_a[0]; gen.a1 = h.cost_a[1]; gen.a2 = h.cost_a[2]; gen.a3 = h.cost_a[3];
  gen.row0 = h.row0;
  minc_kernel<<<148 * 8, 256, 0, s>>>(h.C, h.ldc, gen, h.m, h.n, h.nbands, h.ncells, minc);
}

void launch_slot_meta(const Ctl& h, int slot, bool scan_occ, cudaStream_t s) {
  const Slot& sl = h.slot[slot];
  if (scan_occ) {
    uint8_t* ob = reinterpret_cast<uint8_t*>(h.occ + (int64_t)slot * h.nbands * h.nstrips);
    occ_scan_kernel<<<148 * 8, 256, 0, s>>>(sl.X, h.ldx, h.m, h.n, h.nbands, h.ncells, ob, h.nstrips);
  }
  bounds_kernel<<<64, 256, 0, s>>>(sl.p, sl.q, h.m, h.n, h.nbands, h.ncells, h.pmax + (int64_t)slot * h.nbands,
                                   h.qmax + (int64_t)slot * h.ncells);
}

}  // namespace pdot
