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
#include "pass_ops.cuh"

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
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) screen_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  const int64_t tu = blockIdx.x, tt = blockIdx.y;
  const int s = threadIdx.x & 7, bl = threadIdx.x >> 3;  // strip in tile, band in tile
  const int lane = threadIdx.x & 31;
  const bool with_avg = op == OP_STEP && step_with_avg(c);
  const int64_t band = tt * c.nbt + bl;
  const int64_t strip = tu * kWarps + s;
  const bool valid = bl < c.nbt && band < c.nbands && strip < c.nstrips;
  uint32_t word = 0;
  if (valid) {
    const int64_t sstride = c.nbands * c.nstrips;
    const int64_t ow = band * c.nstrips + strip;
    uint32_t ox = 0, oa = 0, zx = 0, za = 0;
    double P = -INFINITY, Pa = -INFINITY;
    bool bound = false;
    if (op == OP_STEP) {
      ox = __ldcg(c.occ + c.sX * sstride + ow);
      oa = with_avg ? __ldcg(c.occ + c.sAsrc * sstride + ow) : 0u;
      zx = __ldcg(c.occ + c.sXn * sstride + ow);
      za = with_avg ? __ldcg(c.occ + c.sA * sstride + ow) : 0u;
      P = __ldcg(c.pmax + c.sX * c.nbands + band);
      Pa = __ldcg(c.pmax + c.sA * c.nbands + band);
      bound = true;
    } else if (op == OP_DIST) {
      ox = __ldcg(c.occ + c.sCand * sstride + ow);  // X_b = candidate
      oa = __ldcg(c.occ + c.sZ * sstride + ow);     // X_a = anchor
    } else {  // OP_KKT of slot sX
      ox = __ldcg(c.occ + c.sX * sstride + ow);
      P = __ldcg(c.pmax + c.sX * c.nbands + band);
      bound = true;
    }
    // a non-finite step (tau) would turn 0 * inf into NaN: screen nothing
    const bool open = op == OP_STEP && !isfinite(c.tau);
#pragma unroll
    for (int k = 0; k < kCellsPerStrip; ++k) {
      const int64_t cell = strip * kCellsPerStrip + k;
      if (cell >= c.ncells) break;
      const uint32_t bx = (ox >> (8 * k)) & 0xffu, ba = (oa >> (8 * k)) & 0xffu;
      const uint32_t bzx = (zx >> (8 * k)) & 0xffu, bza = (za >> (8 * k)) & 0xffu;
      bool act = bx || ba || open;
      if (bound && !act) {
        const double mc = __ldcg(c.minc + band * c.ncells + cell);
        const double Q = __ldcg(c.qmax + c.sX * c.ncells + cell);
        // !(a <= b) keeps NaN bounds active
        act = !(P + Q <= mc);
        if (op == OP_STEP && !act) {
          const double Qa = __ldcg(c.qmax + c.sA * c.ncells + cell);
          act = !(Pa + Qa <= mc);
        }
      }
      const uint32_t f = (act ? U_ACT : 0u) | (bx ? U_LDX : 0u) | (ba ? U_LDA : 0u) | (bzx ? U_ZX : 0u) |
                         (bza ? U_ZA : 0u);
      word |= f << (8 * k);
    }
    c.unitw[ow] = word;
    if (word) c.ulist[atomicAdd(c.ucount, 1u)] = (uint32_t)ow;
  }
  const bool parts = (word & 0x01010101u) != 0;  // the unit writes partials
  if (parts) atomicOr(c.ubc + strip * c.nbw + (band >> 5), 1u << (band & 31));
  const unsigned bal = __ballot_sync(0xffffffffu, parts);
  // byte (band, tile column): bit s = strip 8 tu + s wrote partials
  if (s == 0 && bl < c.nbt && band < c.nbands) c.ubr[band * c.U + tu] = (uint8_t)((bal >> (lane & 24)) & 0xffu);
}

// ---------------------------------------------------------------------------
// K1: one warp per listed unit (8 rows x 64 columns; lane = column pair).
// ---------------------------------------------------------------------------
struct UnitGeo {
  int64_t band, strip, i0, j;
  int rows;
  bool v0, v1;
};

__device__ __forceinline__ UnitGeo unit_geo(const Ctl& c, uint32_t unit) {
  const int lane = threadIdx.x & 31;
  UnitGeo u;
  u.band = unit / c.nstrips;
  u.strip = unit - u.band * c.nstrips;
  u.i0 = u.band * kBand;
  u.rows = (int)imin64(kBand, c.m - u.i0);
  u.j = u.strip * kStrip + lane * 2;
  u.v0 = u.j < c.n;
  u.v1 = u.j + 1 < c.n;
  return u;
}

// unit row partials of RB rows starting at r0: per-row strip butterflies
template <int NQ, int RB>
__device__ __forceinline__ void unit_rows(const Ctl& c, const UnitGeo& u, double (&rv)[RB * NQ], int r0) {
  const int lane = threadIdx.x & 31;
  constexpr int V = RB * NQ;
  warp_transpose_sum<V>(rv);
  if (transpose_is_writer<V>(lane)) {
    const int idx = transpose_owner_index<V>(lane);
    const int r = r0 + idx / NQ, q = idx % NQ;
    if (r < u.rows) c.urow[(u.strip * kMaxNQ + q) * c.mpad + u.i0 + r] = rv[0];
  }
}

// unit column partials (band partial of the canonical tree) and scalars (band butterfly)
template <int NQ, int NS>
__device__ __forceinline__ void unit_flush(const Ctl& c, const UnitGeo& u, const double (&bacc)[NQ][2],
                                          double (&sacc)[NS]) {
  const int lane = threadIdx.x & 31;
  if (u.v0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      *reinterpret_cast<double2*>(c.ucol + (u.band * kMaxNQ + q) * c.ldx + u.j) = make_double2(bacc[q][0], bacc[q][1]);
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    double x = sacc[s];
#pragma unroll
    for (int msk = 16; msk >= 1; msk >>= 1) x += __shfl_xor_sync(0xffffffffu, x, msk);
    sacc[s] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) c.uscal[(u.band * c.nstrips + u.strip) * kMaxNS + s] = sacc[s];
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// One STEP unit.  Every lane copies its own column pair of the active rows of
// C, X and A into this warp's shared buffer with cp.async (all copies in
// flight at once, no registers held), then computes from shared memory.
template <bool IMPLICIT, bool AVG>
__device__ __forceinline__ void unit_step(const StepOp& op, const Ctl& c, const CostGen& gen, uint32_t unit,
                                          double2* wbuf, unsigned long long& bytes, unsigned long long& cells) {
  constexpr int NQ = StepOp::NQ, NS = StepOp::NS, H = kBand / 2;
  const int lane = threadIdx.x & 31;
  const UnitGeo u = unit_geo(c, unit);
  const uint32_t w = __ldcg(c.unitw + unit);
  const uint32_t cb = (w >> ((lane >> 3) * 8)) & 0xffu;
  const bool act = (cb & U_ACT) && u.v0;
  const bool ldx = act && (cb & U_LDX);
  const bool lda = AVG && act && (cb & U_LDA);
  const bool zx = (cb & U_ZX) && u.v0;
  const bool za = AVG && (cb & U_ZA) && u.v0;
  if ((lane & 7) == 0 && (cb & U_ACT)) cells += 1;
  double2* bc = wbuf + lane;                 // [3][kBand][32] double2, this lane's column
  if (act) {
#pragma unroll
    for (int r = 0; r < kBand; ++r) {
      if (r < u.rows) {
        const int64_t i = u.i0 + r;
        if (!IMPLICIT) cp_async16(bc + (0 * kBand + r) * 32, op.C + i * c.ldc + u.j);
        if (ldx) cp_async16(bc + (1 * kBand + r) * 32, op.X + i * c.ldx + u.j);
        if (lda) cp_async16(bc + (2 * kBand + r) * 32, op.A + i * c.ldx + u.j);
      }
    }
    bytes += (unsigned long long)u.rows * ((IMPLICIT ? 0 : 16) + (ldx ? 16 : 0) + (lda ? 16 : 0));
  }
  const double2 zero2 = make_double2(0.0, 0.0);
  // duals: this lane's columns, and the band's rows broadcast from lanes 0..7
  double q0 = 0.0, q1 = 0.0, qa0 = 0.0, qa1 = 0.0;
  if (act) {
    q0 = op.q[u.j]; qa0 = op.qa[u.j];
    if (u.v1) { q1 = op.q[u.j + 1]; qa1 = op.qa[u.j + 1]; }
  }
  const bool prow = lane < u.rows;
  const double pl = prow ? __ldg(op.p + u.i0 + lane) : 0.0;
  const double pal = prow ? __ldg(op.pa + u.i0 + lane) : 0.0;
  double2 cj0 = zero2, cj1 = zero2;
  if (IMPLICIT) {
    cj0 = gen.col_coord(u.j);
    cj1 = gen.col_coord(u.j + 1);
  }
  double bacc[NQ][2];
#pragma unroll
  for (int q = 0; q < NQ; ++q) bacc[q][0] = bacc[q][1] = 0.0;
  double sacc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
  const bool parts = (w & 0x01010101u) != 0;  // warp-uniform: the unit writes partials
  bool nzx = false, nza = false;
  cp_async_wait_all();  // each lane reads back only what it copied itself
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    double rv[H * NQ];
#pragma unroll
    for (int rr = 0; rr < H; ++rr) {
      const int r = h * H + rr;
      const bool inrow = r < u.rows;
      const bool ok = act && inrow;
      const int64_t i = u.i0 + r;
      const double pi = __shfl_sync(0xffffffffu, pl, r), pai = __shfl_sync(0xffffffffu, pal, r);
      double o0[NQ], o1[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
      if (ok) {
        double2 cc;
        if (IMPLICIT) {
          const double2 rc = gen.row_coord(i);
          cc = make_double2(gen.cost(rc, cj0), gen.cost(rc, cj1));
        } else {
          cc = bc[(0 * kBand + r) * 32];
        }
        const double2 xx = ldx ? bc[(1 * kBand + r) * 32] : zero2;
        const double2 aa = lda ? bc[(2 * kBand + r) * 32] : zero2;
        op.template elem<AVG>(cc.x, xx.x, aa.x, pi, q0, pai, qa0, o0, sacc);
        if (u.v1) op.template elem<AVG>(cc.y, xx.y, aa.y, pi, q1, pai, qa1, o1, sacc);
      }
      const double2 xo = make_double2(o0[2], o1[2]);
      const bool nzr = nz2(xo);
      nzx |= nzr;
      if (inrow && (ok ? (zx || nzr) : zx)) {
        st_stream2(op.Xn + i * c.ldx + u.j, xo);
        bytes += 16;
      }
      if (AVG) {
        const double2 ao = make_double2(o0[3], o1[3]);
        const bool nar = nz2(ao);
        nza |= nar;
        if (inrow && (ok ? (za || nar) : za)) {
          st_stream2(op.An + i * c.ldx + u.j, ao);
          bytes += 16;
        }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        bacc[q][0] += o0[q];
        bacc[q][1] += o1[q];
        rv[rr * NQ + q] = o0[q] + o1[q];
      }
    }
    if (parts) unit_rows<NQ, H>(c, u, rv, h * H);
  }
  __syncwarp();  // the buffer is reused by this warp's next unit
  // occupancy of the unit's 4 output cells (bit patterns, so -0.0 counts)
  const unsigned mx = __ballot_sync(0xffffffffu, nzx);
  const unsigned ma = __ballot_sync(0xffffffffu, nza);
  if (lane == 0) {
    uint32_t wx = 0, wa = 0;
#pragma unroll
    for (int k = 0; k < kCellsPerStrip; ++k) {
      wx |= ((mx >> (8 * k)) & 0xffu) ? (1u << (8 * k)) : 0u;
      wa |= ((ma >> (8 * k)) & 0xffu) ? (1u << (8 * k)) : 0u;
    }
    const int64_t sstride = c.nbands * c.nstrips;
    c.occ[c.sXn * sstride + unit] = wx;
    if (AVG) c.occ[c.sA * sstride + unit] = wa;
  }
  if (parts) {
    unit_flush<NQ, NS>(c, u, bacc, sacc);
    if (lane == 0) bytes += (unsigned long long)(2 * NQ * kStrip + NQ * kBand + NS) * 8;
  }
}

// the NQ = 1 ops through the screen: restart distance and the start KKT
template <class Op>
__device__ __noinline__ void unit_generic(const Op& op, const Ctl& c, uint32_t unit, unsigned long long& bytes,
                                          unsigned long long& cells) {
  constexpr int NQ = Op::NQ, NS = Op::NS;
  static_assert(NQ == 1 && Op::RB == kBand, "unit_generic handles the one-quantity ops");
  const int lane = threadIdx.x & 31;
  const UnitGeo u = unit_geo(c, unit);
  const uint32_t w = __ldcg(c.unitw + unit);
  const uint32_t cb = (w >> ((lane >> 3) * 8)) & 0xffu;
  const bool act = (cb & U_ACT) && u.v0;
  if ((lane & 7) == 0 && (cb & U_ACT)) cells += 1;
  Geo g;  // the fields the ops read
  g.m = c.m; g.n = c.n; g.ldc = c.ldc; g.ldx = c.ldx; g.TM = c.TM;
  g.tu = 0; g.tt = 0; g.i0 = u.i0; g.rows = u.rows; g.j = u.j;
  g.v0 = act;
  g.v1 = act && u.v1;
  g.gen.kind = c.C ? 0 : c.cost_kind;
  g.gen.a0 = c.cost_a[0]; g.gen.a1 = c.cost_a[1]; g.gen.a2 = c.cost_a[2]; g.gen.a3 = c.cost_a[3];
  g.gen.row0 = c.row0;
  typename Op::Col cl;
  op.load_col(cl, g);
  typename Op::Frag fr[kBand];
#pragma unroll
  for (int r = 0; r < kBand; ++r)
    if (act && r < u.rows) op.load(fr[r], g, u.i0 + r);
  double bacc[NQ][2] = {{0.0, 0.0}};
  double sacc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
  double rv[kBand * NQ];
#pragma unroll
  for (int r = 0; r < kBand; ++r) {
    double o0[NQ] = {0.0}, o1[NQ] = {0.0};
    if (act && r < u.rows) op.compute(fr[r], g, u.i0 + r, cl, o0, o1, sacc);
    bacc[0][0] += o0[0];
    bacc[0][1] += o1[0];
    rv[r] = o0[0] + o1[0];
  }
  if (act) bytes += 32 * (unsigned long long)u.rows;
  if (w & 0x01010101u) {
    unit_rows<NQ, kBand>(c, u, rv, 0);
    unit_flush<NQ, NS>(c, u, bacc, sacc);
  }
}

__global__ void __launch_bounds__(kThreads, kSparseCtasPerSm) unit_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (!unit_pass(c, op)) return;
  __shared__ unsigned long long red[2][kWarps];
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (blockIdx.x == 0 && threadIdx.x == 0) c.sstat[ST_T0] = globaltimer_ns();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned nunits = __ldcg(c.ucount);
  const unsigned gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  unsigned long long bytes = 0, cells = 0;
  if (op == OP_STEP) {
    const StepOp o = make_step_op(c);
    CostGen gen;
    gen.kind = c.C ? 0 : c.cost_kind;
    gen.a0 = c.cost_a[0]; gen.a1 = c.cost_a[1]; gen.a2 = c.cost_a[2]; gen.a3 = c.cost_a[3];
    gen.row0 = c.row0;
    double2* wbuf = reinterpret_cast<double2*>(smem_raw) + warp * (3 * kBand * 32);
    for (unsigned k = gw; k < nunits; k += nw) {
      const uint32_t unit = __ldcg(c.ulist + k);
      if (o.C) {
        if (o.with_avg) unit_step<false, true>(o, c, gen, unit, wbuf, bytes, cells);
        else unit_step<false, false>(o, c, gen, unit, wbuf, bytes, cells);
      } else {
        if (o.with_avg) unit_step<true, true>(o, c, gen, unit, wbuf, bytes, cells);
        else unit_step<true, false>(o, c, gen, unit, wbuf, bytes, cells);
      }
    }
  } else if (op == OP_DIST) {
    DiffOp o;
    o.Xa = c.slot[c.sZ].X; o.Xb = c.slot[c.sCand].X;
    for (unsigned k = gw; k < nunits; k += nw) unit_generic(o, c, __ldcg(c.ulist + k), bytes, cells);
  } else {
    KktOp o;
    const Slot& sx = c.slot[c.sX];
    o.C = c.C; o.X = sx.X; o.p = sx.p; o.q = sx.q; o.viol = nullptr;
    for (unsigned k = gw; k < nunits; k += nw) unit_generic(o, c, __ldcg(c.ulist + k), bytes, cells);
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
        c.sstat[ST_TILES] += nunits;
        c.sstat[ST_PASSES] += 1;
        // K0 metadata traffic of this pass: min C + 4 occupancy words + unit word per (band, strip)
        c.sstat[ST_META] += (unsigned long long)c.nbands * c.nstrips * (kCellsPerStrip * 8 + 4 * 4 + 4);
      }
      c.sstat[ST_DONE1] = 0;
    }
  }
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

}  // namespace

constexpr size_t kUnitSmem = (size_t)kWarps * 3 * kBand * 32 * sizeof(double2);  // 96 KB

void prepare_sparse_kernel() {
  cudaFuncSetAttribute(generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUnitSmem);
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
    screen_kernel<<<g0, (unsigned)(kWarps * h.nbt), 0, s>>>(ctl_dev, force_op);
    unit_kernel<<<(unsigned)(sms * kSparseCtasPerSm), kThreads, kUnitSmem, s>>>(ctl_dev, force_op);
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
