// Per-element pass operations shared by the dense TMA walker (stream.cu) and the
// block-screened walker (screen.cu): tile geometry, the fused STEP update and
// the rare ops (KKT, distance, rounding), and the per-tile flush of the row,
// column and scalar partials.  See stream.cu for the reduction layout.
//
// Element arithmetic follows the reference expression by expression and the
// library is compiled with -fmad=false, so X+ and the running average are
// bit-identical to numpy given the same (p, q, tau, k):
//   pdhg.py:123-125   X+ = max(0, X - tau*(C - (p_i + q_j)))
//   pdhg.py:125       e  = 2 X+ - X
//   pdhg.py:139       d  = X+ - X
//   pdhg.py:315       A' = A + (X+ - A) / k
//   kkt.py:70-71      viol = max(p_i + q_j - C, 0)
#pragma once

#include "pdot_internal.cuh"

namespace pdot {
namespace {

struct Geo {
  int64_t m, n, ldc, ldx, TM;
  int64_t tu, tt;  // tile column / tile row (local)
  int64_t i0;   // first row of the tile
  int rows;     // rows in this tile
  int64_t j;    // first of this lane's two columns
  bool v0, v1;  // column validity
  CostGen gen;  // implicit cost (gen.kind > 0 when C is generated, not read)
};

// the cost pair (i, j..j+1): streamed from HBM, or generated from coordinates
__device__ __forceinline__ double2 cost_pair(const double* C, const Geo& g, int64_t i) {
  if (C) return ld_stream2(C + i * g.ldc + g.j);
  if (g.gen.kind > 0) {
    const double2 r = g.gen.row_coord(i);
    return make_double2(g.gen.cost(r, g.gen.col_coord(g.j)), g.gen.cost(r, g.gen.col_coord(g.j + 1)));
  }
  return make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// OP_STEP: the fused PDHG trial step (+ running average, + KKT dual violation
// of the input iterate and of its running average).
//   quantities: 0 e = 2X+ - X, 1 d = X+ - X, 2 X+, 3 A'
//   scalars:    0 |d|^2, 1 <C,X+>, 2 <C,A'>, 3 |X+|^2, 4 |viol(p,q)|^2, 5 |viol(pa,qa)|^2
// ---------------------------------------------------------------------------
struct StepOp {
  static constexpr int NQ = 4, NS = 6;
  const double* C;
  const double* X;
  const double* A;
  double* Xn;
  double* An;
  const double* p;
  const double* q;
  const double* pa;
  const double* qa;
  double tau, kd, rkd;
  bool with_avg;  // this pass also writes the (lagged) average matrix

  struct Col { double q0, q1, qa0, qa1; };
  struct Frag { double2 c, x, a; double p, pa; };

  __device__ __forceinline__ void load_col(Col& cl, const Geo& g) const {
    cl.q0 = g.v0 ? q[g.j] : 0.0;
    cl.q1 = g.v1 ? q[g.j + 1] : 0.0;
    cl.qa0 = g.v0 ? qa[g.j] : 0.0;
    cl.qa1 = g.v1 ? qa[g.j + 1] : 0.0;
  }
  // One plan entry.  o = {e, d, X+, A}; s = the six scalar sums.  AVG: this pass
  // also forms the (lagged) running mean of the input iterate; a re-run after a
  // rejected trial does not, and leaves o[3] and s[2] at zero.
  template <bool AVG = true>
  __device__ __forceinline__ void elem(double c, double x, double a, double pi, double qj, double pai,
                                       double qaj, double (&o)[NQ], double (&s)[NS]) const {
    const double pq = pi + qj;                  // apply_At
    const double sres = c - pq;                 // C - A^T(p,q)
    const double xn = relu_np(x - tau * sres);  // projected primal step
    const double d = xn - x;                    // displacement
    const double e = (xn + xn) - x;             // 2 X+ - X  (xn + xn == 2.0*xn exactly)
    const double vc = relu_np(pq - c);          // dual violation, current (p,q)
    const double va = relu_np((pai + qaj) - c); // dual violation, average (pa,qa)
    o[0] = e; o[1] = d; o[2] = xn;
    s[0] = sqr_acc(s[0], d);
    s[1] = mul_acc(s[1], c, xn);
    s[3] = sqr_acc(s[3], xn);
    s[4] = sqr_acc(s[4], vc);
    s[5] = sqr_acc(s[5], va);
    if (AVG) {
      const double an = a + div_by_count(x - a, kd, rkd);  // running mean of the accepted iterate x (lazy)
      o[3] = an;
      s[2] = mul_acc(s[2], c, an);
    } else {
      o[3] = 0.0;
    }
  }
  // masked variant for edge tiles and the unit (no running average) call
  __device__ __forceinline__ void compute(const Frag& fr, const Geo& g, int64_t i, const Col& cl,
                                          double (&o0)[NQ], double (&o1)[NQ], double (&s)[NS]) const {
    if (with_avg) {
      if (g.v0) elem<true>(fr.c.x, fr.x.x, fr.a.x, fr.p, cl.q0, fr.pa, cl.qa0, o0, s);
      if (g.v1) elem<true>(fr.c.y, fr.x.y, fr.a.y, fr.p, cl.q1, fr.pa, cl.qa1, o1, s);
    } else {
      if (g.v0) elem<false>(fr.c.x, fr.x.x, 0.0, fr.p, cl.q0, fr.pa, cl.qa0, o0, s);
      if (g.v1) elem<false>(fr.c.y, fr.x.y, 0.0, fr.p, cl.q1, fr.pa, cl.qa1, o1, s);
    }
    if (g.v0) {
      st_stream2(Xn + i * g.ldx + g.j, make_double2(o0[2], g.v1 ? o1[2] : 0.0));
      if (with_avg) st_stream2(An + i * g.ldx + g.j, make_double2(o0[3], g.v1 ? o1[3] : 0.0));
    }
  }
};

// ---------------------------------------------------------------------------
// OP_KKT: rows/cols of X, <C,X>, |[p+q-C]^+|^2, |X|^2.  C may be null (apply_A).
// Optionally writes the dual-violation matrix (unit kkt_error).
//   quantities: 0 X ; scalars: 0 <C,X>, 1 |viol|^2, 2 |X|^2
// ---------------------------------------------------------------------------
struct KktOp {
  static constexpr int NQ = 1, NS = 3, RB = 8;
  const double* C;
  const double* X;
  const double* p;
  const double* q;
  double* viol;   // optional output (ldx)

  struct Col { double q0, q1; };
  struct Frag { double2 c, x; double p; };

  __device__ __forceinline__ void load_col(Col& cl, const Geo& g) const {
    cl.q0 = (g.v0 && q) ? q[g.j] : 0.0;
    cl.q1 = (g.v1 && q) ? q[g.j + 1] : 0.0;
  }
  __device__ __forceinline__ void load(Frag& fr, const Geo& g, int64_t i) const {
    fr.c = cost_pair(C, g, i);
    fr.x = ld_stream2(X + i * g.ldx + g.j);
    fr.p = p ? __ldg(p + i) : 0.0;
  }
  __device__ __forceinline__ void compute(const Frag& fr, const Geo& g, int64_t i, const Col& cl,
                                          double (&o0)[NQ], double (&o1)[NQ], double (&s)[NS]) const {
    const double v0 = relu_np((fr.p + cl.q0) - fr.c.x);
    const double v1 = relu_np((fr.p + cl.q1) - fr.c.y);
    o0[0] = g.v0 ? fr.x.x : 0.0;
    o1[0] = g.v1 ? fr.x.y : 0.0;
    if (g.v0) {
      s[0] = mul_acc(s[0], fr.c.x, fr.x.x);
      s[1] = sqr_acc(s[1], v0);
      s[2] = sqr_acc(s[2], fr.x.x);
    }
    if (g.v1) {
      s[0] = mul_acc(s[0], fr.c.y, fr.x.y);
      s[1] = sqr_acc(s[1], v1);
      s[2] = sqr_acc(s[2], fr.x.y);
    }
    if (viol && g.v0) st_stream2(viol + i * g.ldx + g.j, make_double2(v0, g.v1 ? v1 : 0.0));
  }
};

// ---------------------------------------------------------------------------
// OP_DIFF / OP_DIST: d = B - A ; rows/cols of d, |d|^2
// ---------------------------------------------------------------------------
struct DiffOp {
  static constexpr int NQ = 1, NS = 1, RB = 8;
  const double* Xa;
  const double* Xb;
  struct Col { int dummy; };
  struct Frag { double2 a, b; };
  __device__ __forceinline__ void load_col(Col&, const Geo&) const {}
  __device__ __forceinline__ void load(Frag& fr, const Geo& g, int64_t i) const {
    fr.a = ld_stream2(Xa + i * g.ldx + g.j);
    fr.b = ld_stream2(Xb + i * g.ldx + g.j);
  }
  __device__ __forceinline__ void compute(const Frag& fr, const Geo& g, int64_t, const Col&,
                                          double (&o0)[NQ], double (&o1)[NQ], double (&s)[NS]) const {
    const double d0 = fr.b.x - fr.a.x;
    const double d1 = fr.b.y - fr.a.y;
    o0[0] = g.v0 ? d0 : 0.0;
    o1[0] = g.v1 ? d1 : 0.0;
    if (g.v0) s[0] = sqr_acc(s[0], d0);
    if (g.v1) s[0] = sqr_acc(s[0], d1);
  }
};

// ---------------------------------------------------------------------------
// OP_ROUND (rounding.py:18-40), three stages over X with row scale rs (vec_a)
// and column scale cs (vec_b):
//   stage 1: Y  = rs_i * X            -> column sums
//   stage 2: Y2 = (rs_i * X) * cs_j   -> row and column sums
//   stage 3: Xf = Y2 + (er_i*ec_j)/tot (tot > 1e-14) -> <C,Xf>, rows/cols, optional write
// rs/cs/er/ec/tot are produced by the finalize kernel between stages.
// ---------------------------------------------------------------------------
struct RoundOp {
  static constexpr int NQ = 1, NS = 1, RB = 8;
  const double* C;
  const double* X;
  const double* rs;
  const double* cs;
  const double* er;
  const double* ec;
  double tot;
  int stage;
  bool correct;
  double* out;
  struct Col { double c0, c1, e0, e1; };
  struct Frag { double2 c, x; double r, e; };
  __device__ __forceinline__ void load_col(Col& cl, const Geo& g) const {
    cl.c0 = (stage >= 2 && g.v0) ? cs[g.j] : 1.0;
    cl.c1 = (stage >= 2 && g.v1) ? cs[g.j + 1] : 1.0;
    cl.e0 = (stage == 3 && g.v0) ? ec[g.j] : 0.0;
    cl.e1 = (stage == 3 && g.v1) ? ec[g.j + 1] : 0.0;
  }
  __device__ __forceinline__ void load(Frag& fr, const Geo& g, int64_t i) const {
    fr.x = ld_stream2(X + i * g.ldx + g.j);
    fr.c = (stage == 3) ? cost_pair(C, g, i) : make_double2(0.0, 0.0);
    fr.r = (stage >= 1) ? __ldg(rs + i) : 1.0;  // stage 0 sums X itself
    fr.e = (stage == 3) ? __ldg(er + i) : 0.0;
  }
  __device__ __forceinline__ double value(double x, double r, double cs_, double e, double ecj) const {
    double y = (stage >= 1) ? r * x : x;
    if (stage >= 2) y = y * cs_;
    if (stage == 3 && correct) y = y + (e * ecj) / tot;
    return y;
  }
  __device__ __forceinline__ void compute(const Frag& fr, const Geo& g, int64_t i, const Col& cl,
                                          double (&o0)[NQ], double (&o1)[NQ], double (&s)[NS]) const {
    const double y0 = value(fr.x.x, fr.r, cl.c0, fr.e, cl.e0);
    const double y1 = value(fr.x.y, fr.r, cl.c1, fr.e, cl.e1);
    o0[0] = g.v0 ? y0 : 0.0;
    o1[0] = g.v1 ? y1 : 0.0;
    if (stage == 3) {
      if (g.v0) s[0] = mul_acc(s[0], fr.c.x, y0);
      if (g.v1) s[0] = mul_acc(s[0], fr.c.y, y1);
      if (out && g.v0) st_stream2(out + i * g.ldx + g.j, make_double2(y0, g.v1 ? y1 : 0.0));
    }
  }
};

// ---------------------------------------------------------------------------
// Canonical reduction tree of a pass.  Every walker reproduces it exactly, so
// the dense TMA walker, the generic walker and the block-screened cell walker
// (screen.cu) give bit-identical partials.  Units: a BAND is 8 rows of a tile,
// a STRIP 64 columns (one warp of the dense walkers, lane = column pair), a
// CELL = band x 16 columns (8 lanes).
//   * column: band partial = ((r0+r1) + (r2+r3)) + ((r4+r5) + (r6+r7)) over
//     the band's rows; tile partial = sum of band partials in band order;
//   * row: lane value o0 + o1; cell value = 8-lane butterfly (masks 1, 2, 4);
//     strip value = (c0 + c1) + (c2 + c3) (masks 8, 16); tile partial = sum of
//     strip values in strip order;
//   * scalar: lane stage partial = sequential over the stage's (2 rows) elements
//     (row 2k col0, col1, row 2k+1 col0, col1) from +0; lane band partial =
//     (s0 + s1) + (s2 + s3); cell value = 8-lane butterfly; strip band value =
//     (c0 + c1) + (c2 + c3); tile scalar = sum over strips of the strip's sum
//     over bands in band order.
// A skipped cell contributes exact +0 terms anywhere in this tree.
// ---------------------------------------------------------------------------
// Band accumulators of the canonical tree, fed once per 2-row STAGE (stage k =
// rows 2k, 2k+1 of the band): column stage sums and the lane's stage scalar
// partials (sequential over the stage's elements from +0) combine as
// (s0 + s1) + (s2 + s3).
template <int NQ, int NS>
struct BandAcc {
  double ca[NQ][2], cb[NQ][2], sa[NS], sb[NS];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int q = 0; q < NQ; ++q) ca[q][0] = ca[q][1] = cb[q][0] = cb[q][1] = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) sa[s] = sb[s] = 0.0;
  }
  // ps = o(row 2k) + o(row 2k+1); sacc = the stage's scalar partials (reset here)
  __device__ __forceinline__ void stage(int k, const double (&ps)[NQ][2], double (&sacc)[NS]) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (k == 0) ca[q][e] = ps[q][e];
        else if (k == 1) ca[q][e] += ps[q][e];
        else if (k == 2) cb[q][e] = ps[q][e];
        else cb[q][e] += ps[q][e];
      }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (k == 0) sa[s] = sacc[s];
      else if (k == 1) sa[s] += sacc[s];
      else if (k == 2) sb[s] = sacc[s];
      else sb[s] += sacc[s];
      sacc[s] = 0.0;
    }
  }
};

// end of a band: band column partial into the tile partial; band scalar
// partials -> warp totals with a transposed butterfly (masks 1..16), lane L
// accumulating the scalar band_scalar_index(L) into ws; reset
template <int NS>
struct ScalPad {
  static constexpr int V = NS <= 1 ? 1 : NS <= 2 ? 2 : NS <= 4 ? 4 : 8;
};
template <int NS>
__device__ __forceinline__ int band_scalar_index() {
  constexpr int M[5] = {1, 2, 4, 8, 16};
  return tsum_index<ScalPad<NS>::V, 5>(M);
}
// lanes holding distinct scalars (the others hold copies)
template <int NS>
__device__ __forceinline__ bool band_scalar_writer() {
  return ((threadIdx.x & 31) >> log2_pow2<ScalPad<NS>::V>()) == 0;
}
template <int NQ, int NS>
__device__ __forceinline__ void band_close(BandAcc<NQ, NS>& ba, double (&cacc)[NQ][2], double& ws) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    cacc[q][0] += ba.ca[q][0] + ba.cb[q][0];
    cacc[q][1] += ba.ca[q][1] + ba.cb[q][1];
  }
  constexpr int V = ScalPad<NS>::V;
  constexpr int M[5] = {1, 2, 4, 8, 16};
  double v[V];
#pragma unroll
  for (int s = 0; s < V; ++s) v[s] = s < NS ? ba.sa[s] + ba.sb[s] : 0.0;
  tsum<V, 5>(v, M);
  ws += v[0];
  ba.reset();
}

// per-tile flush shared by the walkers: column partials (registers -> global),
// scalars (warp totals -> fixed-order sum over warps), row partials (per-warp
// smem entries -> fixed-order sum over warps).
template <int NQ, int NS>
__device__ __forceinline__ void tile_flush(const Ctl& c, const Geo& g, bool worker, double (&cacc)[NQ][2],
                                           double ws, double* rowbuf, double* sbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (worker && g.v0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      *reinterpret_cast<double2*>(c.colpart + (g.tt * NQ + q) * c.ldx + g.j) =
          make_double2(cacc[q][0], cacc[q][1]);
  }
  if (worker && band_scalar_writer<NS>()) {
    const int s = band_scalar_index<NS>();
    if (s < NS) sbuf[warp * 8 + s] = ws;
  }
  __syncthreads();
  const int nrow_vals = g.rows * NQ;
  for (int e = threadIdx.x; e < nrow_vals; e += blockDim.x) {
    const double* b = rowbuf + (size_t)e * kWarps;
    double acc = b[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) acc += b[w];
    const int r = e / NQ, q = e % NQ;
    c.rowpart[(g.tu * NQ + q) * c.m + g.i0 + r] = acc;
  }
  if (threadIdx.x < NS) {
    double acc = sbuf[threadIdx.x];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) acc += sbuf[w * 8 + threadIdx.x];
    c.tilescal[(g.tt * c.U + g.tu) * kMaxNS + threadIdx.x] = acc;
  }
  if (threadIdx.x == 0 && c.tileflag) c.tileflag[g.tt * c.U + g.tu] = 1;
}

__device__ __forceinline__ Geo make_geo(const Ctl& c, bool worker, int64_t tu, int64_t tt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Geo g;
  g.m = c.m; g.n = c.n; g.ldc = c.ldc; g.ldx = c.ldx; g.TM = c.TM;
  g.tu = tu;
  g.tt = tt;
  g.i0 = tt * c.TM;
  g.rows = (int)imin64(c.TM, c.m - g.i0);
  g.j = tu * kTileN + warp * 64 + lane * 2;
  g.v0 = worker && g.j < c.n;
  g.v1 = worker && g.j + 1 < c.n;
  g.gen.kind = c.C ? 0 : c.cost_kind;
  g.gen.a0 = c.cost_a[0]; g.gen.a1 = c.cost_a[1]; g.gen.a2 = c.cost_a[2]; g.gen.a3 = c.cost_a[3];
  g.gen.row0 = c.row0;
  return g;
}

// row values of one batch -> warp butterfly -> this warp's smem row partials
template <int NQ, int RB>
__device__ __forceinline__ void push_rows(double (&rv)[RB * NQ], double* rowbuf, int r0, bool worker) {
  constexpr int V = RB * NQ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_transpose_sum<V>(rv);
  if (worker && transpose_is_writer<V>(lane)) {
    const int idx = transpose_owner_index<V>(lane);
    const int rr = idx / NQ, q = idx % NQ;
    rowbuf[((r0 + rr) * NQ + q) * kWarps + warp] = rv[0];
  }
}

// ---------------------------------------------------------------------------
// generic walker: direct 128-bit loads (all ops; the rare ones use it)
// ---------------------------------------------------------------------------
template <class Op>
__device__ __forceinline__ void tile_pass(const Op& op, const Ctl& c, double* smem, int64_t tu, int64_t tt) {
  constexpr int NQ = Op::NQ, NS = Op::NS, RB = Op::RB;
  constexpr int V = RB * NQ;
  static_assert((V & (V - 1)) == 0 && V <= 32, "RB*NQ must be a power of two <= 32");
  static_assert(RB == kBand, "one batch of the generic walker is one band");
  const int warp = threadIdx.x >> 5;
  const bool worker = warp < kWarps;
  const Geo g = make_geo(c, worker, tu, tt);
  double* rowbuf = smem;                              // [TM][NQ][kWarps]
  double* sbuf = smem + (size_t)c.TM * NQ * kWarps;   // [kWarps][8]
  double cacc[NQ][2];
#pragma unroll
  for (int q = 0; q < NQ; ++q) cacc[q][0] = cacc[q][1] = 0.0;
  BandAcc<NQ, NS> bacc;
  bacc.reset();
  double sacc[NS], ws = 0.0;
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
  typename Op::Col cl;
  if (worker) op.load_col(cl, g);

  for (int r0 = 0; r0 < g.rows; r0 += RB) {
    typename Op::Frag fr[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr)
      if (r0 + rr < g.rows && g.v0) op.load(fr[rr], g, g.i0 + r0 + rr);
    double rv[V];
    double st[NQ][2];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      double o0[NQ], o1[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
      if (r0 + rr < g.rows && g.v0) op.compute(fr[rr], g, g.i0 + r0 + rr, cl, o0, o1, sacc);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (rr & 1) {
          st[q][0] += o0[q];
          st[q][1] += o1[q];
        } else {
          st[q][0] = o0[q];
          st[q][1] = o1[q];
        }
        rv[rr * NQ + q] = o0[q] + o1[q];
      }
      if (rr & 1) bacc.stage(rr >> 1, st, sacc);
    }
    push_rows<NQ, RB>(rv, rowbuf, r0, worker);
    band_close<NQ, NS>(bacc, cacc, ws);
  }
  tile_flush<NQ, NS>(c, g, worker, cacc, ws, rowbuf, sbuf);
}

// ---------------------------------------------------------------------------
// op construction from the control block (shared by both walkers)
// ---------------------------------------------------------------------------
__device__ __forceinline__ StepOp make_step_op(const Ctl& c) {
  StepOp o;
  const Slot& sx = c.slot[c.sX];
  const Slot& sa = c.slot[c.sA];
  o.C = c.C; o.X = sx.X;
  o.A = c.slot[c.sAsrc].X;   // previous average matrix (lazy update input)
  o.An = sa.X;               // average matrix of the current iterate (output)
  o.Xn = c.slot[c.sXn].X;
  o.p = sx.p; o.q = sx.q; o.pa = sa.p; o.qa = sa.q;
  o.tau = c.tau; o.kd = c.kd; o.rkd = c.rkd;
  o.with_avg = c.unit ? c.unit_avg != 0 : c.lagA != 0;
  return o;
}

// the rare ops through the direct-load walker, for tile (tu, tt)
__device__ __forceinline__ void generic_tile(int op, const Ctl& c, double* smem, int64_t tu, int64_t tt) {
  switch (op) {
    case OP_KKT: {
      KktOp o;
      const Slot& sx = c.slot[c.sX];
      const bool has_cost = c.C != nullptr || c.cost_kind > 0;
      o.C = c.C; o.X = sx.X; o.p = has_cost ? sx.p : nullptr; o.q = has_cost ? sx.q : nullptr;
      o.viol = c.kkt_write_viol ? c.viol_out : nullptr;
      tile_pass(o, c, smem, tu, tt);
      break;
    }
    case OP_DIST: {
      DiffOp o;
      o.Xa = c.slot[c.sZ].X; o.Xb = c.slot[c.sCand].X;
      tile_pass(o, c, smem, tu, tt);
      break;
    }
    case OP_DIFF: {
      DiffOp o;
      o.Xa = c.slot[c.sX].X; o.Xb = c.slot[c.sXn].X;
      tile_pass(o, c, smem, tu, tt);
      break;
    }
    case OP_ROUND: {
      RoundOp o;
      o.C = c.C; o.X = c.slot[c.sX].X;
      o.rs = c.vec_a; o.cs = c.vec_b; o.er = c.vec_a + c.m; o.ec = c.vec_b + c.ldx;
      o.tot = c.out[OUT_ROUND_TOTAL]; o.stage = c.round_stage; o.correct = c.out[OUT_ROUND_CORRECT] != 0.0;
      o.out = c.viol_out;
      tile_pass(o, c, smem, tu, tt);
      break;
    }
    default:
      break;
  }
}

}  // namespace
}  // namespace pdot
