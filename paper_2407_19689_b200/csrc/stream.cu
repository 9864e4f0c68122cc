// Streaming pass over the m x n plan (K1 of every PDHG pass).
//
// One CTA owns a TM x 512 tile.  Lane l of warp w owns the column pair
// j = tile_col0 + 64 w + 2 l and walks the tile's rows, so every warp load and
// store is a fully coalesced 512-byte row segment moved with 128-bit accesses.
// Per element it evaluates the op (the fused PDHG step for OP_STEP) and feeds
// NQ row/column sums plus NS scalar sums:
//   * column sums accumulate in registers over the tile's rows and are written
//     once per tile to colpart[tile_row][q][j];
//   * row sums are reduced across the warp with a transposed butterfly (one
//     shuffle per value), combined across the 8 warps through shared memory in
//     fixed order, and written to rowpart[tile_col][q][i];
//   * scalars are reduced per tile into tilescal[tile_row][tile_col][s].
// No atomics: every partial has a fixed home, every sum a fixed order, so the
// pass is bit-reproducible and independent of CTA scheduling.
//
// Element arithmetic follows the reference expression by expression and the
// library is compiled with -fmad=false, so X+ and the running average are
// bit-identical to numpy given the same (p, q, tau, k):
//   pdhg.py:123-125   X+ = max(0, X - tau*(C - (p_i + q_j)))
//   pdhg.py:125       e  = 2 X+ - X
//   pdhg.py:139       d  = X+ - X
//   pdhg.py:315       A' = A + (X+ - A) / k
//   kkt.py:70-71      viol = max(p_i + q_j - C, 0)
#include "pdot_internal.cuh"

namespace pdot {
namespace {

struct Geo {
  int64_t m, n, ldc, ldx, TM;
  int64_t i0;   // first row of the tile
  int rows;     // rows in this tile
  int64_t j;    // first of this lane's two columns
  bool v0, v1;  // column validity
};

// ---------------------------------------------------------------------------
// OP_STEP: the fused PDHG trial step (+ running average, + KKT dual violation
// of the input iterate and of its running average).
//   quantities: 0 e = 2X+ - X, 1 d = X+ - X, 2 X+, 3 A'
//   scalars:    0 |d|^2, 1 <C,X+>, 2 <C,A'>, 3 |X+|^2, 4 |viol(p,q)|^2, 5 |viol(pa,qa)|^2
// ---------------------------------------------------------------------------
struct StepOp {
  static constexpr int NQ = 4, NS = 6, RB = 2;
  const double* C;
  const double* X;
  const double* A;
  double* Xn;
  double* An;
  const double* p;
  const double* q;
  const double* pa;
  const double* qa;
  double tau, kd;
  bool with_avg;

  struct Col { double q0, q1, qa0, qa1; };
  struct Frag { double2 c, x, a; double p, pa; };

  __device__ __forceinline__ void load_col(Col& cl, const Geo& g) const {
    cl.q0 = g.v0 ? q[g.j] : 0.0;
    cl.q1 = g.v1 ? q[g.j + 1] : 0.0;
    cl.qa0 = g.v0 ? qa[g.j] : 0.0;
    cl.qa1 = g.v1 ? qa[g.j + 1] : 0.0;
  }
  __device__ __forceinline__ void load(Frag& fr, const Geo& g, int64_t i) const {
    fr.c = ld_stream2(C + i * g.ldc + g.j);
    fr.x = ld_stream2(X + i * g.ldx + g.j);
    fr.a = with_avg ? ld_stream2(A + i * g.ldx + g.j) : make_double2(0.0, 0.0);
    fr.p = __ldg(p + i);
    fr.pa = __ldg(pa + i);
  }
  __device__ __forceinline__ void elem(double c, double x, double a, double pi, double qj,
                                       double pai, double qaj, bool valid, double (&o)[NQ],
                                       double (&s)[NS], double& xn_out, double& an_out) const {
    const double pq = pi + qj;                 // apply_At
    const double sres = c - pq;                // C - A^T(p,q)
    const double xn = relu_np(x - tau * sres); // projected primal step
    const double e = 2.0 * xn - x;             // extrapolation
    const double d = xn - x;                   // displacement
    const double an = a + (xn - a) / kd;       // running mean (IEEE division)
    const double vc = relu_np(pq - c);         // dual violation, current (p,q)
    const double va = relu_np((pai + qaj) - c);// dual violation, average (pa,qa)
    if (valid) {
      o[0] = e; o[1] = d; o[2] = xn; o[3] = an;
      s[0] = sqr_acc(s[0], d);
      s[1] = mul_acc(s[1], c, xn);
      s[2] = mul_acc(s[2], c, an);
      s[3] = sqr_acc(s[3], xn);
      s[4] = sqr_acc(s[4], vc);
      s[5] = sqr_acc(s[5], va);
      xn_out = xn; an_out = an;
    } else {
      o[0] = o[1] = o[2] = o[3] = 0.0;
      xn_out = 0.0; an_out = 0.0;
    }
  }
  __device__ __forceinline__ void compute(const Frag& fr, const Geo& g, int64_t i, const Col& cl,
                                          double (&o0)[NQ], double (&o1)[NQ], double (&s)[NS]) const {
    double xa, xb, aa, ab;
    elem(fr.c.x, fr.x.x, fr.a.x, fr.p, cl.q0, fr.pa, cl.qa0, g.v0, o0, s, xa, aa);
    elem(fr.c.y, fr.x.y, fr.a.y, fr.p, cl.q1, fr.pa, cl.qa1, g.v1, o1, s, xb, ab);
    if (g.v0) {
      st_stream2(Xn + i * g.ldx + g.j, make_double2(xa, xb));
      if (with_avg) st_stream2(An + i * g.ldx + g.j, make_double2(aa, ab));
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
    fr.c = C ? ld_stream2(C + i * g.ldc + g.j) : make_double2(0.0, 0.0);
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
    fr.c = (stage == 3) ? ld_stream2(C + i * g.ldc + g.j) : make_double2(0.0, 0.0);
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
// generic tile walker
// ---------------------------------------------------------------------------
template <class Op>
__device__ __forceinline__ void tile_pass(const Op& op, const Ctl& c, double* smem) {
  constexpr int NQ = Op::NQ, NS = Op::NS, RB = Op::RB;
  constexpr int V = RB * NQ;  // values per butterfly (power of two)
  static_assert((V & (V - 1)) == 0 && V <= 32, "RB*NQ must be a power of two <= 32");
  constexpr int NSP = (NS <= 1) ? 1 : (NS <= 2) ? 2 : (NS <= 4) ? 4 : 8;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Geo g;
  g.m = c.m; g.n = c.n; g.ldc = c.ldc; g.ldx = c.ldx; g.TM = c.TM;
  g.i0 = (int64_t)blockIdx.y * c.TM;
  g.rows = (int)imin64(c.TM, c.m - g.i0);
  g.j = (int64_t)blockIdx.x * kTileN + warp * 64 + lane * 2;
  g.v0 = g.j < c.n;
  g.v1 = g.j + 1 < c.n;
  const bool warp_live = ((int64_t)blockIdx.x * kTileN + warp * 64) < c.n;

  double* rowbuf = smem;  // [TM][NQ][kWarps]
  double cacc[NQ][2];
#pragma unroll
  for (int q = 0; q < NQ; ++q) cacc[q][0] = cacc[q][1] = 0.0;
  double sacc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;

  typename Op::Col cl;
  op.load_col(cl, g);

  for (int r0 = 0; r0 < g.rows; r0 += RB) {
    typename Op::Frag fr[RB];
    if (warp_live) {
#pragma unroll
      for (int rr = 0; rr < RB; ++rr)
        if (r0 + rr < g.rows && g.v0) op.load(fr[rr], g, g.i0 + r0 + rr);
    }
    double rv[V];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      double o0[NQ], o1[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
      if (warp_live && r0 + rr < g.rows && g.v0) op.compute(fr[rr], g, g.i0 + r0 + rr, cl, o0, o1, sacc);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        cacc[q][0] += o0[q];
        cacc[q][1] += o1[q];
        rv[rr * NQ + q] = o0[q] + o1[q];
      }
    }
    warp_transpose_sum<V>(rv);
    if (transpose_is_writer<V>(lane)) {
      const int idx = transpose_owner_index<V>(lane);
      const int rr = idx / NQ, q = idx % NQ;
      rowbuf[((r0 + rr) * NQ + q) * kWarps + warp] = rv[0];
    }
  }

  // column partials: one 128-bit store per quantity
  if (g.v0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      *reinterpret_cast<double2*>(c.colpart + ((int64_t)blockIdx.y * NQ + q) * c.ldx + g.j) =
          make_double2(cacc[q][0], cacc[q][1]);
  }

  // scalars: warp butterfly, then fixed-order sum over warps
  double sv[NSP];
#pragma unroll
  for (int s = 0; s < NSP; ++s) sv[s] = (s < NS) ? sacc[s] : 0.0;
  warp_transpose_sum<NSP>(sv);
  double* sbuf = smem + (size_t)c.TM * NQ * kWarps;  // [kWarps][NSP]
  if (transpose_is_writer<NSP>(lane)) sbuf[warp * NSP + transpose_owner_index<NSP>(lane)] = sv[0];
  __syncthreads();

  // row partials: combine the 8 warps in order
  const int nrow_vals = g.rows * NQ;
  for (int e = threadIdx.x; e < nrow_vals; e += kThreads) {
    const double* b = rowbuf + (size_t)e * kWarps;
    double acc = b[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) acc += b[w];
    const int r = e / NQ, q = e % NQ;
    c.rowpart[((int64_t)blockIdx.x * NQ + q) * c.m + g.i0 + r] = acc;
  }
  if (threadIdx.x < NS) {
    double acc = sbuf[threadIdx.x];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) acc += sbuf[w * NSP + threadIdx.x];
    c.tilescal[((int64_t)blockIdx.y * c.U + blockIdx.x) * kMaxNS + threadIdx.x] = acc;
  }
}

__global__ void __launch_bounds__(kThreads, 2) stream_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  extern __shared__ double smem[];
  const Ctl& c = *ctlp;
  if (c.done) return;
  const int op = force_op >= 0 ? force_op : c.op;
  switch (op) {
    case OP_STEP: {
      StepOp o;
      const Slot& sx = c.slot[c.sX];
      const Slot& sa = c.slot[c.sA];
      o.C = c.C; o.X = sx.X; o.A = sa.X;
      o.Xn = c.slot[c.sXn].X; o.An = c.slot[c.sAn].X;
      o.p = sx.p; o.q = sx.q; o.pa = sa.p; o.qa = sa.q;
      o.tau = c.tau; o.kd = c.kd; o.with_avg = !c.unit;
      tile_pass(o, c, smem);
      break;
    }
    case OP_KKT: {
      KktOp o;
      const Slot& sx = c.slot[c.sX];
      o.C = c.C; o.X = sx.X; o.p = c.C ? sx.p : nullptr; o.q = c.C ? sx.q : nullptr;
      o.viol = c.kkt_write_viol ? c.viol_out : nullptr;
      tile_pass(o, c, smem);
      break;
    }
    case OP_DIST: {
      DiffOp o;
      o.Xa = c.slot[c.sZ].X; o.Xb = c.slot[c.sCand].X;
      tile_pass(o, c, smem);
      break;
    }
    case OP_DIFF: {
      DiffOp o;
      o.Xa = c.slot[c.sX].X; o.Xb = c.slot[c.sXn].X;
      tile_pass(o, c, smem);
      break;
    }
    case OP_ROUND: {
      RoundOp o;
      o.C = c.C; o.X = c.slot[c.sX].X;
      o.rs = c.vec_a; o.cs = c.vec_b; o.er = c.vec_a + c.m; o.ec = c.vec_b + c.ldx;
      o.tot = c.out[20]; o.stage = c.round_stage; o.correct = c.out[21] != 0.0;
      o.out = c.viol_out;
      tile_pass(o, c, smem);
      break;
    }
    default:
      break;
  }
}

}  // namespace

size_t stream_smem_bytes(int64_t TM) {
  return (size_t)TM * kMaxNQ * kWarps * sizeof(double) + kWarps * 8 * sizeof(double);
}

void launch_stream_pass(const Ctl* ctl_dev, const Ctl& h, int force_op, cudaStream_t s) {
  static bool attr_set = false;
  const size_t smem = stream_smem_bytes(h.TM);
  if (!attr_set) {
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  dim3 grid((unsigned)h.U, (unsigned)h.T);
  stream_kernel<<<grid, kThreads, smem, s>>>(ctl_dev, force_op);
}

}  // namespace pdot
