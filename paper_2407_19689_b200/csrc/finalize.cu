// Finalize kernel (K2 of every pass) and the device-side controller.
//
// Blocks [0, CB) reduce the column partials of 64 columns each; blocks
// [CB, CB+T) reduce the row partials of one row tile each.  Both then apply
// the O(m+n) vector updates of the pass (p+ / q+, the dual running average,
// the KKT primal residuals, ...) and write per-block scalar partials.  The
// last block to finish (ticket counter) reduces those in a fixed order and
// runs the controller: the restart / termination / line-search logic of
// pdhg.py:298-378 on the device, so the host never waits on an iteration.
//
// Reduction order is fixed: the T row tiles are cut into kGroups=8 contiguous
// groups, summed sequentially inside a group and pairwise across groups.  A
// row-sharded multi-GPU run owning whole groups reproduces the same tree.
#include <math.h>
#include <stdio.h>

#include "pdot_internal.cuh"

namespace pdot {
namespace {

constexpr int kColsPerBlock = 128;  // two 64-column halves per lane pair set

// fixed-order block sum of K per-thread values; result valid in thread 0
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red /* [kWarps][K] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int msk = 16; msk >= 1; msk >>= 1) x += __shfl_xor_sync(0xffffffffu, x, msk);
    v[k] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < K) {  // value k summed over the warps in order by thread k
    double acc = red[threadIdx.x];
    for (int w = 1; w < kWarps; ++w) acc += red[w * K + threadIdx.x];
    red[kWarps * K + threadIdx.x] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = red[kWarps * K + k];
  }
  __syncthreads();
}

// sum of count values at p[0], p[stride], ... in order; loads issued 8 at a time
__device__ __forceinline__ double seq_sum(const double* p, int64_t stride, int64_t count) {
  double acc = 0.0;
  for (int64_t k0 = 0; k0 < count; k0 += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (k0 + k < count) ? __ldcg(p + (k0 + k) * stride) : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k0 + k < count) acc += v[k];
  }
  return acc;
}

__device__ __forceinline__ double pair8(const double* g) {
  return ((g[0] + g[1]) + (g[2] + g[3])) + ((g[4] + g[5]) + (g[6] + g[7]));
}

// ---------------------------------------------------------------------------
// peer-memory exchange (c.p2p): per-exchange parity buffers + sequence flags
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long* xcounter(const Ctl& c) {
  return reinterpret_cast<unsigned long long*>(c.xpeer[c.rank] + 2 * (size_t)kGroups * c.gstride) +
         2 * kMaxRanks;
}
__device__ __forceinline__ int64_t xseq_next(const Ctl& c) { return (int64_t)__ldcg(xcounter(c)) + 1; }
__device__ __forceinline__ int xparity(const Ctl& c) { return (int)(xseq_next(c) & 1); }
__device__ __forceinline__ double* xgroups(const Ctl& c, int r) {
  return c.xpeer[r] + (size_t)xparity(c) * kGroups * c.gstride;
}
__device__ __forceinline__ unsigned long long* xflag(const Ctl& c, int r_owner, int r_src) {
  unsigned long long* f = reinterpret_cast<unsigned long long*>(c.xpeer[r_owner] + 2 * (size_t)kGroups * c.gstride);
  return f + xparity(c) * kMaxRanks + r_src;
}
// the group buffer K2b combines: the local exchange buffer of this parity, or gbuf
__device__ __forceinline__ const double* combine_groups(const Ctl& c) {
  return c.p2p ? xgroups(c, c.rank) : c.gbuf;
}
// group partial store: into every rank's buffer (p2p) or the local gbuf
__device__ __forceinline__ void store_group2(const Ctl& c, int64_t off, double2 v) {
  if (c.p2p) {
    for (int r = 0; r < c.nranks; ++r) *reinterpret_cast<double2*>(xgroups(c, r) + off) = v;
  } else {
    *reinterpret_cast<double2*>(c.gbuf + off) = v;
  }
}
__device__ __forceinline__ void store_group1(const Ctl& c, int64_t off, double v) {
  if (c.p2p) {
    for (int r = 0; r < c.nranks; ++r) xgroups(c, r)[off] = v;
  } else {
    c.gbuf[off] = v;
  }
}
// K2a tail: after every group store of this rank (each block fenced at system
// scope), release this exchange's sequence number into every rank's flag word
// for this sender.  Called by one thread.
__device__ __forceinline__ void publish_exchange(const Ctl& c) {
  __threadfence_system();
  const unsigned long long seq = (unsigned long long)xseq_next(c);
  for (int r = 0; r < c.nranks; ++r)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(xflag(c, r, c.rank)), "l"(seq) : "memory");
}
// K2b tail: this exchange is consumed (the same count on every rank)
__device__ __forceinline__ void consume_exchange(const Ctl& c) { *xcounter(c) += 1ull; }

// K2b: wait until every rank has published this exchange (bounded spin)
__device__ void wait_exchange(Ctl& c) {
  if (threadIdx.x == 0) {
    const int64_t want = xseq_next(c);
    const uint64_t t0 = globaltimer_ns();
    for (int r = 0; r < c.nranks; ++r) {
      unsigned long long v;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(xflag(c, c.rank, r)) : "memory");
        if ((int64_t)v >= want) break;
        if (globaltimer_ns() - t0 > 20000000000ull) {  // 20 s: a rank is gone; fail instead of hanging
          atomicExch(&c.xerror, 1);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// column blocks
// ---------------------------------------------------------------------------
// Sum of the column partials of reduction group g over its row tiles, in tile
// order: the within-group order that every GPU count reproduces.
// the flags of up to 32 consecutive tiles (stride apart) as a bit mask
__device__ __forceinline__ uint32_t flag_mask(const uint8_t* f, int64_t stride, int64_t count) {
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < count && __ldg(f + k * stride)) m |= 1u << k;
  return m;
}

// the same mask, formed cooperatively: lane k loads flag k, one ballot (every
// lane of the warp must be active and pass the same arguments)
__device__ __forceinline__ uint32_t warp_flag_mask(const uint8_t* f, int64_t stride, int64_t count) {
  const int lane = threadIdx.x & 31;
  return __ballot_sync(0xffffffffu, lane < count && __ldg(f + lane * stride) != 0);
}

// A lane owns two column pairs of the block: j and j + kColsPerBlock / 2.
constexpr int kHalfCols = 64;
constexpr int kColBatch = 2;  // flagged tiles per round trip (register budget: 2 x 2 x NQ double2;
                              // 3 per round trip: no gain, 4: K2 +2.3 us, spills)

// The work blocks' fixed geometry (set once per handle) as a KERNEL PARAMETER:
// constant-bank operands in the tile-partial loops instead of shared-memory
// loads of the control block.  The same member names as Ctl, so the loops are
// templates over the view (the rare ops pass the control block itself).
struct FGeo {
  int64_t m, n, ldx, T, U, TM, GS, t0, Tg, ncells, nbands, ncolblk;
  const uint8_t* tileflag;
  const double* colpart;
  const double* rowpart;
  const double* tilescal;
  double* rowblk;
  double* colblk;
  double* qmax;
  double* pmax;
  double* sdq;
  double* sdp;
};

template <int NQ, class Cx>
__device__ __forceinline__ void group_column_sum(const Cx& c, int g, int64_t j, double2 (&acc)[2][NQ],
                                                 uint32_t m0 = 0u, bool has_m0 = false) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[h][q] = make_double2(0.0, 0.0);
  const int64_t ta = imax64((int64_t)g * c.GS, c.t0);
  const int64_t tb = imin64(imin64((int64_t)(g + 1) * c.GS, c.Tg), c.t0 + c.T);
  // tiles whose flag is 0 were screened out entirely: their partials are +0;
  // the flags are read first (one per lane, a ballot: the block's columns share
  // their column tile), then the partials of the flagged tiles kColBatch at a time
  const uint8_t* flags = c.tileflag + (imin64(j, c.n - 1) / kTileN);
  const bool v0 = j < c.n, v1 = j + kHalfCols < c.n;
  for (int64_t tc = ta; tc < tb; tc += 32) {
    // (m0: the first 32 flags, read by the caller before waiting for K1b)
    uint32_t m = (has_m0 && tc == ta) ? m0 : warp_flag_mask(flags + (tc - c.t0) * c.U, c.U, tb - tc);
    if (!v0) m = 0u;
    while (m) {
      int tk[kColBatch];
      int cnt = 0;
#pragma unroll
      for (int e = 0; e < kColBatch; ++e) {
        tk[e] = 0;
        if (m) {
          tk[e] = __ffs(m) - 1;
          m &= m - 1;
          cnt = e + 1;
        }
      }
      double2 v[kColBatch][2][NQ];
#pragma unroll
      for (int e = 0; e < kColBatch; ++e)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const double* p = c.colpart + ((tc + tk[e] - c.t0) * NQ + q) * c.ldx + j;
          v[e][0][q] = e < cnt ? __ldcg(reinterpret_cast<const double2*>(p)) : make_double2(0.0, 0.0);
          v[e][1][q] = (e < cnt && v1) ? __ldcg(reinterpret_cast<const double2*>(p + kHalfCols)) : make_double2(0.0, 0.0);
        }
#pragma unroll
      for (int e = 0; e < kColBatch; ++e)
        if (e < cnt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              acc[h][q].x += v[e][h][q].x;
              acc[h][q].y += v[e][h][q].y;
            }
    }
  }
}

// FIN_A: this shard's groups -> gbuf[g][q][j]
template <int NQ>
__device__ void column_group_partials(const Ctl& c, int b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = c.g0 + warp;
  if (g < c.g1) {
    const int64_t j = (int64_t)b * kColsPerBlock + lane * 2;
    double2 acc[2][NQ];
    group_column_sum<NQ>(c, g, j, acc);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (j + h * kHalfCols < c.n) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) store_group2(c, g * c.gstride + q * c.ldx + j + h * kHalfCols, acc[h][q]);
      }
  }
}

// Full column sums = pairwise combination of the 8 group sums (FIN_FUSED: the
// groups are computed here; FIN_B: they come from the exchange buffer).
template <int NQ, class Cx>
__device__ void column_sums(const Ctl& c, const Cx& gx, int b, double (&col)[NQ], int64_t& j_out, double* smem,
                            int mode, uint32_t m0 = 0u, bool has_m0 = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jj = threadIdx.x;
  j_out = (int64_t)b * kColsPerBlock + jj;
  if (mode == FIN_B) {
    if (jj < kColsPerBlock && j_out < c.n) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double g8[kGroups];
#pragma unroll
        for (int gi = 0; gi < kGroups; ++gi) g8[gi] = __ldcg(combine_groups(c) + gi * c.gstride + q * c.ldx + j_out);
        col[q] = pair8(g8);
      }
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q) col[q] = 0.0;
    }
    return;
  }
  const int64_t j = (int64_t)b * kColsPerBlock + lane * 2;
  double2 acc[2][NQ];
  group_column_sum<NQ>(gx, warp, j, acc, m0, has_m0);
  // smem [group][q][kColsPerBlock]
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      smem[(warp * NQ + q) * kColsPerBlock + h * kHalfCols + lane * 2] = acc[h][q].x;
      smem[(warp * NQ + q) * kColsPerBlock + h * kHalfCols + lane * 2 + 1] = acc[h][q].y;
    }
  __syncthreads();
  if (jj < kColsPerBlock) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double g8[kGroups];
#pragma unroll
      for (int gi = 0; gi < kGroups; ++gi) g8[gi] = smem[(gi * NQ + q) * kColsPerBlock + jj];
      col[q] = pair8(g8);
    }
  } else {
#pragma unroll
    for (int q = 0; q < NQ; ++q) col[q] = 0.0;
  }
  __syncthreads();
}

template <int NQ, class Cx>
__device__ void row_sums(const Cx& c, int64_t i, double (&row)[NQ], uint32_t m0 = 0u, bool has_m0 = false) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) row[q] = 0.0;
  // screened-out tiles: partials +0.  A full warp of rows of one row tile
  // forms the flag mask with one ballot; otherwise each thread reads the flags.
  const bool full = __activemask() == 0xffffffffu && c.TM % 32 == 0;
  const uint8_t* flags = c.tileflag + (imin64(i, c.m - 1) / c.TM) * c.U;
  for (int64_t uc = 0; uc < c.U; uc += 32) {
    uint32_t m = (has_m0 && uc == 0) ? m0
                 : full ? warp_flag_mask(flags + uc, 1, c.U - uc)
                        : (i < c.m ? flag_mask(flags + uc, 1, c.U - uc) : 0u);
    if (i >= c.m) m = 0u;
    while (m) {
      int uk[4];
      int cnt = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uk[e] = 0;
        if (m) {
          uk[e] = __ffs(m) - 1;
          m &= m - 1;
          cnt = e + 1;
        }
      }
      double v[4][NQ];
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[e][q] = e < cnt ? __ldcg(c.rowpart + ((uc + uk[e]) * NQ + q) * c.m + i) : 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < cnt)
#pragma unroll
          for (int q = 0; q < NQ; ++q) row[q] += v[e][q];
    }
  }
}

// STEP: the hot path of every screened pass, compiled on its own (the rare ops
// sit out of line in column_block_rare) so that its code is compact
template <bool STEP, class Gx>
__device__ __forceinline__ void column_block_t(Ctl& c, const Gx& gx, int op, int b, double* smem, int mode) {
  double vals[kMaxColScal];
#pragma unroll
  for (int s = 0; s < kMaxColScal; ++s) vals[s] = 0.0;
  int64_t j;
  if constexpr (STEP) {
    // the vectors of this thread's column, loaded before the (long) column sums
    const int64_t jp = (int64_t)b * kColsPerBlock + threadIdx.x;
    const bool own = threadIdx.x < kColsPerBlock && jp < gx.n;
    const double qj = own ? __ldcg(c.slot[c.sX].q + jp) : 0.0;
    const double gj = own ? __ldg(c.g + jp) : 0.0;
    const double qaj = own ? __ldcg(c.slot[c.sA].q + jp) : 0.0;
    const bool srec = c.sr_on && !c.unit;  // slack certificates: this cell's drift counter
    const double dq_old = (srec && own && (threadIdx.x & (kCell - 1)) == 0) ? __ldcg(gx.sdq + jp / kCell) : 0.0;
    // this warp's group's tile flags: K0 wrote them, so they are read before the wait too
    uint32_t m0 = 0u;
    const bool has_m0 = mode == FIN_FUSED;
    if (has_m0) {
      const int g = threadIdx.x >> 5;
      const int64_t ta = imax64((int64_t)g * gx.GS, gx.t0);
      const int64_t tb = imin64(imin64((int64_t)(g + 1) * gx.GS, gx.Tg), gx.t0 + gx.T);
      const int64_t jl = (int64_t)b * kColsPerBlock + (threadIdx.x & 31) * 2;
      m0 = warp_flag_mask(gx.tileflag + (imin64(jl, gx.n - 1) / kTileN) + (ta - gx.t0) * gx.U, gx.U, tb - ta);
    }
    pdl_wait();  // (a programmatic dependent of K1b: its partials from here on; a no-op otherwise)
    double col[4];
    column_sums<4>(c, gx, b, col, j, smem, mode, m0, has_m0);
    double qb = -INFINITY, qab = -INFINITY;  // screening bounds of q+ and the dual average
    double qdr = 0.0;                           // their drift (rounded up)
    if (threadIdx.x < kColsPerBlock && j < gx.n) {
      const double qn = qj + c.sigma * (gj - col[0]);        // pdhg.py:128
      const double dq = qn - qj;                              // pdhg.py:141
      c.slot[c.sXn].q[j] = qn;
      qb = qn;
      if (srec) qdr = absdiff_ru(qn, qj);
      vals[0] = dq * dq;
      vals[1] = dq * col[1];
      const double pcx = col[2] - gj;                         // kkt.py:69
      vals[2] = pcx * pcx;
      vals[4] = gj * qn;
      vals[6] = qn * qn;
      if (!c.unit || c.unit_avg) {
        const double qan = qaj + div_by_count(qn - qaj, c.kd_dual, c.rkd_dual);  // pdhg.py:317
        c.slot[c.sAn].q[j] = qan;
        qab = qan;
        if (srec) qdr = max_nan(qdr, absdiff_ru(qan, qaj));
        const double pca = col[3] - gj;
        vals[3] = pca * pca;
        vals[5] = gj * qan;
      }
    }
    if (threadIdx.x < kColsPerBlock) {  // NaN-propagating maxima over each 16-column cell
      const int lane = threadIdx.x & 31;
      const unsigned gm = 0xffffu << (lane & 16);
#pragma unroll
      for (int msk = 1; msk < kCell; msk <<= 1) {
        qb = max_nan(qb, __shfl_xor_sync(gm, qb, msk));
        qab = max_nan(qab, __shfl_xor_sync(gm, qab, msk));
        if (srec) qdr = max_nan(qdr, __shfl_xor_sync(gm, qdr, msk));
      }
      const int64_t cell = ((int64_t)b * kColsPerBlock + threadIdx.x) / kCell;
      if ((threadIdx.x & (kCell - 1)) == 0 && cell < gx.ncells) {
        gx.qmax[c.sXn * gx.ncells + cell] = qb;
        if (!c.unit || c.unit_avg) gx.qmax[c.sAn * gx.ncells + cell] = qab;
        if (srec) gx.sdq[cell] = __dadd_ru(dq_old, qdr);
      }
    }
  } else if (op == OP_KKT) {
    double col[1];
    column_sums<1>(c, gx, b, col, j, smem, mode);
    if (threadIdx.x < kColsPerBlock && j < gx.n) {
      c.cols_out[j] = col[0];
      if (c.C || c.cost_kind > 0) {
        const Slot& sx = c.slot[c.sX];
        const double qj = sx.q[j], gj = c.g[j];
        const double pc = col[0] - gj;
        vals[0] = pc * pc;
        vals[1] = gj * qj;
        vals[2] = qj * qj;
      }
    }
  } else if (op == OP_DIFF || op == OP_DIST) {
    double col[1];
    column_sums<1>(c, gx, b, col, j, smem, mode);
    if (threadIdx.x < kColsPerBlock && j < gx.n) {
      c.cols_out[j] = col[0];
      const double* qa = (op == OP_DIFF) ? c.slot[c.sX].q : c.slot[c.sZ].q;
      const double* qb = (op == OP_DIFF) ? c.slot[c.sXn].q : c.slot[c.sCand].q;
      const double dq = qb[j] - qa[j];
      vals[0] = dq * dq;
      vals[1] = dq * col[0];
    }
  } else if (op == OP_ROUND) {
    double col[1];
    column_sums<1>(c, gx, b, col, j, smem, mode);
    if (threadIdx.x < kColsPerBlock && j < gx.n) {
      c.cols_out[j] = col[0];
      const double gj = c.g[j];
      if (c.round_stage == 1) {                       // rounding.py:26-28
        c.vec_b[j] = col[0] > 0.0 ? fmin(gj / col[0], 1.0) : 1.0;
      } else if (c.round_stage == 2) {                // rounding.py:34
        const double e = gj - col[0];
        c.vec_b[gx.ldx + j] = e < 0.0 ? 0.0 : e;
      } else if (c.round_stage == 3) {
        vals[0] = gj * c.slot[c.sX].q[j];             // dual objective, pdhg.py:384
        const double pc = col[0] - gj;
        vals[1] = fabs(pc);
      }
    }
  }
  // one scalar partial per 64-column half (the unit of the column-side scalar
  // order): half h = the in-order sum over the 8 warp slots of warps 2h, 2h + 1
  // (the other slots +0), as a 64-column block formed it
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kMaxColScal; ++k) {
      double x = vals[k];
#pragma unroll
      for (int msk = 16; msk >= 1; msk >>= 1) x += __shfl_xor_sync(0xffffffffu, x, msk);
      if (lane == 0) smem[warp * kMaxColScal + k] = x;
    }
    __syncthreads();
    if (threadIdx.x < 2 * kMaxColScal) {
      const int h = threadIdx.x / kMaxColScal, k = threadIdx.x % kMaxColScal;
      double acc = smem[(2 * h) * kMaxColScal + k];
      for (int w = 1; w < kWarps; ++w) acc += (w < 2) ? smem[(2 * h + w) * kMaxColScal + k] : 0.0;
      if ((int64_t)b * 2 + h < gx.ncolblk) gx.colblk[((int64_t)b * 2 + h) * kMaxColScal + k] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// row blocks (one per row tile)
// ---------------------------------------------------------------------------
// Tile scalars of row tile t (sum over its column tiles, in order; screened-out
// tiles are +0), by one warp: the flag masks by ballot, then lanes < ns sum.
template <class Cx>
__device__ __forceinline__ void tile_scalars(const Cx& c, int t, int ns, int nr, int lane, uint32_t m0 = 0u,
                                             bool has_m0 = false) {
  const int tx = lane;
  const uint8_t* flags = c.tileflag + (int64_t)t * c.U;
  double acc = 0.0;
  for (int64_t uc = 0; uc < c.U; uc += 32) {
    uint32_t m = (has_m0 && uc == 0) ? m0 : warp_flag_mask(flags + uc, 1, c.U - uc);
    if (tx >= ns) m = 0u;
    while (m) {
      int uk[8];
      int cnt = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        uk[e] = 0;
        if (m) {
          uk[e] = __ffs(m) - 1;
          m &= m - 1;
          cnt = e + 1;
        }
      }
      double v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        v[e] = e < cnt ? __ldcg(c.tilescal + ((int64_t)t * c.U + uc + uk[e]) * kMaxNS + tx) : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < cnt) acc += v[e];
    }
  }
  if (tx < ns) c.rowblk[(int64_t)t * kMaxRowScal + nr + tx] = acc;
}

template <bool STEP, class Gx>
__device__ __forceinline__ void row_block_t(Ctl& c, const Gx& gx, int op, int t, double* smem) {
  double vals[kMaxRowScal];
#pragma unroll
  for (int s = 0; s < kMaxRowScal; ++s) vals[s] = 0.0;
  const int64_t i0 = (int64_t)t * gx.TM;
  const int rows = (int)imin64(gx.TM, gx.m - i0);
  // row-side scalars / tile scalars of this op
  const int nr = op == OP_STEP ? 7 : op == OP_KKT ? 3 : op == OP_ROUND ? 3 : 2;
  const int ns = op == OP_STEP ? 6 : op == OP_KKT ? 3 : 1;
  // with rows for at most 7 warps, the last warp forms the tile scalars while the
  // others work on the rows (otherwise warp 0 does after them)
  const bool scal_early = gx.TM <= kRedThreads - 32;
  if (scal_early && threadIdx.x >= kRedThreads - 32) {
    const uint32_t m0 = warp_flag_mask(gx.tileflag + (int64_t)t * gx.U, 1, gx.U);  // K0's flags, before the wait
    pdl_wait();
    tile_scalars(gx, t, ns, nr, threadIdx.x & 31, m0, true);
  }
  for (int r = threadIdx.x; r < gx.TM; r += kRedThreads) {
    const int64_t i = i0 + r;
    const bool ok = r < rows;
    if constexpr (STEP) {
      // the vectors of this row, loaded before the (long) row sums
      const double pi = ok ? __ldcg(c.slot[c.sX].p + i) : 0.0;
      const double fi = ok ? __ldg(c.f + i) : 0.0;
      const double pai = ok ? __ldcg(c.slot[c.sA].p + i) : 0.0;
      const bool srec = c.sr_on && !c.unit;  // slack certificates: this band's drift counter
      const double dp_old = (srec && ok && (r & (kBand - 1)) == 0) ? __ldcg(gx.sdp + i / kBand) : 0.0;
      // the row tile's first 32 flags (K0's) before the wait, as row_sums forms them
      const int64_t ir = ok ? i : gx.m;
      const bool fullw = __activemask() == 0xffffffffu && gx.TM % 32 == 0;
      const uint8_t* fl = gx.tileflag + (imin64(ir, gx.m - 1) / gx.TM) * gx.U;
      const uint32_t m0 = fullw ? warp_flag_mask(fl, 1, gx.U) : (ir < gx.m ? flag_mask(fl, 1, gx.U) : 0u);
      pdl_wait();
      double row[4];
      row_sums<4>(gx, ir, row, m0, true);
      double pb = -INFINITY, pab = -INFINITY;  // screening bounds of p+ and the dual average
      double pdr = 0.0;                           // their drift (rounded up)
      if (ok) {
        const double pn = pi + c.sigma * (fi - row[0]);       // pdhg.py:127
        const double dp = pn - pi;                             // pdhg.py:140
        c.slot[c.sXn].p[i] = pn;
        pb = pn;
        if (srec) pdr = absdiff_ru(pn, pi);
        vals[0] += dp * dp;
        vals[1] += dp * row[1];
        const double prx = row[2] - fi;                        // kkt.py:68
        vals[2] += prx * prx;
        vals[4] += fi * pn;
        vals[6] += pn * pn;
        if (!c.unit || c.unit_avg) {
          const double pan = pai + div_by_count(pn - pai, c.kd_dual, c.rkd_dual);  // pdhg.py:316
          c.slot[c.sAn].p[i] = pan;
          pab = pan;
          if (srec) pdr = max_nan(pdr, absdiff_ru(pan, pai));
          const double pra = row[3] - fi;
          vals[3] += pra * pra;
          vals[5] += fi * pan;
        }
      }
      {  // NaN-propagating maxima over each 8-row band (TM is a multiple of 8)
        const int lane = threadIdx.x & 31;
        const unsigned gm = 0xffu << (lane & 24);
#pragma unroll
        for (int msk = 1; msk < kBand; msk <<= 1) {
          pb = max_nan(pb, __shfl_xor_sync(gm, pb, msk));
          pab = max_nan(pab, __shfl_xor_sync(gm, pab, msk));
          if (srec) pdr = max_nan(pdr, __shfl_xor_sync(gm, pdr, msk));
        }
        const int64_t band = i / kBand;
        if ((r & (kBand - 1)) == 0 && band < gx.nbands) {
          gx.pmax[c.sXn * gx.nbands + band] = pb;
          if (!c.unit || c.unit_avg) gx.pmax[c.sAn * gx.nbands + band] = pab;
          if (srec) gx.sdp[band] = __dadd_ru(dp_old, pdr);
        }
      }
    } else if (op == OP_KKT) {
      double row[1];
      row_sums<1>(c, ok ? i : gx.m, row);
      if (ok) {
        c.rows_out[i] = row[0];
        if (c.C || c.cost_kind > 0) {
          const double pi = c.slot[c.sX].p[i], fi = c.f[i];
          const double pr = row[0] - fi;
          vals[0] += pr * pr;
          vals[1] += fi * pi;
          vals[2] += pi * pi;
        }
      }
    } else if (op == OP_DIFF || op == OP_DIST) {
      double row[1];
      row_sums<1>(c, ok ? i : gx.m, row);
      if (ok) {
        c.rows_out[i] = row[0];
        const double* pa = (op == OP_DIFF) ? c.slot[c.sX].p : c.slot[c.sZ].p;
        const double* pb = (op == OP_DIFF) ? c.slot[c.sXn].p : c.slot[c.sCand].p;
        const double dp = pb[i] - pa[i];
        vals[0] += dp * dp;
        vals[1] += dp * row[0];
      }
    } else if (op == OP_ROUND) {
      double row[1];
      row_sums<1>(c, ok ? i : gx.m, row);
      if (ok) {
        c.rows_out[i] = row[0];
        const double fi = c.f[i];
        if (c.round_stage == 0) {                                  // rounding.py:21-24
          c.vec_a[i] = row[0] > 0.0 ? fmin(fi / row[0], 1.0) : 1.0;
        } else if (c.round_stage == 2) {                           // rounding.py:33-35
          const double e = fi - row[0];
          const double er = e < 0.0 ? 0.0 : e;
          c.vec_a[gx.m + i] = er;
          vals[0] += er;
        } else if (c.round_stage == 3) {
          vals[1] += fi * c.slot[c.sX].p[i];
          vals[2] += fabs(row[0] - fi);
        }
      }
    }
  }
  block_sum<kMaxRowScal>(vals, smem);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nr; ++s) gx.rowblk[(int64_t)t * kMaxRowScal + s] = vals[s];
  }
  if (!scal_early && threadIdx.x < 32) {
    pdl_wait();
    tile_scalars(gx, t, ns, nr, threadIdx.x);
  }
}

__device__ __noinline__ void column_block_rare(Ctl& c, int op, int b, double* smem, int mode) {
  column_block_t<false>(c, c, op, b, smem, mode);
}
__device__ __noinline__ void row_block_rare(Ctl& c, int op, int t, double* smem) { row_block_t<false>(c, c, op, t, smem); }

// ---------------------------------------------------------------------------
// controller
// ---------------------------------------------------------------------------
struct Sums {
  double R[kMaxRowScal];  // row side (+ tile scalars): pairwise over the 8 groups
  double K[kMaxColScal];  // column side, over column blocks
  int stop_any;           // a time-limit stop requested on any rank
};

// Row-side scalar s of reduction group g: the group's row tiles split in two
// halves, each summed in tile order, then added.  Shards compute this for
// their own groups (FIN_A); the single-GPU path computes it for all 8.
__device__ __forceinline__ double group_row_scalar(const Ctl& c, int s, int g, int half) {
  const int64_t ga = (int64_t)g * c.GS, gb = imin64((int64_t)(g + 1) * c.GS, c.Tg);
  const int64_t mid = ga + (imax64(gb - ga, 0) + 1) / 2;
  const int64_t a = half ? mid : ga, e = half ? gb : mid;
  return seq_sum(c.rowblk + (a - c.t0) * kMaxRowScal + s, kMaxRowScal, imax64(e - a, 0));
}

__device__ __forceinline__ bool local_stop(const Ctl& c) {
  return c.stop_request || (c.deadline_ns != 0 && globaltimer_ns() > c.deadline_ns);
}

// FIN_A last block: this shard's group scalars (+ its stop vote) -> gbuf
__device__ void group_scalar_partials(Ctl& c) {
  const int tid = threadIdx.x;
  const int s = tid >> 3, gi = tid & 7;
  const int g = c.g0 + gi;
  if (s < kMaxRowScal && g < c.g1) {
    double v = group_row_scalar(c, s, g, 0) + group_row_scalar(c, s, g, 1);
    if (s == kMaxRowScal - 1) v = (g == c.g0 && local_stop(c)) ? 1.0 : 0.0;
    store_group1(c, g * c.gstride + 4 * c.ldx + s, v);
  }
  if (c.p2p) {  // publish after every block's stores (each fenced at system scope before its ticket)
    __syncthreads();
    if (threadIdx.x == 0) publish_exchange(c);
  }
}

// The controller's reduction of the block partials.  Every load is issued
// first and each warp instruction reads whole lines: on the row side warp g
// holds group g (lane = (half, scalar)), on the column side lane = (part,
// scalar).  The order of the additions is fixed: a row group is
// half0 + half1 of in-order tile sums and the groups combine by pair8; a
// column scalar adds its 32 in-order part sums in order.
__device__ __noinline__ void reduce_blocks(const Ctl& c, Sums* S, double* smem, int mode) {
  static_assert(kGroups == kRedThreads / 32 && kMaxRowScal == 16, "row side: warp per group, lane = (half, scalar)");
  static_assert(kMaxColScal == 8 && kRedThreads == 32 * kMaxColScal, "column side: 32 parts x 8 scalars");
  const int tid = threadIdx.x, lane = tid & 31;
  double* gsum = smem;                         // [kGroups][16] row group values
  double* psum = smem + kGroups * kMaxRowScal; // [32][8] column part sums
  const double* rp = nullptr;
  int64_t rcnt = 0;
  if (mode == FIN_FUSED) {
    const int g = tid >> 5, rh = lane >> 4, rs = lane & 15;
    const int64_t ga = (int64_t)g * c.GS, gb = imin64((int64_t)(g + 1) * c.GS, c.Tg);
    const int64_t mid = ga + (imax64(gb - ga, 0) + 1) / 2;
    const int64_t a = rh ? mid : ga, e = rh ? gb : mid;
    rp = c.rowblk + (a - c.t0) * kMaxRowScal + rs;
    rcnt = imax64(e - a, 0);
  }
  const int cs_ = tid & 7, cw = tid >> 3;
  const int64_t per = (c.ncolblk + 31) / 32;
  const int64_t b0 = cw * per, b1 = imin64(c.ncolblk, b0 + per);
  const double* cp = c.colblk + b0 * kMaxColScal + cs_;
  const int64_t ccnt = imax64(b1 - b0, 0);
  double racc = 0.0, cacc = 0.0;
  for (int64_t k0 = 0; k0 < imax64(rcnt, ccnt); k0 += 8) {
    double va[8], vb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      va[k] = (k0 + k < rcnt) ? __ldcg(rp + (k0 + k) * kMaxRowScal) : 0.0;
      vb[k] = (k0 + k < ccnt) ? __ldcg(cp + (k0 + k) * kMaxColScal) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k0 + k < rcnt) racc += va[k];
      if (k0 + k < ccnt) cacc += vb[k];
    }
  }
  if (mode == FIN_FUSED) {
    racc += __shfl_xor_sync(0xffffffffu, racc, 16);  // half0 + half1
    if (lane < 16) gsum[(tid >> 5) * kMaxRowScal + lane] = racc;
  }
  psum[cw * kMaxColScal + cs_] = cacc;
  __syncthreads();
  if (mode == FIN_FUSED && tid < kMaxRowScal) {
    double g8[kGroups];
#pragma unroll
    for (int g = 0; g < kGroups; ++g) g8[g] = gsum[g * kMaxRowScal + tid];
    S->R[tid] = pair8(g8);
  }
  if (tid >= 32 && tid < 32 + kMaxColScal) {
    const int s = tid - 32;
    double v[32];
#pragma unroll
    for (int w = 0; w < 32; ++w) v[w] = psum[w * kMaxColScal + s];
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < 32; ++w) tot += v[w];
    S->K[s] = tot;
  }
  if (mode == FIN_B && tid >= 64 && tid < 64 + kMaxRowScal) {
    const int s = tid - 64;
    double g8[kGroups];
    for (int g = 0; g < kGroups; ++g) g8[g] = __ldcg(combine_groups(c) + g * c.gstride + 4 * c.ldx + s);
    S->R[s] = pair8(g8);
  }
  if (tid == 96) {
    if (mode == FIN_B) {
      double any = 0.0;
      for (int g = 0; g < kGroups; ++g) any += __ldcg(combine_groups(c) + g * c.gstride + 4 * c.ldx + kMaxRowScal - 1);
      S->stop_any = any > 0.0;
    } else {
      S->stop_any = local_stop(c);
    }
  }
  __syncthreads();
}

__device__ void ring_push(Ctl& c, int type, int ia, double x, double y, double z) {
  if (!c.ring) return;
  Event* e = c.ring + (c.ring_head & (kRingCap - 1));
  e->type = type;
  e->ia = ia;
  e->x = x;
  e->y = y;
  e->z = z;
  c.ring_head += 1;
}

// kkt.py:79-85: returns the configured metric, *rel = relative composite
__device__ double kkt_metric(const Ctl& c, double psq, double dsq, double pobj, double dobj, double* rel) {
  const double gap = pobj - dobj;
  const double gr = gap / c.scale_R;
  const double comp = sqrt(psq + dsq + gr * gr);
  const double r = sqrt(psq) / (1.0 + c.marg_norm) + sqrt(dsq) / (1.0 + c.cost_fro) +
                   fabs(gap) / (1.0 + fabs(pobj) + fabs(dobj));
  *rel = r;
  return c.relative ? r : comp;
}

__device__ int pick_free(const Ctl& c, int avoid) {
  for (int s = 0; s < kNSlot; ++s)
    if (s != c.sX && s != c.sA && s != c.sZ && s != c.sB && s != avoid && !(c.lagA && s == c.sAsrc)) return s;
  return -1;  // unreachable with kNSlot = 7 (at most 5 roles + the two outputs)
}

__device__ void prepare_step(Ctl& c) {
  c.sXn = pick_free(c, -1);
  c.sAn = pick_free(c, c.sXn);
  c.tau = c.eta / c.omega;     // pdhg.py:86-87
  c.sigma = c.eta * c.omega;   // pdhg.py:90-91
  c.kd = (double)c.inner;      // lazy matrix average of the current iterate (k >= 1 when lagA)
  c.rkd = c.inner > 0 ? 1.0 / c.kd : 1.0;
  c.kd_dual = (double)(c.inner + 1);  // dual average of the trial iterate (pdhg.py:316-317)
  c.rkd_dual = 1.0 / c.kd_dual;
  c.op = OP_STEP;
}

__device__ void finish(Ctl& c, int reason, int final_slot, double final_rel) {
  c.done = 1;
  c.reason = reason;
  c.sFinal = final_slot;
  c.final_rel = final_rel;
  c.op = OP_NONE;
}

__device__ void fail(Ctl& c, int err) {
  c.done = 1;
  c.error = err;
  c.op = OP_NONE;
}

// pdhg.py:363-376
__device__ void do_restart(Ctl& c, int cand_slot, double cand_kkt) {
  ring_push(c, EV_RESTART, (int)c.inner, cand_kkt, c.omega, 0.0);
  c.outer += 1;
  c.inner = 0;
  // (the slack records stay valid: both new dual pairs are the candidate's, which
  // was one of this pass's two input pairs, and the records bound both of them)
  c.sX = c.sA = c.sZ = c.sAsrc = cand_slot;
  c.lagA = 0;
  c.epoch_kkt = cand_kkt;
  c.prev_cand = cand_kkt;
  c.pending = 0;
}

// pdhg.py:198-222
__device__ bool should_restart(const Ctl& c, double cand) {
  if (!c.adaptive) return cand <= c.beta * c.epoch_kkt;
  if (cand <= c.beta_suff * c.epoch_kkt) return true;
  if (cand <= c.beta_nec * c.epoch_kkt && cand > c.prev_cand) return true;
  return (double)c.inner >= c.beta_art * (double)c.total;
}

// loop-top limit checks, pdhg.py:299-306
__device__ bool limits_hit(Ctl& c, const Sums& S) {
  if (c.total >= c.max_iters) {
    finish(c, R_ITER, c.sB, c.best_rel);
    return true;
  }
  if (S.stop_any) {
    finish(c, R_TIME, c.sB, c.best_rel);
    return true;
  }
  return false;
}

// The long floating-point pieces of a STEP decision (two KKT metrics, the step
// bound, the iterate norm), evaluated by four warps in parallel before the
// single-thread decision chain; same formulas as the in-line code they replace.
struct Pre {
  double kc, rel_cur, ka, rel_avg, bound, nrm;
};

__device__ double kkt_metric(const Ctl& c, double psq, double dsq, double pobj, double dobj, double* rel);

// t_cur: the thread that evaluates the current iterate's metric (0; the dry
// run moves it off thread 0, which runs the decision code meanwhile)
__device__ __noinline__ void precompute_step(const Ctl& c, const Sums& S, Pre* P, int t_cur = 0) {
  const int tid = threadIdx.x;
  if (tid == t_cur && c.pending)
    P->kc = kkt_metric(c, c.pend_psq_cur, S.R[11], c.pend_pobj_cur, c.pend_dobj_cur, &P->rel_cur);
  if (tid == 32 && c.pending) P->ka = kkt_metric(c, S.R[3] + S.K[3], S.R[12], S.R[9], c.pend_dobj_avg, &P->rel_avg);
  if (tid == 64 && c.adaptive) {
    const double dd = S.R[7], dpp = S.R[0], dqq = S.K[0];
    const double numer = c.omega * dd + (dpp + dqq) / c.omega;
    const double denom = 2.0 * fabs(S.R[1] + S.K[1]);
    P->bound = denom <= c.eps_zero ? INFINITY : numer / denom;
  }
  if (tid == 96) P->nrm = sqrt((S.R[10] + S.R[6]) + S.K[6]);
}

__device__ __noinline__ void control_step(Ctl& c, const Sums& S, const Pre& P) {
  // the average matrix of the input iterate, if lagging, was written by this pass
  c.avg_written = c.lagA;
  c.avg_slot = c.sA;
  c.lagA = 0;
  // ---- 1. resolve the KKT of the input iterate (evaluated at pdhg.py:331-378):
  //         current-iterate primal parts from the pass that created it, the
  //         average's primal parts and both dual violations from this pass
  if (c.pending) {
    c.pending = 0;
    const double kc = P.kc, rel_cur = P.rel_cur, ka = P.ka, rel_avg = P.rel_avg;
    const bool take_cur = kc < ka;  // tie -> average (pdhg.py:335-338)
    const int cand_slot = take_cur ? c.sX : c.sA;
    const double cand = take_cur ? kc : ka;
    const double cand_rel = take_cur ? rel_cur : rel_avg;
    // both metrics travel with the candidate: the host can report decision margins
    if (c.trace_level > 0) ring_push(c, EV_CAND, take_cur ? 1 : 0, cand, kc, ka);
    if (cand < c.best_kkt) {  // pdhg.py:342-344 (role alias instead of a copy)
      c.sB = cand_slot;
      c.best_kkt = cand;
      c.best_rel = cand_rel;
    }
    if (cand <= c.tol) {  // pdhg.py:345-348
      finish(c, R_TOL, cand_slot, cand_rel);
      return;
    }
    if (should_restart(c, cand)) {
      if (c.adaptive) {  // need |cand - anchor| first: one distance pass
        c.sCand = cand_slot;
        c.cand_kkt = cand;
        c.cand_rel = cand_rel;
        c.op = OP_DIST;
        return;
      }
      do_restart(c, cand_slot, cand);
      prepare_step(c);  // the speculative trial started from the old iterate: rerun
      return;
    }
    c.prev_cand = cand;
  }
  // ---- 2. loop top
  if (limits_hit(c, S)) return;
  // ---- 3. the trial step of this pass (pdhg.py:230-251)
  double bound = INFINITY;
  if (c.adaptive) {
    bound = P.bound;
    if (!(c.eta <= bound)) {
      c.halvings += 1;
      c.rejected += 1;
      if (c.trace_level > 1) ring_push(c, EV_REJECT, 0, c.eta, bound, 0.0);
      if (c.halvings >= 80) {
        fail(c, E_LINESEARCH);
        return;
      }
      c.eta *= 0.5;
      prepare_step(c);
      return;
    }
  }
  if (c.trace_level > 0) ring_push(c, EV_ACCEPT, c.adaptive, c.eta, bound, 0.0);
  if (c.adaptive && isfinite(bound)) {
    const double grown = 1.05 * c.eta;
    c.eta = bound < grown ? bound : grown;  // min(1.05 eta, bound)
  }
  c.halvings = 0;
  c.total += 1;
  c.inner += 1;
  c.sX = c.sXn;
  c.sAsrc = c.sA;  // its matrix is the previous average; the next pass writes sAn's
  c.sA = c.sAn;
  c.lagA = 1;
  // pdhg.py:319-322
  const double nrm = P.nrm;
  if (!isfinite(nrm)) {
    fail(c, E_NONFINITE);
    return;
  }
  if (nrm > c.scale_R) c.scale_R = nrm;
  if (c.inner % c.kkt_stride == 0) {
    c.pending = 1;
    c.pend_psq_cur = S.R[2] + S.K[2];
    c.pend_pobj_cur = S.R[8];
    c.pend_dobj_cur = S.R[4] + S.K[4];
    c.pend_dobj_avg = S.R[5] + S.K[5];
  }
  prepare_step(c);
}

__device__ __noinline__ void control_dist(Ctl& c, const Sums& S) {
  c.avg_written = 0;
  // pdhg.py:353-362 + primal_weight_update pdhg.py:174-186
  const double dX = sqrt(S.R[2]);
  const double dpq = sqrt(S.R[0] + S.K[0]);
  if (dX > c.eps_zero && dpq > c.eps_zero) {
    if (c.host_omega) {  // pause: the host evaluates omega with libm, then resume_restart
      c.om_dX = dX;
      c.om_dpq = dpq;
      c.omega_wait = 1;
      c.done = 1;
      c.op = OP_NONE;
      return;
    }
    c.omega = exp(c.theta * log(dpq / dX) + (1.0 - c.theta) * log(c.omega));
  }
  do_restart(c, c.sCand, c.cand_kkt);
  prepare_step(c);
}

__device__ __noinline__ void control_start(Ctl& c, const Sums& S) {
  c.avg_written = 0;
  // pdhg.py:278-296
  const double nrm = sqrt((S.R[5] + S.R[2]) + S.K[2]);
  c.scale_R = nrm > 1.0 ? nrm : 1.0;
  const double psq = S.R[0] + S.K[0];
  const double pobj = S.R[3], dsq = S.R[4];
  const double dobj = S.R[1] + S.K[1];
  double rel;
  const double k0 = kkt_metric(c, psq, dsq, pobj, dobj, &rel);
  c.epoch_kkt = c.prev_cand = c.best_kkt = k0;
  c.best_rel = rel;
  c.sA = c.sZ = c.sB = c.sAsrc = c.sX;
  c.lagA = 0;
  c.pending = 0;
  ring_push(c, EV_START, 0, k0, rel, 0.0);
  if (k0 <= c.tol) {
    finish(c, R_TOL, c.sX, rel);
    return;
  }
  prepare_step(c);
}

__device__ __noinline__ void control_unit(Ctl& c, int op, const Sums& S) {
  if (op == OP_KKT) {
    const double psq = S.R[0] + S.K[0];
    const double pobj = S.R[3], dsq = S.R[4];
    const double dobj = S.R[1] + S.K[1];
    double rel;
    const double gap = pobj - dobj;
    const int32_t saved = c.relative;
    c.relative = 0;
    const double comp = kkt_metric(c, psq, dsq, pobj, dobj, &rel);
    c.relative = saved;
    c.out[0] = gap; c.out[1] = comp; c.out[2] = rel; c.out[3] = pobj; c.out[4] = dobj;
    c.out[5] = psq; c.out[6] = dsq; c.out[7] = S.R[5]; c.out[8] = S.R[2]; c.out[9] = S.K[2];
  } else if (op == OP_DIFF) {
    const double dd = S.R[2], dpp = S.R[0], dqq = S.K[0];
    const double numer = c.omega * dd + (dpp + dqq) / c.omega;
    const double denom = 2.0 * fabs(S.R[1] + S.K[1]);
    c.out[0] = denom <= c.eps_zero ? INFINITY : numer / denom;
    c.out[1] = dd; c.out[2] = dpp; c.out[3] = dqq; c.out[4] = S.R[1] + S.K[1];
  } else if (op == OP_STEP) {
    c.out[0] = S.R[7];  // |dX|^2
    c.out[1] = S.R[10]; // |X+|^2
  } else if (op == OP_ROUND) {
    if (c.round_stage == 2) {
      c.out[OUT_ROUND_TOTAL] = S.R[0];                         // total deficit
      c.out[OUT_ROUND_CORRECT] = S.R[0] <= 1e-14 ? 0.0 : 1.0;  // rounding.py:36
    } else if (c.round_stage == 3) {
      c.out[OUT_ROUND_OBJ] = S.R[3];             // <C, X_feas>
      c.out[OUT_ROUND_DUAL] = S.R[1] + S.K[0];   // f.p + g.q
      c.out[OUT_ROUND_L1VIOL] = S.R[2] + S.K[1]; // l1 marginal violation of X_feas
    }
  }
}

// Wait for the tickets of the `nwork` work blocks (run by the controller block).
__device__ __forceinline__ void wait_tickets(const Ctl& c, unsigned nwork) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c.counter) : "memory");
    } while (v < nwork);
  }
  __syncthreads();
}

// Grid: [controller block] + T row blocks + CB column blocks (FIN_B: column
// blocks only; FIN_A: no controller, the last block to finish combines the
// group scalars).  The controller block does no pass work: while the work
// blocks run it executes the decision code once on a scratch copy of the
// control block (so the instructions are in this SM's instruction cache and
// the real run does not fetch them from DRAM), then waits for every ticket.
// PDOT_K2_PROF (measurement builds only): K2 phase times of screened STEP
// passes, summed over a solve and printed by the controller at pass 600.
// [0..3] work blocks: entry -> Ctl copied, -> work done, -> ticket, count;
// [4..8] controller: entry -> copied, -> dry run done, -> tickets seen, -> reduced, -> end;
// [9] max work-block ticket time after the controller's entry
#ifdef PDOT_K2_PROF
__device__ unsigned long long g_k2prof[16];
__device__ unsigned long long g_k2entry;  // controller entry of the running pass
#endif

template <int mode>
__global__ void __launch_bounds__(kRedThreads, 2) finalize_kernel(Ctl* __restrict__ ctlp, int force_op, const FGeo geo) {
  // launched as a programmatic dependent of K1b (pdl_edge("k2")): every block
  // copies the control block (K1b does not write it) before it waits for K1b,
  // and the controller block also runs its dry run first
  if (mode != FIN_FUSED) pdl_wait();
#ifdef PDOT_K2_PROF
  const unsigned long long tq0 = globaltimer_ns();
  unsigned long long tq1 = 0, tq2 = 0, tq3 = 0;
#endif
  __shared__ double smem[kWarps * 4 * kColsPerBlock + 64];
  __shared__ Sums S;
  __shared__ int is_last;
  __shared__ Ctl cs;
  __shared__ Pre pre;
  {
    const Ctl& g = *ctlp;
    if (g.done) return;
    const int op0 = force_op >= 0 ? force_op : g.op;
    if (op0 == OP_NONE) return;
    if (mode == FIN_B && g.p2p) wait_exchange(*ctlp);
  }
  // Every block works on a shared-memory copy of the control block: its fields
  // are then plain shared loads that no global store can alias (the blocks only
  // write through the pointers it holds), and the controller reuses the copy.
  constexpr int kWords = (int)(sizeof(Ctl) / sizeof(unsigned long long));
  unsigned long long* cw = reinterpret_cast<unsigned long long*>(&cs);
  {
    const unsigned long long* gw = reinterpret_cast<const unsigned long long*>(ctlp);
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) cw[i] = __ldcg(gw + i);
  }
  __syncthreads();
  // the work blocks of a STEP pass wait inside column_block_t / row_block_t, after
  // issuing their vector loads (written by the previous pass); the rest wait here
  if (mode == FIN_FUSED && blockIdx.x != 0 && !((force_op >= 0 ? force_op : cs.op) == OP_STEP)) pdl_wait();
  Ctl& c = cs;
  const int op = force_op >= 0 ? force_op : c.op;
  const bool timed = op == OP_STEP && unit_pass(c, op) && c.sstat;  // K2 timing of screened STEP passes
  const int has_ctl = mode == FIN_A ? 0 : 1;
  const unsigned nwork = gridDim.x - has_ctl;
#ifdef PDOT_K2_PROF
  tq1 = globaltimer_ns();
  if (timed && has_ctl && blockIdx.x == 0 && threadIdx.x == 0) g_k2entry = tq0;
#endif
  // screened-STEP statistics of this pass, read at entry by the controller
  // block's last thread (K1 has completed) and accounted after the write-back
  unsigned long long k2_t0 = 0, k1e = 0, k1s = 0, ncl = 0;
  if (has_ctl && blockIdx.x == 0) {
    // pass statistics by the last thread (its load of the K1 end stamp is used
    // only after the dry run: thread 0 starts the dry run without waiting)
    if (timed && threadIdx.x == kRedThreads - 1) {
      k2_t0 = globaltimer_ns();
      k1e = __ldcg(&c.sstat[ST_K1_END]);
      k1s = __ldcg(&c.sstat[ST_T0]);
      ncl = __ldcg(c.ucount);
      c.sstat[ST_K2_T0] = k2_t0;
    }
    if (timed && c.ktl && threadIdx.x == kRedThreads - 1) atomicMin(c.ktl + 6, k2_t0);
#ifndef PDOT_K2_NO_DRYRUN
    if (op == OP_STEP && !c.unit) {
      __shared__ Ctl dry;
      unsigned long long* dw = reinterpret_cast<unsigned long long*>(&dry);
      for (int i = threadIdx.x; i < kWords; i += blockDim.x) dw[i] = cw[i];
      __syncthreads();
      if (threadIdx.x == 0) {
        dry.ring = nullptr;
        dry.status = nullptr;
      }
#ifdef PDOT_K2_PROF
      const unsigned long long td0 = globaltimer_ns();
#endif
#ifndef PDOT_K2_DRY_NORED
      reduce_blocks(dry, &S, smem, mode);  // partials still being written: values unused
#endif
#ifdef PDOT_K2_PROF
      const unsigned long long td1 = globaltimer_ns();
#endif
#ifdef PDOT_K2_PROF
      const unsigned long long td2 = globaltimer_ns();
#endif
      // the decision code and the four metric pieces warm the instruction cache
      // side by side (different warps); the decision runs on metrics that take
      // the common path (candidate kept, no restart, step accepted and grown)
      __shared__ Pre pre_dry;
      if (threadIdx.x == 0) {
        Pre pd;
        pd.kc = pd.ka = dry.epoch_kkt;
        pd.rel_cur = pd.rel_avg = dry.best_rel;
        pd.bound = 2.0 * dry.eta;
        pd.nrm = 1.0;
        control_step(dry, S, pd);
      } else {
        precompute_step(dry, S, &pre_dry, 128);
      }
      __syncthreads();
#ifdef PDOT_K2_PROF
      if (timed && threadIdx.x == 0) {
        g_k2prof[12] += td1 - td0;
        g_k2prof[13] += td2 - td1;
        g_k2prof[14] += globaltimer_ns() - td2;
        g_k2prof[15] += td0 - tq0;
      }
#endif
    }
#endif
#ifdef PDOT_K2_PROF
    tq2 = globaltimer_ns();
#endif
    pdl_wait();
    wait_tickets(c, nwork);
#ifdef PDOT_K2_PROF
    tq3 = globaltimer_ns();
#endif
  } else {
    const int wb = (int)blockIdx.x - has_ctl;  // work block index
    if (timed && c.kdbg && threadIdx.x == 0) c.kdbg[wb * 4 + 0] = globaltimer_ns();
    if (timed) tl_start(c.ktl, 3);
    // row blocks first (they carry the longer chains); FIN_B has column blocks only
    const int64_t nrow_blocks = mode == FIN_B ? 0 : c.T;
    if ((int64_t)wb >= nrow_blocks) {
      const int b = (int)(wb - nrow_blocks);
      if (mode == FIN_A) {
        if (op == OP_STEP) column_group_partials<4>(c, b);
        else column_group_partials<1>(c, b);
      } else {
        if (op == OP_STEP) column_block_t<true>(c, geo, op, b, smem, mode);
        else column_block_rare(c, op, b, smem, mode);
      }
    } else {
      if (op == OP_STEP) row_block_t<true>(c, geo, op, wb, smem);
      else row_block_rare(c, op, wb, smem);
    }
    if (timed && c.kdbg && threadIdx.x == 0) c.kdbg[wb * 4 + 1] = globaltimer_ns();
    if (mode == FIN_A) {
      if (c.p2p) __threadfence_system();  // remote group stores before the ticket
      else __threadfence();
    }
    __syncthreads();
    if (mode != FIN_A) {
      if (threadIdx.x == 0) {
#ifdef PDOT_K2_PROF
        const unsigned long long tw = globaltimer_ns();
#endif
        // the block's partial stores (ordered before this thread by the barrier)
        // are released with the ticket: one acq_rel fence instead of a
        // sequentially consistent fence by every thread
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        atomicAdd(c.counter, 1u);
        if (timed && c.kdbg) c.kdbg[wb * 4 + 2] = globaltimer_ns();
#ifdef PDOT_K2_PROF
        if (timed) {
          const unsigned long long tt = globaltimer_ns();
          atomicAdd(&g_k2prof[0], tq1 - tq0);
          atomicAdd(&g_k2prof[1], tw - tq0);
          atomicAdd(&g_k2prof[2], tt - tq0);
          atomicAdd(&g_k2prof[3], 1ull);
          const unsigned long long ce = *(volatile unsigned long long*)&g_k2entry;
          if (tt > ce) atomicMax(&g_k2prof[9], tt - ce);
        }
#endif
      }
      return;
    }
    if (threadIdx.x == 0) is_last = atomicAdd(c.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    group_scalar_partials(c);
    __syncthreads();
    if (threadIdx.x == 0) *c.counter = 0u;
    return;
  }
  // (wait_tickets: the acquire load of the ticket count, then a barrier)
  const uint64_t t_last = timed ? globaltimer_ns() : 0;
  // the controller works on the shared-memory copy and writes it back
  if (mode == FIN_B && c.p2p && threadIdx.x == 0) cs.xerror = __ldcg(&ctlp->xerror);  // set by wait_exchange
  __syncthreads();
  reduce_blocks(cs, &S, smem, mode);
  if (op == OP_STEP && !cs.unit && !cs.done) {
    precompute_step(cs, S, &pre);
    __syncthreads();
  }
  const uint64_t t_red = timed ? globaltimer_ns() : 0;
  uint64_t t_logic = 0;
  if (threadIdx.x == 0) {
    if (mode == FIN_B && cs.p2p) {
      consume_exchange(cs);
      if (cs.xerror) fail(cs, E_EXCHANGE);
    }
    if (!cs.done && cs.unit) {
      control_unit(cs, op, S);
    } else if (!cs.unit) {
      if (!cs.done) {  // (done here only when this pass's exchange failed)
        cs.passes += 1;
        if (op == OP_STEP) control_step(cs, S, pre);
        else if (op == OP_DIST) control_dist(cs, S);
        else if (op == OP_KKT) control_start(cs, S);
      }
      if (timed) t_logic = globaltimer_ns();
      // publish to the host mirror (read by the host only after the pass's
      // completion event, which orders these mapped-memory writes).  Stores to
      // host memory hold the kernel's completion for a PCIe round trip, so an
      // untraced solve publishes only every 16th pass and whenever the host must
      // act (done, a paused restart); the host polls at graph-batch boundaries and
      // drains the event ring completely once done.
#ifndef PDOT_STATUS_EVERY_PASS
      const bool publish = cs.done || cs.omega_wait || cs.trace_level > 0 || (cs.passes & 15) == 0;
#else
      const bool publish = true;
#endif
      if (cs.status && publish) {
        cs.status->total = cs.total;
        cs.status->outer = cs.outer;
        cs.status->passes = cs.passes;
        cs.status->ring_head = cs.ring_head;
        cs.status->final_slot = cs.sFinal;
        cs.status->reason = cs.reason;
        cs.status->error = cs.error;
        cs.status->done = cs.done;
        cs.status->pause = cs.omega_wait;
      }
    }
  }
  __syncthreads();
  unsigned long long* gwo = reinterpret_cast<unsigned long long*>(ctlp);
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) gwo[i] = cw[i];
  if (timed && threadIdx.x == kRedThreads - 1) {
    // K1 of this pass: first CTA start (ST_T0) -> latest CTA end (ST_K1_END)
    if (k1e > k1s) cs.sstat[ST_K1_NS] += k1e - k1s;
    cs.sstat[ST_K1_END] = 0;
    cs.sstat[ST_TILES] += ncl;
    cs.sstat[ST_PASSES] += 1;
    // K0 tile-level screen of this pass: 32 cell + nbt band maxima (current and
    // average), 4 tile occupancy bytes and the tile's min C per tile (the
    // per-cell screens add theirs in K0)
    cs.sstat[ST_META] += (unsigned long long)cs.T * cs.U * ((32 + cs.nbt) * 2 * 8 + 4 + 8);
    if (k1e != 0 && k2_t0 > k1e) cs.sstat[ST_K1K2] += k2_t0 - k1e;
  }
  if (threadIdx.x == 0) {
    *cs.counter = 0u;
    if (cs.ucount) *cs.ucount = 0u;  // the screened cell and tile lists of this pass are consumed
    if (cs.tcount) *cs.tcount = 0u;
    if (timed && cs.ktl) {  // pass timeline: K2 end, then reset it for the next pass
      unsigned long long* tl = cs.ktl;
      tl[7] = globaltimer_ns();
      for (int k = 0; k < 8; ++k) tl[8 + k] = tl[k];  // keep the last complete pass
#ifdef DBG_K0
      for (int k = 0; k < 5; ++k) tl[25 + k] = tl[16 + k];
      tl[24] = 0ull;
#endif
      for (int k = 0; k < 4; ++k) {
        tl[2 * k] = ~0ull;
        tl[2 * k + 1] = 0ull;
      }
    }
#ifdef PDOT_K2_PROF
    if (timed) {
      const unsigned long long te = globaltimer_ns();
      g_k2prof[4] += tq1 - tq0;
      g_k2prof[5] += tq2 - tq0;
      g_k2prof[6] += tq3 - tq0;
      g_k2prof[7] += t_red - tq0;
      g_k2prof[8] += te - tq0;
      g_k2prof[10] += g_k2prof[9];
      g_k2prof[11] += 1;
      g_k2prof[9] = 0;
      if (cs.passes == 600) {
        const double n = (double)g_k2prof[11], w = (double)g_k2prof[3];
        printf("K2PROF (ns): work blocks entry->copied %.0f, ->work done %.0f, ->ticket %.0f; last ticket after "
               "controller entry %.0f; controller entry->copied %.0f, ->dry run done %.0f, ->tickets seen %.0f, "
               "->reduced %.0f, ->end %.0f\n",
               g_k2prof[0] / w, g_k2prof[1] / w, g_k2prof[2] / w, g_k2prof[10] / n, g_k2prof[4] / n, g_k2prof[5] / n,
               g_k2prof[6] / n, g_k2prof[7] / n, g_k2prof[8] / n);
        printf("K2PROF dry run (ns): entry->start %.0f, reduce %.0f, precompute %.0f, control_step %.0f\n",
               g_k2prof[15] / n, g_k2prof[12] / n, g_k2prof[13] / n, g_k2prof[14] / n);
      }
    }
#endif
    if (timed) {
      const uint64_t t_end = globaltimer_ns();
      cs.sstat[ST_K2_MAIN] += t_last - __ldcg(&cs.sstat[ST_K2_T0]);
      cs.sstat[ST_K2_CTL] += t_end - t_last;
      cs.sstat[ST_T0K0] += t_red - t_last;     // controller: reduction of the block partials
      cs.sstat[ST_T1K0] += t_logic - t_red;    // controller: decisions
      cs.sstat[ST_DONE0] += t_end - t_logic;   // controller: status mirror + control-block write-back
      cs.sstat[ST_K2_END] = globaltimer_ns();
    }
  }
}

// Test hook for the peer-memory exchange protocol with R ranks emulated in ONE
// cooperative launch (every block co-resident, so a spin can never wait on a
// block that is not running; separate launches that wait on one another on one
// GPU are not safe).  Block r plays rank r's pass sequence `rounds` times:
// a rank-dependent delay, its group stores into EVERY rank's exchange buffer
// (store_group1, the K2a path), publish_exchange, then wait_exchange on its
// own flags (the K2b path), a check of all 8 groups' values in its own buffer,
// and consume_exchange.  out[r] = {errors, max ns spent waiting, xerror}.
__global__ void p2p_protocol_kernel(Ctl* ctls, int rounds, unsigned long long delay_ns,
                                    unsigned long long* out) {
  Ctl& c = ctls[blockIdx.x];
  __shared__ unsigned long long waited_max;
  __shared__ int errors;
  if (threadIdx.x == 0) {
    waited_max = 0ull;
    errors = 0;
  }
  __syncthreads();
  constexpr int kVals = 8;
  for (int s = 0; s < rounds; ++s) {
    const double seqv = (double)xseq_next(c);
    // ranks reach their stores at different times: the others' waits really spin
    if (threadIdx.x == 0) {
      const unsigned long long t0 = globaltimer_ns();
      const unsigned long long d = ((unsigned)(s + c.rank) % (unsigned)c.nranks) * delay_ns;
      while (globaltimer_ns() - t0 < d) {
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < (c.g1 - c.g0) * kVals; e += blockDim.x) {
      const int g = c.g0 + e / kVals, j = e % kVals;
      store_group1(c, g * c.gstride + j, seqv * 1e6 + 1000.0 * g + j);
    }
    __syncthreads();
    if (threadIdx.x == 0) publish_exchange(c);
    const unsigned long long w0 = globaltimer_ns();
    wait_exchange(c);  // ends with __syncthreads
    if (threadIdx.x == 0) {
      const unsigned long long w = globaltimer_ns() - w0;
      if (w > waited_max) waited_max = w;
    }
    const double* buf = xgroups(c, c.rank);
    for (int e = threadIdx.x; e < kGroups * kVals; e += blockDim.x) {
      const int g = e / kVals, j = e % kVals;
      if (__ldcv(buf + g * c.gstride + j) != seqv * 1e6 + 1000.0 * g + j) atomicAdd(&errors, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) consume_exchange(c);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x * 3 + 0] = (unsigned long long)errors;
    out[blockIdx.x * 3 + 1] = waited_max;
    out[blockIdx.x * 3 + 2] = (unsigned long long)c.xerror;
  }
}

// The restart that control_dist paused for a host-evaluated omega: set omega,
// then the same restart actions (one thread; the next graph batch continues).
__global__ void resume_restart_kernel(Ctl* ctlp, double omega) {
  Ctl& c = *ctlp;
  c.omega = omega;
  c.omega_wait = 0;
  c.done = 0;
  do_restart(c, c.sCand, c.cand_kkt);
  prepare_step(c);
  if (c.status) {
    c.status->ring_head = c.ring_head;
    c.status->pause = 0;
    c.status->done = 0;
  }
}

}  // namespace

void launch_resume_restart(Ctl* ctl_dev, double omega, cudaStream_t s) {
  resume_restart_kernel<<<1, 1, 0, s>>>(ctl_dev, omega);
}

int launch_p2p_protocol_test(Ctl* ctls_dev, int nranks, int rounds, unsigned long long delay_ns,
                             unsigned long long* out_dev, cudaStream_t s) {
  void* args[] = {&ctls_dev, &rounds, &delay_ns, &out_dev};
  return (int)cudaLaunchCooperativeKernel((const void*)p2p_protocol_kernel, dim3(nranks), dim3(128), args, 0, s);
}

void launch_finalize_pass(Ctl* ctl_dev, const Ctl& h, int force_op, int mode, cudaStream_t s) {
  const FGeo geo{h.m,        h.n,       h.ldx,       h.T,        h.U,        h.TM,       h.GS,   h.t0,
                 h.Tg,       h.ncells,  h.nbands,    h.ncolblk,  h.tileflag, h.colpart,  h.rowpart,
                 h.tilescal, h.rowblk,  h.colblk,    h.qmax,     h.pmax,     h.sdq,      h.sdp};
  // + 1: the controller block (FIN_FUSED, FIN_B)
  const unsigned blocks = (unsigned)(mode == FIN_B ? h.CB + 1 : mode == FIN_A ? h.CB + h.T : h.CB + h.T + 1);
  if (mode == FIN_FUSED && pdl_edge("k2")) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kRedThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, finalize_kernel<FIN_FUSED>, ctl_dev, force_op, geo);
  } else if (mode == FIN_FUSED) finalize_kernel<FIN_FUSED><<<blocks, kRedThreads, 0, s>>>(ctl_dev, force_op, geo);
  else if (mode == FIN_A) finalize_kernel<FIN_A><<<blocks, kRedThreads, 0, s>>>(ctl_dev, force_op, geo);
  else finalize_kernel<FIN_B><<<blocks, kRedThreads, 0, s>>>(ctl_dev, force_op, geo);
}

}  // namespace pdot
