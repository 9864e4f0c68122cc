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
#include "pass_ops.cuh"

namespace pdot {
namespace {

// ---------------------------------------------------------------------------
// TMA walker for the hot STEP op.  Warp kWarps is the producer: one elected
// lane streams each stage (kStageRows rows of C, X and A for the tile's 512
// columns, 4 KB per row per matrix) into a kStages-deep shared-memory ring with
// cp.async.bulk + mbarrier transaction counts, evict-first in L2.  The 8
// consumer warps read their 128-bit column pair from shared memory, run the
// fused update, store X+ / A' straight to HBM and release the slot.  Loads are
// thereby always kStages-1 stages ahead of the math, independent of registers.
// ---------------------------------------------------------------------------
#ifndef PDOT_STAGES
#define PDOT_STAGES 6
#endif
#ifndef PDOT_MINB
#define PDOT_MINB 1
#endif
constexpr int kStages = PDOT_STAGES;
constexpr int kStageRows = 2;
constexpr int kRowBytes = kTileN * 8;                  // 4096
constexpr int kStageBytes = kStageRows * 3 * kRowBytes;  // 24576
constexpr int kBarBytes = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <bool IMPLICIT, bool AVG>
__device__ __forceinline__ void step_tma(const StepOp& op, const Ctl& c, unsigned char* smem) {
  constexpr int NQ = StepOp::NQ, NS = StepOp::NS, R = kStageRows;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool worker = warp < kWarps;
  Geo g = make_geo(c, worker, blockIdx.x, blockIdx.y);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kStages;
  unsigned char* stages = smem + kBarBytes;
  double* pbuf = reinterpret_cast<double*>(stages + kStages * kStageBytes);  // p, pa of the tile rows
  double* pabuf = pbuf + c.TM;
  double* rowbuf = pabuf + c.TM;
  double* sbuf = rowbuf + (size_t)c.TM * NQ * kWarps;
  const int nst = (g.rows + R - 1) / R;
  const int64_t col0 = (int64_t)blockIdx.x * kTileN;
  const int64_t vcols = imin64(kTileN, c.n - col0);
  const uint32_t rowbytes = (uint32_t)(((vcols + 1) & ~1LL) * 8);
  const uint32_t pbytes = (uint32_t)(((g.rows + 1) & ~1) * 8);
  constexpr bool implicit_c = IMPLICIT;       // cost generated in registers (g.gen)
  const int kfirst = implicit_c ? 1 : 0;      // first streamed matrix (0 = C)
  const int nmat = AVG ? 3 : 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double cacc[NQ][2];
#pragma unroll
  for (int q = 0; q < NQ; ++q) cacc[q][0] = cacc[q][1] = 0.0;
  BandAcc<NQ, NS> bacc;
  bacc.reset();
  double sacc[NS], ws = 0.0;
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
  constexpr int kStagesPerBand = kBand / R;

  if (!worker) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      const double* src[3] = {implicit_c ? nullptr : op.C + g.i0 * c.ldc + col0, op.X + g.i0 * c.ldx + col0,
                              op.A + g.i0 * c.ldx + col0};
      const int64_t ld[3] = {c.ldc, c.ldx, c.ldx};
      for (int it = 0; it < nst; ++it) {
        const int s = it % kStages;
        if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) + 1) & 1);
        const int nr = min(R, g.rows - it * R);
        uint32_t tx = (uint32_t)(nr * (nmat - kfirst)) * rowbytes;
        if (it == 0) tx += 2 * pbytes;
        mbar_expect_tx(&full[s], tx);
        if (it == 0) {
          bulk_g2s(pbuf, op.p + g.i0, pbytes, &full[0], pol);
          bulk_g2s(pabuf, op.pa + g.i0, pbytes, &full[0], pol);
        }
        unsigned char* dst = stages + s * kStageBytes;
        for (int r = 0; r < nr; ++r) {
          const int64_t row = (int64_t)it * R + r;
          for (int k = kfirst; k < nmat; ++k)
            bulk_g2s(dst + (r * 3 + k) * kRowBytes, src[k] + row * ld[k], rowbytes, &full[s], pol);
        }
      }
    }
  } else {
    StepOp::Col cl;
    op.load_col(cl, g);
    const int off = (warp * 64 + lane * 2) * 8;  // byte offset of the column pair in a staged row
    double2 cj0 = make_double2(0.0, 0.0), cj1 = make_double2(0.0, 0.0);  // column coordinates (implicit C)
    double2 rcoord = make_double2(0.0, 0.0);                            // current row's coordinates
    if (implicit_c) {
      cj0 = g.gen.col_coord(g.j);
      cj1 = g.gen.col_coord(g.j + 1);
      rcoord = g.gen.row_coord(g.i0);
    }
    const bool fast = g.rows == c.TM && vcols == kTileN;
    if (fast) {
      // full tile: no masks, running output pointers
      double* xo = op.Xn + g.i0 * c.ldx + g.j;
      double* ao = op.An + g.i0 * c.ldx + g.j;
      // a full tile has whole bands: unroll the band's 4 stages so the stage
      // index of the band accumulators is a compile-time constant
      for (int it0 = 0; it0 < nst; it0 += kStagesPerBand) {
#pragma unroll
       for (int k = 0; k < kStagesPerBand; ++k) {
        const int it = it0 + k;
        const int s = it % kStages;
        mbar_wait(&full[s], (it / kStages) & 1);
        const unsigned char* st = stages + s * kStageBytes;
        double rv[R * NQ];
        double ps[NQ][2];  // 2-row stage sum of the column band partial
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          double2 cc;
          if (implicit_c) {
            cc = make_double2(g.gen.cost(rcoord, cj0), g.gen.cost(rcoord, cj1));
            g.gen.next_row(rcoord);
          } else {
            cc = *reinterpret_cast<const double2*>(st + (rr * 3 + 0) * kRowBytes + off);
          }
          const double2 xx = *reinterpret_cast<const double2*>(st + (rr * 3 + 1) * kRowBytes + off);
          const double2 aa = AVG ? *reinterpret_cast<const double2*>(st + (rr * 3 + 2) * kRowBytes + off)
                                 : make_double2(0.0, 0.0);
          const double pi = pbuf[it * R + rr], pai = pabuf[it * R + rr];
          double o0[NQ], o1[NQ];
          op.template elem<AVG>(cc.x, xx.x, aa.x, pi, cl.q0, pai, cl.qa0, o0, sacc);
          op.template elem<AVG>(cc.y, xx.y, aa.y, pi, cl.q1, pai, cl.qa1, o1, sacc);
          st_stream2(xo, make_double2(o0[2], o1[2]));
          if (AVG) st_stream2(ao, make_double2(o0[3], o1[3]));
          xo += c.ldx;
          ao += c.ldx;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            if (rr == 0) {
              ps[q][0] = o0[q];
              ps[q][1] = o1[q];
            } else {
              ps[q][0] += o0[q];
              ps[q][1] += o1[q];
            }
            rv[rr * NQ + q] = o0[q] + o1[q];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        push_rows<NQ, R>(rv, rowbuf, it * R, true);
        bacc.stage(k, ps, sacc);
       }
        band_close<NQ, NS>(bacc, cacc, ws);
      }
    } else {
      for (int it = 0; it < nst; ++it) {
        const int s = it % kStages;
        mbar_wait(&full[s], (it / kStages) & 1);
        const unsigned char* st = stages + s * kStageBytes;
        double rv[R * NQ];
        double ps[NQ][2];  // 2-row stage sum of the column band partial
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int r = it * R + rr;
          double o0[NQ], o1[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
          if (r < g.rows && g.v0) {
            StepOp::Frag fr;
            if (implicit_c) {
              fr.c = make_double2(g.gen.cost(rcoord, cj0), g.gen.cost(rcoord, cj1));
              g.gen.next_row(rcoord);
            } else {
              fr.c = *reinterpret_cast<const double2*>(st + (rr * 3 + 0) * kRowBytes + off);
            }
            fr.x = *reinterpret_cast<const double2*>(st + (rr * 3 + 1) * kRowBytes + off);
            fr.a = AVG ? *reinterpret_cast<const double2*>(st + (rr * 3 + 2) * kRowBytes + off)
                       : make_double2(0.0, 0.0);
            fr.p = pbuf[r];
            fr.pa = pabuf[r];
            op.compute(fr, g, g.i0 + r, cl, o0, o1, sacc);
          }
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            if (rr == 0) {
              ps[q][0] = o0[q];
              ps[q][1] = o1[q];
            } else {
              ps[q][0] += o0[q];
              ps[q][1] += o1[q];
            }
            rv[rr * NQ + q] = o0[q] + o1[q];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        push_rows<NQ, R>(rv, rowbuf, it * R, true);
        bacc.stage(it % kStagesPerBand, ps, sacc);
        if ((it % kStagesPerBand) == kStagesPerBand - 1 || it == nst - 1) band_close<NQ, NS>(bacc, cacc, ws);
      }
    }
  }
  tile_flush<NQ, NS>(c, g, worker, cacc, ws, rowbuf, sbuf);
}

__global__ void __launch_bounds__(kBlockThreads, PDOT_MINB) stream_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const Ctl& c = *ctlp;
  if (c.done) return;
  const int op = force_op >= 0 ? force_op : c.op;
  switch (op) {
    case OP_STEP: {
      const StepOp o = make_step_op(c);
      if (o.C) {
        if (o.with_avg) step_tma<false, true>(o, c, smem_raw);
        else step_tma<false, false>(o, c, smem_raw);
      } else {
        if (o.with_avg) step_tma<true, true>(o, c, smem_raw);
        else step_tma<true, false>(o, c, smem_raw);
      }
      break;
    }
    case OP_KKT:
    case OP_DIST:
    case OP_DIFF:
    case OP_ROUND:
      generic_tile(op, c, smem, blockIdx.x, blockIdx.y);
      break;
    default:
      break;
  }
}

}  // namespace

size_t stream_smem_bytes(int64_t TM) {
  const size_t rowbuf = (size_t)TM * kMaxNQ * kWarps * sizeof(double) + kWarps * 8 * sizeof(double);
  return kBarBytes + (size_t)kStages * kStageBytes + 2 * TM * sizeof(double) + rowbuf;
}

void prepare_stream_kernel() {
  // per device: called from pdot_create_shard with the handle's device current
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
}

void launch_stream_pass(const Ctl* ctl_dev, const Ctl& h, int force_op, cudaStream_t s) {
  const size_t smem = stream_smem_bytes(h.TM);
  dim3 grid((unsigned)h.U, (unsigned)h.T);
  stream_kernel<<<grid, kBlockThreads, smem, s>>>(ctl_dev, force_op);
}

}  // namespace pdot
