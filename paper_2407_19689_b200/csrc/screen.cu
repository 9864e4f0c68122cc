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
// K0: screening
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) screen_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (op != OP_STEP) return;
  const int64_t tu = blockIdx.x, tt = blockIdx.y;
  const int s = threadIdx.x & 7, bl = threadIdx.x >> 3;  // strip in tile, band in tile
  const bool with_avg = step_with_avg(c);
  const int64_t band = tt * c.nbt + bl;
  const int64_t strip = tu * kWarps + s;
  uint32_t word = 0;
  if (bl < c.nbt && band < c.nbands && strip < c.nstrips) {
    const int64_t sstride = c.nbands * c.nstrips;
    const int64_t ow = band * c.nstrips + strip;
    const uint32_t ox = __ldcg(c.occ + c.sX * sstride + ow);
    const uint32_t oa = with_avg ? __ldcg(c.occ + c.sAsrc * sstride + ow) : 0u;
    const uint32_t zx = __ldcg(c.occ + c.sXn * sstride + ow);
    const uint32_t za = with_avg ? __ldcg(c.occ + c.sA * sstride + ow) : 0u;
    const double P = __ldcg(c.pmax + c.sX * c.nbands + band);
    const double Pa = __ldcg(c.pmax + c.sA * c.nbands + band);
    // a non-finite step (tau) would turn 0 * inf into NaN: screen nothing
    const bool finite_step = isfinite(c.tau);
#pragma unroll
    for (int k = 0; k < kCellsPerStrip; ++k) {
      const int64_t cell = strip * kCellsPerStrip + k;
      if (cell >= c.ncells) break;
      const double Q = __ldcg(c.qmax + c.sX * c.ncells + cell);
      const double Qa = __ldcg(c.qmax + c.sA * c.ncells + cell);
      const double mc = __ldcg(c.minc + band * c.ncells + cell);
      const uint32_t bx = (ox >> (8 * k)) & 0xffu, ba = (oa >> (8 * k)) & 0xffu;
      const uint32_t bzx = (zx >> (8 * k)) & 0xffu, bza = (za >> (8 * k)) & 0xffu;
      // !(a <= b) keeps NaN bounds active
      const bool act = bx || ba || !(P + Q <= mc) || !(Pa + Qa <= mc) || !finite_step;
      const uint32_t f = (act ? U_ACT : 0u) | (bx ? U_LDX : 0u) | (ba ? U_LDA : 0u) | (bzx ? U_ZX : 0u) |
                         (bza ? U_ZA : 0u);
      word |= f << (8 * k);
    }
  }
  if (bl < c.nbt) c.unitw[((tt * c.U + tu) * kWarps + s) * c.nbt + bl] = word;
  const int any = __syncthreads_or(word != 0u);
  if (threadIdx.x == 0) {
    c.tileflag[tt * c.U + tu] = any ? 1 : 0;
    if (any) c.tlist[atomicAdd(c.tcount, 1u)] = (int32_t)(tt * c.U + tu);
  }
}

// the rare ops (start KKT, restart distance, unit calls, rounding) kept out of
// line so their registers do not crowd the screened STEP path
__device__ __noinline__ void generic_tile_call(int op, const Ctl& c, double* smem, int64_t tu, int64_t tt) {
  generic_tile(op, c, smem, tu, tt);
}

// ---------------------------------------------------------------------------
// K1: screened STEP over one tile (same partial layout as the dense walker)
// ---------------------------------------------------------------------------
template <bool IMPLICIT, bool AVG>
__device__ __forceinline__ void screened_tile(const StepOp& op, const Ctl& c, double* smem, int64_t tu, int64_t tt,
                                              unsigned long long& bytes, unsigned long long& cells) {
  constexpr int NQ = StepOp::NQ, NS = StepOp::NS, H = kBand / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Geo g = make_geo(c, true, tu, tt);
  double* rowbuf = smem;                             // [TM][NQ][kWarps]
  double* sbuf = smem + (size_t)c.TM * NQ * kWarps;  // [kWarps][8]
  const int nb = (g.rows + kBand - 1) / kBand;
  const uint32_t w = lane < nb ? __ldcg(c.unitw + ((tt * c.U + tu) * kWarps + warp) * c.nbt + lane) : 0u;
  const unsigned bandmask = __ballot_sync(0xffffffffu, w != 0u);
  StepOp::Col cl;
  op.load_col(cl, g);
  double cacc[NQ][2];
#pragma unroll
  for (int q = 0; q < NQ; ++q) cacc[q][0] = cacc[q][1] = 0.0;
  double sacc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) sacc[s] = 0.0;
  const int cellsh = (lane >> 3) * 8;
  const int64_t sstride = c.nbands * c.nstrips;
  const int64_t strip = tu * kWarps + warp;
  double2 cj0 = make_double2(0.0, 0.0), cj1 = make_double2(0.0, 0.0);
  if (IMPLICIT) {
    cj0 = g.gen.col_coord(g.j);
    cj1 = g.gen.col_coord(g.j + 1);
  }
  const double2 zero2 = make_double2(0.0, 0.0);
#pragma unroll 1
  for (int b = 0; b < nb; ++b) {
    const int r0 = b * kBand;
    if (!((bandmask >> b) & 1u)) {
      // every cell of this band is +0 for this warp: its row partials are +0
      rowbuf[((r0 + (lane >> 2)) * NQ + (lane & 3)) * kWarps + warp] = 0.0;
      continue;
    }
    const uint32_t cb = (__shfl_sync(0xffffffffu, w, b) >> cellsh) & 0xffu;
    const bool act = (cb & U_ACT) && g.v0;
    const bool ldx = act && (cb & U_LDX);
    const bool lda = AVG && act && (cb & U_LDA);
    const bool zx = (cb & U_ZX) && g.v0;
    const bool za = AVG && (cb & U_ZA) && g.v0;
    bool nzx = false, nza = false;
    if ((lane & 7) == 0 && (cb & U_ACT)) cells += 1;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int rh = r0 + h * H;
      double2 cc[H], xx[H], aa[H];
      double pr[H], par[H];
#pragma unroll
      for (int rr = 0; rr < H; ++rr) {
        const int r = rh + rr;
        const bool ok = act && r < g.rows;
        const int64_t i = g.i0 + r;
        if (IMPLICIT) {
          const double2 rc = g.gen.row_coord(i);
          cc[rr] = ok ? make_double2(g.gen.cost(rc, cj0), g.gen.cost(rc, cj1)) : zero2;
        } else {
          cc[rr] = ok ? ld_stream2(op.C + i * g.ldc + g.j) : zero2;
        }
        xx[rr] = (ok && ldx) ? ld_stream2(op.X + i * g.ldx + g.j) : zero2;
        aa[rr] = (ok && lda) ? ld_stream2(op.A + i * g.ldx + g.j) : zero2;
        pr[rr] = ok ? __ldg(op.p + i) : 0.0;
        par[rr] = ok ? __ldg(op.pa + i) : 0.0;
        if (ok) bytes += (IMPLICIT ? 0 : 16) + (ldx ? 16 : 0) + (lda ? 16 : 0);
      }
      double rv[H * NQ];
#pragma unroll
      for (int rr = 0; rr < H; ++rr) {
        const int r = rh + rr;
        const bool inrow = r < g.rows;
        const bool ok = act && inrow;
        const int64_t i = g.i0 + r;
        double o0[NQ], o1[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) o0[q] = o1[q] = 0.0;
        if (ok) {
          op.template elem<AVG>(cc[rr].x, xx[rr].x, aa[rr].x, pr[rr], cl.q0, par[rr], cl.qa0, o0, sacc);
          if (g.v1) op.template elem<AVG>(cc[rr].y, xx[rr].y, aa[rr].y, pr[rr], cl.q1, par[rr], cl.qa1, o1, sacc);
        }
        const double2 xo = make_double2(o0[2], o1[2]);
        const bool nzr = nz2(xo);
        nzx |= nzr;
        if (inrow && (ok ? (zx || nzr) : zx)) {
          st_stream2(op.Xn + i * g.ldx + g.j, xo);
          bytes += 16;
        }
        if (AVG) {
          const double2 ao = make_double2(o0[3], o1[3]);
          const bool nar = nz2(ao);
          nza |= nar;
          if (inrow && (ok ? (za || nar) : za)) {
            st_stream2(op.An + i * g.ldx + g.j, ao);
            bytes += 16;
          }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          cacc[q][0] += o0[q];
          cacc[q][1] += o1[q];
          rv[rr * NQ + q] = o0[q] + o1[q];
        }
      }
      push_rows<NQ, H>(rv, rowbuf, rh, true);
    }
    // occupancy of the band's 4 output cells (bit patterns, so -0.0 counts)
    const unsigned mx = __ballot_sync(0xffffffffu, nzx);
    const unsigned ma = __ballot_sync(0xffffffffu, nza);
    if (lane == 0) {
      uint32_t wx = 0, wa = 0;
#pragma unroll
      for (int k = 0; k < kCellsPerStrip; ++k) {
        wx |= ((mx >> (8 * k)) & 0xffu) ? (1u << (8 * k)) : 0u;
        wa |= ((ma >> (8 * k)) & 0xffu) ? (1u << (8 * k)) : 0u;
      }
      const int64_t ow = (tt * c.nbt + b) * c.nstrips + strip;
      c.occ[c.sXn * sstride + ow] = wx;
      if (AVG) c.occ[c.sA * sstride + ow] = wa;
    }
  }
  tile_flush<NQ, NS>(c, g, true, cacc, sacc, rowbuf, sbuf);
  if (threadIdx.x == 0) bytes += (unsigned long long)(NQ * kTileN + NQ * g.rows + NS) * 8;
}

__global__ void __launch_bounds__(kThreads, kSparseCtasPerSm) sparse_kernel(const Ctl* __restrict__ ctlp, int force_op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const Ctl& c = *ctlp;
  if (c.done || !c.screen) return;
  const int op = force_op >= 0 ? force_op : c.op;
  if (op != OP_STEP) {
    for (int64_t t = blockIdx.x; t < c.T * c.U; t += gridDim.x) {
      generic_tile_call(op, c, smem, t % c.U, t / c.U);
      __syncthreads();
    }
    return;
  }
  __shared__ unsigned long long red[2][kWarps];
  if (blockIdx.x == 0 && threadIdx.x == 0) c.sstat[ST_T0] = globaltimer_ns();
  const StepOp o = make_step_op(c);
  const unsigned ntiles = __ldcg(c.tcount);
  unsigned long long bytes = 0, cells = 0;
  for (unsigned k = blockIdx.x; k < ntiles; k += gridDim.x) {
    const int32_t tile = __ldcg(c.tlist + k);
    const int64_t tu = tile % c.U, tt = tile / c.U;
    if (o.C) {
      if (o.with_avg) screened_tile<false, true>(o, c, smem, tu, tt, bytes, cells);
      else screened_tile<false, false>(o, c, smem, tu, tt, bytes, cells);
    } else {
      if (o.with_avg) screened_tile<true, true>(o, c, smem, tu, tt, bytes, cells);
      else screened_tile<true, false>(o, c, smem, tu, tt, bytes, cells);
    }
    __syncthreads();
  }
  // statistics: one atomic per CTA, then the last CTA stamps the end time
#pragma unroll
  for (int msk = 16; msk >= 1; msk >>= 1) {
    bytes += __shfl_xor_sync(0xffffffffu, bytes, msk);
    cells += __shfl_xor_sync(0xffffffffu, cells, msk);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
      c.sstat[ST_K1_NS] += t1 - __ldcg(&c.sstat[ST_T0]);
      c.sstat[ST_TILES] += ntiles;
      c.sstat[ST_PASSES] += 1;
      c.sstat[ST_DONE1] = 0;
      // K0 metadata traffic of this pass: min C + 4 occupancy words + unit word per (band, strip)
      c.sstat[ST_META] += (unsigned long long)c.nbands * c.nstrips * (kCellsPerStrip * 8 + 4 * 4 + 4);
    }
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

void prepare_sparse_kernel() {
  cudaFuncSetAttribute(sparse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
}

static size_t sparse_smem_bytes(int64_t TM) {
  return (size_t)TM * kMaxNQ * kWarps * sizeof(double) + kWarps * 8 * sizeof(double);
}

void launch_screened_pass(const Ctl* ctl_dev, const Ctl& h, int force_op, cudaStream_t s) {
  dim3 g0((unsigned)h.U, (unsigned)h.T);
  screen_kernel<<<g0, (unsigned)(kWarps * h.nbt), 0, s>>>(ctl_dev, force_op);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = h.T * h.U;
  const unsigned grid = (unsigned)imin64(tiles, (int64_t)sms * kSparseCtasPerSm);
  sparse_kernel<<<grid, kThreads, sparse_smem_bytes(h.TM), s>>>(ctl_dev, force_op);
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
