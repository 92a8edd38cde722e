// gemm_pass.cu -- the streaming tall-skinny passes over A.
//
//   NN form (K2):  C (M x N) = Aop (M x K) * B (K x N),  Aop(m,k) = f(A[m*lda + k])
//                  used for the sketch Y = A Omega (Eq. YAQ; Alg. 4
//                  step 3), the power pass Y = A Q (Alg. 2 step 4),
//                  and the small-K products Y R^-1, Q U~, Q_B J (Eq. UQU).
//   TN form (K3):  C (M x N) = Aop^T ...  Aop(m,k) = f(A[k*lda + m])
//                  used for Z = A^T Q (Alg. 2 step 3), B^T = A^T Q
//                  (Eq. BQA; Alg. 4 step 10) and Gram Y^T Y.
//   f(a) = (a - c[col]) * rs[col] with col = the column index of A (implicit
//   centring/scaling for rpca, Alg. 6), identity when c, rs are null.
//
// Design (B200, FP64): tcgen05 has no f64 kind, so the MMA is the warp-level
// DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), 37 TFLOP/s measured on this
// pool (profiles/peaks_box.json).  A work unit is (row block of BM = 128 rows
// of C, k-tile of BK = 32); the units are split evenly over a persistent grid
// of one CTA per SM ("stream-K"), so there is no wave quantisation whatever
// the shape; row blocks split between CTAs are summed inside the kernel.  A CTA streams its contiguous range of units through a 3-stage
// cp.async (LDGSTS) shared-memory ring with zero-fill for ragged edges; the 8
// warps = 4 (M, 32 rows) x 2 (N halves) keep all N <= 128 columns of C in
// registers and double-buffer their DMMA fragments.  A row block finished
// entirely inside one CTA is written directly; a row block shared by several
// CTAs is summed in CTA order by the CTA holding its first k-tile, from
// partials the later CTAs publish with release/acquire flags (deterministic,
// no FP64 atomics: SURVEY H4).  A is read from HBM exactly
// once per pass; B (Omega / Q, <= 5 MB) is re-read from L2.
#include "common.cuh"
#include "kernels.h"

namespace rsvd {

constexpr int BM = 128, BK = 32, STAGES = 3, GEMM_THREADS = 256;
constexpr int A_NN_LD = BK + 4;      // [BM][BK+4]  (row = m); stride = 4 (mod 16) doubles
constexpr int A_TN_LD = BM + 4;      // [BK][BM+4]  (row = k)
constexpr int B_LDMAX = 132;         // [BK][N + pad], N + pad = 4 (mod 16)
constexpr int NMAX = 128;

template <typename TA>
struct GemmSmem {
  static constexpr int a_stage_elems_nn = BM * A_NN_LD;
  static constexpr int a_stage_elems_tn = BK * A_TN_LD;
  static constexpr int a_stage_elems = a_stage_elems_nn > a_stage_elems_tn ? a_stage_elems_nn : a_stage_elems_tn;
  static constexpr int b_stage_elems = BK * B_LDMAX;
  static constexpr size_t bytes =
      (size_t)STAGES * (a_stage_elems * sizeof(TA) + b_stage_elems * sizeof(double) + 2 * BK * sizeof(double));
};

struct GemmArgs {
  const void* A; int64_t lda;
  const double* B; int64_t ldb;
  double* C; int64_t ldc;           // final output
  double* P;                        // stream-K partials [grid][BM][N] (a CTA's leading segment)
  unsigned* flags; unsigned epoch;  // per-CTA "partial published" flags (value = launch epoch)
  const double* c; const double* rs;
  int64_t M, K; int N, Nout;
  int64_t KT, units;                // k-tiles per row block, total units
  int grid;
  bool a_vec;                       // A rows 16-byte aligned (vector cp.async)
};

// first unit of CTA c when `units` are split evenly over `grid` CTAs
// (units * grid < 2^63 for every shape this library accepts)
__host__ __device__ inline int64_t unit_lo(int64_t units, int grid, int c) {
  return (units * (int64_t)c) / grid;
}

__global__ void epoch_bump_kernel(unsigned* ctr) { ++*ctr; }   // the next pass's stream-K epoch (kernels.h)

template <typename TA, bool TRANS, int TMAX, bool CENT>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_pass_kernel(GemmArgs g) {
  const unsigned epoch = g.flags ? *reinterpret_cast<const volatile unsigned*>(g.flags + kEpochSlot) : 0u;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using S = GemmSmem<TA>;
  TA* As = reinterpret_cast<TA*>(smem_raw);
  double* Bs = reinterpret_cast<double*>(smem_raw + (size_t)STAGES * S::a_stage_elems * sizeof(TA));
  double* Cs = Bs + (size_t)STAGES * S::b_stage_elems;       // per-stage centring: c then rs (BK each)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const int N = g.N;
  // 64-bit fragment loads are served per half-warp (16 lanes x 8 B): a row stride of
  // 4 (mod 16) doubles makes the 4 x 4 (row, column) lanes of a half-warp hit 16
  // distinct bank pairs (one wavefront per half-warp).
  const int ldbs = N + ((4 - N) & 15);
  const int tile_begin = wn * TMAX;          // N = 16 * TMAX: each warp owns TMAX n8 tiles
  const int64_t KT = g.KT;
  const int64_t u_lo = unit_lo(g.units, g.grid, blockIdx.x);
  const int64_t u_hi = unit_lo(g.units, g.grid, blockIdx.x + 1);
  const int64_t nun = u_hi - u_lo;
  const TA* A = reinterpret_cast<const TA*>(g.A);
  const bool centre = CENT && g.c != nullptr;
  const bool scale = CENT && g.rs != nullptr;
  const bool avec = g.a_vec;

  // Per-thread cp.async chunk descriptors, computed once: a thread always moves
  // the same (row, column) chunk slots of a stage; only the tile offsets advance.
  constexpr int EPC = 16 / sizeof(TA);                       // elements per 16-byte chunk
  constexpr int A_CHUNKS = (BM * BK / EPC) / GEMM_THREADS;
  const int a_cpr = TRANS ? BM / EPC : BK / EPC;             // chunks per smem row
  int a_r[A_CHUNKS], a_c[A_CHUNKS];
#pragma unroll
  for (int c = 0; c < A_CHUNKS; ++c) {
    const int id = tid + c * GEMM_THREADS;
    a_r[c] = id / a_cpr;
    a_c[c] = (id % a_cpr) * EPC;
  }

  auto load_stage = [&](int stage, int64_t u) {
    const int64_t mb = u / KT, kt = u - mb * KT;
    const int64_t m0 = mb * BM, k0 = kt * BK;
    TA* as = As + stage * S::a_stage_elems;
    double* bs = Bs + stage * S::b_stage_elems;
    if (!avec) {
      // unaligned rows: element-wise cp.async (same results, slower)
      for (int e = tid; e < BM * BK; e += GEMM_THREADS) {
        int r, cc; int64_t gm, gk;
        if (!TRANS) { r = e / BK; cc = e % BK; gm = m0 + r; gk = k0 + cc; }
        else { r = e / BM; cc = e % BM; gk = k0 + r; gm = m0 + cc; }
        const bool ok = gm < g.M && gk < g.K;
        const TA* src = ok ? (TRANS ? A + gk * g.lda + gm : A + gm * g.lda + gk) : A;
        TA* dst = TRANS ? as + r * A_TN_LD + cc : as + r * A_NN_LD + cc;
        if (sizeof(TA) == 8) cp_async8(dst, src, ok ? 8 : 0);
        else cp_async4(dst, src, ok ? 4 : 0);
      }
    } else {
#pragma unroll
      for (int c = 0; c < A_CHUNKS; ++c) {
        int64_t gm, gk, lim;
        if (!TRANS) { gm = m0 + a_r[c]; gk = k0 + a_c[c]; lim = g.K - gk; }
        else { gk = k0 + a_r[c]; gm = m0 + a_c[c]; lim = g.M - gm; }
        int valid = 0;
        if (gm < g.M && gk < g.K) valid = (int)(lim < EPC ? lim : EPC);
        const TA* src = valid ? A + (TRANS ? gk * g.lda + gm : gm * g.lda + gk) : A;
        cp_async16(as + a_r[c] * (TRANS ? A_TN_LD : A_NN_LD) + a_c[c], src, valid * (int)sizeof(TA));
      }
    }
    // B: BK rows x N cols (N % 16 == 0, ldb even => 16-byte chunks of 2 doubles)
    const int CPRB = N >> 1;
    for (int ch = tid; ch < BK * CPRB; ch += GEMM_THREADS) {
      const int r = ch / CPRB, cc = (ch - r * CPRB) * 2;
      const int64_t gk = k0 + r;
      const bool ok = gk < g.K;
      cp_async16(bs + r * ldbs + cc, ok ? g.B + gk * g.ldb + cc : g.B, ok ? 16 : 0);
    }
    if (!TRANS && CENT) {
      double* cs = Cs + stage * 2 * BK;
      if (tid < BK) {
        const int64_t gk = k0 + tid;
        cs[tid] = (centre && gk < g.K) ? g.c[gk] : 0.0;
        cs[BK + tid] = (scale && gk < g.K) ? g.rs[gk] : 1.0;
      }
    }
  };

  double acc[4][TMAX][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TMAX; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // TN centring: c / rs depend on the output row (= column of A)
  double crow[4], srow[4];
  auto set_rows = [&](int64_t m0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gm = m0 + wm * 32 + i * 8 + gq;
      crow[i] = (TRANS && centre && gm < g.M) ? g.c[gm] : 0.0;
      srow[i] = (TRANS && scale && gm < g.M) ? g.rs[gm] : 1.0;
    }
  };

  // In-kernel stream-K fix-up (deterministic, no FP64 atomics: SURVEY H4).  A
  // row-block segment is (i) the whole row block -> written directly; (ii) a
  // continuation (starts after the row block's first k-tile; always the CTA's
  // first segment) -> partial P[cta] + release flag; (iii) the head of a row
  // block that continues into later CTAs (always the CTA's last segment) ->
  // acquire the later CTAs' partials in CTA order, add, write.  Waits only
  // point to higher CTAs, which publish their partial first: no deadlock with
  // the whole grid resident (grid <= #SMs, one CTA per SM).
  auto epilogue = [&](int64_t mb, int64_t seg_start, int64_t seg_end) {
    const int64_t m0 = mb * BM;
    const int64_t rb_lo = mb * KT, rb_hi = rb_lo + KT;
    if (seg_start > rb_lo) {
      double* pb = g.P + (int64_t)blockIdx.x * BM * N;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rloc = wm * 32 + i * 8 + gq;
#pragma unroll
        for (int j = 0; j < TMAX; ++j) {
          const int col = (tile_begin + j) * 8 + 2 * tq;
          *reinterpret_cast<double2*>(pb + rloc * N + col) = make_double2(acc[i][j][0], acc[i][j][1]);
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(g.flags + blockIdx.x), "r"(epoch) : "memory");
      return;
    }
    if (seg_end < rb_hi) {
      for (int c = blockIdx.x + 1; c < g.grid && unit_lo(g.units, g.grid, c) < rb_hi; ++c) {
        unsigned f;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(g.flags + c) : "memory");
        } while (f != epoch);
        const double* pb = g.P + (int64_t)c * BM * N;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rloc = wm * 32 + i * 8 + gq;
#pragma unroll
          for (int j = 0; j < TMAX; ++j) {
            const int col = (tile_begin + j) * 8 + 2 * tq;
            const double2 v = *reinterpret_cast<const double2*>(pb + rloc * N + col);
            acc[i][j][0] += v.x;
            acc[i][j][1] += v.y;
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rloc = wm * 32 + i * 8 + gq;
      const int64_t gm = m0 + rloc;
#pragma unroll
      for (int j = 0; j < TMAX; ++j) {
        const int col = (tile_begin + j) * 8 + 2 * tq;
        if (gm < g.M) {
          if (col < g.Nout) g.C[gm * g.ldc + col] = acc[i][j][0];
          if (col + 1 < g.Nout) g.C[gm * g.ldc + col + 1] = acc[i][j][1];
        }
        acc[i][j][0] = acc[i][j][1] = 0.0;
      }
    }
  };

  if (CENT && TRANS && nun > 0) set_rows((u_lo / KT) * BM);

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nun) load_stage(s, u_lo + s);
    cp_async_commit();
  }

  for (int64_t it = 0; it < nun; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t pf = it + STAGES - 1;
      if (pf < nun) load_stage((int)(pf % STAGES), u_lo + pf);
      cp_async_commit();
    }
    const int stage = (int)(it % STAGES);
    const TA* as = As + stage * S::a_stage_elems;
    const double* bs = Bs + stage * S::b_stage_elems;
    const double* cs = Cs + stage * 2 * BK;
    // fragments for k-step kk + 4 are loaded (into the other register set)
    // before the DMMAs of k-step kk are issued: no register reuse stalls
    double af[2][4], bf[2][TMAX];
    auto load_frags = [&](int buf, int kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 32 + i * 8 + gq;
        double v;
        if (!TRANS) {
          v = (double)as[r * A_NN_LD + kk + tq];
          if (CENT) {
            if (centre) v -= cs[kk + tq];
            if (scale) v *= cs[BK + kk + tq];
          }
        } else {
          v = (double)as[(kk + tq) * A_TN_LD + r];
          if (CENT) {
            if (centre) v -= crow[i];
            if (scale) v *= srow[i];
          }
        }
        af[buf][i] = v;
      }
#pragma unroll
      for (int j = 0; j < TMAX; ++j) bf[buf][j] = bs[(kk + tq) * ldbs + (tile_begin + j) * 8 + gq];
    };
    load_frags(0, 0);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      if (ks + 1 < BK / 4) load_frags((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int j = 0; j < TMAX; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma884(acc[i][j][0], acc[i][j][1], af[ks & 1][i], bf[ks & 1][j]);
    }
    // end of a row-block segment: write it out (directly if this CTA covered
    // all of its k-tiles, else as a partial for the fix-up)
    const int64_t u = u_lo + it;
    const int64_t mb = u / KT, kt = u - mb * KT;
    if (kt == KT - 1 || it == nun - 1) {
      const int64_t seg_start = (mb * KT > u_lo) ? mb * KT : u_lo;
      epilogue(mb, seg_start, u + 1);
      if (CENT && TRANS && it + 1 < nun) set_rows((mb + 1) * BM);
    }
  }
  cp_async_wait<0>();
}

template <typename TA, bool TRANS, int TMAX>
static cudaError_t launch_one(const GemmArgs& g, cudaStream_t st) {
  const bool cent = g.c != nullptr || g.rs != nullptr;
  auto kfn = cent ? gemm_pass_kernel<TA, TRANS, TMAX, true> : gemm_pass_kernel<TA, TRANS, TMAX, false>;
  const size_t smem = GemmSmem<TA>::bytes;
  const cudaError_t e = smem_optin(kfn);
  if (e != cudaSuccess) return e;
  kfn<<<g.grid, GEMM_THREADS, smem, st>>>(g);
  return cudaGetLastError();
}

template <typename TA, bool TRANS>
static cudaError_t dispatch_tmax(const GemmArgs& g, cudaStream_t st) {
  switch (g.N / 16) {
    case 1: return launch_one<TA, TRANS, 1>(g, st);
    case 2: return launch_one<TA, TRANS, 2>(g, st);
    case 3: return launch_one<TA, TRANS, 3>(g, st);
    case 4: return launch_one<TA, TRANS, 4>(g, st);
    case 5: return launch_one<TA, TRANS, 5>(g, st);
    case 6: return launch_one<TA, TRANS, 6>(g, st);
    case 7: return launch_one<TA, TRANS, 7>(g, st);
    case 8: return launch_one<TA, TRANS, 8>(g, st);
    default: return cudaErrorInvalidValue;
  }
}

// persistent grid: one CTA per SM, but at least kMinUnits k-tiles per CTA so
// that the pipeline fill and the partial write-out stay amortised
constexpr int64_t kMinUnits = 8;
int gemm_choose_grid(int64_t M, int64_t K, int num_sms) {
  const int64_t mblocks = ceil_div(M, BM);
  const int64_t units = mblocks * ceil_div(K, BK);
  int64_t gsz = units / kMinUnits;
  if (gsz < mblocks) gsz = mblocks;                          // short K: one row block per CTA
  if (gsz > num_sms) gsz = num_sms;
  if (gsz < 1) gsz = 1;
  return (int)gsz;
}

size_t gemm_partial_bytes(int N, int grid) { return (size_t)grid * BM * (size_t)N * sizeof(double); }

cudaError_t gemm_pass(const GemmCall& c, cudaStream_t st) {
  if (c.N % 16 != 0 || c.N > NMAX || c.N < 16 || (c.ldb & 1)) return cudaErrorInvalidValue;
  if (c.M <= 0 || c.K <= 0) return cudaErrorInvalidValue;
  GemmArgs g;
  g.A = c.A; g.lda = c.lda; g.B = c.B; g.ldb = c.ldb; g.C = c.C; g.ldc = c.ldc; g.P = c.P;
  g.c = c.center; g.rs = c.rscale; g.M = c.M; g.K = c.K; g.N = c.N; g.Nout = c.Nout;
  g.flags = c.flags;
  g.KT = ceil_div(c.K, BK);
  g.units = ceil_div(c.M, BM) * g.KT;
  g.grid = gemm_choose_grid(c.M, c.K, c.grid > 0 ? c.grid : 148);
  {
    const size_t es = c.a_f32 ? 4 : 8;
    g.a_vec = ((uintptr_t)c.A % 16 == 0) && ((c.lda * es) % 16 == 0);
  }
  if (g.grid > 1 && (c.P == nullptr || c.flags == nullptr)) return cudaErrorInvalidValue;
  if (c.flags) {
    epoch_bump_kernel<<<1, 1, 0, st>>>(c.flags + kEpochSlot);
    ++g_kernel_launches;
  }
  cudaError_t e;
  if (c.a_f32) e = c.trans ? dispatch_tmax<float, true>(g, st) : dispatch_tmax<float, false>(g, st);
  else e = c.trans ? dispatch_tmax<double, true>(g, st) : dispatch_tmax<double, false>(g, st);
  ++g_kernel_launches;
  if (e != cudaSuccess) return e;
  return e;
}

}  // namespace rsvd
