// K9 — execution of the tiled-Cholesky task DAG on one B200 (fp64).
//
// No reference counterpart: the reference only *simulates* these kernels
// (sim.py:135-164 with kernel_time from a calibration table). This is the
// "execution of the partitioned DAG" leg of the hot path (SURVEY §8(a) last
// row, App. D): the task DAG of gen.cholesky_tasks runs as ONE persistent
// kernel per GPU; every CTA pulls work items from device-side ready queues,
// and a finishing task releases its successors by atomic dependency counters.
//
// Layout: the matrix is stored as tiles of b x b (b = 512) doubles, tile
// (i, j) (i >= j) contiguous and row-major at tiles + (i*T + j)*b*b.
//
// Work items (all dense math on DMMA, mma.sync m16n8k8 f64 — fp64 has no
// tcgen05 kind; DMMA and DFMA both peak at ~37 TF/s measured on this part):
//   GEMM(i,j,k)  16 items: 128x128 block of A_ij -= A_ik A_jk^T (K = 512)
//   SYRK(i,k)    10 items: lower 128x128 blocks of A_ii -= A_ik A_ik^T
//   TRSM(i,k)     4 items: a 128-row block of A_ik <- A_ik L_kk^-T, by block
//                          columns: R = A - X L^T (GEMM), X = R Dinv^T (GEMM)
//   POTRF(k)      1 item : blocked Cholesky of A_kk by 128-column blocks
//                          (GEMM updates, 128x128 diagonal factor + inverse
//                          in shared memory, panel X = A Dinv^T), keeping
//                          the 4 inverted diagonal blocks Dinv[k] for TRSM.
// Operands stream into shared memory by TMA (cp.async.bulk.tensor, 128-byte
// hardware swizzle) through a ring of mbarrier-tracked stages: one thread
// issues a stage's two tile loads, every warp waits on the stage's full
// barrier and releases it on its empty barrier — no CTA-wide barrier per k
// chunk. Other data produced inside the kernel is read with L1-bypassing
// loads (ld.cg): L1 is not coherent across SMs; a proxy fence orders those
// generic-proxy writes before the async-proxy (TMA) reads.
#include "common.cuh"
#include <cuda.h>
#include <vector>

namespace {

constexpr int B = 512;        // tile size
constexpr int BB = 128;       // block size of the MMA engine
constexpr int KC = 16;        // k chunk per pipeline stage
constexpr int STAGES = 4;
constexpr int THREADS = 256;  // 8 warps: 2 (M) x 4 (N), warp tile 64 x 32
constexpr int STAGE_DBL = 2 * BB * KC;                 // A + B doubles per stage
constexpr int SMEM_GEMM = STAGES * STAGE_DBL * 8;      // 96 KB
constexpr unsigned STAGE_BYTES = STAGE_DBL * 8;        // 32 KB: two 128 x 16 fp64 boxes
constexpr int SMEM_DIAG = (BB * BB + 3 * 32 * 32) * 8;  // 152 KB (diagonal block + scratch)
constexpr int SMEM_BYTES = SMEM_DIAG > SMEM_GEMM ? SMEM_DIAG : SMEM_GEMM;

enum { K_POTRF = 0, K_TRSM = 1, K_SYRK = 2, K_GEMM = 3 };
constexpr int kMaxRanks = 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// element (r, k) of a [BB][KC] stage box written by TMA with the 128-byte
// swizzle: the 16-byte chunk k / 2 of row r sits at chunk (k / 2) ^ (r & 7),
// so the 8 rows x 4 columns of a fragment load hit 32 distinct doubles of
// the bank space (2 wavefronts, the minimum for 8-byte lanes)
__device__ __forceinline__ int sw(int r, int k) {
  return r * KC + ((((k >> 1) ^ (r & 7)) << 1) | (k & 1));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// The stage ring's barriers (static shared memory: the dynamic buffer is
// reused by the diagonal factor) and the CTA's running chunk count (the same
// in every thread): chunk g uses stage g % STAGES, parity (g / STAGES) & 1.
struct Pipe {
  uint64_t *full, *empty;
  uint32_t seq;
  const CUtensorMap *tm_tiles, *tm_dinv;
  const double *tiles, *dinv;
};

// TMA box coordinates (column, row) of the 128-row operand starting at p
// (tiles: ld = B, the 2D view [T*T*B][B]; Dinv blocks: ld = BB, [T*4*BB][BB])
__device__ __forceinline__ void box_of(const Pipe &P, const double *p, int ld,
                                       const CUtensorMap *&map, int &col, int &row) {
  const int64_t off = ld == B ? p - P.tiles : p - P.dinv;
  map = ld == B ? P.tm_tiles : P.tm_dinv;
  row = (int)(off / ld);
  col = (int)(off % ld);
}

// C[128x128] (ld ldc) = (mode 0) C - A B^T  |  (mode 1) A B^T, K % 16 == 0.
// A, B: pointers to row 0 of the 128-row operand blocks (in the tile array,
// ld = B, or among the inverted diagonal blocks, ld = BB). K may be 0 (no-op
// for mode 0). Ends with __syncthreads (safe to overwrite A/B/C after).
__device__ void mma_block(Pipe &P, double *smem, const double *A, int lda, const double *Bm,
                          int ldb, int K, double *C, int ldc, int mode) {
  if (K == 0 && mode == 0) return;  // nothing to subtract
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;
  const int nk = K / KC;
  const CUtensorMap *ma, *mb;
  int ca, ra, cbx, rbx;
  box_of(P, A, lda, ma, ca, ra);
  box_of(P, Bm, ldb, mb, cbx, rbx);
  const uint32_t g0 = P.seq;
  // chunk c of this block: A box (ca + c*KC, ra), B box (cbx + c*KC, rbx)
  auto issue = [&](int c) {
    const uint32_t g = g0 + c, st = g % STAGES;
    if (g >= STAGES) mbar_wait(P.empty + st, ((g / STAGES) & 1) ^ 1);  // slot released
    double *dst = smem + st * STAGE_DBL;
    mbar_expect_tx(P.full + st, STAGE_BYTES);
    tma_load_2d(dst, ma, ca + c * KC, ra, P.full + st);
    tma_load_2d(dst + BB * KC, mb, cbx + c * KC, rbx, P.full + st);
  };
  if (threadIdx.x == 0) {
    // generic-proxy writes (epilogues of this and other CTAs, the diagonal
    // factor's shared-memory use) before the async-proxy reads and writes
    asm volatile("fence.proxy.async;" ::: "memory");
    for (int c = 0; c < STAGES - 1 && c < nk; ++c) issue(c);
  }
  for (int kc = 0; kc < nk; ++kc) {
    if (threadIdx.x == 0 && kc + STAGES - 1 < nk) issue(kc + STAGES - 1);
    const uint32_t g = g0 + kc, st = g % STAGES;
    mbar_wait(P.full + st, (g / STAGES) & 1);
    const double *As = smem + st * STAGE_DBL, *Bs = As + BB * KC;
#pragma unroll
    for (int ks = 0; ks < KC; ks += 8) {
      double a[4][4], b[4][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r = wm + mt * 16 + gid;
        a[mt][0] = As[sw(r, ks + tig)];
        a[mt][1] = As[sw(r + 8, ks + tig)];
        a[mt][2] = As[sw(r, ks + tig + 4)];
        a[mt][3] = As[sw(r + 8, ks + tig + 4)];
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int r = wn + nt * 8 + gid;
        b[nt][0] = Bs[sw(r, ks + tig)];
        b[nt][1] = Bs[sw(r, ks + tig + 4)];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], a[mt], b[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(P.empty + st);  // this warp is done with the stage
  }
  P.seq = g0 + nk;
  __syncthreads();  // every read of A/B done before C (possibly aliasing A) is written
  // epilogue by 16-row slab: the slab's 8 loads of C are issued together
  // (one round trip instead of eight: a store may alias the next load, so
  // interleaved load/store pairs would serialise), then updated and stored
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    double2 o[4][2];
    if (mode == 0) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm + mt * 16 + gid + 8 * h, c = wn + nt * 8 + 2 * tig;
          o[nt][h] = __ldcg((const double2 *)(C + (size_t)r * ldc + c));
        }
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wm + mt * 16 + gid + 8 * h, c = wn + nt * 8 + 2 * tig;
        double2 v;
        if (mode == 0) {
          v.x = o[nt][h].x - acc[mt][nt][2 * h];
          v.y = o[nt][h].y - acc[mt][nt][2 * h + 1];
        } else {
          v.x = acc[mt][nt][2 * h];
          v.y = acc[mt][nt][2 * h + 1];
        }
        __stcg((double2 *)(C + (size_t)r * ldc + c), v);
      }
  }
  __syncthreads();
}

// 128x128 diagonal block in shared memory:
//  A) Cholesky, right-looking by columns with every thread (see below);
//  B) Dinv = L^-1: warp s inverts diagonal 32x32 block s (lane = column), then
//     off-diagonal 32x32 blocks by increasing distance d = bi - bj:
//     Linv[bi][bj] = -Linv[bi][bi] * sum_{m=bj}^{bi-1} L[bi][m] Linv[m][bj].
// L goes back to D (zeros above the diagonal), Dinv to global (128x128).
__device__ void diag_factor(double *sm, double *D, int ldd, double *Dinv, int *fail,
                            unsigned long long *st = nullptr) {
  long long t0 = clock64();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *scr = sm + BB * BB;
  for (int e = tid; e < BB * BB; e += THREADS) sm[e] = __ldcg(D + (size_t)(e / BB) * ldd + e % BB);
  __syncthreads();
  // A) right-looking column Cholesky, every thread on every column: each
  // thread takes the pivot's square root itself, scales its share of the
  // column below it (kept twice: in place, and as a contiguous vector for
  // conflict-free reads), then the rank-1 update of the trailing lower
  // triangle in 16 x 16 thread tiles: 2 barriers per column (the former
  // one-warp 32x32 factor + per-row panel solves took ~4x longer)
  double *colv = scr;  // [BB] the current column
  const int ti = tid >> 4, tl = tid & 15;
  for (int j = 0; j < BB; ++j) {
    double d = sm[j * BB + j];
    if (!(d > 0.0)) {
      if (tid == 0) *fail = 1;
      d = 1.0;
    }
    const double djj = sqrt(d);
    for (int i = j + 1 + tid; i < BB; i += THREADS) {
      const double v = sm[i * BB + j] / djj;
      sm[i * BB + j] = v;
      colv[i] = v;
    }
    __syncthreads();
    if (tid == 0) sm[j * BB + j] = djj;
    for (int i = j + 1 + ti; i < BB; i += 16) {
      const double lij = colv[i];
      for (int l = j + 1 + tl; l <= i; l += 16) sm[i * BB + l] -= lij * colv[l];
    }
    __syncthreads();
  }
  if (st && tid == 0) atomicAdd(st + 11, (unsigned long long)(clock64() - t0));
  t0 = clock64();
  for (int e = tid; e < BB * BB; e += THREADS) {
    const int i = e / BB, l = e % BB;
    __stcg(D + (size_t)i * ldd + l, l <= i ? sm[e] : 0.0);
  }
  // B1: diagonal blocks of the inverse (warp s, lane = column)
  if (warp < 4) {
    const int o = 32 * warp, c = lane;
    double x[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) x[r] = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      if (r < c) continue;
      double v = (r == c) ? 1.0 : 0.0;
      const double *lr = sm + (o + r) * BB + o;
#pragma unroll
      for (int m = 0; m < r; ++m)
        if (m >= c) v -= lr[m] * x[m];
      x[r] = v / lr[r];
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) __stcg(Dinv + (size_t)(o + r) * BB + o + c, x[r]);
  }
  // zero the strictly upper 32x32 blocks
  for (int e = tid; e < BB * BB; e += THREADS) {
    const int i = e / BB, l = e % BB;
    if ((l >> 5) > (i >> 5)) __stcg(Dinv + e, 0.0);
  }
  __threadfence_block();
  __syncthreads();
  if (st && tid == 0) atomicAdd(st + 12, (unsigned long long)(clock64() - t0));
  t0 = clock64();
  // B2: off-diagonal blocks by distance
  for (int d = 1; d < 4; ++d) {
    const int nb = 4 - d;
    // T_b = sum_{m = bj*32}^{bi*32 - 1} L[bi*32 + r][m] Linv[m][bj*32 + c]
    for (int e = tid; e < nb * 1024; e += THREADS) {
      const int b = e >> 10, r = (e >> 5) & 31, c = e & 31;
      const int bj = b, bi = b + d;
      const double *lr = sm + (bi * 32 + r) * BB;
      // 8 independent L2 reads in flight (Dinv was just written by this CTA)
      double acc = 0.0;
      for (int m0 = bj * 32; m0 < bi * 32; m0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(Dinv + (size_t)(m0 + u) * BB + bj * 32 + c);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += lr[m0 + u] * v[u];
      }
      scr[e] = acc;
    }
    __syncthreads();
    // Linv[bi][bj] = -Linv[bi][bi] T_b   (Linv[bi][bi] lower: q <= r)
    for (int e = tid; e < nb * 1024; e += THREADS) {
      const int b = e >> 10, r = (e >> 5) & 31, c = e & 31;
      const int bj = b, bi = b + d;
      double acc = 0.0;
      const double *lrow = Dinv + (size_t)(bi * 32 + r) * BB + bi * 32;
      for (int q0 = 0; q0 <= r; q0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = q0 + u <= r ? __ldcg(lrow + q0 + u) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u <= r) acc += v[u] * scr[(b << 10) + (q0 + u) * 32 + c];
      }
      __stcg(Dinv + (size_t)(bi * 32 + r) * BB + bj * 32 + c, -acc);
    }
    __threadfence_block();
    __syncthreads();
  }
  if (st && tid == 0) atomicAdd(st + 13, (unsigned long long)(clock64() - t0));
}

struct Task {
  int8_t kind;
  int16_t i, j, k;
};

struct ExecArgs {
  CUtensorMap tm_tiles;  // TMA view of the tiles: [T*T*B rows][B] fp64, box 128 x 16
  CUtensorMap tm_dinv;   // TMA view of the inverted diagonal blocks: [T*4*BB][BB]
  double *tiles;     // T*T tiles (lower used)
  double *dinv;      // T * 4 * 128*128 inverted diagonal blocks
  int T;
  int n_tasks;
  const int8_t *kind;
  const int16_t *ti, *tj, *tk;
  const int64_t *succ_ptr;
  const int32_t *succ;
  int32_t *pending;     // [n_tasks] unmet dependencies
  int32_t *items_left;  // [n_tasks]
  // two queues: 0 urgent (panel critical path), 1 normal
  int64_t *q[2];
  unsigned long long *head, *tail;  // [2] each
  unsigned long long *done;         // finished items
  unsigned long long total_items;
  int *fail;
  unsigned long long *stats;  // optional: [kind*2] cycles, [kind*2+1] items; [8..13] POTRF phases; [14] idle
  // partitioned execution (nranks > 1): tasks owned by other ranks are
  // completed there; their output tiles arrive by peer stores and their ids
  // through this rank's inbox ring
  int rank, nranks;
  const int8_t *owner;
  double *peer_tiles[kMaxRanks];
  double *peer_dinv[kMaxRanks];
  long long *peer_inbox[kMaxRanks];
  unsigned long long *peer_inbox_tail[kMaxRanks];
  long long *inbox;                 // own ring (= peer_inbox[rank])
  unsigned long long *inbox_tail;   // own (= peer_inbox_tail[rank])
  unsigned long long *inbox_head;   // own, local claims
  unsigned long long *copies;       // tiles sent (evidence: = K2 transfer count)
};

__device__ __forceinline__ int n_items_of(int kind) {
  return kind == K_POTRF ? 1 : kind == K_TRSM ? 4 : kind == K_SYRK ? 10 : 16;
}

__device__ __forceinline__ int urgent(const ExecArgs &E, int t) {
  const int kd = E.kind[t];
  return kd == K_POTRF || kd == K_TRSM || E.tj[t] == E.tk[t] + 1;
}

__device__ void push_task(const ExecArgs &E, int t) {
  const int qi = urgent(E, t) ? 0 : 1;
  const int n = n_items_of(E.kind[t]);
  const unsigned long long pos = atomicAdd(&E.tail[qi], (unsigned long long)n);
  for (int it = 0; it < n; ++it)
    atomicExch((unsigned long long *)&E.q[qi][pos + it], (unsigned long long)(((int64_t)t << 8) | it));
}

__device__ double *tile(const ExecArgs &E, int i, int j) {
  return E.tiles + ((size_t)i * E.T + j) * (size_t)B * B;
}

__device__ __forceinline__ void stat_add(const ExecArgs &E, int idx, unsigned long long v) {
  if (E.stats && threadIdx.x == 0) atomicAdd(&E.stats[idx], v);
}

__device__ void run_item(const ExecArgs &E, Pipe &P, double *smem, int t, int it) {
  const int kd = E.kind[t], i = E.ti[t], j = E.tj[t], k = E.tk[t];
  if (kd == K_GEMM) {
    const int rb = it >> 2, cb = it & 3;
    mma_block(P, smem, tile(E, i, k) + (size_t)rb * BB * B, B, tile(E, j, k) + (size_t)cb * BB * B, B,
              B, tile(E, i, j) + (size_t)rb * BB * B + cb * BB, B, 0);
  } else if (kd == K_SYRK) {
    // lower blocks (rb, cb), rb >= cb, enumerated row by row
    int rb = 0, rem = it;
    while (rem > rb) { rem -= rb + 1; ++rb; }
    const int cb = rem;
    mma_block(P, smem, tile(E, i, k) + (size_t)rb * BB * B, B, tile(E, i, k) + (size_t)cb * BB * B, B,
              B, tile(E, i, i) + (size_t)rb * BB * B + cb * BB, B, 0);
  } else if (kd == K_TRSM) {
    // row block rb of A_ik: X = A L_kk^-T by block columns
    const int rb = it;
    double *Aik = tile(E, i, k) + (size_t)rb * BB * B;
    const double *Lkk = tile(E, k, k);
    for (int cb = 0; cb < B / BB; ++cb) {
      // R = A[:, cb] - X[:, :cb] L[cb, :cb]^T
      mma_block(P, smem, Aik, B, Lkk + (size_t)cb * BB * B, B, cb * BB, Aik + cb * BB, B, 0);
      // X[:, cb] = R Dinv_cb^T (in place)
      mma_block(P, smem, Aik + cb * BB, B, E.dinv + ((size_t)k * 4 + cb) * BB * BB, BB, BB,
                Aik + cb * BB, B, 1);
    }
  } else {  // POTRF(k): blocked by 128 columns
    double *Akk = tile(E, k, k);
    for (int cb = 0; cb < B / BB; ++cb) {
      long long c0 = clock64();
      for (int rb = cb; rb < B / BB; ++rb)  // A[rb, cb] -= L[rb, :cb] L[cb, :cb]^T
        mma_block(P, smem, Akk + (size_t)rb * BB * B, B, Akk + (size_t)cb * BB * B, B, cb * BB,
                  Akk + (size_t)rb * BB * B + cb * BB, B, 0);
      long long c1 = clock64();
      double *dinv = E.dinv + ((size_t)k * 4 + cb) * BB * BB;
      diag_factor(smem, Akk + (size_t)cb * BB * B + cb * BB, B, dinv, E.fail, E.stats);
      long long c2 = clock64();
      for (int rb = cb + 1; rb < B / BB; ++rb)  // panel: X = A Dinv^T
        mma_block(P, smem, Akk + (size_t)rb * BB * B + cb * BB, B, dinv, BB, BB,
                  Akk + (size_t)rb * BB * B + cb * BB, B, 1);
      long long c3 = clock64();
      stat_add(E, 8, c1 - c0);
      stat_add(E, 9, c2 - c1);
      stat_add(E, 10, c3 - c2);
    }
  }
}

// releases the local successors of task t (any rank's task) — thread 0 only
__device__ void release_local(const ExecArgs &E, int t) {
  for (int64_t e = E.succ_ptr[t]; e < E.succ_ptr[t + 1]; ++e) {
    const int s = E.succ[e];
    if (E.nranks > 1 && E.owner[s] != E.rank) continue;
    if (atomicSub(&E.pending[s], 1) == 1) push_task(E, s);
  }
}

// output tile of task t: GEMM (i,j), SYRK (i,i), TRSM (i,k), POTRF (k,k)
__device__ __forceinline__ size_t out_tile_offset(const ExecArgs &E, int t) {
  const int kd = E.kind[t], i = E.ti[t], j = E.tj[t], k = E.tk[t];
  const int r = kd == K_POTRF ? k : i;
  const int c = kd == K_GEMM ? j : (kd == K_SYRK ? i : k);
  return ((size_t)r * E.T + c) * (size_t)B * B;
}

// all threads: copy t's output (and Dinv[k] for POTRF) into rank q's buffers
__device__ void send_output(const ExecArgs &E, int t, int q) {
  const size_t off = out_tile_offset(E, t);
  const double2 *src = (const double2 *)(E.tiles + off);
  double2 *dst = (double2 *)(E.peer_tiles[q] + off);
  for (int e = threadIdx.x; e < B * B / 2; e += THREADS) dst[e] = __ldcg(src + e);
  if (E.kind[t] == K_POTRF) {
    const size_t doff = (size_t)E.tk[t] * 4 * BB * BB;
    const double2 *ds = (const double2 *)(E.dinv + doff);
    double2 *dd = (double2 *)(E.peer_dinv[q] + doff);
    for (int e = threadIdx.x; e < 4 * BB * BB / 2; e += THREADS) dd[e] = __ldcg(ds + e);
  }
}

__global__ void __launch_bounds__(THREADS, 1) exec_kernel(const __grid_constant__ ExecArgs E) {
  extern __shared__ __align__(1024) double smem[];
  __shared__ __align__(8) uint64_t s_full[STAGES], s_empty[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Pipe P{s_full, s_empty, 0u, &E.tm_tiles, &E.tm_dinv, E.tiles, E.dinv};
  __shared__ long long s_item;
  __shared__ unsigned s_mask;
  while (true) {
    if (threadIdx.x == 0) {
      long long got = -1;
      int spins = 0;
      while (got < 0) {
        for (int qi = 0; qi < 2 && got < 0; ++qi) {
          unsigned long long h = *(volatile unsigned long long *)&E.head[qi];
          unsigned long long tl = *(volatile unsigned long long *)&E.tail[qi];
          if (h < tl && atomicCAS(&E.head[qi], h, h + 1) == h) {
            volatile long long *slot = (volatile long long *)&E.q[qi][h];
            long long v;
            while ((v = *slot) < 0) __nanosleep(20);
            got = v;
          }
        }
        if (got < 0 && E.nranks > 1) {  // remote completions: release local successors
          unsigned long long h = *(volatile unsigned long long *)E.inbox_head;
          unsigned long long tl = *(volatile unsigned long long *)E.inbox_tail;
          if (h < tl && atomicCAS(E.inbox_head, h, h + 1) == h) {
            volatile long long *slot = (volatile long long *)&E.inbox[h];
            long long v;
            int w = 0;
            while ((v = *slot) < 0 && ++w < (1 << 28)) __nanosleep(20);
            if (v < 0) { atomicMax(E.fail, 2); continue; }
            __threadfence_system();  // acquire: the peer's tile stores precede its post
            release_local(E, (int)v);
            continue;
          }
        }
        if (got < 0) {
          if (*(volatile unsigned long long *)E.done >= E.total_items) { got = -2; break; }
          if (*(volatile int *)E.fail >= 2) { got = -2; break; }  // another CTA gave up
          __nanosleep(spins < 64 ? 32 : 256);
          // watchdog: ~30 s without any work means a lost dependency (e.g. a
          // peer that never posts) — fail loudly instead of hanging the GPU
          if (++spins > (1 << 27)) {
            atomicMax(E.fail, 2);
            got = -2;
            break;
          }
        }
      }
      s_item = got;
    }
    __syncthreads();
    const long long item = s_item;
    __syncthreads();
    if (item == -2) break;
    const int t = (int)(item >> 8), it = (int)(item & 0xff);
    const long long c0 = clock64();
    run_item(E, P, smem, t, it);
    stat_add(E, E.kind[t] * 2, clock64() - c0);
    stat_add(E, E.kind[t] * 2 + 1, 1);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int last = atomicSub(&E.items_left[t], 1) == 1;
      unsigned mask = 0;
      if (last) {  // task complete: release successors, collect remote owners
        __threadfence();
        release_local(E, t);
        if (E.nranks > 1)
          for (int64_t e = E.succ_ptr[t]; e < E.succ_ptr[t + 1]; ++e) {
            const int q = E.owner[E.succ[e]];
            if (q != E.rank) mask |= 1u << q;
          }
      }

      s_mask = mask;
    }
    __syncthreads();
    if (s_mask) {  // one copy per (producer, destination rank), then post
      for (int q = 0; q < E.nranks; ++q)
        if ((s_mask >> q) & 1u) send_output(E, t, q);
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0)
        for (int q = 0; q < E.nranks; ++q)
          if ((s_mask >> q) & 1u) {
            const unsigned long long pos = atomicAdd_system(E.peer_inbox_tail[q], 1ull);
            atomicExch_system((unsigned long long *)&E.peer_inbox[q][pos], (unsigned long long)t);
            atomicAdd(E.copies, 1ull);
          }
    }
    if (threadIdx.x == 0) atomicAdd(E.done, 1ull);
  }
}

// tiled <-> row-major conversion (lower tiles only); blockIdx.y = tile
// TMA descriptors of the two operand arrays (driver entry point fetched
// through the runtime: no -lcuda link): 128 rows x 16 fp64 boxes, 128-byte
// swizzle, L2 promotion of 128-byte lines.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tensor_maps(ExecArgs *E, double *tiles, double *dinv, int T) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    HS_CHECK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    HS_REQUIRE(fn && q == cudaDriverEntryPointSuccess, HS_ECUDA, "cuTensorMapEncodeTiled missing");
    encode = (EncodeTiledFn)fn;
  }
  const cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)BB}, estr[2] = {1, 1};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)T * T * B};
    const cuuint64_t strides[1] = {(cuuint64_t)B * sizeof(double)};
    const CUresult r = encode(&E->tm_tiles, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, tiles, dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HS_REQUIRE(r == CUDA_SUCCESS, HS_ECUDA, "tile tensor map: CUresult %d", (int)r);
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)BB, (cuuint64_t)T * 4 * BB};
    const cuuint64_t strides[1] = {(cuuint64_t)BB * sizeof(double)};
    const CUresult r = encode(&E->tm_dinv, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dinv, dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HS_REQUIRE(r == CUDA_SUCCESS, HS_ECUDA, "Dinv tensor map: CUresult %d", (int)r);
  }
  return HS_OK;
}

__global__ void pack_kernel(double *A, int n, int T, double *tiles, int to_tiles) {
  const int tl = blockIdx.y;
  int ti = 0;
  while ((ti + 1) * (ti + 2) / 2 <= tl) ++ti;
  const int tj = tl - ti * (ti + 1) / 2;
  double *tp = tiles + ((size_t)ti * T + tj) * B * B;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B * B; e += gridDim.x * blockDim.x) {
    const int r = e / B, c = e % B;
    const size_t gi = (size_t)(ti * B + r) * n + (tj * B + c);
    if (to_tiles)
      tp[e] = A[gi];
    else
      A[gi] = (ti == tj && c > r) ? 0.0 : tp[e];
  }
}

}  // namespace

extern "C" int hs_chol_pack(double *A, int32_t n, int32_t b, double *tiles, int32_t to_tiles,
                            void *stream) {
  HS_REQUIRE(b == B && n % B == 0, HS_EINVAL, "tile size must be %d and divide n", B);
  const int T = n / B;
  cudaStream_t s = (cudaStream_t)stream;
  pack_kernel<<<dim3(16, T * (T + 1) / 2), 256, 0, s>>>(A, n, T, tiles, to_tiles);
  HS_CHECK_LAUNCH();
  return HS_OK;
}

extern "C" int hs_chol_execute(double *tiles, double *dinv, int32_t T, int32_t n_tasks,
                               const int8_t *kind, const int16_t *ti, const int16_t *tj,
                               const int16_t *tk, const int64_t *succ_ptr, const int32_t *succ,
                               const int32_t *indeg, int32_t grid_ctas, int32_t *fail_host,
                               void *stream) {
  return hs_chol_execute_stats(tiles, dinv, T, n_tasks, kind, ti, tj, tk, succ_ptr, succ, indeg,
                               grid_ctas, fail_host, nullptr, stream);
}

extern "C" int hs_chol_execute_stats(double *tiles, double *dinv, int32_t T, int32_t n_tasks,
                                     const int8_t *kind, const int16_t *ti, const int16_t *tj,
                                     const int16_t *tk, const int64_t *succ_ptr,
                                     const int32_t *succ, const int32_t *indeg, int32_t grid_ctas,
                                     int32_t *fail_host, unsigned long long *stats, void *stream) {
  return hs_chol_execute_part(tiles, dinv, T, n_tasks, kind, ti, tj, tk, succ_ptr, succ, indeg,
                              nullptr, grid_ctas, fail_host, stats, nullptr, stream);
}

extern "C" int hs_chol_execute_part(double *tiles, double *dinv, int32_t T, int32_t n_tasks,
                                    const int8_t *kind, const int16_t *ti, const int16_t *tj,
                                    const int16_t *tk, const int64_t *succ_ptr,
                                    const int32_t *succ, const int32_t *indeg,
                                    const hs_chol_peers_t *peers, int32_t grid_ctas,
                                    int32_t *fail_host, unsigned long long *stats,
                                    unsigned long long *copies_dev, void *stream) {
  HS_REQUIRE(tiles && dinv && kind && succ_ptr && indeg, HS_EINVAL, "hs_chol_execute: null argument");
  const int nranks = peers ? peers->nranks : 1;
  const int rank = peers ? peers->rank : 0;
  HS_REQUIRE(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks, HS_ELIMIT,
             "ranks must be 1..%d", kMaxRanks);
  HS_REQUIRE(nranks == 1 || (peers->owner && peers->inbox[rank] && peers->ctl[rank]), HS_EINVAL,
             "partitioned execution needs owner, inbox and ctl buffers");
  cudaStream_t s = (cudaStream_t)stream;
  // host copies of the small task table to size the queues and seed them
  std::vector<int8_t> hk(n_tasks), hown(n_tasks, 0);
  std::vector<int32_t> hin(n_tasks);
  std::vector<int16_t> hj(n_tasks), hkk(n_tasks);
  HS_CHECK_CUDA(cudaMemcpyAsync(hk.data(), kind, n_tasks, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(hin.data(), indeg, n_tasks * 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(hj.data(), tj, n_tasks * 2, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(hkk.data(), tk, n_tasks * 2, cudaMemcpyDeviceToHost, s));
  if (nranks > 1)
    HS_CHECK_CUDA(cudaMemcpyAsync(hown.data(), peers->owner, n_tasks, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  auto items = [](int kd) { return kd == K_POTRF ? 1 : kd == K_TRSM ? 4 : kd == K_SYRK ? 10 : 16; };
  unsigned long long cap[2] = {1, 1}, total = 0;
  std::vector<int64_t> q0, q1;  // seeds (owned tasks ready at start)
  std::vector<int32_t> left(n_tasks);
  for (int t = 0; t < n_tasks; ++t) {
    const int n = items(hk[t]);
    left[t] = n;
    if (hown[t] != rank) continue;
    const int qi = (hk[t] == K_POTRF || hk[t] == K_TRSM || hj[t] == hkk[t] + 1) ? 0 : 1;
    cap[qi] += n;
    total += n;
    if (hin[t] == 0)
      for (int it = 0; it < n; ++it) (qi ? q1 : q0).push_back(((int64_t)t << 8) | it);
  }
  hs::Scratch<int64_t> qa, qb;
  hs::Scratch<int32_t> pending, items_left, fail;
  hs::Scratch<unsigned long long> ctr;
  HS_CHECK_CUDA(qa.alloc(cap[0], s));
  HS_CHECK_CUDA(qb.alloc(cap[1], s));
  HS_CHECK_CUDA(pending.alloc(n_tasks, s));
  HS_CHECK_CUDA(items_left.alloc(n_tasks, s));
  HS_CHECK_CUDA(fail.alloc(1, s));
  HS_CHECK_CUDA(ctr.alloc(8, s));
  HS_CHECK_CUDA(cudaMemsetAsync(qa, 0xff, cap[0] * 8, s));
  HS_CHECK_CUDA(cudaMemsetAsync(qb, 0xff, cap[1] * 8, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(pending, indeg, n_tasks * 4, cudaMemcpyDeviceToDevice, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(items_left, left.data(), n_tasks * 4, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemsetAsync(fail, 0, 4, s));
  // head[2], tail[2], done, copies, -, -
  unsigned long long c0[8] = {0, 0, q0.size(), q1.size(), 0, 0, 0, 0};
  HS_CHECK_CUDA(cudaMemcpyAsync(ctr, c0, sizeof c0, cudaMemcpyHostToDevice, s));
  if (!q0.empty())
    HS_CHECK_CUDA(cudaMemcpyAsync(qa, q0.data(), q0.size() * 8, cudaMemcpyHostToDevice, s));
  if (!q1.empty())
    HS_CHECK_CUDA(cudaMemcpyAsync(qb, q1.data(), q1.size() * 8, cudaMemcpyHostToDevice, s));
  ExecArgs E;
  memset(&E, 0, sizeof E);
  {
    int rc = make_tensor_maps(&E, tiles, dinv, T);
    if (rc) return rc;
  }
  E.tiles = tiles; E.dinv = dinv; E.T = T; E.n_tasks = n_tasks;
  E.kind = kind; E.ti = ti; E.tj = tj; E.tk = tk; E.succ_ptr = succ_ptr; E.succ = succ;
  E.pending = pending; E.items_left = items_left;
  E.q[0] = qa; E.q[1] = qb;
  E.head = ctr.p; E.tail = ctr.p + 2; E.done = ctr.p + 4;
  E.copies = copies_dev ? copies_dev : ctr.p + 5;
  E.total_items = total;
  E.fail = fail;
  E.stats = stats;
  E.rank = rank;
  E.nranks = nranks;
  if (nranks > 1) {
    E.owner = peers->owner;
    for (int q = 0; q < nranks; ++q) {
      E.peer_tiles[q] = peers->tiles[q];
      E.peer_dinv[q] = peers->dinv[q];
      E.peer_inbox[q] = peers->inbox[q];
      E.peer_inbox_tail[q] = peers->ctl[q];
    }
    E.inbox = peers->inbox[rank];
    E.inbox_tail = peers->ctl[rank];
    E.inbox_head = peers->ctl[rank] + 1;
  }
  HS_CHECK_CUDA(cudaFuncSetAttribute(exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SMEM_BYTES));
  const int grid = grid_ctas > 0 ? grid_ctas : hs::sm_count();
  {
    hs::Prof P("cholesky_exec", s, 0.0);
    exec_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(E);
  }
  HS_CHECK_LAUNCH();
  if (fail_host) {  // synchronous only when the caller asks for the status
    int32_t f = 0;
    HS_CHECK_CUDA(cudaMemcpyAsync(&f, fail, 4, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    *fail_host = f;
    HS_REQUIRE(f < 2, HS_EDEADLOCK, "partitioned execution lost a dependency (watchdog)");
  }
  return HS_OK;
}

// IPC-shareable buffers are separate cudaMalloc allocations: a handle refers
// to an allocation's base, so sub-allocations (e.g. from a caching allocator)
// cannot be shared by pointer.
extern "C" int hs_ipc_alloc(int64_t bytes, void **dev_ptr) {
  HS_CHECK_CUDA(cudaMalloc(dev_ptr, bytes > 0 ? bytes : 1));
  return HS_OK;
}

extern "C" int hs_ipc_free(void *dev_ptr) {
  HS_CHECK_CUDA(cudaFree(dev_ptr));
  return HS_OK;
}

extern "C" int hs_memset_async(void *dev_ptr, int32_t byte_value, int64_t bytes, void *stream) {
  HS_CHECK_CUDA(cudaMemsetAsync(dev_ptr, byte_value, bytes, (cudaStream_t)stream));
  return HS_OK;
}

extern "C" int hs_ipc_handle(void *dev_ptr, char *handle64) {
  cudaIpcMemHandle_t h;
  HS_CHECK_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle64, &h, sizeof h);
  return HS_OK;
}

extern "C" int hs_ipc_open(const char *handle64, void **dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  HS_CHECK_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return HS_OK;
}

extern "C" int hs_ipc_close(void *dev_ptr) {
  HS_CHECK_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return HS_OK;
}
