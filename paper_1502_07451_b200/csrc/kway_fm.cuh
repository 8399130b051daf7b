// K5/K6 on small levels — CTA-resident Fiduccia–Mattheyses for the k-way
// partitioner (included by kway.cu; uses G, part_t and mix32 from there).
//
// The reference's partitioner is FM (partition.py:137-220): every pass moves
// vertices one at a time, best gain first, through negative-gain stretches,
// remembers the best prefix by the key (out of balance, cut) and rolls the
// rest back (partition.py:169-170, 206-219); a start comes from a greedy
// balanced fill (partition.py:223-255) under several orders
// (partition.py:280-295). This file is that algorithm generalised to k parts
// and to weighted coarse graphs, one CTA per candidate partition:
//
//   * candidate state lives on-chip: part ids and move locks in shared
//     memory, the connectivity rows conn[v][p] (weight of v's edges into part
//     p) in shared memory when n*k*4 bytes fit, else in global memory read
//     through L2 (ld.cg; updates are atomics, so L1 could hold stale lines);
//   * a step is one block-wide arg-max over every unlocked vertex of
//     (gain, per-pass hash) among the balance-admissible moves, then the
//     move's neighbour rows are updated by all threads;
//   * balance: part p must stay within [lo_p, hi_p]; a move is admissible
//     if the state after it is in bounds or strictly less out of bounds
//     (the k-way form of partition.py:193-196); prefix key = (violation,
//     cut) as partition.py:169-170;
//   * a pass stops after `stall` moves without a new best prefix (the
//     reference moves every vertex; the early stop is METIS's and changes
//     only how far a pass looks, not what it accepts);
//   * initial partitions: recursive bisection inside the CTA — greedy graph
//     growing from a hashed seed (frontier vertex of best gain first, stop at
//     the side's target weight) then 2-way FM passes, down to k parts — and
//     a final k-way FM over all parts. Candidates differ by their hash salt.
// Every sum is an integer and every tie breaks on a hash of (salt, vertex,
// pass), so a candidate is a pure function of (graph, start, salt).
#pragma once

constexpr int kFmThreads = 512;
constexpr int kFmMaxN = 4096;  // per-vertex state of a level lives in shared memory

struct FmArgs {
  G g;
  int k;
  const int64_t *hi, *lo;  // global k-way bounds [k]
  const double *cum;       // cumulative target fractions [k+1]
  double tol_split;        // relative slack of each bisection's sides
  part_t *parts;           // [C][n] candidate parts (in for refine, out always)
  int32_t *conn_g;         // [C][n*k] rows in global memory (null: shared memory)
  int32_t *trail;          // [C][n] moves of the current pass (v * 64 + old part)
  int64_t *cut;            // [C] out: integer cut (each undirected edge once)
  int64_t *viol;           // [C] out: total weight outside the k-way bounds
  int n_init;              // candidates [0, n_init) start from recursive bisection
  uint64_t salt;
  int passes, stall;
  long long *stats;        // [C][8] (HS_KWAY_TRACE): moves, passes, rolled back,
                           // scan clocks, move clocks, grow steps, total clocks
};

// shared-memory bytes of the per-vertex state (conn rows excluded):
// tie hash, weight (4 B), part, lock, dirty, best target (1 B)
__host__ __device__ constexpr int64_t fm_vertex_bytes(int n) {
  return 12 * (int64_t)((n + 15) & ~15);
}

struct FmCand {
  unsigned long long key;  // 0 = none
  int v, q;                // q = target | own << 8
};

__device__ __forceinline__ FmCand fm_better(const FmCand &a, const FmCand &b) {
  if (a.key != b.key) return a.key > b.key ? a : b;
  return a.v <= b.v ? a : b;
}

// Per-move cost. A step of the reference's FM is "the best admissible move
// of all unlocked vertices" (partition.py:176-200). Rescanning every
// (vertex, part) pair per move with the full violation arithmetic made a
// step cost ~20 us on a 3.6k-vertex level. Here every vertex keeps its best
// target by gain (bq: the lowest part of maximal connectivity), refreshed
// only when its row or its part changed (dirty flag, set by the move that
// changed it, cleared by the vertex's scanning thread). In the balanced state
// a move is admissible iff the vertex weight fits the own part's give and the
// target's room (two subtractions), so a vertex whose best target has room is
// decided with one row read; otherwise the full row is scanned with the same
// cheap test. The chosen move is exactly the full scan's. Every thread holds
// the pass scalars in registers (they follow from the broadcast winner), part
// weights alternate between two buffers, so a move costs one barrier for the
// arg-max and one after the neighbour rows are updated. Rollbacks touch
// distinct vertices (each moves at most once per pass) and run in parallel.
template <bool SM>
struct FmCta {
  const FmArgs &A;
  int n, k;
  part_t *part;     // shared
  uint8_t *lock;    // shared
  uint8_t *dirty;   // shared: best target stale
  uint8_t *bq;      // shared: best target by gain
  uint32_t *hs;     // shared: per-pass tie hash
  int32_t *vws;     // shared: vertex weights
  int32_t *conn;    // shared or global rows
  int32_t *trail;   // global
  int64_t *pw, *pw2, *bhi, *blo;  // shared [kMaxParts]
  FmCand *s_red;    // [2][32]
  int rb = 0;       // s_red buffer of the next reduction
  int32_t wmin = 0; // smallest vertex weight of the level
  int pa, pb;       // active pair (pa < 0: k-way)

  __device__ FmCta(const FmArgs &a) : A(a) {}

  __device__ __forceinline__ int32_t cget(int64_t i) const {
    if constexpr (SM) return conn[i];
    else return __ldcg(conn + i);
  }
  __device__ __forceinline__ void cadd(int64_t i, int32_t d) const { atomicAdd(conn + i, d); }

  __device__ __forceinline__ int64_t over(int p, int64_t x) const {
    int64_t o = 0;
    if (x > bhi[p]) o += x - bhi[p];
    if (x < blo[p]) o += blo[p] - x;
    return o;
  }
  __device__ __forceinline__ bool active(int p) const { return pa < 0 || p == pa || p == pb; }
  // total violation after moving weight w from `own` to `q` (part weights P)
  __device__ __forceinline__ int64_t viol_after(int64_t viol, const int64_t *P, int own, int q,
                                                int64_t w) const {
    return viol - over(own, P[own]) - over(q, P[q]) + over(own, P[own] - w) + over(q, P[q] + w);
  }
  __device__ int64_t viol_now() const {
    int64_t s = 0;
    for (int p = 0; p < k; ++p)
      if (active(p)) s += over(p, pw[p]);
    return s;
  }

  // block-wide arg-max; every thread gets the winner. One barrier: the
  // partials alternate between two buffers, so a reduction never overwrites
  // the slots a slow warp may still read from the previous one.
  __device__ FmCand reduce(FmCand c) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int off = 16; off; off >>= 1) {
      FmCand o;
      o.key = __shfl_xor_sync(0xffffffffu, c.key, off);
      o.v = __shfl_xor_sync(0xffffffffu, c.v, off);
      o.q = __shfl_xor_sync(0xffffffffu, c.q, off);
      c = fm_better(c, o);
    }
    FmCand *buf = s_red + rb * 32;
    rb ^= 1;
    if (lane == 0) buf[wid] = c;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    c = lane < nw ? buf[lane] : FmCand{0ull, INT_MAX, 0};
    for (int off = 16; off; off >>= 1) {
      FmCand o;
      o.key = __shfl_xor_sync(0xffffffffu, c.key, off);
      o.v = __shfl_xor_sync(0xffffffffu, c.v, off);
      o.q = __shfl_xor_sync(0xffffffffu, c.q, off);
      c = fm_better(c, o);
    }
    return c;
  }

  __device__ int64_t block_sum(int64_t x) {
    __shared__ long long s_sum[32];
    for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += s_sum[i];
      s_sum[0] = t;
    }
    __syncthreads();
    const int64_t r = s_sum[0];
    __syncthreads();
    return r;
  }

  // best target of v by gain (lowest part among the maximal rows)
  __device__ __forceinline__ void refresh(int v) {
    const int own = part[v];
    const int64_t r = (int64_t)v * k;
    int best = -1;
    int32_t cb = INT_MIN;
    for (int q = 0; q < k; ++q) {
      if (q == own) continue;
      const int32_t c = cget(r + q);
      if (c > cb) { cb = c; best = q; }
    }
    bq[v] = (uint8_t)best;
    dirty[v] = 0;
  }

  // neighbour rows of v for its move from -> to (threads t0, t0 + nt, ...)
  __device__ __forceinline__ void rows(int v, int from, int to, int t0, int nt) {
    const G &g = A.g;
    const int64_t b = g.xbeg[v];
    const int d = g.deg[v];
    for (int j = t0; j < d; j += nt) {
      const int u = __ldg(g.adj + b + j);
      const int w = g.ew(b + j);
      cadd((int64_t)u * k + from, -w);
      cadd((int64_t)u * k + to, w);
      dirty[u] = 1;
    }
  }

  // part[v]: from -> to. The caller synchronises afterwards.
  __device__ void move(int v, int from, int to) {
    if (threadIdx.x == 0) {
      const int64_t w = vws[v];
      part[v] = (part_t)to;
      pw[from] -= w;
      pw[to] += w;
      dirty[v] = 1;
    }
    rows(v, from, to, threadIdx.x, blockDim.x);
  }

  // conn rows, best targets and part weights from scratch
  __device__ void build() {
    const G &g = A.g;
    __shared__ int32_t s_wmin;
    for (int p = threadIdx.x; p < k; p += blockDim.x) pw[p] = 0;
    if (threadIdx.x == 0) s_wmin = INT_MAX;
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      int32_t *row = conn + (int64_t)v * k;
      for (int q = 0; q < k; ++q) row[q] = 0;
      const int64_t b = g.xbeg[v];
      const int d = g.deg[v];
      for (int j = 0; j < d; ++j) {
        const int u = __ldg(g.adj + b + j);
        row[part[u]] += g.ew(b + j);  // row v is this thread's alone
      }
      vws[v] = g.vw[v];
      atomicMin(&s_wmin, g.vw[v]);
      atomicAdd((unsigned long long *)&pw[part[v]], (unsigned long long)(int64_t)g.vw[v]);
    }
    __syncthreads();
    wmin = s_wmin;
    for (int v = threadIdx.x; v < n; v += blockDim.x) refresh(v);
    __syncthreads();
  }

  __device__ __forceinline__ uint32_t hsh(int v, int pass) const {
    return mix32(A.salt ^ ((uint64_t)(uint32_t)v * 0x9E3779B97F4A7C15ull) ^
                 ((uint64_t)(uint32_t)pass << 40));
  }

  __device__ __forceinline__ FmCand cand(int v, int own, int q, int64_t gain) const {
    FmCand c;
    c.key = ((unsigned long long)(gain + (1ll << 31)) << 32) | hs[v];
    c.v = v;
    c.q = q | own << 8;
    return c;
  }

  // best admissible move of this thread's vertices (violation viol, part
  // weights P): for each vertex the admissible target of largest gain,
  // lowest part id on ties; in the balanced state targets with an empty row
  // are skipped (partition.py:176-200 generalised to k parts)
  __device__ FmCand scan(int64_t viol, const int64_t *P) {
    FmCand best{0ull, INT_MAX, 0};
    // parts with room for the lightest vertex: the only possible targets in
    // the balanced state (usually a few: FM fills parts to their bounds)
    uint64_t roomy = 0;
    if (viol == 0 && pa < 0)
      for (int q = 0; q < k; ++q)
        if (bhi[q] - P[q] >= wmin) roomy |= 1ull << q;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      if (dirty[v]) refresh(v);
      if (lock[v]) continue;
      const int own = part[v];
      if (!active(own)) continue;
      const int64_t wv = vws[v];
      const int64_t r = (int64_t)v * k;
      if (pa >= 0) {  // 2-way step of a bisection: the pair's other side only
        const int q = own == pa ? pb : pa;
        const int32_t c_q = cget(r + q);
        if (viol == 0 && c_q == 0) continue;
        const int64_t nv = viol_after(viol, P, own, q, wv);
        if (!(nv == 0 || nv < viol)) continue;
        best = fm_better(best, cand(v, own, q, (int64_t)c_q - cget(r + own)));
        continue;
      }
      const int32_t c_own = cget(r + own);
      if (viol == 0) {
        if (wv > P[own] - blo[own]) continue;  // the own part cannot give wv
        const int qb = bq[v];
        const int32_t c_b = cget(r + qb);
        if (c_b == 0) continue;  // interior: every row to another part is 0
        if (wv <= bhi[qb] - P[qb]) {  // the best target has room: it is the answer
          best = fm_better(best, cand(v, own, qb, (int64_t)c_b - c_own));
          continue;
        }
        int q1 = -1;
        int32_t c1 = 0;
        // the other parts with room, ascending (strict > keeps the lowest id)
        for (uint64_t m = roomy & ~(1ull << own) & ~(1ull << qb); m; m &= m - 1) {
          const int q = __ffsll((long long)m) - 1;
          const int32_t c_q = cget(r + q);
          if (c_q > c1 && wv <= bhi[q] - P[q]) { c1 = c_q; q1 = q; }
        }
        if (q1 >= 0) best = fm_better(best, cand(v, own, q1, (int64_t)c1 - c_own));
        continue;
      }
      for (int q = 0; q < k; ++q) {  // out of balance: the violation test per target
        if (q == own) continue;
        const int64_t nv = viol_after(viol, P, own, q, wv);
        if (!(nv == 0 || nv < viol)) continue;
        best = fm_better(best, cand(v, own, q, (int64_t)cget(r + q) - c_own));
      }
    }
    return best;
  }

  // One FM pass (the active pair, or all parts); true if the prefix key
  // improved (partition.py:169-170, 206-219).
  __device__ bool pass(int pass_no) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      lock[v] = 0;
      hs[v] = hsh(v, pass_no);
    }
    __syncthreads();
    long long *st = A.stats ? A.stats + 8 * blockIdx.x : nullptr;
    if (st && threadIdx.x == 0) st[1] += 1;
    // every thread tracks the pass scalars (identical everywhere)
    int64_t viol = viol_now(), cur = 0, best_cur = 0, best_viol = viol;
    int moves = 0, best_len = 0, since = 0;
    int64_t *P = pw, *Q = pw2;
    while (true) {
      const long long t0 = st ? clock64() : 0;
      const FmCand c = reduce(scan(viol, P));
      if (st && threadIdx.x == 0) st[3] += clock64() - t0;
      if (c.key == 0ull) break;
      const int v = c.v, q = c.q & 0xff, own = c.q >> 8;
      const int64_t gain = (int64_t)(c.key >> 32) - (1ll << 31);
      const int64_t w = vws[v];
      viol = viol_after(viol, P, own, q, w);
      cur -= gain;
      ++moves;
      bool done = false;
      if (viol < best_viol || (viol == best_viol && cur < best_cur)) {
        best_viol = viol;
        best_cur = cur;
        best_len = moves;
        since = 0;
      } else if (++since > A.stall) {
        done = true;
      }
      for (int x = threadIdx.x; x < k; x += blockDim.x)
        Q[x] = P[x] - (x == own ? w : 0) + (x == q ? w : 0);
      if (threadIdx.x == 0) {
        lock[v] = 1;
        trail[moves - 1] = v * 64 + own;
        part[v] = (part_t)q;
        dirty[v] = 1;
      }
      const long long t1 = st ? clock64() : 0;
      rows(v, own, q, threadIdx.x, blockDim.x);
      __syncthreads();
      if (st && threadIdx.x == 0) {
        st[4] += clock64() - t1;
        st[0] += 1;
      }
      int64_t *t = P;
      P = Q;
      Q = t;
      if (done) break;
    }
    if (P != pw)
      for (int x = threadIdx.x; x < k; x += blockDim.x) pw[x] = P[x];
    __syncthreads();
    const int keep = best_len;
    if (st && threadIdx.x == 0) st[2] += moves - keep;
    // roll back the moves past the best prefix: distinct vertices, and row
    // updates commute, so one warp per move in parallel
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int m = keep + wid; m < moves; m += nw) {
      const int code = trail[m];
      const int v = code >> 6, old = code & 63;
      const int from = part[v];
      __syncwarp();  // every lane read part[v] before lane 0 rewrites it
      rows(v, from, old, lane, 32);
      if (lane == 0) {
        const unsigned long long w = (unsigned long long)(int64_t)vws[v];
        part[v] = (part_t)old;
        atomicAdd((unsigned long long *)&pw[from], 0ull - w);
        atomicAdd((unsigned long long *)&pw[old], w);
        dirty[v] = 1;
      }
    }
    __syncthreads();
    return keep > 0;
  }

  __device__ void refine(int passes, int pass0) {
    for (int p = 0; p < passes; ++p)
      if (!pass(pass0 + p)) break;
  }

  // Greedy graph growing of side b out of side a (the range's vertices all
  // hold part a): a hashed seed, then the best-gain frontier vertex, until b
  // holds its target weight.
  __device__ void grow(int a, int b, int64_t tgt_b, int salt_no) {
    while (true) {
      const bool first = pw[b] == 0;
      FmCand best{0ull, INT_MAX, 0};
      for (int v = threadIdx.x; v < n; v += blockDim.x) {
        if (part[v] != a) continue;
        FmCand c;
        if (first) {
          c.key = 1ull << 32 | hsh(v, salt_no);
        } else {
          const int32_t cb = cget((int64_t)v * k + b), ca = cget((int64_t)v * k + a);
          const int64_t gain = (int64_t)cb - ca;
          // frontier first (bit 63), then gain (31 bits), then the hash
          int64_t gc = gain + (1ll << 30);
          gc = gc < 0 ? 0 : (gc > (1ll << 31) - 1 ? (1ll << 31) - 1 : gc);
          const unsigned long long gb = (unsigned long long)gc;
          c.key = (cb > 0 ? 1ull << 63 : 0ull) | gb << 32 | hsh(v, salt_no);
        }
        c.v = v;
        c.q = b;
        best = fm_better(best, c);
      }
      FmCand c = reduce(best);
      if (c.key == 0ull) break;
      const int64_t w = vws[c.v];
      // stop when taking the vertex overshoots more than stopping undershoots
      const bool enough = !first && pw[b] + w - tgt_b > tgt_b - pw[b];
      __syncthreads();  // pw[b] read by every thread before move() changes it
      if (enough) break;
      move(c.v, a, b);
      __syncthreads();
      if (A.stats && threadIdx.x == 0) A.stats[8 * blockIdx.x + 5] += 1;
      if (pw[b] >= tgt_b) break;
    }
  }

  __device__ void bisect_all(int passes) {
    __shared__ int s_r0[2 * kMaxParts], s_r1[2 * kMaxParts];  // every range of the split tree: 2k - 1
    __shared__ int s_head, s_tail;
    if (threadIdx.x == 0) {
      s_r0[0] = 0;
      s_r1[0] = k;
      s_head = 0;
      s_tail = 1;
    }
    __syncthreads();
    int split_no = 0;
    while (s_head < s_tail) {
      const int p0 = s_r0[s_head], p1 = s_r1[s_head];
      __syncthreads();
      if (threadIdx.x == 0) ++s_head;
      if (p1 - p0 >= 2) {
        const int pm = p0 + (p1 - p0) / 2;
        const double ta = A.cum[pm] - A.cum[p0], tb = A.cum[p1] - A.cum[pm];
        const int64_t ws = pw[p0];
        const int64_t tgt_b = (int64_t)llround((double)ws * (tb / (ta + tb)));
        const int64_t tgt_a = ws - tgt_b;
        const int64_t slack = (int64_t)floor(A.tol_split * (double)ws);
        __syncthreads();
        if (threadIdx.x == 0) {
          bhi[p0] = tgt_a + slack;
          blo[p0] = tgt_a - slack;
          bhi[pm] = tgt_b + slack;
          blo[pm] = tgt_b - slack;
          s_r0[s_tail] = p0;
          s_r1[s_tail] = pm;
          s_r0[s_tail + 1] = pm;
          s_r1[s_tail + 1] = p1;
          s_tail += 2;
        }
        __syncthreads();
        grow(p0, pm, tgt_b, 1000 + split_no);
        pa = p0;
        pb = pm;
        refine(passes, 2000 + 64 * split_no);
        pa = pb = -1;
        ++split_no;
      }
      __syncthreads();
    }
  }

  __device__ void set_global_bounds() {
    for (int p = threadIdx.x; p < k; p += blockDim.x) {
      bhi[p] = A.hi[p];
      blo[p] = A.lo[p];
    }
    __syncthreads();
  }
};

template <bool SM>
__global__ void __launch_bounds__(kFmThreads) fm_kernel(FmArgs A) {
  extern __shared__ __align__(16) unsigned char fm_dyn[];
  __shared__ int64_t pw[kMaxParts], pw2[kMaxParts], bhi[kMaxParts], blo[kMaxParts];
  __shared__ FmCand s_red[64];
  const int n = A.g.n, k = A.k, c = blockIdx.x;
  const long long t_start = clock64();
  const int64_t n16 = (n + 15) & ~15;
  FmCta<SM> C(A);
  C.n = n;
  C.k = k;
  C.hs = (uint32_t *)fm_dyn;
  C.vws = (int32_t *)(fm_dyn + 4 * n16);
  C.part = (part_t *)(fm_dyn + 8 * n16);
  C.lock = fm_dyn + 9 * n16;
  C.dirty = fm_dyn + 10 * n16;
  C.bq = fm_dyn + 11 * n16;
  C.conn = SM ? (int32_t *)(fm_dyn + fm_vertex_bytes(n)) : A.conn_g + (int64_t)c * n * k;
  C.trail = A.trail + (int64_t)c * n;
  C.pw = pw; C.pw2 = pw2; C.bhi = bhi; C.blo = blo;
  C.s_red = s_red;
  C.pa = C.pb = -1;
  part_t *gp = A.parts + (int64_t)c * n;
  const bool init = c < A.n_init;
  for (int v = threadIdx.x; v < n; v += blockDim.x) C.part[v] = init ? (part_t)0 : gp[v];
  __syncthreads();
  C.build();
  if (init && k > 1) {
    C.bisect_all(A.passes);
    C.set_global_bounds();
  } else {
    C.set_global_bounds();
  }
  C.refine(A.passes, 0);
  // outputs: parts, cut (from the rows), violation
  int64_t cut2 = 0;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    const int own = C.part[v];
    gp[v] = C.part[v];
    for (int q = 0; q < k; ++q)
      if (q != own) cut2 += C.cget((int64_t)v * k + q);
  }
  cut2 = C.block_sum(cut2);
  if (threadIdx.x == 0) {
    int64_t vsum = 0;
    for (int p = 0; p < k; ++p) vsum += C.over(p, pw[p]);
    A.cut[c] = cut2 / 2;
    A.viol[c] = vsum;
    if (A.stats) A.stats[8 * c + 6] = clock64() - t_start;
  }
}

// winner = min (violation, cut, candidate index); copied into out
__global__ void fm_pick(const int64_t *viol, const int64_t *cut, int C, const part_t *parts, int n,
                        part_t *out, int32_t *winner) {
  __shared__ int s_best;
  if (threadIdx.x == 0) {
    int b = 0;
    for (int c = 1; c < C; ++c)
      if (viol[c] < viol[b] || (viol[c] == viol[b] && cut[c] < cut[b])) b = c;
    s_best = b;
    if (winner) *winner = b;
  }
  __syncthreads();
  const part_t *src = parts + (int64_t)s_best * n;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    out[v] = src[v];
}

__global__ void fm_fill_copies(const part_t *cur, int n, part_t *parts, int c0, int copies) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)copies * n;
       i += (int64_t)gridDim.x * blockDim.x)
    parts[(int64_t)c0 * n + i] = cur[i % n];
}

__global__ void fm_fill_starts(const int32_t *starts, int64_t count, part_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (part_t)starts[i];
}
