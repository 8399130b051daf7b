// Team-per-vertex kernels of the k-way partitioner (included by kway.cu).
//
// A "team" is T consecutive lanes of a warp (T in {8, 16, 32}) working on
// one vertex; the host picks T from the level's average degree so that the
// fine levels (degree ~20) keep most lanes busy and the dense coarse levels
// use whole warps. Vertex loops advance warp-uniformly so every team of a
// warp takes part in the width-T shuffles.
#pragma once

template <int T>
__device__ __forceinline__ int team_lane() { return T == 1 ? 0 : (threadIdx.x & 31) % T; }

template <int T>
__device__ __forceinline__ int team_sum(int x) {
  for (int off = T / 2; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off, T);
  return x;  // valid in team lane 0
}

template <int T>
__device__ __forceinline__ unsigned long long team_sum64(unsigned long long x) {
  for (int off = T / 2; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off, T);
  return x;
}

template <int T>
__device__ __forceinline__ int team_or(int x) {
  for (int off = T / 2; off; off >>= 1) x |= __shfl_xor_sync(0xffffffffu, x, off, T);
  return x;  // valid in every lane
}

// arg-max over (gain, part): larger gain, then smaller part; bp < 0 = none
template <int T>
__device__ __forceinline__ void team_argmax(int &bg, int &bp) {
  for (int off = T / 2; off; off >>= 1) {
    int og = __shfl_down_sync(0xffffffffu, bg, off, T);
    int op = __shfl_down_sync(0xffffffffu, bp, off, T);
    if (op >= 0 && (bp < 0 || og > bg || (og == bg && op < bp))) { bg = og; bp = op; }
  }
}

// Warp-aggregated append: every lane calls it (uniformly); lanes with
// `take` get a slot in list[] (order unspecified, content deterministic).
__device__ __forceinline__ void warp_append(bool take, int value, int32_t *list, int32_t *count) {
  unsigned m = __ballot_sync(0xffffffffu, take);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int leader = __ffs(m) - 1, base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (take) list[base + __popc(m & ((1u << lane) - 1))] = value;
}

constexpr int kTeamBlock = 256;
constexpr int kAppendBuf = 256;  // per-warp staging slots for list appends

// Per-warp staged append: entries gather in shared memory and are flushed to
// the global list with one atomic per ~kAppendBuf entries (a global atomic
// per warp-iteration made the list counter an L2 hotspot).
struct WarpAppender {
  int32_t *buf;  // kAppendBuf slots of this warp
  int n = 0;     // warp-uniform fill level
  __device__ void push(bool take, int value, int32_t *list, int32_t *count) {
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    if (n + 32 > kAppendBuf) flush(list, count);
    if (take) buf[n + __popc(m & ((1u << lane) - 1))] = value;
    n += __popc(m);
    __syncwarp();
  }
  __device__ void flush(int32_t *list, int32_t *count) {
    if (!n) return;
    const int lane = threadIdx.x & 31;
    __syncwarp();
    int base = 0;
    if (lane == 0) base = atomicAdd(count, n);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane; i < n; i += 32) list[base + i] = buf[i];
    n = 0;
    __syncwarp();
  }
};

// Per-vertex refinement state packed in one word so the afterburner gathers
// 4 bytes per neighbour: part (bits 0-6), candidate part + 1 (bits 7-13, 0 =
// none), candidate gain clipped to [0, 2^18) (bits 14-31).
__device__ __forceinline__ uint32_t pack_state(int part, int cand, int gain) {
  uint32_t g = gain <= 0 ? 0u : (gain >= (1 << 18) ? (1u << 18) - 1 : (uint32_t)gain);
  return (g << 14) | ((uint32_t)(cand + 1) << 7) | (uint32_t)part;
}
__device__ __forceinline__ int st_part(uint32_t s) { return (int)(s & 127u); }
__device__ __forceinline__ int st_cand(uint32_t s) { return (int)((s >> 7) & 127u) - 1; }
__device__ __forceinline__ int st_gain(uint32_t s) { return (int)(s >> 14); }

// Candidate move per vertex (K6): best strictly positive gain into a part that
// can take it; candidates are appended to `list`.
// KR > 0: per-part connectivity lives in KR registers per lane (k <= KR),
// summed across the team with xor shuffles — no shared-memory atomics (those
// serialised whenever a vertex's neighbours share a part, the common case).
// KR == 0: shared-memory accumulators for larger k.
// U: adjacency entries in flight per lane (private-counter path).
template <int T, int KR, int U = 4>
__global__ void __launch_bounds__(kTeamBlock)
refine_cand_t(G g, const part_t *part, int k, const int64_t *pw, const int64_t *hi,
              const int64_t *lo, Rep<uint32_t> st, int32_t *list, int32_t *count,
              const int32_t *run, const part_t *gp, int32_t wconst, Conn cache,
              const int32_t *bands) {
  if (run && !*run) return;
  // bands (optional): the partition is still id-range bands (bands[q] = first
  // global id of part q, bands[k+1] != 0 when that holds): a neighbour's part
  // is then a 6-step search in shared memory instead of a gather
  __shared__ int32_t s_band[kMaxParts + 1];
  __shared__ int s_use_bands;
  if (threadIdx.x == 0) s_use_bands = bands != nullptr && bands[k + 1] != 0;
  if (bands)
    for (int p = threadIdx.x; p <= k; p += blockDim.x) s_band[p] = bands[p];
  __syncthreads();
  const bool use_bands = s_use_bands != 0;
  const bool bands_unit = use_bands && k <= 8 && wconst == 1 && gp == nullptr;
  // k <= 8: the bounds live in registers and a part is a sum of 7 compares
  int kb[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) kb[q] = (use_bands && q < k && k <= 8) ? s_band[q] : INT_MAX;
  auto part_of = [&](int u) -> int {
    if (!use_bands) return (int)__ldg(part + u);
    if (k <= 8) {
      int q = 0;
#pragma unroll
      for (int i = 1; i < 8; ++i) q += u >= kb[i];
      return q;
    }
    int q = 0;
    for (int st2 = 32; st2; st2 >>= 1)
      if (q + st2 < k && s_band[q + st2] <= u) q += st2;
    return q;
  };
  __shared__ int32_t conn_s[KR != 0 ? 1 : kTeamBlock / T][kMaxParts];
  // KR < 0: per-lane private counters, [part][thread] so every lane hits its
  // own bank; zeroed here and re-zeroed by the lanes that reduce them
  __shared__ int32_t priv_s[KR < 0 ? -KR : 1][kTeamBlock];
  if constexpr (KR < 0) {
    for (int i = threadIdx.x; i < (-KR) * kTeamBlock; i += blockDim.x) (&priv_s[0][0])[i] = 0;
  }
  // part weights and bounds are read for every vertex: keep them on chip
  // (global reads of these few lines made one L2 slice the bottleneck)
  __shared__ int64_t s_pw[kMaxParts], s_hi[kMaxParts], s_lo[kMaxParts];
  __shared__ int32_t s_app[kTeamBlock / 32][kAppendBuf];
  for (int p = threadIdx.x; p < k; p += blockDim.x) {
    s_pw[p] = pw[p];
    s_hi[p] = hi[p];
    s_lo[p] = lo[p];
  }
  __syncthreads();
  WarpAppender app{s_app[threadIdx.x >> 5]};
  const int lane = team_lane<T>();
  const int64_t step = (int64_t)warps_total() * (32 / T);
  for (int64_t vb = (int64_t)warp_id_global() * (32 / T); vb < g.n; vb += step) {
    const int v = (int)(vb + (threadIdx.x & 31) / T);
    const bool valid = v < g.n;
    int own = 0, bnd = 0, bg = 0, bp = -1;
    int32_t vwv = 0;
    int64_t b = 0;
    int d = 0;
    if (valid) {
      own = part[g.v0 + v];
      vwv = g.vw[v];
      b = g.xbeg[v];
      d = g.deg[v];
    }
    if constexpr (KR < 0) {
      const int tcol = threadIdx.x, base_col = threadIdx.x - lane;
      if (bands_unit) {
        // band start, unit weights, k <= 8: per-lane suffix counters in
        // registers (ge[i] = neighbours with id >= band i's start), summed
        // over the team with shuffles; every lane then holds the vertex's
        // eight part counts and picks the move itself (ascending parts,
        // strict >: the largest gain, ties to the smaller part, as
        // team_argmax) — no shared-memory columns, no per-part team loop
        int ge[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ge[i] = 0;
        for (int j0 = lane; j0 < d; j0 += U * T) {
          int u[U];
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int j = j0 + q * T;
            u[q] = j < d ? __ldg(g.adj + b + j) : -1;
          }
#pragma unroll
          for (int q = 0; q < U; ++q) {
            ge[0] += u[q] >= 0;
#pragma unroll
            for (int i = 1; i < 8; ++i) ge[i] += u[q] >= kb[i];
          }
        }
        int cnt[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          int x = ge[q] - (q < 7 ? ge[q + 1] : 0);
          for (int off = T / 2; off; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off, T);
          cnt[q] = q < k ? x : 0;
        }
        int cown = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cown = q == own ? cnt[q] : cown;
          bnd |= q != own && cnt[q] > 0;
        }
        const bool can = valid && bnd && s_pw[own] - vwv >= s_lo[own];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (can && q < k && q != own && s_pw[q] + vwv <= s_hi[q] && cnt[q] - cown > bg) {
            bg = cnt[q] - cown;
            bp = q;
          }
        }
        if (cache.p && valid) {
          if (cache.kc * cache.cw == 8 && cache.cw == 1) {  // one 8-byte row
            unsigned long long row = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) row |= (unsigned long long)(cnt[q] & 0xff) << (8 * q);
            if (lane == 0) st_keep2(reinterpret_cast<unsigned long long *>(cache.p) + v, row,
                                    l2_keep());
          } else {
            for (int q = lane; q < k; q += T) cache.set(v, q, cnt[q]);
          }
        }
      } else {
      for (int j0 = lane; j0 < d; j0 += U * T) {
        int w[U], p[U];
        if (gp) {
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int j = j0 + q * T;
            p[q] = j < d ? (int)gp[b + j] : -1;
            w[q] = j < d ? (wconst ? wconst : __ldg(g.wgt + b + j)) : 0;
          }
        } else {
          int u[U];
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int j = j0 + q * T;
            u[q] = j < d ? __ldg(g.adj + b + j) : -1;
            w[q] = j < d ? g.ew(b + j) : 0;
          }
#pragma unroll
          for (int q = 0; q < U; ++q) p[q] = u[q] >= 0 ? part_of(u[q]) : -1;
        }
#pragma unroll
        for (int q = 0; q < U; ++q)
          if (p[q] >= 0) {
            bnd |= p[q] != own;
            priv_s[p[q]][tcol] += w[q];
          }
      }
      __syncwarp();
      bnd = team_or<T>(bnd);
      // every lane reads the own-part row (rotated columns: distinct banks)
      int cown = 0;
      for (int c = 0; c < T; ++c) cown += priv_s[own][base_col + ((c + lane) & (T - 1))];
      __syncwarp();
      // lane handles parts lane, lane + T, ...: team total, then re-zero
      const bool can = valid && bnd && s_pw[own] - vwv >= s_lo[own];
      // 8-byte rows (8 one-byte counters, config 4): the team assembles the
      // row in registers and one lane stores it (one 8-byte store instead of
      // eight byte stores per vertex)
      const bool row8 = cache.p && cache.kc * cache.cw == 8 && cache.cw == 1;
      unsigned long long row = 0;
      for (int q = lane; q < k; q += T) {
        int cq = 0;
        for (int c = 0; c < T; ++c) {
          const int col = base_col + ((c + lane) & (T - 1));
          cq += priv_s[q][col];
          priv_s[q][col] = 0;
        }
        if (row8) row |= (unsigned long long)(cq & 0xff) << (8 * q);
        else if (cache.p && valid) cache.set(v, q, cq);  // connectivity cache row
        if (can && q != own && s_pw[q] + vwv <= s_hi[q]) {
          const int gain = cq - cown;
          if (gain > bg) { bg = gain; bp = q; }  // ascending q: ties keep the smaller part
        }
      }
      if (row8) {
        for (int off = T / 2; off; off >>= 1) row |= __shfl_xor_sync(0xffffffffu, row, off, T);
        if (valid && lane == 0) st_keep2(reinterpret_cast<unsigned long long *>(cache.p) + v, row,
                                         l2_keep());
      }
      __syncwarp();
      team_argmax<T>(bg, bp);
      }
    } else if constexpr (KR > 0) {
      // PK = 2: two 16-bit counters per register (host guarantees every
      // vertex's weighted degree < 2^16 on this level); PK = 1: 32-bit.
      constexpr int PK = KR == 8 ? 2 : 1;
      constexpr int NR = KR / PK;
      uint32_t c[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) c[i] = 0;
      // 4 neighbours per lane in flight: independent adj loads, then gathers
      for (int j0 = lane; j0 < d; j0 += 4 * T) {
        int w[4], p[4];
        if (gp) {  // ghost parts: one coalesced byte per entry, no gather
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = j0 + q * T;
            p[q] = j < d ? (int)gp[b + j] : own;
            w[q] = j < d ? (wconst ? wconst : __ldg(g.wgt + b + j)) : 0;
          }
        } else {
          int u[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = j0 + q * T;
            u[q] = j < d ? __ldg(g.adj + b + j) : -1;
            w[q] = j < d ? g.ew(b + j) : 0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) p[q] = u[q] >= 0 ? part_of(u[q]) : own;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bnd |= p[q] != own;
          const int idx = PK == 2 ? (p[q] >> 1) : p[q];
          const uint32_t val = PK == 2 ? ((uint32_t)w[q] << ((p[q] & 1) << 4)) : (uint32_t)w[q];
#pragma unroll
          for (int i = 0; i < NR; ++i) c[i] += (idx == i) ? val : 0u;
        }
      }
#pragma unroll
      for (int i = 0; i < NR; ++i)
        for (int off = T / 2; off; off >>= 1) c[i] += __shfl_xor_sync(0xffffffffu, c[i], off, T);
      bnd = team_or<T>(bnd);
      // lane q of the team evaluates parts q, q+T, ... (T >= 8 >= k for KR = 8)
      auto conn_of = [&](int p) -> int {
        uint32_t r = 0;
#pragma unroll
        for (int i = 0; i < NR; ++i) r = ((PK == 2 ? (p >> 1) : p) == i) ? c[i] : r;
        return PK == 2 ? (int)((r >> ((p & 1) << 4)) & 0xffffu) : (int)r;
      };
      if (valid && bnd && s_pw[own] - vwv >= s_lo[own]) {
        const int cown = conn_of(own);
        for (int pp = lane; pp < k; pp += T) {
          if (pp == own || s_pw[pp] + vwv > s_hi[pp]) continue;
          const int gain = conn_of(pp) - cown;
          if (gain > bg || (gain == bg && bp >= 0 && pp < bp)) { bg = gain; bp = pp; }
        }
      }
      team_argmax<T>(bg, bp);
    } else {
      int32_t *conn = conn_s[threadIdx.x / T];
      for (int p = lane; p < k; p += T) conn[p] = 0;
      __syncwarp();
      for (int j = lane; j < d; j += T) {
        int p = part_of(g.adj[b + j]);
        bnd |= p != own;
        atomicAdd(&conn[p], g.ew(b + j));
      }
      __syncwarp();
      bnd = team_or<T>(bnd);
      if (valid && bnd && s_pw[own] - vwv >= s_lo[own])
        for (int p = lane; p < k; p += T) {
          if (p == own || s_pw[p] + vwv > s_hi[p]) continue;
          int gain = conn[p] - conn[own];
          if (gain > bg || (gain == bg && bp >= 0 && p < bp)) { bg = gain; bp = p; }
        }
      team_argmax<T>(bg, bp);
      __syncwarp();
    }
    const bool writer = valid && lane == 0;
    const int c = (bp >= 0 && bg > 0) ? bp : -1;
    if (writer) st.put(g.v0 + v, pack_state(own, c, bg));
    app.push(writer && c >= 0, v, list, count);
  }
  app.flush(list, count);
}

// Candidate moves from the connectivity cache (cache[v][q] = weight of v's
// edges into part q, kept exact by every applied move): the same choice as
// refine_cand_t without scanning the adjacency. One thread per vertex.
template <int KC, int CW>
__global__ void __launch_bounds__(kTeamBlock, 6)  // <= 40 registers: the loop is latency-bound
refine_cached(G g, const part_t *part, int k, const int64_t *pw, const int64_t *hi,
              const int64_t *lo, Rep<uint32_t> st, int32_t *list, int32_t *count,
              const int32_t *run, const uint8_t *cache, int64_t *flows) {
  if (run && !*run) return;
  // room of every part in 32 bits (total vertex weight < 2^31): a move of
  // weight w may enter q iff w <= s_in[q] and leave p iff w <= s_out[p]
  __shared__ int32_t s_in[KC], s_out[KC];
  __shared__ unsigned long long sf[2 * KC];
  __shared__ int32_t s_app[kTeamBlock / 32][kAppendBuf];
  auto room = [](int64_t r) -> int32_t {
    return r < 0 ? -1 : (r > (int64_t)INT32_MAX ? INT32_MAX : (int32_t)r);
  };
  for (int p = threadIdx.x; p < KC; p += blockDim.x) {
    s_in[p] = p < k ? room(hi[p] - pw[p]) : -1;
    s_out[p] = p < k ? room(pw[p] - lo[p]) : -1;
  }
  for (int p = threadIdx.x; p < 2 * KC; p += blockDim.x) sf[p] = 0;
  __syncthreads();
  // flows != nullptr: the pre-plan's candidate flows, fused (register
  // counters per thread; a thread's partial sums stay below the total weight)
  uint32_t fo[KC], fi[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) fo[q] = fi[q] = 0;
  WarpAppender app{s_app[threadIdx.x >> 5]};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < g.n; base += stride) {
    const int v = (int)(base + threadIdx.x);
    const bool valid = v < g.n;
    int bg = 0, bp = -1, own = 0;
    if (valid) {
      own = part[g.v0 + v];
      const int32_t vwv = g.vw[v];
      int c[KC];
      conn_row<KC, CW>(cache, v, c);
      int cown = 0, other = 0;
#pragma unroll
      for (int q = 0; q < KC; ++q) {
        if (q == own) cown = c[q];
        else if (q < k) other |= c[q];
      }
      if (other && vwv <= s_out[own]) {
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          if (q == own || vwv > s_in[q]) continue;  // s_in = -1 past k
          const int gain = c[q] - cown;
          if (gain > bg) { bg = gain; bp = q; }
        }
      }
      if (flows && bp >= 0 && bg > 0) {
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          fo[q] += own == q ? (uint32_t)vwv : 0u;
          fi[q] += bp == q ? (uint32_t)vwv : 0u;
        }
      }
    }
    const int cand = (bp >= 0 && bg > 0) ? bp : -1;
    if (valid) st.put(g.v0 + v, pack_state(own, cand, bg));
    app.push(valid && cand >= 0, v, list, count);
  }
  app.flush(list, count);
  if (flows) {
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      unsigned long long a = fo[q], b = fi[q];
      for (int off = 16; off; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
      }
      if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(&sf[q], a);
        if (b) atomicAdd(&sf[KC + q], b);
      }
    }
    __syncthreads();
    for (int p = threadIdx.x; p < k; p += blockDim.x) {
      if (sf[p]) atomicAdd((unsigned long long *)&flows[p], sf[p]);
      if (sf[KC + p]) atomicAdd((unsigned long long *)&flows[k + p], sf[KC + p]);
    }
  }
}

// refine_cached for 8-byte cache rows (k <= 8, 1-byte counters) on one GPU,
// four consecutive vertices per thread and step: parts (4 x 1 B), vertex
// weights (16 B; none when every vertex weighs vconst), cache rows (2 x 16 B)
// and states (16 B) move as vector accesses. The scalar kernel is issue
// bound (ncu: 71% issue slots), so the best move is found with byte-SIMD:
// counters of the parts a move may enter (room >= weight) masked in two
// words, own part zeroed, max byte by __vmaxu4, first part holding it by
// __vcmpeq4 + ffs — the scalar loop's choice (strictly larger gain wins, so
// the smallest part among equal maxima). Same decisions and appended set.
__global__ void __launch_bounds__(kTeamBlock, 6)
refine_cached_v4(G g, const part_t *part, int k, const int64_t *pw, const int64_t *hi,
                 const int64_t *lo, uint32_t *st, int32_t *list, int32_t *count,
                 const int32_t *run, const uint8_t *cache, int64_t *flows, int32_t vconst) {
  constexpr int KC = 8;
  if (run && !*run) return;
  __shared__ int32_t s_in[KC], s_out[KC];
  __shared__ unsigned long long sf[2 * KC];
  __shared__ int32_t s_app[kTeamBlock / 32][kAppendBuf];
  auto room = [](int64_t r) -> int32_t {
    return r < 0 ? -1 : (r > (int64_t)INT32_MAX ? INT32_MAX : (int32_t)r);
  };
  for (int p = threadIdx.x; p < KC; p += blockDim.x) {
    s_in[p] = p < k ? room(hi[p] - pw[p]) : -1;
    s_out[p] = p < k ? room(pw[p] - lo[p]) : -1;
  }
  for (int p = threadIdx.x; p < 2 * KC; p += blockDim.x) sf[p] = 0;
  __syncthreads();
  int32_t in_[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) in_[q] = s_in[q];
  // byte masks of the parts a vertex of weight w may enter
  auto enter_mask = [&](int32_t w, uint32_t &mlo, uint32_t &mhi) {
    mlo = mhi = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (w <= in_[q]) mlo |= 0xffu << (8 * q);
      if (w <= in_[q + 4]) mhi |= 0xffu << (8 * q);
    }
  };
  uint32_t clo = 0, chi = 0;
  if (vconst) enter_mask(vconst, clo, chi);
  uint32_t fo[KC], fi[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) fo[q] = fi[q] = 0;
  WarpAppender app{s_app[threadIdx.x >> 5]};
  const int64_t n4 = ((int64_t)g.n + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n4; base += stride) {
    const int64_t t = base + threadIdx.x;
    const int v0 = (int)(4 * t);
    const bool full = v0 + 3 < g.n;
    uint32_t pk = 0, rw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int32_t vw4[4] = {vconst, vconst, vconst, vconst};
    if (full) {
      pk = __ldg(reinterpret_cast<const uint32_t *>(part) + t);
      if (!vconst) {
        const int4 w = __ldg(reinterpret_cast<const int4 *>(g.vw) + t);
        vw4[0] = w.x; vw4[1] = w.y; vw4[2] = w.z; vw4[3] = w.w;
      }
      const uint64_t keep = l2_keep();
      const uint4 a = ld_keep4(reinterpret_cast<const uint4 *>(cache) + 2 * t, keep);
      const uint4 b = ld_keep4(reinterpret_cast<const uint4 *>(cache) + 2 * t + 1, keep);
      rw[0] = a.x; rw[1] = a.y; rw[2] = a.z; rw[3] = a.w;
      rw[4] = b.x; rw[5] = b.y; rw[6] = b.z; rw[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int v = v0 + i;
        if (v < g.n) {
          pk |= (uint32_t)(uint8_t)part[v] << (8 * i);
          vw4[i] = g.vw[v];
          const uint2 x = __ldg(reinterpret_cast<const uint2 *>(cache) + v);
          rw[2 * i] = x.x;
          rw[2 * i + 1] = x.y;
        }
      }
    }
    uint32_t out[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int v = v0 + i;
      const bool valid = v < g.n;
      const int own = (int)((pk >> (8 * i)) & 0xffu);
      const uint32_t lo32 = rw[2 * i], hi32 = rw[2 * i + 1];
      const uint32_t own_lo = own < 4 ? 0xffu << (8 * own) : 0u;
      const uint32_t own_hi = own >= 4 ? 0xffu << (8 * (own - 4)) : 0u;
      const int cown = (int)(((own < 4 ? lo32 : hi32) >> (8 * (own & 3))) & 0xffu);
      const int32_t vwv = vw4[i];
      int bg = 0, bp = -1;
      // counters of parts >= k are never written (0): no k mask needed
      if (valid && ((lo32 & ~own_lo) | (hi32 & ~own_hi)) && vwv <= s_out[own]) {
        uint32_t mlo = clo, mhi = chi;
        if (!vconst) enter_mask(vwv, mlo, mhi);
        const uint32_t a = lo32 & mlo & ~own_lo, b = hi32 & mhi & ~own_hi;
        uint32_t x = __vmaxu4(a, b);
        x = __vmaxu4(x, x >> 16);
        x = __vmaxu4(x, x >> 8);
        const int m = (int)(x & 0xffu);
        if (m > cown) {
          const uint32_t rep = (uint32_t)m * 0x01010101u;
          const uint32_t ea = __vcmpeq4(a, rep), eb = __vcmpeq4(b, rep);
          bp = ea ? (__ffs(ea) - 1) >> 3 : 4 + ((__ffs(eb) - 1) >> 3);
          bg = m - cown;
        }
      }
      if (flows && bp >= 0) {
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          fo[q] += own == q ? (uint32_t)vwv : 0u;
          fi[q] += bp == q ? (uint32_t)vwv : 0u;
        }
      }
      out[i] = pack_state(own, bp, bg);
      app.push(valid && bp >= 0, v, list, count);
    }
    if (full) {
      reinterpret_cast<uint4 *>(st)[t] = make_uint4(out[0], out[1], out[2], out[3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (v0 + i < g.n) st[v0 + i] = out[i];
    }
  }
  app.flush(list, count);
  if (flows) {
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      unsigned long long a = fo[q], b = fi[q];
      for (int off = 16; off; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
      }
      if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(&sf[q], a);
        if (b) atomicAdd(&sf[KC + q], b);
      }
    }
    __syncthreads();
    for (int p = threadIdx.x; p < k; p += blockDim.x) {
      if (sf[p]) atomicAdd((unsigned long long *)&flows[p], sf[p]);
      if (sf[KC + p]) atomicAdd((unsigned long long *)&flows[k + p], sf[KC + p]);
    }
  }
}

// Cut from the connectivity cache: sum over vertices of the weight into other
// parts (each cut edge counted from both ends).
template <int KC, int CW>
__global__ void cut_cached(G g, const part_t *part, int k, const uint8_t *cache,
                           unsigned long long *cut2) {
  unsigned long long local = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int own = part[g.v0 + v];
    int c[KC];
    conn_row<KC, CW>(cache, v, c);
#pragma unroll
    for (int q = 0; q < KC; ++q)
      if (q < k && q != own) local += (unsigned long long)c[q];
  }
  for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cut2, local);
}

// Keeps the connectivity cache exact for one applied move of v (own -> dest).
__device__ __forceinline__ void cache_move(const G &g, const Conn &cache, int v, int own,
                                           int dest) {
  const int64_t b = g.xbeg[v];
  const int d = g.deg[v];
  for (int j = 0; j < d; ++j)
    cache.move(__ldg(g.adj + b + j) - g.v0, own, dest, g.ew(b + j));
}

// Warp-cooperative form: every lane calls it; lanes with v >= 0 moved v
// (own -> dest). The warp walks each moved vertex's list together
// (coalesced adjacency reads, parallel atomics).
__device__ __forceinline__ void cache_move_warp(const G &g, const Conn &cache, int v, int own,
                                                int dest) {
  unsigned m = __ballot_sync(0xffffffffu, v >= 0);
  const int lane = threadIdx.x & 31;
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int vv = __shfl_sync(0xffffffffu, v, src);
    const int o = __shfl_sync(0xffffffffu, own, src);
    const int de = __shfl_sync(0xffffffffu, dest, src);
    const int64_t b = g.xbeg[vv];
    const int d = g.deg[vv];
    for (int j = lane; j < d; j += 32) cache.move(__ldg(g.adj + b + j) - g.v0, o, de, g.ew(b + j));
  }
}

// The same, flattened: the warp's moved vertices' neighbour lists are one
// sequence (prefix of degrees in shared memory), so every lane works on every
// step and the adjacency loads of different vertices overlap instead of
// running vertex by vertex.
struct MoveScratch {
  int64_t b[8][32];
  int pre[8][32];
  int od[8][32];
};
__device__ __forceinline__ void cache_move_flat(const G &g, const Conn &cache, int v, int own,
                                                int dest, MoveScratch &ms) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int d = 0;
  int64_t b = 0;
  if (v >= 0) {
    b = g.xbeg[v];
    d = g.deg[v];
  }
  int inc = d;
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  const int tot = __shfl_sync(0xffffffffu, inc, 31);
  if (tot == 0) return;
  ms.b[w][lane] = b;
  ms.pre[w][lane] = inc - d;
  ms.od[w][lane] = (own << 16) | (dest & 0xffff);
  __syncwarp();
  // kU entries per lane in flight: the neighbour-id loads of one step are
  // independent, so their latencies overlap (the loop is load-latency bound)
  constexpr int kU = 4;
  for (int f0 = lane; f0 < tot; f0 += 32 * kU) {
    int64_t jj[kU];
    int odv[kU], uu[kU], ww[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int f = f0 + q * 32;
      jj[q] = -1;
      odv[q] = 0;
      if (f < tot) {
        int t = 0;
#pragma unroll
        for (int st = 16; st; st >>= 1)
          if (ms.pre[w][t + st] <= f) t += st;
        jj[q] = ms.b[w][t] + (f - ms.pre[w][t]);
        odv[q] = ms.od[w][t];
      }
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      uu[q] = jj[q] >= 0 ? ld_once(g.adj + jj[q]) : 0;
      ww[q] = jj[q] >= 0 ? g.ew(jj[q]) : 0;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q)
      if (jj[q] >= 0) cache.move(uu[q] - g.v0, odv[q] >> 16, odv[q] & 0xffff, ww[q]);
  }
  __syncwarp();
}

// Warp-aggregated s[key] += val over the lanes with key >= 0 (one shared
// atomic per distinct key instead of one per lane; |partial sums| < 2^31
// because the total vertex weight is).
__device__ __forceinline__ void warp_add_by_key(long long *s, int key, int val) {
  unsigned rem = __ballot_sync(0xffffffffu, key >= 0);
  while (rem) {
    const int src = __ffs(rem) - 1;
    const int kk = __shfl_sync(0xffffffffu, key, src);
    const unsigned grp = __ballot_sync(0xffffffffu, key == kk);
    const int sum = __reduce_add_sync(0xffffffffu, key == kk ? val : 0);
    if ((threadIdx.x & 31) == src) atomicAdd((unsigned long long *)&s[kk], (unsigned long long)(long long)sum);
    rem &= ~grp;
  }
}

// Jet-style afterburner over the candidate list: a move survives only if it
// still gains assuming every higher-priority (gain, then smaller id)
// neighbouring candidate moved. Confirmed moves land in conf[i] and in the
// planned flows (flows[p] out of p, flows[k+q] into q); nconf counts them.
template <int T>
__global__ void __launch_bounds__(kTeamBlock, 6)  // <= 40 registers: occupancy for the gathers
afterburner_t(G g, const uint32_t *st, const int32_t *list, const int32_t *count, int k,
              int32_t *conf, int64_t *flows, int32_t *nconf, const int32_t *run) {
  if (run && !*run) return;
  __shared__ unsigned long long sf[2 * kMaxParts];
  __shared__ int s_n;
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) sf[p] = 0;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const int lane = team_lane<T>();
  const int total = *count;
  const int64_t step = (int64_t)warps_total() * (32 / T);
  int local = 0;
  for (int64_t ib = (int64_t)warp_id_global() * (32 / T); ib < total; ib += step) {
    const int64_t i = ib + (threadIdx.x & 31) / T;
    const bool valid = i < total;
    int delta = 0, v = 0, dest = -1, own = 0;
    if (valid) v = list[i];
    const bool live = valid && v >= 0;  // v < 0: dropped by the pre-plan thinning
    if (live) {
      const uint32_t sv = st[g.v0 + v];
      dest = st_cand(sv);
      own = st_part(sv);
      const int gv = st_gain(sv);
      const int64_t b = g.xbeg[v];
      const int d = g.deg[v];
      constexpr int AU = 4;  // entries in flight per lane (8 spills under the 40-register cap)
      for (int j0 = lane; j0 < d; j0 += AU * T) {
        int u[AU], w[AU];
        uint32_t su[AU];
#pragma unroll
        for (int q = 0; q < AU; ++q) {
          const int j = j0 + q * T;
          u[q] = j < d ? ld_once(g.adj + b + j) : -1;
          w[q] = j < d ? g.ew(b + j) : 0;
        }
#pragma unroll
        for (int q = 0; q < AU; ++q) su[q] = u[q] >= 0 ? __ldg(st + u[q]) : 0u;
#pragma unroll
        for (int q = 0; q < AU; ++q) {
          if (u[q] < 0) continue;
          int pu = st_part(su[q]);
          const int cu = st_cand(su[q]);
          if (cu >= 0) {
            const int gu = st_gain(su[q]);
            if (gu > gv || (gu == gv && u[q] < g.v0 + v)) pu = cu;
          }
          delta += (pu == dest ? w[q] : 0) - (pu == own ? w[q] : 0);
        }
      }
    }
    delta = team_sum<T>(delta);
    if (valid && lane == 0) {
      const bool ok = live && delta > 0;
      conf[i] = ok ? dest : -1;
      if (ok) {
        const unsigned long long w = (unsigned long long)g.vw[v];
        atomicAdd(&sf[own], w);
        atomicAdd(&sf[k + dest], w);
        ++local;
      }
    }
  }
  if (local) atomicAdd(&s_n, local);
  __syncthreads();
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x)
    if (sf[p]) atomicAdd((unsigned long long *)&flows[p], sf[p]);
  if (threadIdx.x == 0 && s_n) atomicAdd(nconf, s_n);
}

// First id of every part when the parts are non-decreasing in the vertex id
// (the band start of `range_parts`): bands[q] for q < k, bands[k] = n, and
// bands[k+1] cleared if some part[v] < part[v-1]. Caller sets bands[k+1] != 0.
__global__ void band_starts(int n, const part_t *part, int k, int32_t *bands) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int a = v == 0 ? -1 : (int)part[v - 1], b = part[v];
    if (b < a) bands[k + 1] = 0;
    for (int q = a + 1; q <= b; ++q) bands[q] = (int32_t)v;
    if (v == n - 1)
      for (int q = b + 1; q <= k; ++q) bands[q] = n;
  }
}

// Pre-plan of a refinement pass: the part flows every candidate
// would cause, before the afterburner... k <= KC: per-thread register
// counters (selects, no indexing), warp-reduced, one shared atomic per warp
// and counter (shared atomics on k addresses serialised: 0.25 ms a pass).
template <int KC>
__global__ void __launch_bounds__(256) cand_flows_reg(const uint32_t *st, const int32_t *list,
                                                      const int32_t *count, const int32_t *vw,
                                                      int k, int64_t *flows, const int32_t *run,
                                                      int32_t v0) {
  if (run && !*run) return;
  __shared__ unsigned long long sf[2 * KC];
  for (int p = threadIdx.x; p < 2 * KC; p += blockDim.x) sf[p] = 0;
  __syncthreads();
  unsigned long long out[KC], in[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) out[q] = in[q] = 0;
  const int total = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = list[i];
    const uint32_t sv = st[v0 + v];
    const unsigned long long w = (unsigned long long)vw[v];
    const int own = st_part(sv), dest = st_cand(sv);
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      out[q] += own == q ? w : 0ull;
      in[q] += dest == q ? w : 0ull;
    }
  }
#pragma unroll
  for (int q = 0; q < KC; ++q) {
    for (int off = 16; off; off >>= 1) {
      out[q] += __shfl_down_sync(0xffffffffu, out[q], off);
      in[q] += __shfl_down_sync(0xffffffffu, in[q], off);
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      if (out[q]) atomicAdd(&sf[q], out[q]);
      if (in[q]) atomicAdd(&sf[KC + q], in[q]);
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < k; p += blockDim.x) {
    if (sf[p]) atomicAdd((unsigned long long *)&flows[p], sf[p]);
    if (sf[KC + p]) atomicAdd((unsigned long long *)&flows[k + p], sf[KC + p]);
  }
}

__global__ void cand_flows(const uint32_t *st, const int32_t *list, const int32_t *count,
                           const int32_t *vw, int k, int64_t *flows, const int32_t *run,
                           int32_t v0) {
  if (run && !*run) return;
  __shared__ unsigned long long sf[2 * kMaxParts];
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) sf[p] = 0;
  __syncthreads();
  const int total = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = list[i];
    const uint32_t sv = st[v0 + v];
    const unsigned long long w = (unsigned long long)vw[v];
    atomicAdd(&sf[st_part(sv)], w);
    atomicAdd(&sf[k + st_cand(sv)], w);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x)
    if (sf[p]) atomicAdd((unsigned long long *)&flows[p], sf[p]);
}

// ...and the thinning it implies, applied to the candidates themselves: a
// candidate is kept with probability prob[own] * prob[k + dest] (hash coin of
// (salt, v)); a dropped one loses its candidate mark (neighbours see it stay),
// kept ones are compacted into kept[] (order irrelevant: the afterburner and
// apply work per entry), so the afterburner neither evaluates dropped moves
// nor assumes they happen.
__global__ void thin_cands(Rep<uint32_t> st, int32_t v0, const int32_t *list, const int32_t *count,
                           const double *prob, int k, uint64_t salt, const int32_t *run,
                           int32_t *kept, int32_t *kept_count, int64_t *flows) {
  // flows (read by the pre-plan, which has finished) are zeroed here for the
  // afterburner's confirmed-move sums
  if (blockIdx.x == 0)
    for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) flows[p] = 0;
  if (run && !*run) return;
  __shared__ double s_prob[2 * kMaxParts];
  __shared__ int32_t s_app[8][kAppendBuf];  // 256 threads
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) s_prob[p] = prob[p];
  __syncthreads();
  WarpAppender app{s_app[threadIdx.x >> 5]};
  const int total = *count;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < total; base += stride) {
    const int64_t i = base + threadIdx.x;  // warp-uniform trip count (appender)
    int v = -1;
    bool keep = false;
    if (i < total) {
      v = list[i];
      const uint32_t sv = st.p[0][v0 + v];
      const double pr = s_prob[st_part(sv)] * s_prob[k + st_cand(sv)];
      const uint64_t gv = (uint64_t)(v0 + v);
      keep = pr >= 1.0 ||
             (double)mix32(salt ^ (gv * 0x9E3779B97F4A7C15ull)) < pr * 4294967296.0;
      if (!keep) st.put(gv, sv & 127u);  // own part, no candidate (every replica)
    }
    app.push(keep, v, kept, kept_count);
  }
  app.flush(kept, kept_count);
}

// Applies confirmed moves of the list, each kept with probability
// prob[own] * prob[k + dest] (hash of (salt, v): deterministic thinning).
__global__ void apply_list(const int32_t *list, const int32_t *count, const int32_t *conf,
                           const int32_t *vw, const double *prob, int k, uint64_t salt,
                           int32_t v0, const part_t *part, Rep<part_t> prep, int64_t *pw,
                           const int32_t *run, const int64_t *xbeg, const int32_t *deg,
                           const int32_t *twin, part_t *gp, G g, Conn cache,
                           int32_t *moved) {
  if (run && !*run) return;
  __shared__ long long s[kMaxParts];
  __shared__ double s_prob[2 * kMaxParts];
  __shared__ MoveScratch ms;  // 256 threads = 8 warps
  for (int p = threadIdx.x; p < k; p += blockDim.x) s[p] = 0;
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) s_prob[p] = prob[p];
  __syncthreads();
  const int total = *count;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < total; base += stride) {
    const int64_t i = base + threadIdx.x;  // warp-uniform trip count (cache updates below)
    int v = -1, own = 0, dest = i < total ? conf[i] : -1;
    if (dest >= 0) {
      v = list[i];
      own = part[v0 + v];
      const double pr = s_prob[own] * s_prob[k + dest];
      const uint64_t gv = (uint64_t)(v0 + v);
      if (pr < 1.0 && (double)mix32(salt ^ (gv * 0x9E3779B97F4A7C15ull)) >= pr * 4294967296.0)
        v = -1;
    }
    int wv = 0;
    if (v >= 0) {
      prep.put(v0 + v, (part_t)dest);
      if (gp)  // keep the ghost copies in the neighbours' lists current
        for (int64_t j = xbeg[v], e = xbeg[v] + deg[v]; j < e; ++j) gp[twin[j]] = (part_t)dest;
      wv = vw[v];
    }
    if (moved) {  // profiling: applied moves (warp-aggregated)
      const unsigned mm = __ballot_sync(0xffffffffu, v >= 0);
      if ((threadIdx.x & 31) == 0 && mm) atomicAdd(moved, __popc(mm));
    }
    warp_add_by_key(s, v >= 0 ? dest : -1, wv);
    warp_add_by_key(s, v >= 0 ? own : -1, -wv);
    if (cache.p) cache_move_flat(g, cache, v, own, dest, ms);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < k; p += blockDim.x)
    if (s[p]) atomicAdd((unsigned long long *)&pw[p], (unsigned long long)s[p]);
}

// Heavy-edge proposals (K3) with teams: prop[u] = best unmatched neighbour,
// fav[u] = best neighbour overall (for two-hop pairing).
// list != nullptr: only the *count vertices of list (the still-unmatched
// ones after round 0) are visited.
template <int T>
__global__ void __launch_bounds__(kTeamBlock)
propose_t(G g, const uint32_t *mw, int32_t *prop, int32_t *fav, uint64_t salt,
          int32_t max_vw, const int32_t *list, const int32_t *count, int32_t vconst,
          bool uniform) {
  const int lane = team_lane<T>();
  const int64_t step = (int64_t)warps_total() * (32 / T);
  const int nv = list ? *count : g.n;
  for (int64_t ub = (int64_t)warp_id_global() * (32 / T); ub < nv; ub += step) {
    const int ui = (int)(ub + (threadIdx.x & 31) / T);
    const int u = ui < nv ? (list ? list[ui] : ui) : g.n;
    const bool live = u < g.n && !(mw[u] >> 31);
    float br = -1.f, fr = -1.f;
    int bv = -1, fv = -1;
    uint32_t bh = 0, fh = 0;
    if (live) {
      const int64_t b = g.xbeg[u];
      const int d = g.deg[u];
      const int32_t vu = (int32_t)(mw[u] & 0x7fffffffu);
      constexpr int PU = 2;  // entries in flight per lane (4 measured no faster)
      for (int j0 = lane; j0 < d; j0 += PU * T) {
        int vq[PU], wq[PU];
        uint32_t mq[PU];
#pragma unroll
        for (int q = 0; q < PU; ++q) {
          const int j = j0 + q * T;
          vq[q] = j < d ? __ldg(g.adj + b + j) - g.v0 : -1;  // local index
          wq[q] = j < d ? g.ew(b + j) : 0;
        }
        // vconst != 0: first round with uniform vertex weights — every vertex
        // is unmatched and weighs vconst, so no per-neighbour gather
#pragma unroll
        for (int q = 0; q < PU; ++q)
          mq[q] = (unsigned)vq[q] < (unsigned)g.n ? (vconst ? (uint32_t)vconst : __ldg(mw + vq[q]))
                                                  : 0x80000000u;
#pragma unroll
        for (int q = 0; q < PU; ++q) {
        const int v = vq[q];
        // sharded: matching pairs vertices of one rank only (local contraction)
        if ((unsigned)v >= (unsigned)g.n || v == u) continue;
        const uint32_t wv = mq[q];
        const int32_t vv = (int32_t)(wv & 0x7fffffffu);
        if (vu + vv > max_vw) continue;
        // uniform edge and vertex weights: every rating is equal (hash decides)
        float r = uniform ? 1.f : rating(wq[q], vu, vv);
        uint32_t h = edge_hash32(g.v0 + u, g.v0 + v, (uint32_t)salt);
        if (fav && (r > fr || (r == fr && (h > fh || (h == fh && v < fv))))) {
          fr = r; fh = h; fv = v;
        }
        if (wv >> 31) continue;  // already matched
        if (r > br || (r == br && (h > bh || (h == bh && v < bv)))) { br = r; bh = h; bv = v; }
        }
      }
    }
    for (int off = T / 2; off; off >>= 1) {
      float orr = __shfl_down_sync(0xffffffffu, br, off, T);
      uint32_t oh = __shfl_down_sync(0xffffffffu, bh, off, T);
      int ov = __shfl_down_sync(0xffffffffu, bv, off, T);
      if (ov >= 0 && (bv < 0 || orr > br || (orr == br && (oh > bh || (oh == bh && ov < bv))))) {
        br = orr; bh = oh; bv = ov;
      }
      orr = __shfl_down_sync(0xffffffffu, fr, off, T);
      oh = __shfl_down_sync(0xffffffffu, fh, off, T);
      ov = __shfl_down_sync(0xffffffffu, fv, off, T);
      if (ov >= 0 && (fv < 0 || orr > fr || (orr == fr && (oh > fh || (oh == fh && ov < fv))))) {
        fr = orr; fh = oh; fv = ov;
      }
    }
    if (u < g.n && lane == 0) {
      prop[u] = live ? bv : -1;
      if (fav) fav[u] = live ? fv : -1;
    }
  }
}

template <int T>
__global__ void __launch_bounds__(kTeamBlock)
cut_t(G g, const part_t *part, unsigned long long *cut2) {
  const int lane = team_lane<T>();
  const int64_t step = (int64_t)warps_total() * (32 / T);
  unsigned long long local = 0;
  for (int64_t vb = (int64_t)warp_id_global() * (32 / T); vb < g.n; vb += step) {
    const int v = (int)(vb + (threadIdx.x & 31) / T);
    if (v >= g.n) continue;
    const int pv = part[g.v0 + v];
    const int64_t b = g.xbeg[v];
    const int d = g.deg[v];
    for (int j = lane; j < d; j += T)
      if (part[g.adj[b + j]] != pv) local += (unsigned long long)g.ew(b + j);
  }
  for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cut2, local);
}

// Team sizes (lanes per vertex), measured on config 4 (degree ~20,
// tools/sweep_kway.py): sparse levels take 2-lane teams for the candidate
// scan (2 lanes x 4 entries in flight beat 4x4 by 0.18 ms/pass, 1x8 and 8x4)
// and the afterburner (2 beat 8 by 0.15 ms/pass); denser levels 16 or 32.
// The band-start pass 0 (register fast path) runs one lane per vertex with 8
// entries in flight instead (kway.cu, 0.55 -> 0.43 ms at config 4).
inline int team_for(const G &g) {
  const double avg = g.n ? (double)g.nnz / (double)g.n : 0.0;
  return avg <= 24.0 ? 2 : (avg <= 64.0 ? 16 : 32);
}
inline int refine_team_for(const G &g) { return team_for(g); }
inline int after_team_for(const G &g) { return team_for(g); }

// refine_cand_t<T, KR>: KR = 8 / 16 register accumulators, 0 = shared memory
#define HS_REFINE_DISPATCH(T_, K_, PACK16_, GRID, ...)                          \
  do {                                                                           \
    if ((K_) <= 16) {  /* private shared-memory counters per lane */             \
      if ((T_) == 1) refine_cand_t<1, -16, 8><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);   \
      else if ((T_) == 2) refine_cand_t<2, -16, 4><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);   \
      else if ((T_) == 16) refine_cand_t<16, -16><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);\
      else refine_cand_t<32, -16><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);               \
    } else {                                                                     \
      if ((T_) == 8) refine_cand_t<8, 0><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);        \
      else if ((T_) == 16) refine_cand_t<16, 0><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__); \
      else refine_cand_t<32, 0><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);                 \
    }                                                                            \
  } while (0)

#define HS_TEAM_DISPATCH(T_, KERNEL, GRID, ...)                                  \
  do {                                                                           \
    if ((T_) == 2) KERNEL<2><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);           \
    else if ((T_) == 4) KERNEL<4><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);      \
    else if ((T_) == 8) KERNEL<8><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);      \
    else if ((T_) == 16) KERNEL<16><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);    \
    else KERNEL<32><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);                    \
  } while (0)

// ---- device-side pass control (no host round trip per pass) ----
// ctl layout (int32): [0] list count, [1] confirmed/planned moves,
// [2] ACTIVE (refinement continues), [3] APPLY (this pass applies moves),
// [4] passes done, [5] OVER (some part above its bound), [6] unused.
enum { CTL_COUNT = 0, CTL_NCONF = 1, CTL_ACTIVE = 2, CTL_APPLY = 3, CTL_PASSES = 4, CTL_OVER = 5,
       CTL_KEPT = 10, CTL_MOVED = 11 };

// mode 0 (refine): thinning keeps the expected post-move weight of every
// part inside [lo, hi]; refinement stops once < 0.5% of vertices improve.
// mode 1 (rebalance): move just the excess of over-full parts into the room
// left below the targets of the others.
__global__ void plan_kernel(int k, int n, int mode, const int64_t *flows, const int64_t *pw,
                            const int64_t *hi, const int64_t *lo, const int64_t *target,
                            double *prob, int32_t *ctl) {
  const int p = threadIdx.x;
  const bool gate = mode != 1 ? ctl[CTL_ACTIVE] != 0 : ctl[CTL_OVER] != 0;
  const int nconf = ctl[CTL_NCONF];
  __syncthreads();
  if (!gate) {
    if (p == 0 && mode != 2) ctl[CTL_APPLY] = 0;
    return;
  }
  if (p < k) {
    const double out = (double)flows[p], in = (double)flows[k + p];
    double po = 1.0, pi = 1.0;
    if (mode == 1) {
      if (out > 0) po = fmin(1.0, (double)(pw[p] - target[p]) / out);
      if (in > 0) pi = fmin(1.0, (double)(target[p] - pw[p]) / in);
    } else {
      const double room_in = (double)(hi[p] - pw[p]), room_out = (double)(pw[p] - lo[p]);
      if (in > 0 && in > room_in) pi = room_in / in;
      if (out > 0 && out > room_out) po = room_out / out;
    }
    prob[p] = fmax(0.0, po);
    prob[k + p] = fmax(0.0, pi);
  }
  if (p == 0 && mode == 2) ctl[CTL_KEPT] = 0;  // the thinning's list count
  if (p == 0 && mode != 2) {  // mode 2: pre-plan, probabilities only
    ctl[CTL_APPLY] = nconf > 0;
    if (mode == 0) {
      if (nconf > 0) ctl[CTL_PASSES] += 1;
      ctl[CTL_ACTIVE] = (int64_t)nconf * 200 > (int64_t)n;
    }
  }
}

__global__ void balance_check(int k, const int64_t *pw, const int64_t *hi, int32_t *ctl) {
  if (threadIdx.x == 0) {
    int over = 0;
    for (int p = 0; p < k; ++p) over |= pw[p] > hi[p];
    ctl[CTL_OVER] = over;
  }
}
