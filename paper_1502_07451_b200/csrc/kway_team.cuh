// Team-per-vertex kernels of the k-way partitioner (included by kway.cu).
//
// A "team" is T consecutive lanes of a warp (T in {8, 16, 32}) working on
// one vertex; the host picks T from the level's average degree so that the
// fine levels (degree ~20) keep most lanes busy and the dense coarse levels
// use whole warps. Vertex loops advance warp-uniformly so every team of a
// warp takes part in the width-T shuffles.
#pragma once

template <int T>
__device__ __forceinline__ int team_lane() { return (threadIdx.x & 31) % T; }

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
template <int T>
__global__ void __launch_bounds__(kTeamBlock)
refine_cand_t(G g, const part_t *part, int k, const int64_t *pw, const int64_t *hi,
              const int64_t *lo, uint32_t *st, int32_t *list, int32_t *count, const int32_t *run) {
  if (run && !*run) return;
  __shared__ int32_t conn_s[kTeamBlock / T][kMaxParts];
  // part weights and bounds are read for every vertex: keep them on chip
  // (global reads of these few lines made one L2 slice the bottleneck)
  __shared__ int64_t s_pw[kMaxParts], s_hi[kMaxParts], s_lo[kMaxParts];
  for (int p = threadIdx.x; p < k; p += blockDim.x) {
    s_pw[p] = pw[p];
    s_hi[p] = hi[p];
    s_lo[p] = lo[p];
  }
  __syncthreads();
  const int lane = team_lane<T>();
  int32_t *conn = conn_s[threadIdx.x / T];
  const int64_t step = (int64_t)warps_total() * (32 / T);
  for (int64_t vb = (int64_t)warp_id_global() * (32 / T); vb < g.n; vb += step) {
    const int v = (int)(vb + (threadIdx.x & 31) / T);
    const bool valid = v < g.n;
    for (int p = lane; p < k; p += T) conn[p] = 0;
    __syncwarp();
    int own = 0, bnd = 0;
    if (valid) {
      own = part[v];
      const int64_t b = g.xbeg[v];
      const int d = g.deg[v];
      for (int j = lane; j < d; j += T) {
        int p = part[g.adj[b + j]];
        bnd |= p != own;
        atomicAdd(&conn[p], g.wgt[b + j]);
      }
    }
    __syncwarp();
    bnd = team_or<T>(bnd);
    int bg = 0, bp = -1;
    if (valid && bnd) {
      const int32_t vwv = g.vw[v];
      if (s_pw[own] - vwv >= s_lo[own])
        for (int p = lane; p < k; p += T) {
          if (p == own || s_pw[p] + vwv > s_hi[p]) continue;
          int gain = conn[p] - conn[own];
          if (gain > bg || (gain == bg && bp >= 0 && p < bp)) { bg = gain; bp = p; }
        }
    }
    team_argmax<T>(bg, bp);
    const bool writer = valid && lane == 0;
    const int c = (bp >= 0 && bg > 0) ? bp : -1;
    if (writer) st[v] = pack_state(own, c, bg);
    warp_append(writer && c >= 0, v, list, count);
    __syncwarp();
  }
}

// Jet-style afterburner over the candidate list: a move survives only if it
// still gains assuming every higher-priority (gain, then smaller id)
// neighbouring candidate moved. Confirmed moves land in conf[i] and in the
// planned flows (flows[p] out of p, flows[k+q] into q); nconf counts them.
template <int T>
__global__ void __launch_bounds__(kTeamBlock)
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
    if (valid) {
      v = list[i];
      const uint32_t sv = st[v];
      dest = st_cand(sv);
      own = st_part(sv);
      const int gv = st_gain(sv);
      const int64_t b = g.xbeg[v];
      const int d = g.deg[v];
      for (int j = lane; j < d; j += T) {
        int u = g.adj[b + j];
        const uint32_t su = st[u];
        int pu = st_part(su);
        int cu = st_cand(su);
        if (cu >= 0) {
          int gu = st_gain(su);
          if (gu > gv || (gu == gv && u < v)) pu = cu;
        }
        int w = g.wgt[b + j];
        delta += (pu == dest ? w : 0) - (pu == own ? w : 0);
      }
    }
    delta = team_sum<T>(delta);
    if (valid && lane == 0) {
      const bool ok = delta > 0;
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

// Applies confirmed moves of the list, each kept with probability
// prob[own] * prob[k + dest] (hash of (salt, v): deterministic thinning).
__global__ void apply_list(const int32_t *list, const int32_t *count, const int32_t *conf,
                           const int32_t *vw, const double *prob, int k, uint64_t salt,
                           part_t *part, int64_t *pw, const int32_t *run) {
  if (run && !*run) return;
  __shared__ long long s[kMaxParts];
  __shared__ double s_prob[2 * kMaxParts];
  for (int p = threadIdx.x; p < k; p += blockDim.x) s[p] = 0;
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) s_prob[p] = prob[p];
  __syncthreads();
  const int total = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int dest = conf[i];
    if (dest < 0) continue;
    const int v = list[i];
    const int own = part[v];
    const double pr = s_prob[own] * s_prob[k + dest];
    if (pr < 1.0 &&
        (double)mix32(salt ^ ((uint64_t)v * 0x9E3779B97F4A7C15ull)) >= pr * 4294967296.0)
      continue;
    part[v] = dest;
    atomicAdd((unsigned long long *)&s[dest], (unsigned long long)(long long)vw[v]);
    atomicAdd((unsigned long long *)&s[own], (unsigned long long)(-(long long)vw[v]));
  }
  __syncthreads();
  for (int p = threadIdx.x; p < k; p += blockDim.x)
    if (s[p]) atomicAdd((unsigned long long *)&pw[p], (unsigned long long)s[p]);
}

// Heavy-edge proposals (K3) with teams: prop[u] = best unmatched neighbour,
// fav[u] = best neighbour overall (for two-hop pairing).
template <int T>
__global__ void __launch_bounds__(kTeamBlock)
propose_t(G g, const uint32_t *mw, int32_t *prop, int32_t *fav, uint64_t salt,
          int32_t max_vw) {
  const int lane = team_lane<T>();
  const int64_t step = (int64_t)warps_total() * (32 / T);
  for (int64_t ub = (int64_t)warp_id_global() * (32 / T); ub < g.n; ub += step) {
    const int u = (int)(ub + (threadIdx.x & 31) / T);
    const bool live = u < g.n && !(mw[u] >> 31);
    float br = -1.f, fr = -1.f;
    int bv = -1, fv = -1;
    uint32_t bh = 0, fh = 0;
    if (live) {
      const int64_t b = g.xbeg[u];
      const int d = g.deg[u];
      const int32_t vu = (int32_t)(mw[u] & 0x7fffffffu);
      for (int j = lane; j < d; j += T) {
        int v = g.adj[b + j];
        if (v == u) continue;
        const uint32_t wv = mw[v];
        const int32_t vv = (int32_t)(wv & 0x7fffffffu);
        if (vu + vv > max_vw) continue;
        float r = rating(g.wgt[b + j], vu, vv);
        uint32_t h = edge_hash32(u, v, (uint32_t)salt);
        if (fav && (r > fr || (r == fr && (h > fh || (h == fh && v < fv))))) {
          fr = r; fh = h; fv = v;
        }
        if (wv >> 31) continue;  // already matched
        if (r > br || (r == br && (h > bh || (h == bh && v < bv)))) { br = r; bh = h; bv = v; }
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
    const int pv = part[v];
    const int64_t b = g.xbeg[v];
    const int d = g.deg[v];
    for (int j = lane; j < d; j += T)
      if (part[g.adj[b + j]] != pv) local += (unsigned long long)g.wgt[b + j];
  }
  for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cut2, local);
}

inline int team_for(const G &g) {
  const double avg = g.n ? (double)g.nnz / (double)g.n : 0.0;
  return avg <= 24.0 ? 8 : (avg <= 64.0 ? 16 : 32);
}

#define HS_TEAM_DISPATCH(T_, KERNEL, GRID, ...)                                  \
  do {                                                                           \
    if ((T_) == 8) KERNEL<8><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);           \
    else if ((T_) == 16) KERNEL<16><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);    \
    else KERNEL<32><<<GRID, kTeamBlock, 0, s>>>(__VA_ARGS__);                    \
  } while (0)

// ---- device-side pass control (no host round trip per pass) ----
// ctl layout (int32): [0] list count, [1] confirmed/planned moves,
// [2] ACTIVE (refinement continues), [3] APPLY (this pass applies moves),
// [4] passes done, [5] OVER (some part above its bound), [6] unused.
enum { CTL_COUNT = 0, CTL_NCONF = 1, CTL_ACTIVE = 2, CTL_APPLY = 3, CTL_PASSES = 4, CTL_OVER = 5 };

// mode 0 (refine): thinning keeps the expected post-move weight of every
// part inside [lo, hi]; refinement stops once < 0.5% of vertices improve.
// mode 1 (rebalance): move just the excess of over-full parts into the room
// left below the targets of the others.
__global__ void plan_kernel(int k, int n, int mode, const int64_t *flows, const int64_t *pw,
                            const int64_t *hi, const int64_t *lo, const int64_t *target,
                            double *prob, int32_t *ctl) {
  const int p = threadIdx.x;
  const bool gate = mode == 0 ? ctl[CTL_ACTIVE] != 0 : ctl[CTL_OVER] != 0;
  const int nconf = ctl[CTL_NCONF];
  __syncthreads();
  if (!gate) {
    if (p == 0) ctl[CTL_APPLY] = 0;
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
  if (p == 0) {
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
