// K8 — batched discrete-event simulation of the CPU+GPU machine.
//
// Restates sim.simulate (reference pkg/src/hetsched/sim.py:68-204) with the
// three built-in policies (policies.py:19-99) for a batch of independent
// (graph, policy, machine) triples. One thread runs one simulation; the
// event loop is inherently serial, the batch is the parallel axis.
//
// Bit-exactness: the reference only uses fp64 `+` and `max` on times, and
// this file is compiled with --fmad=false; every max() below keeps Python's
// "first argument unless the second is strictly greater" semantics and every
// sum runs in the reference's order (ascending predecessor id).
//
// Heap: a worker runs at most one kernel, so the reference's (end, seq, kid,
// wid) heap holds at most W entries; the batch popped at time t is "all busy
// workers whose end == t", re-sorted by kernel id exactly as sim.py:190 does,
// so the seq tie-breaker never matters and a linear scan over W replaces it.
#include "common.cuh"

namespace {

constexpr double kAbsent = -1.0;  // arrival sentinel: item not on that memory node

__device__ __forceinline__ double pmax(double a, double b) { return b > a ? b : a; }

struct SimArgs {
  hs_dag_batch_t g;
  int policy;
  const int8_t *pin;
  int C, G;
  double *makespan;
  int64_t *tcount, *tbytes, *kpd;
  double *busy;
  int32_t *status;
  hs_event_t *ev;
  const int64_t *ev_off;
  int64_t *ev_count;
  // scratch (global node / edge index space of the batch)
  int32_t *pending;  // [N]
  int32_t *qnext;    // [N]
  int32_t *ready;    // [N]
  double *arr;       // [2*(N+M)]
  // per-worker state, [batch][W] (any worker count, MachineModel has no cap)
  double *w_free, *w_end, *w_est;
  int32_t *w_kid, *w_qh, *w_qt;
  int8_t *w_busy;
};

struct Sim {
  // graph view (local indices)
  int n, root;
  const int64_t *out_ptr, *in_ptr;
  const int32_t *out_dst, *in_src, *in_eid;
  const double *w_cpu, *w_gpu, *w_xfer;
  const int64_t *bytes;
  const int8_t *pin;
  int32_t *pending, *qnext, *ready;
  double *arr;
  int64_t root_e0;  // first out-edge of the root
  // machine
  int C, W, policy;
  // per-worker state (this simulation's rows of the [batch][W] scratch)
  double *free_time, *run_end, *est_free;
  int32_t *run_kid, *qhead, *qtail;
  int8_t *busyw;
  double bus_free, est_bus;
  // outputs
  int64_t tcount, tbytes, kpd[2], finished;
  double busy_ms[2], makespan;
  hs_event_t *ev;
  int64_t ev_n, ev_cap;

  __device__ int mem_of(int w) const { return w < C ? 0 : 1; }
  // item index: d{u} -> u, d0.v -> n + (edge - root_e0)
  __device__ int64_t item_of(int u, int64_t e) const {
    return u == root ? (int64_t)n + (e - root_e0) : (int64_t)u;
  }
  __device__ void emit(double t, int kind, int a, int b, int res) {
    if (ev && ev_n < ev_cap) {
      hs_event_t x;
      x.time = t; x.kind = kind; x.a = a; x.b = b; x.resource = res;
      ev[ev_n] = x;
    }
    ev_n++;
  }
  __device__ void q_push(int q, int kid) {
    qnext[kid] = -1;
    if (qtail[q] < 0) qhead[q] = kid; else qnext[qtail[q]] = kid;
    qtail[q] = kid;
  }
  __device__ int q_pop(int q) {
    int k = qhead[q];
    if (k >= 0) {
      qhead[q] = qnext[k];
      if (qhead[q] < 0) qtail[q] = -1;
    }
    return k;
  }

  // sim.py:122-133 — item arrivals on the finishing worker's memory node,
  // then successors whose last input just arrived, inserted sorted into ready.
  __device__ void mark_done(int nid, double t, int mem, int &nready) {
    finished++;
    for (int64_t e = out_ptr[nid]; e < out_ptr[nid + 1]; ++e)
      arr[2 * item_of(nid, e) + mem] = t;
    for (int64_t e = out_ptr[nid]; e < out_ptr[nid + 1]; ++e) {
      int s = out_dst[e];
      if (--pending[s] == 0) {
        int i = nready++;
        while (i > 0 && ready[i - 1] > s) { ready[i] = ready[i - 1]; --i; }
        ready[i] = s;
      }
    }
  }

  // policies.py:19-99 on_ready
  __device__ void on_ready(int kid, double t) {
    if (policy == 0) { q_push(0, kid); return; }
    if (policy == 2) { q_push(pin[kid] ? 1 : 0, kid); return; }
    // dmda (policies.py:52-74)
    double best_est = 0.0, best_avail = 0.0, best_xfer = 0.0;
    int best_w = -1;
    for (int w = 0; w < W; ++w) {
      int mem = mem_of(w);
      double dur = mem == 0 ? w_cpu[kid] : w_gpu[kid];
      double xfer = 0.0;
      for (int64_t j = in_ptr[kid]; j < in_ptr[kid + 1]; ++j) {
        int u = in_src[j];
        int64_t e = in_eid[j];
        if (arr[2 * item_of(u, e) + mem] == kAbsent) xfer = xfer + w_xfer[e];
      }
      double avail = (xfer == 0.0) ? t : pmax(pmax(est_bus, bus_free), t) + xfer;
      double fr = pmax(pmax(est_free[w], free_time[w]), t);
      double est = pmax(fr, avail) + dur;
      if (best_w < 0 || est < best_est) {
        best_est = est; best_w = w; best_avail = avail; best_xfer = xfer;
      }
    }
    q_push(best_w, kid);
    est_free[best_w] = best_est;
    if (best_xfer != 0.0) est_bus = best_avail;
  }

  __device__ int next_for_worker(int w) {
    if (policy == 0) return q_pop(0);
    if (policy == 2) return q_pop(mem_of(w));
    return q_pop(w);
  }

  // sim.py:135-164
  __device__ void start_kernel(int kid, int w, double t) {
    int mem = mem_of(w);
    double avail = t;
    for (int64_t j = in_ptr[kid]; j < in_ptr[kid + 1]; ++j) {
      int u = in_src[j];
      int64_t e = in_eid[j];
      int64_t it = item_of(u, e);
      double a = arr[2 * it + mem];
      if (a != kAbsent) { avail = pmax(avail, a); continue; }
      double s = pmax(bus_free, t);
      double en = s + w_xfer[e];
      bus_free = en;
      arr[2 * it + mem] = en;
      int ea = u, eb = (u == root) ? (int)out_dst[e] : -1;
      emit(s, 0, ea, eb, -1);
      emit(en, 1, ea, eb, -1);
      tcount++;
      tbytes += bytes[e];
      avail = pmax(avail, en);
    }
    double dur = mem == 0 ? w_cpu[kid] : w_gpu[kid];
    double st = pmax(t, avail);
    double en = st + dur;
    emit(st, 2, kid, -1, w);
    emit(en, 3, kid, -1, w);
    busy_ms[mem] = busy_ms[mem] + dur;
    kpd[mem]++;
    free_time[w] = en;
    busyw[w] = true;
    run_end[w] = en;
    run_kid[w] = kid;
    makespan = pmax(makespan, en);
  }

  // sim.py:166-176
  __device__ void dispatch(double t) {
    bool assigned = true;
    while (assigned) {
      assigned = false;
      for (int w = 0; w < W; ++w) {
        if (busyw[w] || free_time[w] > t) continue;
        int kid = next_for_worker(w);
        if (kid >= 0) { start_kernel(kid, w, t); assigned = true; }
      }
    }
  }
};

__global__ void des_kernel(SimArgs A) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.g.batch) return;
  const int64_t n0 = A.g.node_off[b], n1 = A.g.node_off[b + 1];
  const int64_t e0 = A.g.edge_off[b];
  Sim S;
  S.n = (int)(n1 - n0);
  S.root = A.g.root[b];
  S.out_ptr = A.g.out_ptr + n0 + b;
  S.in_ptr = A.g.in_ptr + n0 + b;
  S.out_dst = A.g.out_dst + e0;
  S.in_src = A.g.in_src + e0;
  S.in_eid = A.g.in_eid + e0;
  S.w_cpu = A.g.w_cpu + n0;
  S.w_gpu = A.g.w_gpu + n0;
  S.w_xfer = A.g.w_xfer + e0;
  S.bytes = A.g.bytes + e0;
  S.pin = A.pin ? A.pin + n0 : nullptr;
  S.pending = A.pending + n0;
  S.qnext = A.qnext + n0;
  S.ready = A.ready + n0;
  S.arr = A.arr + 2 * (n0 + e0);
  S.root_e0 = S.out_ptr[S.root];
  S.C = A.C;
  S.W = A.C + A.G;
  S.policy = A.policy;
  S.bus_free = 0.0;
  S.est_bus = 0.0;
  S.tcount = 0; S.tbytes = 0; S.kpd[0] = S.kpd[1] = 0; S.finished = 0;
  S.busy_ms[0] = S.busy_ms[1] = 0.0;
  S.makespan = 0.0;
  S.ev = A.ev ? A.ev + A.ev_off[b] : nullptr;
  S.ev_cap = A.ev ? A.ev_off[b + 1] - A.ev_off[b] : 0;
  S.ev_n = 0;
  {
    const int64_t o = (int64_t)b * S.W;
    S.free_time = A.w_free + o; S.run_end = A.w_end + o; S.est_free = A.w_est + o;
    S.run_kid = A.w_kid + o; S.qhead = A.w_qh + o; S.qtail = A.w_qt + o; S.busyw = A.w_busy + o;
  }
  for (int w = 0; w < S.W; ++w) {
    S.free_time[w] = 0.0; S.busyw[w] = false; S.est_free[w] = 0.0;
    S.qhead[w] = -1; S.qtail[w] = -1; S.run_end[w] = 0.0; S.run_kid[w] = -1;
  }
  const int n = S.n;
  const int64_t m = A.g.edge_off[b + 1] - e0;
  for (int v = 0; v < n; ++v) S.pending[v] = (int32_t)(S.in_ptr[v + 1] - S.in_ptr[v]);
  for (int64_t i = 0; i < 2 * (n + m); ++i) S.arr[i] = kAbsent;

  // sim.py:178-181 — the root finishes at t=0 on the host
  int nready = 0;
  S.mark_done(S.root, 0.0, 0, nready);
  for (int i = 0; i < nready; ++i) S.on_ready(S.ready[i], 0.0);
  S.dispatch(0.0);

  // sim.py:183-195
  while (true) {
    double t = 0.0;
    bool any = false;
    for (int w = 0; w < S.W; ++w)
      if (S.busyw[w] && (!any || S.run_end[w] < t)) { t = S.run_end[w]; any = true; }
    if (!any) break;
    nready = 0;
    // the popped batch, in ascending kernel id (kid is unique per entry)
    int last = -1;
    while (true) {
      int pick = -1;
      for (int w = 0; w < S.W; ++w)
        if (S.busyw[w] && S.run_end[w] == t && S.run_kid[w] > last &&
            (pick < 0 || S.run_kid[w] < S.run_kid[pick]))
          pick = w;
      if (pick < 0) break;
      last = S.run_kid[pick];
      S.busyw[pick] = false;
      S.mark_done(last, t, S.mem_of(pick), nready);
    }
    for (int i = 0; i < nready; ++i) S.on_ready(S.ready[i], t);
    S.dispatch(t);
  }

  A.makespan[b] = S.makespan;
  A.tcount[b] = S.tcount;
  A.tbytes[b] = S.tbytes;
  A.busy[2 * b] = S.busy_ms[0];
  A.busy[2 * b + 1] = S.busy_ms[1];
  A.kpd[2 * b] = S.kpd[0];
  A.kpd[2 * b + 1] = S.kpd[1];
  A.status[b] = (S.finished == n) ? 0 : HS_EDEADLOCK;
  if (A.ev_count) A.ev_count[b] = S.ev_n;
}

}  // namespace

extern "C" int hs_simulate_batch(const hs_dag_batch_t *g, int policy, const int8_t *pin,
                                 int32_t cpu_workers, int32_t gpu_workers,
                                 double *makespan, int64_t *transfer_count,
                                 int64_t *transfer_bytes, double *busy, int64_t *kpd,
                                 int32_t *status, hs_event_t *ev, const int64_t *ev_off,
                                 int64_t *ev_count, void *stream) {
  HS_REQUIRE(g && g->batch >= 0, HS_EINVAL, "hs_simulate_batch: null batch");
  HS_REQUIRE(policy >= 0 && policy <= 2, HS_EPOLICY, "unknown policy id %d", policy);
  HS_REQUIRE(policy != 2 || pin, HS_EINVAL, "gp policy needs a pin map");
  HS_REQUIRE(cpu_workers >= 0 && gpu_workers >= 0 && cpu_workers + gpu_workers > 0 &&
                 (int64_t)cpu_workers + gpu_workers <= (1 << 24),
             HS_ELIMIT, "worker counts must be >= 0, total in 1..2^24");
  HS_REQUIRE(!ev || ev_off, HS_EINVAL, "events need ev_off");
  if (g->batch == 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  hs::sm_count();
  int64_t N = g->total_nodes, M = g->total_edges;
  hs::Scratch<int32_t> pending, qnext, ready;
  hs::Scratch<double> arr;
  HS_CHECK_CUDA(pending.alloc(N, s));
  HS_CHECK_CUDA(qnext.alloc(N, s));
  HS_CHECK_CUDA(ready.alloc(N, s));
  HS_CHECK_CUDA(arr.alloc(2 * (N + M), s));
  const int64_t BW = (int64_t)g->batch * (cpu_workers + gpu_workers);
  hs::Scratch<double> wd;
  hs::Scratch<int32_t> wi;
  hs::Scratch<int8_t> wb;
  HS_CHECK_CUDA(wd.alloc(3 * BW, s));
  HS_CHECK_CUDA(wi.alloc(3 * BW, s));
  HS_CHECK_CUDA(wb.alloc(BW, s));
  SimArgs A;
  A.w_free = wd.p; A.w_end = wd.p + BW; A.w_est = wd.p + 2 * BW;
  A.w_kid = wi.p; A.w_qh = wi.p + BW; A.w_qt = wi.p + 2 * BW;
  A.w_busy = wb.p;
  A.g = *g;
  A.policy = policy; A.pin = pin; A.C = cpu_workers; A.G = gpu_workers;
  A.makespan = makespan; A.tcount = transfer_count; A.tbytes = transfer_bytes;
  A.busy = busy; A.kpd = kpd; A.status = status;
  A.ev = ev; A.ev_off = ev_off; A.ev_count = ev_count;
  A.pending = pending; A.qnext = qnext; A.ready = ready; A.arr = arr;
  // one simulation per thread: small blocks spread the batch over every SM
  // (4096 simulations -> 128 blocks of 32 instead of 64 blocks of 64)
  int block = 32;
  while (block < 128 && (int64_t)g->batch >= (int64_t)block * 2 * 2 * hs::sm_count()) block *= 2;
  {
    // every graph's CSR + weights read once, scratch state initialised once
    hs::Prof P("des", s, 40.0 * N + 36.0 * M);
    des_kernel<<<(g->batch + block - 1) / block, block, 0, s>>>(A);
  }
  HS_CHECK_LAUNCH();
  return HS_OK;
}
