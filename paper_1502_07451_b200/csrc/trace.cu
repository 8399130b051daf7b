// Trace products from the DES's device event buffer:
//
//   hs_trace_sort     the reference's event order (sim.py:200-201): by time,
//                     then xfer_start < xfer_end < kernel_start < kernel_end,
//                     then the subject compared AS A STRING ("10" < "9";
//                     "d5" < "d5.3" < "d50"), then the resource name as a
//                     string ("bus" < "cpu10" < "cpu2" < "gpu0");
//   hs_trace_metrics  metrics(trace) (sim.py:207-236) recomputed from the
//                     sorted events: busy time per device summed in event
//                     order (the reference's sequential fp64 adds), kernels
//                     per device, transfer count, makespan.
//
// The sort is LSD over stable radix passes (CUB onesweep): the resource
// rank, the subject in 15-character chunks (4 bits per character: end 0,
// '-' 1, '.' 2, digits 3-12; the kind rides above the most significant
// chunk), then the time (IEEE bits of a non-negative double order like the
// value). Transfer subjects drop their common "d" prefix: the kind is
// compared first, so a transfer subject is only ever compared with another.
#include "common.cuh"
#include <cstring>
#include <cub/device/device_radix_sort.cuh>

namespace {

constexpr int kChunkChars = 15;

__device__ __forceinline__ int dec_len(int64_t x) {
  int len = x < 0 ? 1 : 0;
  uint64_t u = x < 0 ? (uint64_t)(-(x + 1)) + 1 : (uint64_t)x;
  do {
    ++len;
    u /= 10;
  } while (u);
  return len;
}

// writes the 4-bit codes of str(x) into c[pos..], returns the new pos
__device__ __forceinline__ int dec_codes(int64_t x, uint8_t *c, int pos) {
  if (x < 0) c[pos++] = 1;
  uint64_t u = x < 0 ? (uint64_t)(-(x + 1)) + 1 : (uint64_t)x;
  char tmp[20];
  int n = 0;
  do {
    tmp[n++] = (char)(u % 10);
    u /= 10;
  } while (u);
  while (n) c[pos++] = (uint8_t)(3 + tmp[--n]);
  return pos;
}

__device__ __forceinline__ int subject_len(const hs_event_t &e, const int64_t *ids) {
  if (e.kind >= 2) return dec_len(ids[e.a]);
  return dec_len(ids[e.a]) + (e.b >= 0 ? 1 + dec_len(ids[e.b]) : 0);
}

__global__ void max_subject_len(const hs_event_t *ev, int64_t count, const int64_t *ids,
                                int32_t *out) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, subject_len(ev[i], ids));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// key of pass `what` for the event at perm[i]: -2 resource rank, -1 time,
// c >= 0 subject chunk c (kind above chunk 0)
__global__ void pass_keys(const hs_event_t *ev, const int32_t *perm, int64_t count,
                          const int64_t *ids, const int32_t *res_rank, int what,
                          uint64_t *keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const hs_event_t e = ev[perm ? perm[i] : i];
    uint64_t k;
    if (what == -2) {
      k = (uint64_t)res_rank[e.resource + 1];
    } else if (what == -1) {
      k = (uint64_t)__double_as_longlong(e.time);
    } else {
      uint8_t c[48];
      int n = dec_codes(ids[e.a], c, 0);
      if (e.kind < 2 && e.b >= 0) {
        c[n++] = 2;
        n = dec_codes(ids[e.b], c, n);
      }
      k = 0;
      for (int j = 0; j < kChunkChars; ++j) {
        const int p = what * kChunkChars + j;
        k = k << 4 | (p < n ? c[p] : 0u);
      }
      if (what == 0) k |= (uint64_t)e.kind << 60;
    }
    keys[i] = k;
  }
}

// per sorted position: the duration of a kernel_end (end - its start), the
// device (0 CPU, 1 GPU); start times are indexed by the kernel's node
__global__ void kernel_starts(const hs_event_t *ev, int64_t count, double *start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (ev[i].kind == 2) start[ev[i].a] = ev[i].time;
}

__global__ void end_durations(const hs_event_t *ev, const int32_t *perm, int64_t count,
                              int32_t cpu_workers, const double *start, double *dur,
                              int8_t *dev, unsigned long long *acc) {
  unsigned long long n_cpu = 0, n_gpu = 0, n_x = 0, mk = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const hs_event_t e = ev[perm[i]];
    int8_t d = -1;
    if (e.kind == 3) {
      d = e.resource < cpu_workers ? 0 : 1;
      dur[i] = e.time - start[e.a];
      (d ? n_gpu : n_cpu) += 1;
      const unsigned long long tb = (unsigned long long)__double_as_longlong(e.time);
      mk = tb > mk ? tb : mk;  // non-negative doubles order like their bits
    } else if (e.kind == 1) {
      ++n_x;
    }
    dev[i] = d;
  }
  atomicAdd(acc + 0, n_cpu);
  atomicAdd(acc + 1, n_gpu);
  atomicAdd(acc + 2, n_x);
  atomicMax(acc + 3, mk);
}

// busy[dev] += dur in sorted event order: one warp, 32 positions per step
// loaded together, the adds applied in order by lane 0
__global__ void busy_sums(const double *dur, const int8_t *dev, int64_t count, double *busy) {
  const int lane = threadIdx.x;
  double b0 = 0.0, b1 = 0.0;
  for (int64_t base = 0; base < count; base += 32) {
    const int64_t i = base + lane;
    const int8_t d = i < count ? dev[i] : (int8_t)-1;
    const double x = (i < count && d >= 0) ? dur[i] : 0.0;
    for (int j = 0; j < 32; ++j) {
      const int8_t dj = __shfl_sync(0xffffffffu, d, j);
      const double xj = __shfl_sync(0xffffffffu, x, j);
      if (dj == 0) b0 = b0 + xj;
      else if (dj == 1) b1 = b1 + xj;
    }
  }
  if (lane == 0) {
    busy[0] = b0;
    busy[1] = b1;
  }
}

}  // namespace

extern "C" int hs_trace_sort(const hs_event_t *ev, int64_t count, const int64_t *ids,
                             const int32_t *res_rank, int32_t *perm, void *stream) {
  HS_REQUIRE(count >= 0, HS_EINVAL, "hs_trace_sort: negative count");
  HS_REQUIRE(count == 0 || (ev && ids && res_rank && perm), HS_EINVAL,
             "hs_trace_sort: null argument");
  HS_REQUIRE(count < (1ll << 31), HS_ELIMIT, "hs_trace_sort: at most 2^31 - 1 events");
  if (count == 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  hs::Scratch<int32_t> mx, p2;
  hs::Scratch<uint64_t> k1, k2;
  HS_CHECK_CUDA(mx.alloc(1, s));
  HS_CHECK_CUDA(p2.alloc(count, s));
  HS_CHECK_CUDA(k1.alloc(count, s));
  HS_CHECK_CUDA(k2.alloc(count, s));
  HS_CHECK_CUDA(cudaMemsetAsync(mx, 0, 4, s));
  const int grid = hs::grid_for(count, 256);
  max_subject_len<<<grid, 256, 0, s>>>(ev, count, ids, mx);
  HS_CHECK_LAUNCH();
  int32_t maxlen = 0;
  HS_CHECK_CUDA(cudaMemcpyAsync(&maxlen, mx, 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  const int chunks = (maxlen + kChunkChars - 1) / kChunkChars;
  {
    const int rc0 = hs::iota32(perm, count, s);
    if (rc0) return rc0;
  }
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint64_t *)k1, (uint64_t *)k2,
                                  (int32_t *)perm, (int32_t *)p2, (int)count, 0, 64, s);
  hs::Scratch<uint8_t> tmp;
  HS_CHECK_CUDA(tmp.alloc(tmp_bytes, s));
  // least significant first: resource, subject chunks (last to first), time
  int32_t *cur = perm, *nxt = p2;
  auto pass = [&](int what, int bits) -> int {
    pass_keys<<<grid, 256, 0, s>>>(ev, cur, count, ids, res_rank, what, k1);
    HS_CHECK_LAUNCH();
    size_t tb = tmp_bytes;
    HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs((void *)tmp, tb, (uint64_t *)k1,
                                                  (uint64_t *)k2, cur, nxt, (int)count, 0,
                                                  bits, s));
    hs::count_launch();
    int32_t *t = cur;
    cur = nxt;
    nxt = t;
    return HS_OK;
  };
  int rc = pass(-2, 32);
  for (int c = chunks - 1; rc == HS_OK && c >= 0; --c) rc = pass(c, 64);
  if (rc == HS_OK) rc = pass(-1, 64);
  if (rc) return rc;
  if (cur != perm)
    HS_CHECK_CUDA(cudaMemcpyAsync(perm, cur, count * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  return HS_OK;
}

extern "C" int hs_trace_metrics(const hs_event_t *ev, const int32_t *perm, int64_t count,
                                int32_t n_nodes, int32_t cpu_workers, double *out_host,
                                void *stream) {
  HS_REQUIRE(count >= 0 && n_nodes >= 0 && out_host, HS_EINVAL, "hs_trace_metrics: bad argument");
  for (int i = 0; i < 6; ++i) out_host[i] = 0.0;
  if (count == 0) return HS_OK;
  HS_REQUIRE(ev && perm, HS_EINVAL, "hs_trace_metrics: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  hs::Scratch<double> start, dur, busy;
  hs::Scratch<int8_t> dev;
  hs::Scratch<unsigned long long> acc;
  HS_CHECK_CUDA(start.alloc(n_nodes > 0 ? n_nodes : 1, s));
  HS_CHECK_CUDA(dur.alloc(count, s));
  HS_CHECK_CUDA(busy.alloc(2, s));
  HS_CHECK_CUDA(dev.alloc(count, s));
  HS_CHECK_CUDA(acc.alloc(4, s));
  HS_CHECK_CUDA(cudaMemsetAsync(acc, 0, 32, s));
  const int grid = hs::grid_for(count, 256);
  kernel_starts<<<grid, 256, 0, s>>>(ev, count, start);
  HS_CHECK_LAUNCH();
  end_durations<<<grid, 256, 0, s>>>(ev, perm, count, cpu_workers, start, dur, dev, acc);
  HS_CHECK_LAUNCH();
  busy_sums<<<1, 32, 0, s>>>(dur, dev, count, busy);
  HS_CHECK_LAUNCH();
  unsigned long long a[4];
  double b[2];
  HS_CHECK_CUDA(cudaMemcpyAsync(a, acc, sizeof a, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(b, busy, sizeof b, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  double mk;
  memcpy(&mk, &a[3], sizeof mk);
  out_host[0] = mk;               // makespan
  out_host[1] = (double)a[2];     // transfer count (xfer_end events)
  out_host[2] = b[0];             // busy CPU
  out_host[3] = b[1];             // busy GPU
  out_host[4] = (double)a[0];     // kernels on CPU
  out_host[5] = (double)a[1];     // kernels on GPU
  return HS_OK;
}
