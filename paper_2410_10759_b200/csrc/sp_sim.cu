// K4: FIFO capacity-queue replay (reference: throughput_sim.py:207-256).
//
// One thread replays one independent run (a (stream, capacity) pair); a
// Monte-Carlo sweep launches tens of thousands of runs at once.  The waiting
// queue of the reference is always the contiguous index range [head, next)
// of arrivals, so only the in-service min-heap needs storage: a per-run
// binary heap of (finish_ms, seq, request) in the caller's workspace, keyed
// lexicographically on (finish, seq) exactly like the reference's heapq
// tuples (seq is unique, so the pop order is fully determined; any heap
// arity gives it -- this one is 4-ary).
#include <algorithm>

#include "sp_internal.cuh"
#include "np_random.cuh"

namespace sp {
namespace {

struct HeapEntry {
  double finish;
  int32_t seq;
  int32_t req;
};

__device__ __forceinline__ bool less(const HeapEntry& a, const HeapEntry& b) {
  return a.finish < b.finish || (a.finish == b.finish && a.seq < b.seq);
}

// 4-ary heap: half the depth of a binary one; a node's four children are
// adjacent (one or two 32-B sectors), loaded back to back before comparing,
// so a sift-down level costs one memory latency.  Keys are unique (seq), so
// every valid heap pops the same order.
__device__ void heap_push(HeapEntry* h, int64_t& size, HeapEntry e) {
  int64_t c = size++;
  while (c > 0) {
    const int64_t p = (c - 1) >> 2;
    const HeapEntry pe = h[p];
    if (!less(e, pe)) break;
    h[c] = pe;
    c = p;
  }
  h[c] = e;
}

// (root_finish: the new root's finish time after the pop, INFINITY if empty)
// A node's four children h[4c+1 .. 4c+4] are one 64-B aligned group (the
// run's heap starts 3 entries into a 64-B aligned block): two 256-bit loads.
struct __align__(32) EntryPair {
  HeapEntry a, b;
};
__device__ HeapEntry heap_pop(HeapEntry* h, int64_t& size, double& root_finish) {
  const HeapEntry top = h[0];
  const HeapEntry last = h[--size];
  root_finish = size > 0 ? last.finish : INFINITY;
  int64_t c = 0;
  while (true) {
    const int64_t f = 4 * c + 1;
    if (f >= size) break;
    const int nv = (int)min((int64_t)4, size - f);  // children past the end are not in the heap
    HeapEntry c0, c1, c2, c3;
    if (nv == 4) {
      const EntryPair* g = reinterpret_cast<const EntryPair*>(h + f);
      const EntryPair p0 = g[0], p1 = g[1];
      c0 = p0.a, c1 = p0.b, c2 = p1.a, c3 = p1.b;
    } else {  // the last, partial group: only entries of the heap are read
      c0 = h[f];
      c1 = h[f + min(1, nv - 1)];
      c2 = h[f + min(2, nv - 1)];
      c3 = h[f + min(3, nv - 1)];
    }
    // the minimum child by selects (no indexed array: it would live in local memory)
    HeapEntry best = c0;
    int bi = 0;
    if (nv > 1 && less(c1, best)) best = c1, bi = 1;
    if (nv > 2 && less(c2, best)) best = c2, bi = 2;
    if (nv > 3 && less(c3, best)) best = c3, bi = 3;
    if (!less(best, last)) break;
    if (c == 0) root_finish = best.finish;
    h[c] = best;
    c = f + bi;
  }
  if (size > 0) h[c] = last;
  return top;
}

__global__ void sim_replay_kernel(sp_sim_batch b, sp_sim_out o, HeapEntry* heap_ws) {
  const int64_t run = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (run >= b.n_runs) return;
  const int64_t lo = b.run_off[run];
  const int64_t n = b.run_off[run + 1] - lo;
  const double* arr = b.arrival_ms + lo;
  const double* dem = b.demand + lo;
  const double* dur = b.duration_ms + lo;
  double* admit = o.admit_ms + lo;
  // a run never holds more than n in service; its heap starts 3 entries into
  // a 64-B aligned block (children groups aligned), 8 spare entries per run
  HeapEntry* h = heap_ws + (((lo + 8 * run) + 3) & ~(int64_t)3) + 3;
  const double cap = b.capacity[run];
  const double eps = dmul(1e-9, cap);
  double free_cap = cap;
  int64_t hsize = 0, head = 0, next = 0;
  int32_t seq = 0;
  int32_t status = SP_OK;
  int64_t dead = -1;
  // the heap's root finish, the next arrival and the FIFO head's demand stay
  // in registers: every global access is divergent across a warp's runs (one
  // run per lane), so the replay is bound by load instructions, not math.
  // (admit needs no initialisation: a run that completes admits every
  // request; a deadlocked run's admit times are not reported)
  double top_f = INFINITY;
  double t_arr = n > 0 ? arr[0] : INFINITY;
  double need = n > 0 ? dem[0] : 0.0;  // dem[head]
  while (next < n || hsize > 0) {
    double now;
    if (top_f <= t_arr) {  // completions before equal-time arrivals (top_f is INFINITY when empty)
      const HeapEntry e = heap_pop(h, hsize, top_f);
      now = e.finish;
      free_cap = dadd(free_cap, dem[e.req]);
    } else {
      now = t_arr;
      ++next;
      t_arr = next < n ? arr[next] : INFINITY;
    }
    while (head < next) {
      if (need <= dadd(free_cap, eps)) {
        admit[head] = now;
        free_cap = dadd(free_cap, -need);
        HeapEntry e;
        e.finish = dadd(now, dur[head]);
        e.seq = seq++;
        e.req = (int32_t)head;
        heap_push(h, hsize, e);
        top_f = e.finish < top_f ? e.finish : top_f;  // the root is the minimum finish
        ++head;
        if (head < n) need = dem[head];
      } else {
        if (need > dadd(cap, eps)) {
          status = SP_ERR_DEADLOCK;
          dead = head;
        }
        break;
      }
    }
    if (status != SP_OK) break;
  }
  o.status[run] = status;
  if (o.deadlock_req) o.deadlock_req[run] = dead;
  if (status != SP_OK) return;
  // waits, max, numpy-order mean, sequential cumsum (throughput_sim.py:122-130, 247)
  double mx = -INFINITY, run_sum = 0.0;
  const bool per_request = o.wait_ms || o.cum_wait_ms;
  if (per_request || !o.mean_wait_ms) {
    for (int64_t k = 0; k < n; ++k) {
      const double w = dadd(admit[k], -arr[k]);
      if (o.wait_ms) o.wait_ms[lo + k] = w;
      if (o.cum_wait_ms) {
        run_sum = (k == 0) ? w : dadd(run_sum, w);
        o.cum_wait_ms[lo + k] = run_sum;
      }
      mx = (w > mx || w != w) ? w : mx;
    }
  }
  if (o.mean_wait_ms) {
    // (without per-request outputs the max rides along the sum's single pass:
    // np_sum reads every element exactly once)
    const double s = np_sum(
        [&](int64_t k) {
          const double w = dadd(admit[k], -arr[k]);
          if (!per_request) mx = (w > mx || w != w) ? w : mx;
          return w;
        },
        n);
    o.mean_wait_ms[run] = n ? ddiv(s, (double)n) : 0.0;
  }
  if (o.max_wait_ms) o.max_wait_ms[run] = n ? mx : 0.0;
}

// One thread per skeleton: numpy's default_rng(seed) draws in numpy's order
// (np_random.cuh; throughput_sim.py:179-186): the exponential inter-arrival
// gaps summed left to right (np.cumsum), then the table-row picks, then the
// execution counts.  The three phases draw from the same stream, so a thread
// generates its skeleton start to end.
__global__ void skeleton_kernel(const int64_t* seeds, const int64_t* lo, const int64_t* hi, int64_t n,
                                int64_t horizon, double scale, int64_t exec_max, double* arrival_ms,
                                int32_t* choice, int32_t* exec_count, int32_t* status) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t a = lo[r], span = hi[r] - a;
  if (span < 1) {
    if (status) status[r] = SP_ERR_INVALID;
    return;
  }
  nprand::Pcg64 g = nprand::pcg64_from_seed((uint64_t)seeds[r]);
  double* arr = arrival_ms + r * horizon;
  double run = 0.0;
  for (int64_t k = 0; k < horizon; ++k) {
    const double e = dmul(scale, nprand::standard_exponential(g));
    run = k == 0 ? e : dadd(run, e);
    arr[k] = run;
  }
  int32_t* ch = choice + r * horizon;
  for (int64_t k = 0; k < horizon; ++k) ch[k] = (int32_t)(nprand::integers(g, 0, span) + a);
  int32_t* ex = exec_count + r * horizon;
  for (int64_t k = 0; k < horizon; ++k) ex[k] = (int32_t)nprand::integers(g, 1, exec_max + 1);
  if (status) status[r] = SP_OK;
}

__global__ void segment_sum_kernel(const double* x, const int64_t* off, int64_t n_seg, double* out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_seg) return;
  const double* a = x + off[k];
  out[k] = np_sum([&](int64_t i) { return a[i]; }, off[k + 1] - off[k]);
}

}  // namespace
}  // namespace sp

using namespace sp;

extern "C" {

int sp_segment_sum(const double* x, const int64_t* seg_off, int64_t n_seg, double* out, void* stream) {
  if (n_seg < 0 || (n_seg > 0 && (!x || !seg_off || !out))) {
    set_error(SP_ERR_INVALID, "sp_segment_sum: bad arguments");
    return SP_ERR_INVALID;
  }
  if (n_seg == 0) return SP_OK;
  segment_sum_kernel<<<(unsigned)((n_seg + 127) / 128), 128, 0, (cudaStream_t)stream>>>(x, seg_off, n_seg,
                                                                                       out);
  return launch_check("segment_sum_kernel launch");
}

int sp_sim_skeletons(const int64_t* seeds, const int64_t* choice_lo, const int64_t* choice_hi, int64_t n,
                     int64_t horizon, double scale, int64_t exec_max, double* arrival_ms, int32_t* choice,
                     int32_t* exec_count, int32_t* status, void* stream) {
  if (n < 0 || horizon < 0 || exec_max < 1 || exec_max >= ((int64_t)1 << 31) ||
      (n > 0 && (!seeds || !choice_lo || !choice_hi)) ||
      (n > 0 && horizon > 0 && (!arrival_ms || !choice || !exec_count))) {
    set_error(SP_ERR_INVALID, "sp_sim_skeletons: bad arguments");
    return SP_ERR_INVALID;
  }
  if (n == 0) return SP_OK;
  skeleton_kernel<<<(unsigned)((n + 63) / 64), 64, 0, (cudaStream_t)stream>>>(
      seeds, choice_lo, choice_hi, n, horizon, scale, exec_max, arrival_ms, choice, exec_count, status);
  return launch_check("skeleton_kernel launch");
}

size_t sp_sim_workspace_bytes(const sp_sim_batch* b) {
  if (!b) return 0;
  return sizeof(HeapEntry) * (size_t)std::max<int64_t>(1, b->total_requests + 8 * b->n_runs + 8);
}

int sp_sim_replay(const sp_sim_batch* b, sp_sim_out* o, void* ws, size_t ws_bytes, void* stream) {
  if (!b || !o || b->n_runs < 0 || (b->n_runs > 0 && (!b->run_off || !b->capacity || !o->admit_ms ||
                                                      !o->status))) {
    set_error(SP_ERR_INVALID, "sp_sim_replay: bad arguments");
    return SP_ERR_INVALID;
  }
  if (b->n_runs == 0) return SP_OK;
  const size_t need = sp_sim_workspace_bytes(b);
  if (!ws || ws_bytes < need) {
    set_required_workspace(need);
    set_error(SP_ERR_WORKSPACE, "sp_sim_replay needs %zu B of heap workspace", need);
    return SP_ERR_WORKSPACE;
  }
  sim_replay_kernel<<<(unsigned)((b->n_runs + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      *b, *o, (HeapEntry*)ws);
  return launch_check("sim_replay_kernel launch");
}

}  // extern "C"
