// K1: cost-table kernel (reference: cost_model.py:137-192, 305-329 and
// problem.py:58-115, 188-222).
//
// One warp per request; lanes stride over the request's layers.  Every
// (request, layer) cell is independent: the boundary bytes of layer k are the
// output bytes of layer k-1 (cost_model.py:327), recomputed in place.  Integer
// FLOP counts are exact int64 (the reference uses Python ints); every float
// operation is an explicit round-to-nearest op so nvcc cannot contract it.
#include <algorithm>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr double kSnapRelTol = 1e-9;  // problem.py:28 _SNAP_REL_TOL
constexpr int64_t kBytesPerElement = 4;  // cost_model.py:17
constexpr int64_t kSoftmaxFlops = 5;     // cost_model.py:18

struct LayerCost {
  double flops;  // float(flop_of_layer)
  double r;      // float(flops or memory)
  double out;    // float(output_bytes)
};

__device__ inline int64_t eff_seq(int64_t seq_len, int64_t div) {
  // cost_model.py:137-138 (positive operands: floor division; the common
  // divisor 1 skips the 64-bit division routine)
  return max((int64_t)1, div == 1 ? seq_len : seq_len / div);
}

__device__ inline double poly(const double* c, double s) {
  // cost_model.py:141-143: quad * s * s + lin * s + const, left to right
  return dadd(dadd(dmul(dmul(c[0], s), s), dmul(c[1], s)), c[2]);
}

__device__ LayerCost layer_cost(const sp_models& M, int64_t e, int64_t seq_len, bool memory) {
  const int kind = M.kind[e];
  const int64_t d = M.hidden_dim[e];
  const int64_t s = eff_seq(seq_len, M.seq_divisor[e]);
  LayerCost lc;
  // flop_of_layer, cost_model.py:146-165
  int64_t fi = 0;
  bool custom = false;
  switch (kind) {
    case SP_ATTENTION: fi = 8 * s * d * d + 4 * s * s * d + kSoftmaxFlops * s * s * M.heads[e]; break;
    case SP_FEED_FORWARD: fi = 4 * s * d * M.ffn_dim[e]; break;
    case SP_LAYER_NORM: fi = 5 * s * d; break;
    case SP_EMBEDDING: fi = 2 * s * d; break;
    case SP_CLASSIFIER: fi = 2 * s * d * M.out_dim[e]; break;
    default: custom = true;
  }
  lc.flops = custom ? poly(M.flop_coeffs + 3 * e, (double)s) : (double)fi;
  // memory_of_layer, cost_model.py:168-177
  if (!memory) {
    lc.r = lc.flops;
  } else if (custom) {
    if (M.has_mem_coeffs[e]) {
      lc.r = poly(M.mem_coeffs + 3 * e, (double)s);
    } else {
      const double c[3] = {0.0, (double)(kBytesPerElement * d), 0.0};
      lc.r = poly(c, (double)s);
    }
  } else {
    int64_t m = s * d * kBytesPerElement;
    if (kind == SP_ATTENTION) m += s * s * M.heads[e] * kBytesPerElement;
    lc.r = (double)m;
  }
  // output_bytes, cost_model.py:180-187
  if (kind == SP_CLASSIFIER) lc.out = (double)(M.out_dim[e] * kBytesPerElement);
  else if (custom && M.has_out_bytes[e]) lc.out = dmul(M.out_bytes_per_token[e], (double)s);
  else lc.out = (double)(s * d * kBytesPerElement);
  return lc;
}

// problem.py:68-76: snap q to the nearest integer when within 1e-9 relative
__device__ inline double snap(double q) {
  const double n = rint(q);  // Python round(): half to even
  const double tol = dmul(kSnapRelTol, fmax(1.0, fabs(n)));
  return fabs(dadd(q, -n)) <= tol ? n : q;
}

// error flags gathered per request, in the order integerize() would raise
enum : uint32_t { F_NEG = 1, F_NAN = 2, F_INF = 4, F_OVF = 8 };

__device__ inline uint32_t classify(double t) {
  if (t != t) return F_NAN;
  if (isinf(t)) return t < 0 ? (F_NEG | F_INF) : F_INF;
  return t < 0 ? F_NEG : 0u;
}

// problem.py:79-92 to_units for one element; flags unit-count overflow
__device__ inline int64_t to_units(double t, double unit, bool paper, uint32_t& flags) {
  const double q = snap(ddiv(t, unit));
  const double v = paper ? floor(dadd(q, 0.5)) : ceil(q);
  if (!(v >= -9.2233720368547758e18 && v < 9.2233720368547758e18)) {
    if (v == v && !isinf(v)) flags |= F_OVF;
    return 0;
  }
  return (int64_t)v;
}

struct ReqView {
  int64_t seq_len;
  double cfps, sfps, up, down, prop, deadline, unit;
  uint8_t flags;
};

__device__ inline ReqView load_req(const sp_requests& q, int64_t k) {
  ReqView v;
  v.seq_len = q.seq_len ? q.seq_len[k] : 1;
  v.cfps = q.client_fps ? q.client_fps[k] : 1.0;
  v.sfps = q.server_fps ? q.server_fps[k] : 1.0;
  v.up = q.uplink_bps ? q.uplink_bps[k] : 1.0;
  v.down = q.downlink_bps ? q.downlink_bps[k] : 1.0;
  v.prop = q.propagation_s ? q.propagation_s[k] : 0.0;
  v.deadline = q.deadline_s ? q.deadline_s[k] : 0.0;
  v.unit = q.unit_s ? q.unit_s[k] : 1e-3;
  v.flags = q.flags ? q.flags[k] : 0;
  return v;
}

// per-array error state: flag bits + first non-finite index by kind
struct ArrErr {
  uint32_t neg;
  int64_t first_nan, first_inf;
};

__device__ inline void note(ArrErr& a, double t, int64_t l) {
  const uint32_t c = classify(t);
  if (c & F_NEG) a.neg = 1;
  if ((c & F_NAN) && l < a.first_nan) a.first_nan = l;
  if ((c & F_INF) && l < a.first_inf) a.first_inf = l;
}

__device__ inline void warp_merge(ArrErr& a) {
  for (int o = 16; o > 0; o >>= 1) {
    a.neg |= __shfl_xor_sync(0xffffffffu, a.neg, o);
    a.first_nan = min(a.first_nan, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)a.first_nan, o));
    a.first_inf = min(a.first_inf, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)a.first_inf, o));
  }
}

// status for one array checked by to_units (array-level negativity first, then
// the first element whose round() raises)
__device__ inline int32_t array_status(const ArrErr& a) {
  if (a.neg) return SP_COST_NEGATIVE_TIME;
  if (a.first_nan < a.first_inf) return SP_COST_NAN_TIME;
  if (a.first_inf < a.first_nan) return SP_COST_INF_TIME;
  return SP_COST_OK;
}

// shared integerize body: given per-layer (r, client_s, server_time_s, tau)
template <typename Src>
__device__ void integerize_request(const Src& src, const sp_requests& req, int64_t k, int64_t lo,
                                   int64_t L, bool do_units, sp_cost_table& out) {
  const int lane = threadIdx.x & 31;
  const ReqView q = load_req(req, k);
  const bool paper = q.flags & SP_REQ_PAPER_ROUNDING;
  const bool zst = q.flags & SP_REQ_ZERO_SERVER;
  const int64_t BIG = INT64_MAX;
  ArrErr ec{0, BIG, BIG}, es{0, BIG, BIG}, eu{0, BIG, BIG}, ed{0, BIG, BIG};
  uint32_t ovf = 0, rneg = 0;
  for (int64_t l = lane; l < L; l += 32) {
    double r, cs, ss, tau;
    src(l, r, cs, ss, tau);
    const int64_t o = lo + l;
    if (out.r) out.r[o] = r;
    if (out.client_time_s) out.client_time_s[o] = cs;
    if (out.server_time_s) out.server_time_s[o] = ss;
    if (out.tau_bytes) out.tau_bytes[o] = tau;
    if (!do_units) continue;
    const double se = zst ? 0.0 : ss;
    // problem.py:58-65: ((8 * tau) / bps) + prop
    const double up = dadd(ddiv(dmul(8.0, tau), q.up), q.prop);
    const double dn = dadd(ddiv(dmul(8.0, tau), q.down), q.prop);
    if (out.server_s) out.server_s[o] = se;
    if (out.up_s) out.up_s[o] = up;
    if (out.down_s) out.down_s[o] = dn;
    note(ec, cs, l);
    note(es, se, l);
    note(eu, up, l);
    note(ed, dn, l);
    if (r < 0) rneg = 1;
    const int64_t iu = to_units(cs, q.unit, paper, ovf);
    const int64_t su = to_units(se, q.unit, paper, ovf);
    const int64_t uu = to_units(up, q.unit, paper, ovf);
    const int64_t du = to_units(dn, q.unit, paper, ovf);
    if (out.client_units) out.client_units[o] = iu;
    if (out.server_units) out.server_units[o] = su;
    if (out.up_units) out.up_units[o] = uu;
    if (out.down_units) out.down_units[o] = du;
  }
  if (!do_units) {
    if (lane == 0 && out.status) out.status[k] = SP_COST_OK;
    return;
  }
  warp_merge(ec);
  warp_merge(es);
  warp_merge(eu);
  warp_merge(ed);
  for (int o = 16; o > 0; o >>= 1) {
    ovf |= __shfl_xor_sync(0xffffffffu, ovf, o);
    rneg |= __shfl_xor_sync(0xffffffffu, rneg, o);
  }
  if (lane == 0) {
    // status = array code | budget code << 8 | negative-r << 16, so the host
    // can raise in the reference's order (problem.py:107-115 then :145-165)
    int32_t st = array_status(ec);
    if (!st) st = array_status(es);
    if (!st) st = array_status(eu);
    if (!st) st = array_status(ed);
    if (!st && ovf) st = SP_COST_OVERFLOW;
    // problem.py:95-104 budget_units: floor (conservative) / half-up (paper)
    const double qb = snap(ddiv(q.deadline, q.unit));
    const double wb = paper ? floor(dadd(qb, 0.5)) : floor(qb);
    int64_t W = 0;
    int32_t bst = SP_COST_OK;
    if (wb != wb) bst = SP_COST_NAN_TIME;
    else if (isinf(wb)) bst = SP_COST_INF_TIME;
    else if (wb >= -9.2233720368547758e18 && wb < 9.2233720368547758e18) W = (int64_t)wb;
    else bst = SP_COST_OVERFLOW;
    st |= bst << 8;
    if (rneg) st |= 1 << 16;  // problem.py:151-153
    if (out.budget) out.budget[k] = W;
    if (out.source_at_client) out.source_at_client[k] = (q.flags & SP_REQ_SOURCE_CLIENT) ? 1 : 0;
    if (out.status) out.status[k] = st;
  }
}

__global__ void __launch_bounds__(256, 3) cost_table_kernel(sp_models M, sp_requests req, int32_t integerize, sp_cost_table out) {
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= req.n) return;
  const int32_t m = req.model ? req.model[k] : 0;
  const int64_t e0 = M.layer_off[m];
  const int64_t L = M.layer_off[m + 1] - e0;
  const int64_t lo = out.layer_off[k];
  const ReqView q = load_req(req, k);
  const bool memory = q.flags & SP_REQ_METRIC_MEMORY;
  auto src = [&](int64_t l, double& r, double& cs, double& ss, double& tau) {
    const LayerCost lc = layer_cost(M, e0 + l, q.seq_len, memory);
    r = lc.r;
    // cost_model.py:318-325: flops / flops_per_s (int converted to double first)
    cs = ddiv(lc.flops, q.cfps);
    ss = ddiv(lc.flops, q.sfps);
    // tau = raw input (seq_len * 4) for layer 0, else previous layer's output bytes
    tau = (l == 0) ? (double)(q.seq_len * kBytesPerElement)
                   : layer_cost(M, e0 + l - 1, q.seq_len, false).out;
  };
  integerize_request(src, req, k, lo, L, integerize != 0, out);
}

__global__ void integerize_kernel(sp_profiles P, sp_requests req, sp_cost_table out) {
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= req.n) return;
  const int64_t lo = out.layer_off[k];
  const int64_t L = out.layer_off[k + 1] - lo;
  auto src = [&](int64_t l, double& r, double& cs, double& ss, double& tau) {
    r = P.r[lo + l];
    cs = P.client_time_s[lo + l];
    ss = P.server_time_s[lo + l];
    tau = P.tau_bytes[lo + l];
  };
  integerize_request(src, req, k, lo, L, true, out);
}


// elementwise to_units / budget_units (problem.py:79-104)
__global__ void to_units_kernel(const double* t, int64_t n, double unit, int32_t mode, int64_t* units,
                                int32_t* status) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double v = t[k];
  const uint32_t c = classify(v);
  int32_t st = SP_COST_OK;
  int64_t u = 0;
  if (c & F_NEG) {
    st = SP_COST_NEGATIVE_TIME;
  } else if (c & F_NAN) {
    st = SP_COST_NAN_TIME;
  } else if (c & F_INF) {
    st = SP_COST_INF_TIME;
  } else {
    const double q = snap(ddiv(v, unit));
    const double w = mode == 1 ? floor(dadd(q, 0.5)) : (mode == 2 ? floor(q) : ceil(q));
    if (w >= -9.2233720368547758e18 && w < 9.2233720368547758e18) u = (int64_t)w;
    else st = SP_COST_OVERFLOW;
  }
  units[k] = u;
  if (status) status[k] = st;
}

// single-CTA exclusive scan of per-request layer counts
__global__ void layer_offsets_kernel(sp_models M, sp_requests req, int64_t* off) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry_sh;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    carry_sh = 0;
    off[0] = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < req.n; base += blockDim.x) {
    const int64_t k = base + tid;
    int64_t v = 0;
    if (k < req.n) {
      const int32_t m = req.model ? req.model[k] : 0;
      v = M.layer_off[m + 1] - M.layer_off[m];
    }
    int64_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    int64_t before = carry_sh;
    for (int w = 0; w < wid; ++w) before += warp_tot[w];
    if (k < req.n) off[k + 1] = before + inc;
    __syncthreads();
    if (tid == blockDim.x - 1) carry_sh = before + inc;
    __syncthreads();
  }
}

}  // namespace
}  // namespace sp

using namespace sp;

extern "C" {


int sp_to_units(const double* seconds, int64_t n, double unit_s, int32_t mode, int64_t* units,
                int32_t* status, void* stream) {
  if (n < 0 || (n > 0 && (!seconds || !units)) || mode < 0 || mode > 2) {
    set_error(SP_ERR_INVALID, "sp_to_units: bad arguments");
    return SP_ERR_INVALID;
  }
  if (!(unit_s > 0)) {
    set_error(SP_ERR_INVALID, "unit_s must be positive");
    return SP_ERR_INVALID;
  }
  if (n == 0) return SP_OK;
  to_units_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(seconds, n, unit_s, mode,
                                                                                units, status);
  return launch_check("to_units_kernel launch");
}

int sp_request_layer_offsets(const sp_models* models, const sp_requests* req, int64_t* layer_off,
                             void* stream) {
  if (!models || !req || !layer_off || req->n < 0) {
    set_error(SP_ERR_INVALID, "sp_request_layer_offsets: bad arguments");
    return SP_ERR_INVALID;
  }
  layer_offsets_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(*models, *req, layer_off);
  return launch_check("layer_offsets_kernel launch");
}

int sp_build_cost_table(const sp_models* models, const sp_requests* req, int32_t integerize,
                        sp_cost_table* out, void* stream) {
  if (!models || !req || !out || !out->layer_off || req->n < 0) {
    set_error(SP_ERR_INVALID, "sp_build_cost_table: bad arguments");
    return SP_ERR_INVALID;
  }
  if (req->n == 0) return SP_OK;
  const int64_t threads = req->n * 32;
  cost_table_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      *models, *req, integerize, *out);
  return launch_check("cost_table_kernel launch");
}

int sp_integerize_profiles(const sp_profiles* prof, const sp_requests* req, sp_cost_table* out,
                           void* stream) {
  if (!prof || !req || !out || !out->layer_off || req->n < 0 || !prof->r || !prof->client_time_s ||
      !prof->server_time_s || !prof->tau_bytes) {
    set_error(SP_ERR_INVALID, "sp_integerize_profiles: bad arguments");
    return SP_ERR_INVALID;
  }
  if (req->n == 0) return SP_OK;
  const int64_t threads = req->n * 32;
  integerize_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*prof, *req,
                                                                                         *out);
  return launch_check("integerize_kernel launch");
}

}  // extern "C"
