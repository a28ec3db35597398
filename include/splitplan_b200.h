/*
 * splitplan_b200.h -- C ABI of the B200-native SplitLLM placement engine.
 *
 * The reference (`splitplan`, /root/reference/pkg/src/splitplan) is a pure
 * Python package with no FFI; its "operator API" is the set of module-level
 * functions.  Each entry point below replaces one of them, batched over many
 * independent instances (requests / scenarios), and is what a Python (ctypes),
 * C or C++ host binds.  See INTEGRATION.md for the ctypes stub.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the name ends in `_host`.  The caller owns every buffer; the
 *    library never frees caller memory and keeps no allocations between
 *    calls.  `stream` is a cudaStream_t passed as void*.
 *  - Every function returns an int status (SP_OK == 0).  Nothing throws across
 *    the ABI.  On failure `sp_last_error()` (thread-local) describes it.
 *  - "Infeasible" is a result, not an error (planner.py:104-107): the policy
 *    is all-server with feasible == 0 and its latency computed.
 *  - Instances are batched in CSR form over layers (sp_instances).
 *  - The functions are reentrant across host threads given distinct streams
 *    and workspaces.
 */
#ifndef SPLITPLAN_B200_H
#define SPLITPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 4  /* 2: + sp_plan_dp_devices, sp_plan_dp_workspace_bytes;
                             3: per-partition workspaces, sp_grid_* (one process per
                                device), sp_ipc_*, sp_last_full_workspace;
                             4: sp_plan_dp_async / sp_plan_dp_finish; 256-B aligned
                                workspaces; sp_plan_dp_onewave_bytes */

enum sp_status {
  SP_OK = 0,
  SP_ERR_INVALID = 1,    /* bad argument (wrapper raises ValueError) */
  SP_ERR_CUDA = 2,       /* CUDA runtime error */
  SP_ERR_WORKSPACE = 3,  /* workspace too small; see sp_last_required_workspace() */
  SP_ERR_BACKTRACE = 4,  /* planner.py:168-169/177-178 AssertionError (NaN tables) */
  SP_ERR_DEADLOCK = 5,   /* throughput_sim.py:243-246 CapacityDeadlockError */
  SP_ERR_UNSUPPORTED = 6 /* size outside what the engine handles (e.g. W_eff >= 2^31) */
};

enum sp_prefix_planner { SP_GREEDY = 0, SP_ALL_SERVER = 1, SP_ALL_CLIENT = 2 };

/* A batch of integer placement instances (problem.py:118-185 PlanProblem),
 * CSR over layers: instance k owns layers [layer_off[k], layer_off[k+1]). */
typedef struct sp_instances {
  int64_t n;                      /* number of instances */
  int64_t total_layers;           /* == layer_off[n] */
  const int64_t* layer_off;       /* [n+1] */
  const int64_t* client_units;    /* [total_layers] i_k */
  const int64_t* server_units;    /* [total_layers] s_k */
  const int64_t* up_units;        /* [total_layers] u_k */
  const int64_t* down_units;      /* [total_layers] d_k */
  const double* r;                /* [total_layers] resource value r_k */
  const int64_t* budget;          /* [n] integer budget W */
  const uint8_t* source_at_client;/* [n] 1 = data originates at the client */
  const int8_t* must_end_at;      /* [n] or NULL: -1 free, 0 server, 1 client */
} sp_instances;

/* Planner output (planner.py:42-51 PlacementPolicy), one record per instance. */
typedef struct sp_policies {
  uint8_t* pi;               /* [total_layers] 1 = client, 0 = server */
  double* client_value;      /* [n] numpy-order sum of r over client layers */
  double* server_load;       /* [n] numpy-order sum of r over server layers */
  int64_t* integer_latency;  /* [n] exact unit latency of pi */
  uint8_t* feasible;         /* [n] */
  int32_t* status;           /* [n] SP_OK or SP_ERR_BACKTRACE */
} sp_policies;

/* ---- library ------------------------------------------------------------ */

int sp_abi_version(void);
const char* sp_last_error(void);
/* bytes the last SP_ERR_WORKSPACE call needed */
size_t sp_last_required_workspace(void);
/* after a successful sp_plan_dp: the workspace that would have planned every
 * wave-path instance in ONE wave and kept every back-pointer stage of the
 * whole-GPU ones (no recompute); a caller growing its workspace uses it */
size_t sp_last_full_workspace(void);
/* after sp_plan_dp: instances whose rows outgrew the breakpoint lists and
 * were re-solved on the dense kernels */
int64_t sp_last_dense_fallbacks(void);

/* Instrumentation (thread-local, off by default).  While enabled, every
 * DP-stage kernel launch is bracketed by CUDA events on its stream and every
 * kernel the library launches is counted. sp_profile_collect synchronises
 * the recorded events and returns: total DP-stage kernel ms, DP-stage
 * launches, DP cells and algorithmic DP bytes those launches processed, the
 * count of all library kernel launches, and the DP variant that took the most
 * time (0 = rows in one CTA's SMEM, 1 = rows in cluster DSMEM, 2 = rows in
 * global memory); then resets the counters. */
void sp_profile_enable(int on);
int sp_profile_collect(double* dp_kernel_ms, int64_t* dp_launches, double* dp_cells,
                       double* dp_bytes, int64_t* all_launches, int32_t* dp_variant);

/* ---- planner (planner.py) ---------------------------------------------- */

/* W_eff = min(budget, sum_k max(i_k+d_k, s_k+u_k)) per instance.
 * Replaces planner.py:120-125 `_effective_budget`.  w_eff: device int64[n]. */
int sp_effective_budget(const sp_instances* in, int64_t* w_eff, void* stream);

/* Optimal DP placement for every instance: cost-table prep, the DP stage
 * kernel over the integer budget axis, end-side argmax and back-pointer walk.
 * Replaces planner.py:182-202 `plan_dp` (with :128-143 `build_dp_tables`,
 * :146-179 `_backtrace`, :88-107 `_finish`/`_infeasible`).
 * `ws` is scratch of `ws_bytes` bytes (device, 256-byte aligned as cudaMalloc
 * returns it; SP_ERR_INVALID otherwise); instances are processed in waves that
 * fit it.  SP_ERR_WORKSPACE if a single instance does not fit.
 * Synchronises `stream` once (to size the waves) before returning. */
int sp_plan_dp(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes,
               void* stream);

/* sp_plan_dp in two halves, so that a caller can queue the next batch while
 * this one runs (no stream synchronisation in the first half).
 * sp_plan_dp_async enqueues the device-planned tier (prep, breakpoint lists,
 * walk back, _finish) on `stream` and returns; `pending` is caller-owned
 * PINNED host memory of SP_PENDING_BYTES bytes (8-B aligned) that receives
 * the tier's counters.  When the tier cannot take the batch (workspace,
 * widths) the call runs to completion like sp_plan_dp.  sp_plan_dp_finish
 * waits for the counters (not for the whole stream) and runs the
 * host-planned tiers for the instances left; `in`, `out`, `ws` and
 * `ws_bytes` must be those of the async call, and `ws` untouched in between.
 * The policies are final once sp_plan_dp_finish returned SP_OK and the
 * stream has reached that point. */
#define SP_PENDING_BYTES 64
int sp_plan_dp_async(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream,
                     void* pending);
int sp_plan_dp_finish(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream,
                      void* pending);

/* Workspace sizes for sp_plan_dp on these instances (the `*_workspace_bytes`
 * query of SURVEY.md 8b): min_bytes runs every instance (in waves; whole-GPU
 * instances with checkpoint / recompute), full_bytes plans every wave-path
 * instance in one wave and keeps every back-pointer stage of whole-GPU ones.
 * Runs the prep kernel, so it needs the fixed part of the workspace
 * (n x 48 + total_layers x 40 bytes); SP_ERR_WORKSPACE otherwise, with
 * sp_last_required_workspace().  Synchronises `stream`; launches no DP. */
int sp_plan_dp_workspace_bytes(const sp_instances* in, size_t* min_bytes, size_t* full_bytes, void* ws,
                               size_t ws_bytes, void* stream);

/* sp_plan_dp with HOST pointers in `in` and `out` (the scalar drop-in calls:
 * planner.plan_dp on one problem, planner.py:182-202).  Each side's arrays
 * are expected packed in one host buffer (alignment gaps allowed): the
 * instances travel in one host-to-device copy, the policies back in one
 * device-to-host copy, both through the front of `ws`; then the stream is
 * synchronised.  SP_ERR_UNSUPPORTED when a side spans more than 64 MB. */
int sp_plan_dp_host(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream);

/* sp_plan_prefix with host pointers, the same way (planner.plan_greedy /
 * plan_trivial on one problem, planner.py:205-225). */
int sp_plan_prefix_host(const sp_instances* in, int32_t which, sp_policies* out, void* ws, size_t ws_bytes,
                        void* stream);

/* Host arithmetic only (no device work): the workspace with which sp_plan_dp
 * runs the device-planned breakpoint-list tier of n instances of total_layers
 * stages in ONE wave (fixed part + every instance's store).  A caller sizing
 * its workspace ahead of a call uses it to avoid many small waves. */
size_t sp_plan_dp_onewave_bytes(int64_t n, int64_t total_layers);

/* sp_plan_dp with the capacity axis of huge instances split over devices
 * (SURVEY.md 8(e), cfg5).  Instances that take the whole-GPU path (>= 4M
 * budget columns, or whose back-pointers exceed the workspace) are split
 * along the budget axis into one partition per listed device: partition p
 * runs on devices[p] and keeps EVERYTHING of its columns -- row buffers,
 * progress counters, stage records, checkpoint rows and back-pointers -- in
 * part_ws[p] (device memory of devices[p], part_ws_bytes[p] bytes, owned by
 * the caller).  Each partition mirrors its left neighbour's last columns (the
 * halo) by NVLink peer stores from inside the DP kernel, partitions order
 * their stages through system-scope progress counters, and the backtrack
 * walks the partitions from the right, each reading its own back-pointers
 * and handing (stage, column, side) to its left neighbour when the column
 * leaves its range (planner.py:146-179).  devices[0] must be the current
 * device, which owns `in`, `out`, `ws` and `stream`; a device may be listed
 * more than once.  Other instances are planned in `ws` as by sp_plan_dp.
 * Replaces the same reference functions as sp_plan_dp (planner.py:182-202). */
int sp_plan_dp_devices(const sp_instances* in, sp_policies* out, const int32_t* devices, int32_t n_devices,
                       void* ws, size_t ws_bytes, void* const* part_ws, const size_t* part_ws_bytes,
                       void* stream);

/* Workspace sizes for sp_plan_dp_devices: ws_min for `ws`, and per
 * partition workspace the smallest that runs (checkpoint / recompute) and the
 * one keeping every back-pointer stage.  Runs the prep kernel in `ws` (it
 * needs the fixed part; SP_ERR_WORKSPACE otherwise). */
int sp_plan_dp_devices_workspace_bytes(const sp_instances* in, const int32_t* devices, int32_t n_devices,
                                       size_t* ws_min, size_t* part_min, size_t* part_full, void* ws,
                                       size_t ws_bytes, void* stream);

/* ---- capacity partitions, one process per device ------------------------
 * The same partitioned solve driven by one process per partition (torchrun,
 * one rank per GPU): every rank plans identically, allocates one partition
 * workspace of plan.part_bytes, maps every other rank's workspace into its
 * address space (sp_ipc_export / sp_ipc_import over the process group), and
 * runs the phases in lockstep:
 *   forward:   for seg in 0..nseg-1: reset; barrier; forward(seg, write_ckpt=1,
 *              keep_bp = seg == nseg-1); barrier
 *   end:       the owner partition runs sp_grid_part_end; broadcast state
 *   backtrack: for seg = nseg-1..0: (recompute seg with keep_bp=1 unless it
 *              is the last), then partitions nparts-1..0 in turn run
 *              sp_grid_part_backtrack on the handed-over state
 *   finish:    combine pi (each stage written by exactly one partition) and
 *              evaluate it (sp_evaluate_policy).                              */
typedef struct sp_grid_plan {
  int32_t mode, n_layers, ctas, chunks_per_cta, nparts, seg_stages, nseg, nckpt, sac, owner_part;
  int64_t ncol, part_cols, halo, span, row_words;
  uint64_t rec_off, prog_off, state_off, rows_off, ckpt_off, bp_off, ckpt_bytes, bp_stage, part_bytes;
} sp_grid_plan;

/* Geometry for ONE instance (in->n == 1, layer_off[0] == 0) over `nparts`
 * partitions of at most `ctas_per_part` CTAs (0: all co-resident CTAs of the
 * device) in partition workspaces of `part_ws_bytes`; force_segment > 0 fixes
 * the checkpoint segment length.  ws: scratch for the prep kernel.
 * Synchronises `stream`. */
int sp_grid_plan_make(const sp_instances* in, int32_t nparts, int32_t ctas_per_part, size_t part_ws_bytes,
                      int32_t force_segment, sp_grid_plan* plan, void* ws, size_t ws_bytes, void* stream);
/* stage records and state of a partition workspace (prep kernel into it) */
int sp_grid_part_prepare(const sp_grid_plan* plan, const sp_instances* in, void* part_ws, void* stream);
/* zero the partition's progress counters (before every forward launch, on
 * every partition, before any partition launches) */
int sp_grid_part_reset(const sp_grid_plan* plan, void* part_ws, void* stream);
/* DP stages of segment `seg` on partition `part` (a cooperative launch that
 * spins on its neighbours' counters: every partition of the phase must be
 * launched).  part_ws[nparts]: every partition workspace as mapped here. */
int sp_grid_part_forward(const sp_grid_plan* plan, int32_t part, void* const* part_ws, int32_t seg,
                         int32_t write_ckpt, int32_t keep_bp, void* stream);
/* end side from the final row (owner partition plan->owner_part):
 * state[4] (device) = {column, client side, flag 0 ok / 1 infeasible /
 * 2 backtrace error, next stage} (planner.py:190-200) */
int sp_grid_part_end(const sp_grid_plan* plan, void* owner_ws, int8_t must_end_at, int64_t* state,
                     void* stream);
/* walk segment `seg` through this partition's back-pointers while the column
 * stays in its range; writes pi[stage] (device u8[L]) and advances state */
int sp_grid_part_backtrack(const sp_grid_plan* plan, int32_t part, void* part_ws, int32_t seg, int64_t* state,
                           uint8_t* pi, void* stream);

/* CUDA IPC of a device buffer: a 64-byte handle of its allocation plus the
 * buffer's offset in it; import maps it (returns the buffer and the mapping
 * base to close). */
int sp_ipc_export(const void* dptr, void* handle64, size_t* offset);
int sp_ipc_import(const void* handle64, size_t offset, void** dptr, void** base);
int sp_ipc_close(void* base);

/* Full DP tables of ONE instance (in->n == 1) as float64, row-major
 * [(L+1) x (w_eff+1)], unreachable cells = -inf.  Replaces planner.py:128-143
 * `build_dp_tables`.  w_eff must equal sp_effective_budget()'s value
 * (SP_ERR_INVALID otherwise, before anything is written). */
int sp_build_dp_tables(const sp_instances* in, int64_t w_eff, double* client_table,
                       double* server_table, void* ws, size_t ws_bytes, void* stream);

/* Prefix planners: greedy longest feasible client prefix, all-server,
 * all-client.  Replaces planner.py:205-214 `plan_greedy` and :217-225
 * `plan_trivial`.  `which` is an sp_prefix_planner. */
int sp_plan_prefix(const sp_instances* in, int32_t which, sp_policies* out, void* stream);

/* Exhaustive planner over all 2^L placements (L <= 24; SP_ERR_UNSUPPORTED
 * for longer instances).  Replaces
 * planner.py:228-268 `plan_oracle`: maximum client value among feasible
 * masks, ties to the smallest mask with layer 1 as the MSB. */
int sp_plan_exhaustive(const sp_instances* in, sp_policies* out, void* stream);

/* ---- evaluator (evaluator.py) ------------------------------------------ */

/* Eq. (1) real-valued latency of each policy (evaluator.py:64-78
 * `latency_of`): per-layer terms x(c + (1-x')d) + (1-x)(s + x'u) summed in
 * numpy pairwise order.  Times are [total_layers] float64; latency_s [n]. */
int sp_latency_eq1(const sp_instances* in, const double* client_s, const double* server_s,
                   const double* up_s, const double* down_s, const uint8_t* pi,
                   double* latency_s, void* stream);



/* _finish for caller-supplied placements (planner.py:88-101): fills
 * client_value / server_load (numpy order), integer_latency and feasible of
 * each policy pi.  Also evaluator.py:81-102 server_load_of / client_value_of.
 * ws: >= 4 * total_layers bytes of scratch. */
int sp_evaluate_policy(const sp_instances* in, const uint8_t* pi, sp_policies* out, void* ws,
                       size_t ws_bytes, void* stream);

/* Elementwise integerization of times (problem.py:79-104): mode 0 = cost,
 * conservative (ceil); 1 = paper (floor(q+0.5)), cost or budget; 2 = budget,
 * conservative (floor).  status[k] is an sp_cost_status. */
int sp_to_units(const double* seconds, int64_t n, double unit_s, int32_t mode, int64_t* units,
                int32_t* status, void* stream);

/* ---- cost model + integerization (cost_model.py, problem.py) ------------ */

enum sp_layer_kind {  /* cost_model.py:43-49 LayerKind */
  SP_EMBEDDING = 0, SP_ATTENTION = 1, SP_FEED_FORWARD = 2,
  SP_LAYER_NORM = 3, SP_CLASSIFIER = 4, SP_CUSTOM = 5
};

/* Model specs (cost_model.py:52-106 LayerSpec / ModelSpec), CSR over layer
 * entries: model m owns entries [layer_off[m], layer_off[m+1]). */
typedef struct sp_models {
  int64_t n_models;
  const int64_t* layer_off;         /* [n_models+1] */
  const int32_t* kind;              /* [E] sp_layer_kind */
  const int64_t* hidden_dim;        /* [E] */
  const int64_t* heads;             /* [E] */
  const int64_t* ffn_dim;           /* [E] */
  const int64_t* out_dim;           /* [E] */
  const int64_t* seq_divisor;       /* [E] */
  const double* flop_coeffs;        /* [E*3] custom (quad, lin, const) */
  const double* mem_coeffs;         /* [E*3] custom, valid where has_mem_coeffs */
  const uint8_t* has_mem_coeffs;    /* [E] */
  const double* out_bytes_per_token;/* [E] custom, valid where has_out_bytes */
  const uint8_t* has_out_bytes;     /* [E] */
} sp_models;

enum sp_request_flags {
  SP_REQ_PAPER_ROUNDING = 1,  /* problem.py rounding="paper" (else conservative) */
  SP_REQ_SOURCE_CLIENT = 2,   /* source_at_client */
  SP_REQ_ZERO_SERVER = 4,     /* build_problem zero_server_time */
  SP_REQ_METRIC_MEMORY = 8    /* profile metric="memory" (else "flop") */
};

/* One scenario per request: model x seq_len x devices x link x deadline. */
typedef struct sp_requests {
  int64_t n;
  const int32_t* model;          /* [n] index into sp_models */
  const int64_t* seq_len;        /* [n] */
  const double* client_fps;      /* [n] DeviceSpec.flops_per_s */
  const double* server_fps;      /* [n] */
  const double* uplink_bps;      /* [n] LinkSpec */
  const double* downlink_bps;    /* [n] */
  const double* propagation_s;   /* [n] */
  const double* deadline_s;      /* [n] */
  const double* unit_s;          /* [n] */
  const uint8_t* flags;          /* [n] sp_request_flags */
} sp_requests;

/* Per-layer profiles supplied directly (build_problem from LayerProfile list). */
typedef struct sp_profiles {
  const double* r;               /* [total_layers] */
  const double* client_time_s;
  const double* server_time_s;
  const double* tau_bytes;
} sp_profiles;

/* Cost-table output, CSR over request layers.  Any per-layer pointer may be
 * NULL to skip it.  The integer arrays + r + budget + source_at_client form
 * an sp_instances batch for the planners. */
typedef struct sp_cost_table {
  const int64_t* layer_off;   /* [n+1] from sp_request_layer_offsets */
  int64_t total_layers;
  double* r;                  /* LayerProfile.r */
  double* client_time_s;      /* LayerProfile.client_time_s */
  double* server_time_s;      /* LayerProfile.server_time_s (profiled) */
  double* tau_bytes;          /* LayerProfile.tau_bytes */
  double* server_s;           /* PlanProblem.server_s (0 under zero_server_time) */
  double* up_s;               /* PlanProblem.up_s (problem.py:58-65) */
  double* down_s;             /* PlanProblem.down_s */
  int64_t* client_units;      /* problem.py:79-92 to_units */
  int64_t* server_units;
  int64_t* up_units;
  int64_t* down_units;
  int64_t* budget;            /* [n] problem.py:95-104 budget_units */
  uint8_t* source_at_client;  /* [n] */
  int32_t* status;            /* [n] 0 ok, else (array sp_cost_status)
                                 | (budget sp_cost_status << 8) | (negative r << 16) */
} sp_cost_table;

enum sp_cost_status {
  SP_COST_OK = 0,
  SP_COST_NEGATIVE_TIME = 1,   /* ValueError("times must be >= 0") problem.py:87 */
  SP_COST_NEGATIVE_R = 2,      /* ValueError("r must be >= 0") problem.py:152 */
  SP_COST_NAN_TIME = 3,        /* ValueError from round(nan) problem.py:69 */
  SP_COST_INF_TIME = 4,        /* OverflowError from round(inf) problem.py:69 */
  SP_COST_OVERFLOW = 5         /* unit count beyond int64 */
};

/* layer_off[k+1] = layer_off[k] + L(model[k]); layer_off device int64[n+1]. */
int sp_request_layer_offsets(const sp_models* models, const sp_requests* req,
                             int64_t* layer_off, void* stream);

/* K1: per (request, layer) profile (cost_model.py:305-329 `profile`), link
 * transfer times and integerization (problem.py:58-115, 188-222
 * `build_problem`); integer outputs are skipped when `integerize` == 0. */
int sp_build_cost_table(const sp_models* models, const sp_requests* req, int32_t integerize,
                        sp_cost_table* out, void* stream);

/* build_problem over caller-supplied profiles (problem.py:188-222). */
int sp_integerize_profiles(const sp_profiles* prof, const sp_requests* req,
                           sp_cost_table* out, void* stream);

/* ---- throughput simulator (throughput_sim.py) --------------------------- */

/* Independent replay runs, CSR over requests: run k owns requests
 * [run_off[k], run_off[k+1]) in arrival order (throughput_sim.py:98-106 Stream). */
typedef struct sp_sim_batch {
  int64_t n_runs;
  int64_t total_requests;      /* == run_off[n_runs] (host value) */
  const int64_t* run_off;      /* [n_runs+1] */
  const double* arrival_ms;    /* [total] non-decreasing within a run */
  const double* demand;        /* [total] */
  const double* duration_ms;   /* [total] */
  const double* capacity;      /* [n_runs] */
} sp_sim_batch;

typedef struct sp_sim_out {
  double* admit_ms;      /* [total] */
  double* wait_ms;       /* [total] or NULL */
  double* cum_wait_ms;   /* [total] or NULL: np.cumsum of waits */
  double* max_wait_ms;   /* [n_runs] or NULL */
  double* mean_wait_ms;  /* [n_runs] or NULL: numpy-order mean */
  int32_t* status;       /* [n_runs] SP_OK or SP_ERR_DEADLOCK */
  int64_t* deadlock_req; /* [n_runs] or NULL: FIFO head that can never fit */
} sp_sim_out;

/* Segmented numpy-order sums: out[k] = np.sum(x[seg_off[k]:seg_off[k+1]])
 * (0.0 + pairwise).  Backs np.sum / np.mean in evaluator.py:102 total_r and
 * throughput_sim.py:156,176 (scenario normalisation, capacity). */
int sp_segment_sum(const double* x, const int64_t* seg_off, int64_t n_seg, double* out,
                   void* stream);

/* Heap workspace the replay needs (16 bytes per request + 128 per run). */
size_t sp_sim_workspace_bytes(const sp_sim_batch* b);

/* K4: FIFO admission with a completion min-heap keyed (finish, seq), one
 * thread per run.  Replaces throughput_sim.py:207-256 `simulate_stream`
 * (and the per-variant loop of :264-272 `compare_variants`). */
int sp_sim_replay(const sp_sim_batch* b, sp_sim_out* out, void* ws, size_t ws_bytes,
                  void* stream);

/* Arrival skeletons, one per seed, drawn by numpy's default_rng(seed) stream
 * bit for bit (PCG64 seeded through SeedSequence, numpy's ziggurat
 * exponential, Lemire bounded integers).  Replaces throughput_sim.py:179-186
 * `_skeleton` for a batch of runs:
 *   g = default_rng(seeds[r])
 *   arrival_ms[r, :] = np.cumsum(g.exponential(scale, horizon))
 *   choice[r, :]     = g.integers(0, choice_hi[r] - choice_lo[r], horizon) + choice_lo[r]
 *   exec_count[r, :] = g.integers(1, exec_max + 1, horizon)
 * Outputs are row-major [n, horizon].  seeds[r] >= 0; 1 <= choice_hi[r] -
 * choice_lo[r] <= 2^32 and the rows < 2^31; 1 <= exec_max < 2^31.  status[r]
 * (optional): SP_OK, or SP_ERR_INVALID for a run whose range is empty (numpy
 * raises ValueError there; nothing is written for it). */
int sp_sim_skeletons(const int64_t* seeds, const int64_t* choice_lo, const int64_t* choice_hi,
                     int64_t n, int64_t horizon, double scale, int64_t exec_max,
                     double* arrival_ms, int32_t* choice, int32_t* exec_count, int32_t* status,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLITPLAN_B200_H */
