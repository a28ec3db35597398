// K2 for ONE huge instance over the whole GPU (cfg5): the grid kernel
// (capacity partitions, devices), its in-place variant, and the grid
// end / backtrack / finish kernels of the checkpoint-recompute path.
//
// Fragment of sp_planner.cu: included there inside namespace sp::(anonymous),
// after the declarations it uses; not a standalone header.
#pragma once

// ---------------------------------------------------------------------------
// K2 grid variant: ONE very large instance (L = 1e5 stages x
// W = 1e7 columns) spread over every co-resident CTA of the GPU (cooperative
// launch).  Same producer-warp / bulk-copy / mbarrier-ring structure as the
// streaming kernel, but the per-CTA progress counters live in global memory
// and each producer waits only on the CTAs that own its windows: the owners
// of columns [j0 - max_shift - 16 B, j0 + B) for the rows it reads (RAW) and
// the CTAs that read its block two stages earlier (WAR on the triple-
// buffered rows).  With small per-stage shifts that is just the two
// neighbours, so the GPU runs as a wavefront with no grid-wide barrier.
// A launch advances a range of stages [k_begin, k_begin + k_count) from an
// initial row (the origin row or a checkpoint) and can write the final row
// (a checkpoint) and the range's back-pointers; the host chains launches
// into checkpoint / recompute passes when the full back-pointer table does
// not fit in memory.

constexpr int kMaxParts = 8;

// One huge instance over the whole GPU (or, partitioned, over several GPUs).
// The capacity axis can be split into `nparts` partitions of Gp CTAs each
// (one per device in a multi-GPU run): partition p owns global columns
// [p*Wp, (p+1)*Wp), Wp = Gp*B, keeps its own triple-buffered rows, and
// mirrors the left neighbour's last `halo` columns of every row in front of
// its column 0 -- the halo, written by the neighbour's CTAs with plain
// (peer) stores as they produce those columns.  Dependencies are computed
// in the global CTA index space, so the protocol is the same whether the
// partitions are launched together (one device, emulating several) or one
// per device.
//
// Every buffer of a partition lives in that partition's own workspace (on its
// device): rows, progress counters, checkpoint rows and back-pointers of its
// columns.  Only the halo stores (into the right neighbour's rows), the
// counter polls and the halo part of a checkpoint restart (from the left
// neighbour's checkpoint) touch a neighbour's memory.
struct GridPart {
  uint8_t* rows;          // [3][C|S][NEG pad | halo | Wp | line]
  uint32_t* prog;         // [G] stages completed + 1 (zeroed before a launch)
  uint32_t* bp;           // back-pointers of this launch's stages, local columns, or null
  const void* init;       // row k_begin, local columns [0, Wp): C then S, or null (origin row)
  const void* init_left;  // the left neighbour's row k_begin (same layout), or null
  void* out;              // row k_begin + k_count, local columns: C then S, or null
};

struct GridArgs {
  const StageShift* shifts;  // stage records of the instance (index = stage)
  const int64_t* rv;         // stage values in the value domain
  const int2* reach;         // per stage: first reachable global column of the C / S row it reads
  int k_begin, k_count;      // stage range of this launch
  int ncol;                  // W_eff + 1
  int G, NC;                 // CTAs per partition, chunks per CTA
  int sac;
  int64_t bp_row_words;      // u32 words per stage row of one partition's back-pointers
  int nparts;                // partitions of the capacity axis
  int part_base;             // first partition of this launch
  int launch_parts;          // partitions of this launch (grid = launch_parts x G)
  int sys;                   // partitions on different devices / processes: system-scope ordering
  int halo;                  // mirrored left-neighbour columns (multiple of 128 B)
  GridPart parts[kMaxParts];
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int max_shift(const StageShift& sh) {
  return max(max(sh.i, sh.id), max(sh.s, sh.su));
}

template <int MODE, int T, int E, int NSLOT>
__global__ void __launch_bounds__(T + 32, 2) dp_grid_kernel(GridArgs a) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  constexpr int AL = 16 / (int)sizeof(V);
  constexpr int WIN = CH + AL;
  constexpr int PAD = stream_pad<V, CH>();  // NEG area in front of the halo
  constexpr int LINE = 128 / (int)sizeof(V);
  constexpr int NWARP = T / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NSLOT;
  V* slots = reinterpret_cast<V*>(smem + 256);
  V* negwin = slots + NSLOT * 4 * WIN;  // [WIN] of NEG: windows below the reachable frontier

  const int G = a.G, NC = a.NC;
  const int part = a.part_base + (int)blockIdx.x / G;
  const int q = (int)blockIdx.x % G;
  const int GT = a.nparts * G;  // CTAs over the whole capacity axis
  const int gq = part * G + q;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = NC * CH;
  const int Wp = G * B;
  const int p0 = part * Wp;      // global column of this partition's local column 0
  const int j0 = q * B;          // local
  const int j0g = p0 + j0;       // global
  const int ncol = a.ncol;
  const int H = a.halo;
  const int64_t span = (int64_t)PAD + H + Wp + LINE;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  auto row_of = [&](int p, int buf, int rs) {
    return reinterpret_cast<V*>(a.parts[p].rows) + (int64_t)(buf * 2 + rs) * span + PAD + H;
  };
  auto row = [&](int buf, int rs) { return row_of(part, buf, rs); };
  auto owner = [&](int x) { return min(GT - 1, max(0, x) / B); };  // global CTA of global column x
  // progress counter of global CTA o (in its partition's -- possibly a peer device's -- memory)
  auto prog_of = [&](int o) { return a.parts[o / G].prog + (o % G); };
  auto publish = [&](uint32_t v) {
    if (a.sys) {
      __threadfence_system();
      fence_proxy_async_global();
      st_release_sys(prog_of(gq), v);
    } else {
      __threadfence();
      fence_proxy_async_global();
      st_release_gpu(prog_of(gq), v);
    }
  };
  const V* ic = reinterpret_cast<const V*>(a.parts[part].init);
  const V* il = reinterpret_cast<const V*>(a.parts[part].init_left);
  auto init_at = [&](int x, V& c, V& sv) {  // row k_begin at global column x (>= p0 - H)
    const bool valid = x >= 0 && x < ncol;
    if (ic) {
      // own columns from this partition's checkpoint, halo columns (x < p0)
      // from the left neighbour's
      const V* src = x >= p0 ? ic + (x - p0) : il + (Wp + x - p0);
      c = valid ? src[0] : NEG;
      sv = valid ? src[Wp] : NEG;
    } else {
      c = (valid && a.sac) ? ZERO : NEG;
      sv = (valid && !a.sac) ? ZERO : NEG;
    }
  };

  for (int buf = 0; buf < kRowBufs; ++buf) {
    V* Cb = row(buf, 0);
    V* Sb = row(buf, 1);
    if (q == 0) {
      for (int x = tid - PAD - H; x < -H; x += blockDim.x) Cb[x] = Sb[x] = NEG;  // NEG area
      // halo of buffer 0: row k_begin of the neighbour's last columns (all NEG
      // in partition 0).  Buffers 1 and 2 belong to the neighbour's CTAs, which
      // write them before any read (RAW) -- never touch them here.
      if (buf == 0)
        for (int x = tid - H; x < 0; x += blockDim.x) {
          V c = NEG, sv = NEG;
          if (part > 0) init_at(p0 + x, c, sv);
          Cb[x] = c;
          Sb[x] = sv;
        }
      else if (part == 0)
        for (int x = tid - H; x < 0; x += blockDim.x) Cb[x] = Sb[x] = NEG;
    }
    if (q == G - 1)
      for (int x = Wp + tid; x < Wp + LINE; x += blockDim.x) Cb[x] = Sb[x] = NEG;
    if (buf == 0)
      for (int j = j0 + tid; j < j0 + B; j += blockDim.x) init_at(p0 + j, Cb[j], Sb[j]);
  }
  for (int x = tid; x < WIN; x += blockDim.x) negwin[x] = NEG;
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) publish(1u);  // rows initialised (counter = completed stages + 1)

  if (warp == NWARP) {
    // ---------------- producer warp ----------------
    uint32_t u = 0;
    for (int t = 0; t < a.k_count; ++t) {
      const int k = a.k_begin + t;
      const StageShift sh = a.shifts[k];
      // RAW: owners of the windows read this stage (row t complete => counter >= t + 1)
      const int lo_o = owner(j0g - max_shift(sh) - AL);
      // WAR: CTAs that read this block's target buffers (own rows and the
      // right neighbour's halo copy) two stages ago
      int hi_o = gq;
      if (t >= 2) hi_o = owner(j0g + B - 1 + max_shift(a.shifts[k - 2]) + CH + AL);
      for (int o0 = lo_o; o0 <= hi_o; o0 += 32) {
        const int o = o0 + lane;
        const uint32_t need = o <= gq ? (uint32_t)(t + 1) : (uint32_t)max(t - 1, 0) + 1u;
        // (a watchdog turns a lost partition -- e.g. launches that were not
        // co-scheduled -- into a launch failure instead of a hang)
        const long long t0 = clock64();
        for (uint32_t it = 1;; ++it) {
          const bool ok = o > hi_o || (a.sys ? ld_acquire_sys(prog_of(o)) : ld_acquire_gpu(prog_of(o))) >= need;
          if (__all_sync(0xffffffffu, ok)) break;
          if ((it & 1023u) == 0 && clock64() - t0 > (30ll << 30)) __trap();
        }
      }
      if (lane == 0) {
        fence_proxy_async_global();
        const V* Cc = row(t % kRowBufs, 0);
        const V* Sc = row(t % kRowBufs, 1);
        const V* src[4] = {Cc, Sc, Sc, Cc};
        const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
        const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
        const int mrow[4] = {rch.x, rch.y, rch.y, rch.x};
        for (int c = 0; c < NC; ++c, ++u) {
          const int slot = (int)(u % NSLOT);
          mbar_wait(&empty[slot], ((u / NSLOT) & 1) ^ 1);
          const int c0g = j0g + c * CH, ctop = c0g + CH;
          uint32_t ncopy = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) ncopy += c0g - min(shf[w], ctop) + CH > mrow[w] ? 1u : 0u;
          mbar_expect_tx(&full[slot], ncopy * WIN * sizeof(V));
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int start = c0g - min(shf[w], ctop);
            if (start + CH <= mrow[w]) continue;  // below the reachable frontier: all NEG, no copy
            // Partition 0 keeps NEG in front of column 0 (halo + NEG area), so
            // partially negative windows read it in place.  In later
            // partitions start < 0 only when the shift was clamped (every cell
            // of the window unreachable): read the NEG area.
            const int local = (start < 0 && part > 0) ? -H - PAD : (start & ~(AL - 1)) - p0;
            bulk_g2s(slots + (slot * 4 + w) * WIN, src[w] + local, WIN * sizeof(V), &full[slot]);
          }
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- compute warps ----------------
    const uint64_t pol = evict_first_policy();
    uint32_t u = 0;
    StageShift sh_next = a.shifts[a.k_begin];
    int64_t rbits_next = a.rv[a.k_begin];
    // global columns mirrored into the right neighbour's halo
    const int halo_lo = part + 1 < a.nparts ? p0 + Wp - H : INT_MAX;
    for (int t = 0; t < a.k_count; ++t) {
      const StageShift sh = sh_next;
      const int64_t rbits = rbits_next;
      if (t + 1 < a.k_count) {
        sh_next = a.shifts[a.k_begin + t + 1];
        rbits_next = a.rv[a.k_begin + t + 1];
      }
      const V rk = MODE == VM_INT32 ? (V)(int32_t)rbits : (V)__longlong_as_double(rbits);
      V* Cn = row((t + 1) % kRowBufs, 0);
      V* Sn = row((t + 1) % kRowBufs, 1);
      uint32_t* bpp = a.parts[part].bp;
      uint32_t* bprow = bpp ? bpp + (int64_t)t * a.bp_row_words + warp * bp_words(MODE) : nullptr;
      const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
      // every cell of row t+1 below both frontiers is unreachable
      const int64_t next_front = a.reach ? min(min((int64_t)rch.x + sh.i, (int64_t)rch.y + sh.id),
                                               min((int64_t)rch.y + sh.s, (int64_t)rch.x + sh.su))
                                         : 0;
      for (int c = 0; c < NC; ++c, ++u) {
        const int slot = (int)(u % NSLOT);
        const int c0 = j0 + c * CH;       // local
        const int c0g = p0 + c0, ctop = c0g + CH;
        const int sa = c0g - min(sh.i, ctop), sb = c0g - min(sh.id, ctop);
        const int sc = c0g - min(sh.s, ctop), sd = c0g - min(sh.su, ctop);
        const V* ws = slots + slot * 4 * WIN + tid;
        const V* pca = (sa + CH > rch.x ? ws + 0 * WIN : negwin + tid) + (sa & (AL - 1));
        const V* pcb = (sb + CH > rch.y ? ws + 1 * WIN : negwin + tid) + (sb & (AL - 1));
        const V* psa = (sc + CH > rch.y ? ws + 2 * WIN : negwin + tid) + (sc & (AL - 1));
        const V* psb = (sd + CH > rch.x ? ws + 3 * WIN : negwin + tid) + (sd & (AL - 1));
        mbar_wait(&full[slot], (u / NSLOT) & 1);
        V cn[E], sn[E];
        CellFlags f[E];
        const bool dead = (int64_t)ctop <= next_front;  // whole chunk unreachable: NEG, no back-pointers
        if (dead) {
#pragma unroll
          for (int e = 0; e < E; ++e) cn[e] = sn[e] = NEG;
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0g + e * T + tid;
            f[e] = cell_update<MODE, V>(pca[e * T], pcb[e * T], psa[e * T], psb[e * T], rk, j >= sh.i,
                                        j >= sh.id, j >= sh.s, j >= sh.su, cn[e], sn[e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (bprow && !dead) {
          uint32_t* bpc = bprow + (c0 >> 5) * bp_words(MODE);  // local column groups
#pragma unroll
          for (int e = 0; e < E; ++e) emit_bp_stream<MODE>(bpc + e * (T / 32) * bp_words(MODE), f[e], pol);
        }
        V* qc = Cn + c0 + tid;
        V* qs = Sn + c0 + tid;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          qc[e * T] = cn[e];
          qs[e * T] = sn[e];
        }
        if (ctop > halo_lo) {  // the right neighbour mirrors these columns
          V* hc = row_of(part + 1, (t + 1) % kRowBufs, 0) - (p0 + Wp);
          V* hs = row_of(part + 1, (t + 1) % kRowBufs, 1) - (p0 + Wp);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0g + e * T + tid;
            if (j >= halo_lo) {
              hc[j] = cn[e];
              hs[j] = sn[e];
            }
          }
        }
      }
      named_barrier(1, T);
      if (tid == 0) publish((uint32_t)(t + 2));
    }
    // the range's final row (this CTA's own block: its own writes)
    if (a.parts[part].out) {
      named_barrier(1, T);
      V* oc = reinterpret_cast<V*>(a.parts[part].out);
      const V* Cf = row(a.k_count % kRowBufs, 0);
      const V* Sf = row(a.k_count % kRowBufs, 1);
      for (int j = j0 + tid; j < j0 + B; j += T) {
        oc[j] = Cf[j];
        oc[Wp + j] = Sf[j];
      }
    }
  }
}

// End of the forward pass of a grid-solved instance: the end side from the
// final row's last cell (planner.py:190-200), read from the checkpoint of
// the partition owning column W_eff (`last`: its C row then S row, Wp values
// each), or the infeasible policy.  state = {j, client side, flag (0 ok,
// 1 infeasible, 2 backtrace error), next stage to decide}.
__global__ void grid_end_kernel(InstInfo* info, int64_t p0, int64_t Wp, int L, int must_val,
                                const int8_t* must_ptr, const void* last, int64_t* state) {
  const InstInfo inf = *info;
  const int64_t jl = inf.w_eff - p0;  // local column in the owning partition
  double ec, es;
  if (inf.mode == VM_INT32) {
    ec = to_f64(reinterpret_cast<const int32_t*>(last)[jl], inf.scale);
    es = to_f64(reinterpret_cast<const int32_t*>(last)[Wp + jl], inf.scale);
  } else {
    ec = reinterpret_cast<const double*>(last)[jl];
    es = reinterpret_cast<const double*>(last)[Wp + jl];
  }
  info->end_c = ec;
  info->end_s = es;
  const int must = must_ptr ? (int)*must_ptr : must_val;
  if (must == 1) es = -INFINITY;
  else if (must == 0) ec = -INFINITY;
  const double pmax = (es > ec) ? es : ec;
  state[0] = inf.w_eff;
  state[1] = ec >= es ? 1 : 0;
  state[2] = pmax == -INFINITY ? 1 : 0;
  state[3] = L - 1;
}

// Walk the back-pointers of ONE capacity partition (global columns
// [p0, p0 + Wp)) through one segment of stages [k_begin, k_begin + k_count),
// from state {j, side, flag, next stage k}, writing pi[k] (stage-indexed).
// The walk stops when j leaves the partition to the left -- the state is
// then handed to the left neighbour, which continues from stage k -- or at
// the segment's first stage.  j never grows, so one pass over the partitions
// from right to left finishes a segment.  Same decisions as backtrack_kernel
// (planner.py:146-179).  bp: this partition's back-pointers of the segment,
// stage rows of row_words u32 over local columns.
__global__ void grid_backtrack_part_kernel(const StageShift* shifts, const uint32_t* bp, int64_t row_words,
                                           int mode, int k_begin, int k_count, int64_t p0, int64_t* state,
                                           uint8_t* pi) {
  if (state[2] != 0) return;  // infeasible or failed: nothing to walk
  int64_t j = state[0];
  bool client = state[1] != 0;
  int k = (int)state[3];
  const int nw = bp_words(mode);
  for (; k >= k_begin && j >= p0; --k) {
    const int t = k - k_begin;
    const int64_t jl = j - p0;
    const uint32_t* grp = bp + (int64_t)t * row_words + (jl >> 5) * nw;
    const uint32_t bit = 1u << (jl & 31);
    const bool c_stay = grp[0] & bit, s_stay = grp[1] & bit;
    const bool c_sw = nw == 4 ? (grp[2] & bit) != 0 : !c_stay;
    const bool s_sw = nw == 4 ? (grp[3] & bit) != 0 : !s_stay;
    const StageShift sh = shifts[k];
    if (client) {
      pi[k] = 1;
      if (c_stay) {
        j -= sh.i;
      } else if (c_sw) {
        j -= sh.id;
        client = false;
      } else {
        state[2] = 2;
        return;
      }
    } else {
      pi[k] = 0;
      if (s_stay) {
        j -= sh.s;
      } else if (s_sw) {
        j -= sh.su;
        client = true;
      } else {
        state[2] = 2;
        return;
      }
    }
  }
  state[0] = j;
  state[1] = client ? 1 : 0;
  state[3] = k;
}

// ---------------------------------------------------------------------------
// _finish (planner.py:88-101) for a placement already written to pi

__device__ void finish_policy(const sp_instances& in, int64_t inst, int64_t lo, int L,
                              int32_t* idx, sp_policies& out, bool feasible_hint, bool hint_value) {
  const uint8_t* pi = out.pi + lo;
  const bool sac = in.source_at_client[inst] != 0;
  int64_t lat = 0;
  int prev = sac ? 1 : 0;
  int n1 = 0;
  for (int k = 0; k < L; ++k) {
    const int x = pi[k];
    if (x) {
      lat += in.client_units[lo + k] + (prev == 0 ? in.down_units[lo + k] : 0);
      ++n1;
    } else {
      lat += in.server_units[lo + k] + (prev == 1 ? in.up_units[lo + k] : 0);
    }
    prev = x;
  }
  int a = 0, b = n1;
  for (int k = 0; k < L; ++k) {
    if (pi[k]) idx[a++] = k;
    else idx[b++] = k;
  }
  const double* r = in.r + lo;
  const double cv = np_sum([&](int64_t m) { return r[idx[m]]; }, n1);
  const double sl = np_sum([&](int64_t m) { return r[idx[n1 + m]]; }, L - n1);
  out.client_value[inst] = cv;
  out.server_load[inst] = sl;
  out.integer_latency[inst] = lat;
  out.feasible[inst] = feasible_hint ? (hint_value ? 1 : 0) : (lat <= in.budget[inst] ? 1 : 0);
}


// _finish of one grid-solved instance; state[2]: 0 ok, 1 infeasible, 2 backtrace error
__global__ void grid_finish_kernel(sp_instances in, int64_t inst, const int64_t* state,
                                   int32_t* idx_scratch, sp_policies out) {
  const int64_t lo = in.layer_off[inst];
  const int L = (int)(in.layer_off[inst + 1] - lo);
  if (state[2] == 2) {  // planner.py:168-169 / 177-178 AssertionError
    out.status[inst] = SP_ERR_BACKTRACE;
    return;
  }
  if (state[2] == 1)
    for (int k = 0; k < L; ++k) out.pi[lo + k] = 0;
  finish_policy(in, inst, lo, L, idx_scratch + lo, out, state[2] == 1, false);
  out.status[inst] = SP_OK;
}

