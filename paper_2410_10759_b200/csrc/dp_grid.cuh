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
struct GridArgs {
  const StageShift* shifts;  // stage records of the instance (index = stage)
  const int64_t* rv;         // stage values in the value domain
  const int2* reach;         // per stage: first reachable global column of the C / S row it reads
  int k_begin, k_count;      // stage range of this launch
  int ncol;                  // W_eff + 1
  int G, NC;                 // CTAs per partition, chunks per CTA
  int sac;
  const void* init_c;        // row k_begin, ncol values each, or null: origin row
  const void* init_s;
  void* out_c;               // row k_begin + k_count, or null
  void* out_s;
  uint32_t* bp;              // back-pointers of the range's stages, or null
  int64_t bp_row_words;
  uint32_t* progs[kMaxParts];  // per partition: [G] stages completed + 1 (zeroed)
  int nparts;                // partitions of the capacity axis
  int part_base;             // first partition of this launch
  int launch_parts;          // partitions of this launch (grid = launch_parts x G)
  int sys;                   // partitions on different devices: system-scope ordering
  int halo;                  // mirrored left-neighbour columns (multiple of 128 B)
  uint8_t* rows[kMaxParts];  // per partition: [3][C|S][NEG pad | halo | Wp | line]
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

__device__ __forceinline__ int max_shift(const StageShift& sh) {
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
    return reinterpret_cast<V*>(a.rows[p]) + (int64_t)(buf * 2 + rs) * span + PAD + H;
  };
  auto row = [&](int buf, int rs) { return row_of(part, buf, rs); };
  auto owner = [&](int x) { return min(GT - 1, max(0, x) / B); };  // global CTA of global column x
  // progress counter of global CTA o (in its partition's -- possibly a peer device's -- memory)
  auto prog_of = [&](int o) { return a.progs[o / G] + (o % G); };
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
  const V* ic = reinterpret_cast<const V*>(a.init_c);
  const V* is = reinterpret_cast<const V*>(a.init_s);
  auto init_at = [&](int x, V& c, V& sv) {  // row k_begin at global column x
    const bool valid = x >= 0 && x < ncol;
    if (ic) {
      c = valid ? ic[x] : NEG;
      sv = valid ? is[x] : NEG;
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
      uint32_t* bprow = a.bp ? a.bp + (int64_t)t * a.bp_row_words + warp * bp_words(MODE) : nullptr;
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
          uint32_t* bpc = bprow + (c0g >> 5) * bp_words(MODE);
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
    if (a.out_c) {
      named_barrier(1, T);
      V* oc = reinterpret_cast<V*>(a.out_c);
      V* os = reinterpret_cast<V*>(a.out_s);
      const V* Cf = row(a.k_count % kRowBufs, 0);
      const V* Sf = row(a.k_count % kRowBufs, 1);
      for (int j = j0 + tid; j < j0 + B && p0 + j < ncol; j += T) {
        oc[p0 + j] = Cf[j];
        os[p0 + j] = Sf[j];
      }
    }
  }
}

// End of the forward pass of a grid-solved instance: the end side from the
// final row's last cell (planner.py:190-200), or the infeasible policy.
// state = {j, client side, infeasible}.
// ---------------------------------------------------------------------------
// K2 grid variant with ONE row buffer (single partition, every stage's
// shifts <= the halo width): the rows of a 1e7-column instance are 80 MB
// instead of 240 MB with three buffers, so they stay in L2 instead of
// streaming through HBM (profiles/r01/dp_grid_ncu_summary.json: 15.5 B/cell
// of DRAM traffic with three buffers).  Each CTA updates its block IN PLACE,
// chunks top-down: every predecessor window of chunk c lies below the top of
// chunk c (reads go left), so the chunks above c that already hold the new
// row are never read again this stage, and window copies already sit in
// shared-memory slots before chunk c stores over them.  Nobody else reads the
// main buffer: the right neighbour takes this block's last `hw` columns from
// a small per-CTA halo buffer (3 stage slots) written alongside the row.
// Producer waits per stage: own and left neighbour finished the previous
// stage (RAW), right neighbour finished the stage two back (WAR on the halo
// slot this stage overwrites).
struct GridInplaceArgs {
  const StageShift* shifts;
  const int64_t* rv;
  const int2* reach;
  int k_begin, k_count;
  int ncol, G, NC, sac, hw;  // hw: halo columns (multiple of 128 B, <= B)
  const void* init_c;
  const void* init_s;
  void* out_c;
  void* out_s;
  uint32_t* bp;
  int64_t bp_row_words;
  uint32_t* prog;  // [G] completed stages + 1 (zeroed)
  uint8_t* rows;   // [C|S][PAD | G*B | line]
  uint8_t* halo;   // [G][3][C|S][hw]
  int row_hint;    // 1: row stores with an L2 evict_last policy (SPLITPLAN_ROW_EVICT_LAST)
};

template <int MODE, int T, int E, int NSLOT>
__global__ void __launch_bounds__(T + 32, 2) dp_grid_inplace_kernel(GridInplaceArgs a) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  constexpr int AL = 16 / (int)sizeof(V);
  constexpr int WIN = CH + AL;
  constexpr int PAD = stream_pad<V, CH>();
  constexpr int LINE = 128 / (int)sizeof(V);
  constexpr int NWARP = T / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NSLOT;
  V* slots = reinterpret_cast<V*>(smem + 256);
  V* negwin = slots + NSLOT * 4 * WIN;  // [WIN] of NEG: windows below the reachable frontier

  const int G = a.G, NC = a.NC;
  const int q = (int)blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = NC * CH;
  const int Wt = G * B;
  const int j0 = q * B;
  const int ncol = a.ncol, hw = a.hw;
  const int64_t span = (int64_t)PAD + Wt + LINE;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  V* const Cm = reinterpret_cast<V*>(a.rows) + PAD;          // C row, column 0
  V* const Sm = reinterpret_cast<V*>(a.rows) + span + PAD;   // S row, column 0
  // halo of CTA o, stage slot t % 3: columns [o*B + B - hw, o*B + B) of row t
  auto halo = [&](int o, int slot, int rs) {
    return reinterpret_cast<V*>(a.halo) + ((int64_t)(o * 3 + slot) * 2 + rs) * hw;
  };
  const V* ic = reinterpret_cast<const V*>(a.init_c);
  const V* is = reinterpret_cast<const V*>(a.init_s);

  // row k_begin in the main buffer, its top hw columns in halo slot 0, NEG pads
  for (int x = j0 + tid; x < j0 + B; x += blockDim.x) {
    const bool valid = x < ncol;
    V c, s;
    if (ic) {
      c = valid ? ic[x] : NEG;
      s = valid ? is[x] : NEG;
    } else {
      c = (valid && a.sac) ? ZERO : NEG;
      s = (valid && !a.sac) ? ZERO : NEG;
    }
    Cm[x] = c;
    Sm[x] = s;
    if (x >= j0 + B - hw) {
      halo(q, 0, 0)[x - (j0 + B - hw)] = c;
      halo(q, 0, 1)[x - (j0 + B - hw)] = s;
    }
  }
  if (q == 0)
    for (int x = tid - PAD; x < 0; x += blockDim.x) Cm[x] = Sm[x] = NEG;
  if (q == G - 1)
    for (int x = Wt + tid; x < Wt + LINE; x += blockDim.x) Cm[x] = Sm[x] = NEG;
  for (int x = tid; x < WIN; x += blockDim.x) negwin[x] = NEG;
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    fence_proxy_async_global();
    st_release_gpu(&a.prog[q], 1u);
  }

  if (warp == NWARP) {
    // ---------------- producer warp ----------------
    uint32_t u = 0;
    for (int t = 0; t < a.k_count; ++t) {
      const StageShift sh = a.shifts[a.k_begin + t];
      // lane 0: own block (row t complete), lane 1: left neighbour (its halo
      // of row t), lane 2: right neighbour (finished stage t - 2: halo slot reuse)
      const int o = lane == 0 ? q : (lane == 1 ? q - 1 : q + 1);
      const bool watch = lane < 3 && o >= 0 && o < G;
      const uint32_t need = lane < 2 ? (uint32_t)(t + 1) : (uint32_t)max(t - 1, 0) + 1u;
      const long long t0 = clock64();
      for (uint32_t it = 1;; ++it) {
        if (__all_sync(0xffffffffu, !watch || ld_acquire_gpu(&a.prog[o]) >= need)) break;
        if ((it & 1023u) == 0 && clock64() - t0 > (30ll << 30)) __trap();
      }
      if (lane == 0) {
        fence_proxy_async_global();
        const V* hc = q > 0 ? halo(q - 1, t % 3, 0) - (j0 - hw) : nullptr;  // index by global column
        const V* hs = q > 0 ? halo(q - 1, t % 3, 1) - (j0 - hw) : nullptr;
        const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
        const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
        const int mrow[4] = {rch.x, rch.y, rch.y, rch.x};
        for (int c = NC - 1; c >= 0; --c, ++u) {
          const int slot = (int)(u % NSLOT);
          mbar_wait(&empty[slot], ((u / NSLOT) & 1) ^ 1);
          const int c0 = j0 + c * CH, ctop = c0 + CH;
          uint32_t ncopy = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) ncopy += c0 - min(shf[w], ctop) + CH > mrow[w] ? 1u : 0u;
          mbar_expect_tx(&full[slot], ncopy * WIN * sizeof(V));
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const bool cw = w == 0 || w == 3;
            const int start = c0 - min(shf[w], ctop);
            if (start + CH <= mrow[w]) continue;  // below the reachable frontier: all NEG, no copy
            V* dst = slots + (slot * 4 + w) * WIN;
            if (q == 0 || start < 0) {  // partition start: NEG pad in front of column 0
              const int sa = start < 0 && q > 0 ? -PAD : (start & ~(AL - 1));
              bulk_g2s(dst, (cw ? Cm : Sm) + sa, WIN * sizeof(V), &full[slot]);
              continue;
            }
            const int sa = start & ~(AL - 1);
            const int split = min(max(j0 - sa, 0), WIN);  // values from the left halo
            if (split > 0)
              bulk_g2s(dst, (cw ? hc : hs) + sa, split * sizeof(V), &full[slot]);
            if (split < WIN)
              bulk_g2s(dst + split, (cw ? Cm : Sm) + sa + split, (WIN - split) * sizeof(V), &full[slot]);
          }
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- compute warps ----------------
    const uint64_t pol = evict_first_policy();
    const uint64_t rpol = evict_last_policy();
    uint32_t u = 0;
    StageShift sh_next = a.shifts[a.k_begin];
    int64_t rbits_next = a.rv[a.k_begin];
    const int hlo = j0 + B - hw;  // first column mirrored into this CTA's halo
    for (int t = 0; t < a.k_count; ++t) {
      const StageShift sh = sh_next;
      const int64_t rbits = rbits_next;
      if (t + 1 < a.k_count) {
        sh_next = a.shifts[a.k_begin + t + 1];
        rbits_next = a.rv[a.k_begin + t + 1];
      }
      const V rk = MODE == VM_INT32 ? (V)(int32_t)rbits : (V)__longlong_as_double(rbits);
      V* const hc = halo(q, (t + 1) % 3, 0) - hlo;
      V* const hs = halo(q, (t + 1) % 3, 1) - hlo;
      uint32_t* bprow = a.bp ? a.bp + (int64_t)t * a.bp_row_words + warp * bp_words(MODE) : nullptr;
      const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
      const int64_t next_front = a.reach ? min(min((int64_t)rch.x + sh.i, (int64_t)rch.y + sh.id),
                                               min((int64_t)rch.y + sh.s, (int64_t)rch.x + sh.su))
                                         : 0;
      for (int c = NC - 1; c >= 0; --c, ++u) {
        const int slot = (int)(u % NSLOT);
        const int c0 = j0 + c * CH, ctop = c0 + CH;
        const int sa = c0 - min(sh.i, ctop), sb = c0 - min(sh.id, ctop);
        const int sc = c0 - min(sh.s, ctop), sd = c0 - min(sh.su, ctop);
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
            const int j = c0 + e * T + tid;
            f[e] = cell_update<MODE, V>(pca[e * T], pcb[e * T], psa[e * T], psb[e * T], rk, j >= sh.i,
                                        j >= sh.id, j >= sh.s, j >= sh.su, cn[e], sn[e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (bprow && !dead) {
          uint32_t* bpc = bprow + (c0 >> 5) * bp_words(MODE);
#pragma unroll
          for (int e = 0; e < E; ++e) emit_bp_stream<MODE>(bpc + e * (T / 32) * bp_words(MODE), f[e], pol);
        }
        V* qc = Cm + c0 + tid;
        V* qs = Sm + c0 + tid;
        if (a.row_hint) {  // keep the rows ahead of the streamed back-pointers in L2
#pragma unroll
          for (int e = 0; e < E; ++e) {
            st_hint(qc + e * T, cn[e], rpol);
            st_hint(qs + e * T, sn[e], rpol);
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            qc[e * T] = cn[e];
            qs[e * T] = sn[e];
          }
        }
        if (ctop > hlo) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0 + e * T + tid;
            if (j >= hlo) {
              hc[j] = cn[e];
              hs[j] = sn[e];
            }
          }
        }
      }
      named_barrier(1, T);
      if (tid == 0) {
        __threadfence();
        fence_proxy_async_global();
        st_release_gpu(&a.prog[q], (uint32_t)(t + 2));
      }
    }
    if (a.out_c) {
      named_barrier(1, T);
      V* oc = reinterpret_cast<V*>(a.out_c);
      V* os = reinterpret_cast<V*>(a.out_s);
      for (int j = j0 + tid; j < j0 + B && j < ncol; j += T) {
        oc[j] = Cm[j];
        os[j] = Sm[j];
      }
    }
  }
}

__global__ void grid_end_kernel(sp_instances in, InstInfo* info, int64_t inst, const void* last_c,
                                const void* last_s, int64_t* state) {
  const InstInfo inf = info[inst];
  const int64_t jl = inf.w_eff;
  double ec, es;
  if (inf.mode == VM_INT32) {
    ec = to_f64(reinterpret_cast<const int32_t*>(last_c)[jl], inf.scale);
    es = to_f64(reinterpret_cast<const int32_t*>(last_s)[jl], inf.scale);
  } else {
    ec = reinterpret_cast<const double*>(last_c)[jl];
    es = reinterpret_cast<const double*>(last_s)[jl];
  }
  info[inst].end_c = ec;
  info[inst].end_s = es;
  const int8_t must = in.must_end_at ? in.must_end_at[inst] : (int8_t)-1;
  if (must == 1) es = -INFINITY;
  else if (must == 0) ec = -INFINITY;
  const double pmax = (es > ec) ? es : ec;
  state[0] = jl;
  state[1] = ec >= es ? 1 : 0;
  state[2] = pmax == -INFINITY ? 1 : 0;
}

// Walk one segment of back-pointers (stages k_begin + k_count - 1 .. k_begin)
// from state {j, side}, writing pi; the same decisions as backtrack_kernel.
__global__ void grid_backtrack_kernel(sp_instances in, int64_t inst, const StageShift* shifts,
                                      const uint32_t* bp, int64_t row_words, int mode, int k_begin,
                                      int k_count, int64_t* state, sp_policies out) {
  const int64_t lo = in.layer_off[inst];
  int64_t j = state[0];
  bool client = state[1] != 0;
  const int nw = bp_words(mode);
  uint8_t* pi = out.pi + lo;
  for (int t = k_count - 1; t >= 0; --t) {
    const int k = k_begin + t;
    const uint32_t* grp = bp + (int64_t)t * row_words + (j >> 5) * nw;
    const uint32_t bit = 1u << (j & 31);
    const bool c_stay = grp[0] & bit, s_stay = grp[1] & bit;
    const bool c_sw = nw == 4 ? (grp[2] & bit) != 0 : !c_stay;
    const bool s_sw = nw == 4 ? (grp[3] & bit) != 0 : !s_stay;
    const StageShift sh = shifts[lo + k];
    if (client) {
      pi[k] = 1;
      if (c_stay) {
        j -= sh.i;
      } else if (c_sw) {
        j -= sh.id;
        client = false;
      } else {
        out.status[inst] = SP_ERR_BACKTRACE;
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
        out.status[inst] = SP_ERR_BACKTRACE;
        state[2] = 2;
        return;
      }
    }
  }
  state[0] = j;
  state[1] = client ? 1 : 0;
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
  if (state[2] == 2) return;  // status already set
  if (state[2] == 1)
    for (int k = 0; k < L; ++k) out.pi[lo + k] = 0;
  finish_policy(in, inst, lo, L, idx_scratch + lo, out, state[2] == 1, false);
  out.status[inst] = SP_OK;
}

