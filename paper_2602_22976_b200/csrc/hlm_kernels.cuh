// hlm_kernels.cuh -- sm_100a kernels of the local-max matching round (CRCW variant), the exact
// tie path, loader helpers, result assembly and verification.  Included by hlm_engine.cu only.
// Kernel roles and the reference phases they replace: see hlm_types.cuh and DESIGN.md.
#pragma once
#include <cooperative_groups.h>

#include "hlm_types.cuh"

namespace hlmb {

// ---------------------------------------------------------------------------------------------
// Round kernels, class 0: one thread per edge (size <= kLargeEdge), ITEMS edges per thread and
// tile.  D > 0: uniform edge size, one 64/128-bit pin load per edge; D == 0: runtime offsets.
// ---------------------------------------------------------------------------------------------
#ifndef HLM_SWEEP_MIN_BLOCKS
#define HLM_SWEEP_MIN_BLOCKS 5  // d = 2: 48 registers for the four in-flight batches of a warp
#endif
#ifndef HLM_SIMPLE_MIN_BLOCKS
#define HLM_SIMPLE_MIN_BLOCKS 8  // later-round sweep of d = 2, 4: 32 registers, 64 warps per SM
#endif
#ifndef HLM_SWEEP_MIN_BLOCKS_D4
#define HLM_SWEEP_MIN_BLOCKS_D4 3
#endif
#ifndef HLM_SWEEP_MIN_BLOCKS_D8
#define HLM_SWEEP_MIN_BLOCKS_D8 2
#endif
#ifndef HLM_MIN_BLOCKS
#define HLM_MIN_BLOCKS 6  // ragged-size sweep: 40 registers (8 CTAs/SM spill: config 3 38.2 -> 36.3 ms)
#endif

__device__ __forceinline__ uint32_t region_count(const RoundParams& P, bool ident, const uint32_t* cnt,
                                                 uint32_t seg) {
  if (!ident) return __ldcg(cnt + seg);  // written by the previous sweep (same launch in the fused kernel)
  const uint64_t b = static_cast<uint64_t>(seg) * P.seg_cap;
  return b >= P.m ? 0u : static_cast<uint32_t>(min(static_cast<uint64_t>(P.seg_cap), P.m - b));
}

// One warp claims `gran` consecutive regions of the id space per ticket (no block barrier anywhere
// in a sweep).  Same-address atomics retire at roughly one per nanosecond, so a kernel that takes
// 75 K tickets cannot finish in less than ~60 us: sweeps over short lists claim 8 regions at a time.
// Static-first mode (the check kernel): the first ticket of a warp is its own index in the grid, no
// atomic, and the dynamic tickets follow behind the grid's warp count, so a short list costs the
// warps that find nothing no atomic at all.  The sweeps do not use it: their first claims measured
// slower that way on long lists, and the extra state spills in the 32-register kernel.
__device__ __forceinline__ uint32_t grid_warp() { return blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); }
__device__ __forceinline__ uint32_t claim_region(uint32_t* ticket, uint32_t lane, bool static_first) {
  uint32_t seg = 0;
  if (lane == 0) seg = atomicAdd(ticket, 1u);
  return __shfl_sync(0xffffffffu, seg, 0) + (static_first ? gridDim.x * (blockDim.x >> 5) : 0u);
}
constexpr uint32_t kCoarseClaim = 8;
__device__ __forceinline__ uint32_t claim_granularity(const RoundParams& P, uint32_t list_len) {
  // keep several tickets per resident warp (dynamic balance) while the list is long
  return list_len > (P.m >> 3) ? 1u : (list_len > (P.m >> 5) ? 2u : (list_len > (P.m >> 7) ? 4u : kCoarseClaim));
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) { return __reduce_add_sync(0xffffffffu, x); }

// Round 2 on a first-pin sorted instance: the first pins of a region lie in a known id interval
// (consecutive edges of a hub share one vertex).  If every vertex of that interval died in round 1
// the region is dropped without reading a pin: after degree renumbering the sorted order starts
// with the hubs, which are almost always matched in round 1 (round 2 of config 2: 1.89 -> 1.72 ms;
// the same test per 32-edge batch costs more than it saves).
// `first` .. `first + count` are edges of one region, first a multiple of 32
__device__ __forceinline__ bool span_all_dead(const RoundParams& P, uint32_t first, uint32_t count, uint32_t lane) {
  if (!P.bat_pin0) return false;
  const uint32_t lo = __ldg(P.bat_pin0 + (first >> 5)), hi = __ldg(P.bat_pin0 + ((first + count + 31u) >> 5));
  if (hi < lo || hi - lo >= 32u) return false;
  const bool ok = lane > hi - lo || is_dead(P, lo + lane);
  return __all_sync(0xffffffffu, ok);
}

// MERGED (fused kernel, d = 2 / 4): the filter word of a vertex is the high half of its 64-bit key in place --
// no second array and no second atomic per deposit.  An instance this small keeps vkey (8 B per vertex) in L2,
// which is what the separate 4-byte array exists for elsewhere; round 1 of config 1 is bound by the L2's
// atomic rate (8 M atomicMax -> 4 M: 50 -> 27 us).  A covered vertex holds all-ones in both halves.
__device__ __forceinline__ const uint32_t* top_half(const RoundParams& P, uint32_t v) {
  return reinterpret_cast<const uint32_t*>(P.vkey + v) + 1;  // little-endian: the high word
}
template <bool MERGED>
__device__ __forceinline__ uint32_t ld_top_x(const RoundParams& P, uint32_t v) {
  if constexpr (!MERGED) return ld_top(P, v);
  else return v < P.hot_vtop ? __ldca(top_half(P, v)) : __ldcg(top_half(P, v));
}
template <bool MERGED>
__device__ __forceinline__ bool deposit_key_x(const RoundParams& P, uint32_t v, unsigned long long key, uint32_t cur) {
  if constexpr (!MERGED) return deposit_key(P, v, key, cur);
  else {
    if (cur > static_cast<uint32_t>(key >> 32)) return false;
    return atomicMax(P.vkey + v, key) == key;
  }
}
template <bool MERGED>
__device__ __forceinline__ void mark_dead_x(const RoundParams& P, uint32_t v) {
  if constexpr (!MERGED) mark_dead(P, v);
  else {
    P.vkey[v] = ~0ull;
    atomicOr(P.dead + (v >> 5), 1u << (v & 31));
  }
}

// ---------------------------------------------------------------------------------------------
// Round sweep, uniform edge size D (2, 4, 8): one thread per edge, one 64/128-bit pin load per
// edge, software-pipelined over the 32-edge batches of a warp's region.
//
// A batch goes through four stages, one per step, so that every global-memory round trip of
// batch t overlaps the work of its neighbours instead of stalling the warp (the sweep was
// latency-bound with four dependent waits per batch: profiles/ncu_c2_r01_baseline.md):
//   A  (batch t+3)  load the list id and the pins (streaming, evict-first); round 1 also loads
//                   the caller id and the base weight here, because every edge survives
//   B  (batch t+2)  gather the 32-bit filter word vtop[v] of every pin (L2-resident)
//   C1 (batch t+1)  a pin with kTopDead kills the edge (the reference's deactivation phase,
//                   local_max_par.hpp:229-248); survivors are compacted into the next list and
//                   fetch caller id + base weight
//   C2 (batch t)    key of the edge (weight refresh, :126-135), atomicMax at the pins where it can
//                   still raise the maximum (vertex argmax, :137-159), candidate list for the
//                   check kernel.  (Keeping the returning atomics' results in registers for a
//                   later step was measured and dropped: the compiler copies them at once, and the
//                   extra registers cost a CTA per SM.)
// The four batches live in four statically named register sets (the loop is unrolled by four and
// the roles rotate), so no value that is still in flight is ever moved or touched early.
// R1: the kernel launched for round 1 (identity list in and out, no dead vertices yet).
// ---------------------------------------------------------------------------------------------
template <int D>
struct SweepSlot {
  uint32_t e;
  bool live;
  PinVec<D> pv;
  uint32_t cur[D];
  uint32_t oid;  // caller's id of the edge (before id_base)
  double base;
};

template <int D>
struct SweepState {
  uint32_t out_off, cand_off, local_deact;
  uint32_t q_head, q_n;  // deposit queue of the warp (ring of kDepositRing entries)
  bool tie;
};

// Deposit queue (round 1): only a few percent of the pins still raise a vertex maximum, so a batch
// issued its returning atomicMax with one or two active lanes and then waited for it -- half of the
// stall samples of the round-1 sweep (profiles/ncu_c2_r01_final.md).  The (vertex, key) pairs that
// need the atomic are queued per warp in shared memory and issued 32 at a time: one wait per 32
// deposits instead of one per batch and pin.  A deposit may now happen later than its batch; the
// filter words other warps read in the meantime are stale-low, which the pre-filter allows.
constexpr uint32_t kDepositRing = 64;
struct DepositQueue {
  unsigned long long key[kDepositRing];
  uint32_t v[kDepositRing];
};
#ifndef HLM_DEPOSIT_QUEUE
#define HLM_DEPOSIT_QUEUE 1
#endif

template <int D, bool VMAX, bool R1>
struct SweepCtx {
  const RoundParams& P;
  uint32_t r, tag, lane, lt_mask;
  bool in_ident, out_ident, peek, dead_first;
  const uint32_t* __restrict__ in;
  uint32_t* __restrict__ out;
  uint32_t seg_base, cnt;
  DepositQueue* q;
  static constexpr bool kQueue = R1 && HLM_DEPOSIT_QUEUE;

  // issue the first `take` queued deposits, one per lane
  __device__ __forceinline__ void flush(SweepState<D>& st, uint32_t take) const {
    if (lane < take) {
      const uint32_t slot = (st.q_head + lane) & (kDepositRing - 1u);
      const unsigned long long key = q->key[slot];
      const uint32_t v = q->v[slot];
      const unsigned long long old = atomicMax(P.vkey + v, key);
      atomicMax(P.vtop + v, static_cast<uint32_t>(key >> 32));
      st.tie |= (old == key);
    }
    st.q_head += take;
    st.q_n -= take;
    __syncwarp();
  }

  // one pipeline step: stage A on `a`, B on `b`, C1 on `c1`, C2 on `c2`
  __device__ __forceinline__ void step(uint32_t it, SweepSlot<D>& a, SweepSlot<D>& b, SweepSlot<D>& c1,
                                       SweepSlot<D>& c2, SweepState<D>& st) const {
    // ---- stage B: filter words of batch it-1
#pragma unroll
    for (int i = 0; i < D; ++i) b.cur[i] = 0u;
    if (peek && b.live) {
      if (dead_first) {
#pragma unroll
        for (int i = 0; i < D; ++i) b.cur[i] = (is_dead(P, b.pv.v[i]) ? kTopDead : 0u);
      } else {
#pragma unroll
        for (int i = 0; i < D; ++i) b.cur[i] = ld_top(P, b.pv.v[i]);
      }
    }
    // ---- stage A: ids and pins of batch it
    {
      const uint32_t idx = it * 32u + lane;
      a.live = idx < cnt;  // false for the drain steps
      if (a.live) {
        a.e = in_ident ? seg_base + idx : __ldcs(in + seg_base + idx);
        a.pv = load_pins_stream<D>(P.csr.pins, a.e);
        if (R1) {
          a.oid = P.orig ? __ldcs(P.orig + a.e) : a.e;
          a.base = base_of_stream(P, a.e);
        }
      }
    }
    // ---- stage C1: batch it-2
    if (!R1) {
      if (c1.live) {
        bool dead_any = false;
#pragma unroll
        for (int i = 0; i < D; ++i) dead_any |= (c1.cur[i] == kTopDead);
        if (dead_any) {
          c1.live = false;
          ++st.local_deact;
        }
      }
      if (!out_ident) {  // order-preserving warp compaction into the next round's list
        const uint32_t ballot = __ballot_sync(0xffffffffu, c1.live);
        if (c1.live) __stcs(out + seg_base + st.out_off + __popc(ballot & lt_mask), c1.e);
        st.out_off += __popc(ballot);
      }
      if (VMAX && c1.live) {
        c1.oid = P.orig ? __ldg(P.orig + c1.e) : c1.e;
        c1.base = base_of(P, c1.e);
        if (dead_first) {  // only the survivors pay for the (HBM-resident) filter words
#pragma unroll
          for (int i = 0; i < D; ++i) c1.cur[i] = ld_top(P, c1.pv.v[i]);
        }
      }
    }
    // ---- stage C2: batch it-3
    if constexpr (VMAX) {
      bool cand = false;
      unsigned long long key = 0ull;
      uint32_t need = 0u;  // bit i: pin i still needs the atomic (queued form)
      if (c2.live) {
        key = priority_key(P.stream, P.ks, c2.oid + P.id_base, r, c2.base, tag);
        const uint32_t hi = static_cast<uint32_t>(key >> 32);
        bool lost = false;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          if constexpr (kQueue) need |= (c2.cur[i] > hi ? 0u : 1u) << i;
          else st.tie |= deposit_key(P, c2.pv.v[i], key, c2.cur[i]);
          lost |= c2.cur[i] > hi;  // a larger key was already there: cannot win this round
        }
        cand = !lost;
      }
      if constexpr (kQueue) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const bool mine = (need >> i) & 1u;
          const uint32_t nb = __ballot_sync(0xffffffffu, mine);
          if (nb) {
            if (mine) {
              const uint32_t slot = (st.q_head + st.q_n + __popc(nb & lt_mask)) & (kDepositRing - 1u);
              q->key[slot] = key;
              q->v[slot] = c2.pv.v[i];
            }
            st.q_n += __popc(nb);
            __syncwarp();
            if (st.q_n >= 32u) flush(st, 32u);
          }
        }
      }
      // edges that may still win go to the (dense) candidate list of the check kernel
      const uint32_t ballot = __ballot_sync(0xffffffffu, cand);
      if (cand) P.cand_ids[seg_base + st.cand_off + __popc(ballot & lt_mask)] = c2.e;
      st.cand_off += __popc(ballot);
    }
  }
};

template <int D>
struct SweepTuning {  // CTAs per SM = register budget of the four in-flight batches (48 / 80 / 128 registers)
  static constexpr int kMinBlocks = D == 2 ? HLM_SWEEP_MIN_BLOCKS : (D == 4 ? HLM_SWEEP_MIN_BLOCKS_D4 : HLM_SWEEP_MIN_BLOCKS_D8);
};

// STRIDED: regions are dealt out by warp index (warp, warp + grid warps, ...) instead of by ticket -- the
// fused kernel of small instances, where thousands of same-address ticket atomics (one per ns) would cost
// more than the sweep
template <int D, bool VMAX, bool R1, bool STRIDED = false>
__device__ __forceinline__ void sweep_uniform_body(const RoundParams& P, DepositQueue* s_queue) {
  static_assert(!R1 || VMAX, "round 1 without keys has nothing to do");
  Ctrl* c = P.ctrl;
  const uint32_t par = c->parity;
  SweepCtx<D, VMAX, R1> X{P};
  X.q = &s_queue[SweepCtx<D, VMAX, R1>::kQueue ? (threadIdx.x >> 5) : 0];
  X.r = c->round;
  X.tag = round_tag(P.ks, X.r);
  X.lane = threadIdx.x & 31;
  X.lt_mask = (1u << X.lane) - 1u;
  X.in_ident = R1 || X.r <= 2;   // rounds 1 and 2 read the identity list
  X.out_ident = R1 || X.r == 1;  // round 1 keeps every edge: nothing to write
  X.peek = X.r > 1 || P.ks.precheck;
  X.dead_first = !R1 && X.r > 1 && P.dead_first;
  X.in = P.seg_ids[par];
  X.out = P.seg_ids[par ^ 1];
  const uint32_t* __restrict__ in_cnt = P.seg_cnt[par];
  uint32_t* __restrict__ out_cnt = P.seg_cnt[par ^ 1];
  uint32_t local_kept = 0;
  SweepState<D> st;
  st.local_deact = 0;
  st.q_head = st.q_n = 0;
  st.tie = false;

  const uint32_t gran = R1 ? 1u : claim_granularity(P, c->active_prev);
  uint32_t next_claim = grid_warp();
  for (uint32_t seg = 0, seg_end = 0;; ++seg) {
    if (seg == seg_end) {
      if constexpr (STRIDED) {
        seg = next_claim * gran;
        next_claim += gridDim.x * kWarpsPerBlock;
      } else {
        seg = claim_region(&c->ticket_f, X.lane, false) * gran;
      }
      seg_end = seg + gran;
    }
    if (seg >= P.nseg) break;
    X.cnt = region_count(P, X.in_ident, in_cnt, seg);
    X.seg_base = seg * P.seg_cap;
    if (!R1 && X.r == 2 && X.cnt && span_all_dead(P, X.seg_base, X.cnt, X.lane)) {
      if (X.lane == 0) {
        out_cnt[seg] = 0;
        if (VMAX) P.cand_cnt[seg] = 0;
        st.local_deact += X.cnt;
      }
      continue;
    }
    const uint32_t steps = ((X.cnt + 31u) >> 5) + 3u;
    st.out_off = 0;
    st.cand_off = 0;
    SweepSlot<D> s0, s1, s2, s3;
    s0.live = s1.live = s2.live = s3.live = false;
    if (X.cnt) {
      for (uint32_t it = 0; it < steps; it += 4u) {
        X.step(it, s0, s3, s2, s1, st);
        X.step(it + 1u, s1, s0, s3, s2, st);
        X.step(it + 2u, s2, s1, s0, s3, st);
        X.step(it + 3u, s3, s2, s1, s0, st);
      }
    }
    if (X.lane == 0) {
      const uint32_t kept = X.out_ident ? X.cnt : st.out_off;
      out_cnt[seg] = kept;
      if (VMAX) P.cand_cnt[seg] = st.cand_off;
      local_kept += kept;
    }
  }
  if constexpr (SweepCtx<D, VMAX, R1>::kQueue) {
    if (st.q_n) X.flush(st, st.q_n);
  }
  const uint32_t d = warp_sum(st.local_deact);
  if (X.lane == 0) {
    if (d) atomicAdd(P.deact_cnt + (X.r - 1), d);
    if (local_kept) atomicAdd(&c->active_small, local_kept);
  }
  if (st.tie) c->tie_flag = 1u;
}

template <int D, bool VMAX, bool R1>
__global__ void __launch_bounds__(kBlock, SweepTuning<D>::kMinBlocks) k_sweep_uniform(const RoundParams P) {
  __shared__ DepositQueue s_queue[SweepCtx<D, VMAX, R1>::kQueue ? kWarpsPerBlock : 1];
  sweep_uniform_body<D, VMAX, R1>(P, s_queue);
}

// Non-pipelined form of the same sweep: one batch per warp at a time, 32 registers, 64 resident
// warps per SM.  Latency is hidden by occupancy instead of by the per-warp pipeline.
template <int D, bool VMAX, bool STRIDED = false>
__device__ __forceinline__ void sweep_uniform_simple_body(const RoundParams& P) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const bool in_ident = r <= 2;
  const bool out_ident = r == 1;
  const bool peek = r > 1 || P.ks.precheck;
  const bool dead_first = r > 1 && P.dead_first;
  const uint32_t* __restrict__ in = P.seg_ids[par];
  const uint32_t* __restrict__ in_cnt = P.seg_cnt[par];
  uint32_t* __restrict__ out = P.seg_ids[par ^ 1];
  uint32_t* __restrict__ out_cnt = P.seg_cnt[par ^ 1];
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t local_deact = 0, local_kept = 0;
  bool tie = false;
  const uint32_t gran = claim_granularity(P, c->active_prev);
  uint32_t next_claim = grid_warp();
  for (uint32_t seg = 0, seg_end = 0;; ++seg) {
    if (seg == seg_end) {
      if constexpr (STRIDED) {
        seg = next_claim * gran;
        next_claim += gridDim.x * kWarpsPerBlock;
      } else {
        seg = claim_region(&c->ticket_f, lane, false) * gran;
      }
      seg_end = seg + gran;
    }
    if (seg >= P.nseg) break;
    const uint32_t cnt = region_count(P, in_ident, in_cnt, seg);
    const uint32_t seg_base = seg * P.seg_cap;
    uint32_t out_off = 0, cand_off = 0;
    if (r == 2 && cnt && span_all_dead(P, seg_base, cnt, lane)) {
      if (lane == 0) {
        out_cnt[seg] = 0;
        if (VMAX) P.cand_cnt[seg] = 0;
        local_deact += cnt;
      }
      continue;
    }
    for (uint32_t t0 = 0; t0 < cnt; t0 += 32u) {
      const uint32_t idx = t0 + lane;
      bool survive = idx < cnt, cand = false;
      uint32_t e = 0;
      PinVec<D> pv;
      uint32_t cur[D];
#pragma unroll
      for (int i = 0; i < D; ++i) cur[i] = 0u;
      if (survive) {
        e = in_ident ? seg_base + idx : __ldcs(in + seg_base + idx);
        pv = load_pins_stream<D>(P.csr.pins, e);
        if (peek) {
          // first pin first (coalesced: the edges are sorted by it); about half of the edges that
          // die are already decided here and never issue the random gathers of their other pins
          bool dead_any = false;
          if (dead_first) {
#pragma unroll
            for (int i = 0; i < D; ++i) dead_any |= is_dead(P, pv.v[i]);
            if (VMAX && !dead_any) {
#pragma unroll
              for (int i = 0; i < D; ++i) cur[i] = ld_top(P, pv.v[i]);
            }
          } else {
            cur[0] = ld_top(P, pv.v[0]);
            dead_any = cur[0] == kTopDead;
            if (!dead_any) {
#pragma unroll
              for (int i = 1; i < D; ++i) cur[i] = ld_top(P, pv.v[i]);
#pragma unroll
              for (int i = 1; i < D; ++i) dead_any |= (cur[i] == kTopDead);
            }
          }
          if (dead_any) {
            survive = false;
            ++local_deact;
          }
        }
      }
      if constexpr (VMAX) {
        if (survive) {
          const unsigned long long key = priority_key(P.stream, P.ks, edge_gid(P, e), r, base_of(P, e), tag);
          const uint32_t hi = static_cast<uint32_t>(key >> 32);
          bool lost = false;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            tie |= deposit_key(P, pv.v[i], key, cur[i]);
            lost |= cur[i] > hi;
          }
          cand = !lost;
        }
      }
      if (!out_ident) {
        const uint32_t ballot = __ballot_sync(0xffffffffu, survive);
        if (survive) __stcs(out + seg_base + out_off + __popc(ballot & lt_mask), e);
        out_off += __popc(ballot);
      }
      if constexpr (VMAX) {
        const uint32_t ballot = __ballot_sync(0xffffffffu, cand);
        if (cand) P.cand_ids[seg_base + cand_off + __popc(ballot & lt_mask)] = e;
        cand_off += __popc(ballot);
      }
    }
    if (lane == 0) {
      const uint32_t kept = out_ident ? cnt : out_off;
      out_cnt[seg] = kept;
      if (VMAX) P.cand_cnt[seg] = cand_off;
      local_kept += kept;
    }
  }
  const uint32_t d = warp_sum(local_deact);
  if (lane == 0) {
    if (d) atomicAdd(P.deact_cnt + (r - 1), d);
    if (local_kept) atomicAdd(&c->active_small, local_kept);
  }
  if (tie) c->tie_flag = 1u;
}

// The sweep of the fused small-instance kernel: the same decisions as the plain sweep, ITEMS batches of a
// region per step with the loads of all of them issued together.  A small instance is latency-bound -- the
// resident warps each walk a few batches one dependent L2 round trip after the other (config 1: 6.6 batches
// per warp, ~5 trips each) -- so the trips of ITEMS batches overlap.  Regions by warp index (no tickets);
// deactivation always on the dead bitmap (identical to the kTopDead test: mark_dead sets both).
template <int D, int ITEMS, bool MERGED>
__device__ __forceinline__ void sweep_uniform_ilp_body(const RoundParams& P) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const bool in_ident = r <= 2;
  const bool out_ident = r == 1;
  const bool peek = r > 1 || P.ks.precheck;
  const uint32_t* in = P.seg_ids[par];
  const uint32_t* in_cnt = P.seg_cnt[par];
  uint32_t* out = P.seg_ids[par ^ 1];
  uint32_t* out_cnt = P.seg_cnt[par ^ 1];
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t local_deact = 0, local_kept = 0;
  bool tie = false;
  const uint32_t gran = claim_granularity(P, c->active_prev);
  const uint32_t stride = gridDim.x * kWarpsPerBlock * gran;
  for (uint32_t first = grid_warp() * gran; first < P.nseg; first += stride) {
    const uint32_t last = min(P.nseg, first + gran);
    for (uint32_t seg = first; seg < last; ++seg) {
      const uint32_t cnt = region_count(P, in_ident, in_cnt, seg);
      const uint32_t seg_base = seg * P.seg_cap;
      uint32_t out_off = 0, cand_off = 0;
      if (r == 2 && cnt && span_all_dead(P, seg_base, cnt, lane)) {
        if (lane == 0) {
          out_cnt[seg] = 0;
          P.cand_cnt[seg] = 0;
          local_deact += cnt;
        }
        continue;
      }
      for (uint32_t t0 = 0; t0 < cnt; t0 += 32u * ITEMS) {
        uint32_t e[ITEMS];
        bool live[ITEMS], cand[ITEMS];
        PinVec<D> pv[ITEMS];
        uint32_t cur[ITEMS][D];
        unsigned long long key[ITEMS];
        // every load below is unconditional (lanes past the end read the region's first edge): no branch
        // separates the loads of the ITEMS batches
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t idx = t0 + k * 32u + lane;
          live[k] = idx < cnt;
          const uint32_t pos = seg_base + (live[k] ? idx : 0u);
          e[k] = in_ident ? pos : __ldcs(in + pos);
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) pv[k] = load_pins_stream<D>(P.csr.pins, e[k]);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
#pragma unroll
          for (int i = 0; i < D; ++i) cur[k][i] = 0u;
        if (peek) {
          bool dead_any[ITEMS];
#pragma unroll
          for (int k = 0; k < ITEMS; ++k) {
            dead_any[k] = false;
#pragma unroll
            for (int i = 0; i < D; ++i) dead_any[k] |= is_dead(P, pv[k].v[i]);
          }
#pragma unroll
          for (int k = 0; k < ITEMS; ++k)
            if (live[k] && dead_any[k]) {
              live[k] = false;
              ++local_deact;
            }
#pragma unroll
          for (int k = 0; k < ITEMS; ++k)
            if (live[k]) {
#pragma unroll
              for (int i = 0; i < D; ++i) cur[k][i] = ld_top_x<MERGED>(P, pv[k].v[i]);
            }
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          key[k] = 0ull;
          if (live[k]) key[k] = priority_key(P.stream, P.ks, edge_gid(P, e[k]), r, base_of(P, e[k]), tag);
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          cand[k] = false;
          if (live[k]) {
            const uint32_t hi = static_cast<uint32_t>(key[k] >> 32);
            bool lost = false;
#pragma unroll
            for (int i = 0; i < D; ++i) {
              tie |= deposit_key_x<MERGED>(P, pv[k].v[i], key[k], cur[k][i]);
              lost |= cur[k][i] > hi;
            }
            cand[k] = !lost;
          }
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {  // batches in list order
          if (!out_ident) {
            const uint32_t ballot = __ballot_sync(0xffffffffu, live[k]);
            if (live[k]) __stcs(out + seg_base + out_off + __popc(ballot & lt_mask), e[k]);
            out_off += __popc(ballot);
          }
          const uint32_t ballot = __ballot_sync(0xffffffffu, cand[k]);
          if (cand[k]) P.cand_ids[seg_base + cand_off + __popc(ballot & lt_mask)] = e[k];
          cand_off += __popc(ballot);
        }
      }
      if (lane == 0) {
        const uint32_t kept = out_ident ? cnt : out_off;
        out_cnt[seg] = kept;
        P.cand_cnt[seg] = cand_off;
        local_kept += kept;
      }
    }
  }
  const uint32_t d = warp_sum(local_deact);
  if (lane == 0) {
    if (d) atomicAdd(P.deact_cnt + (r - 1), d);
    if (local_kept) atomicAdd(&c->active_small, local_kept);
  }
  if (tie) c->tie_flag = 1u;
}

template <int D, bool VMAX>
__global__ void __launch_bounds__(kBlock, HLM_SIMPLE_MIN_BLOCKS) k_sweep_uniform_simple(const RoundParams P) {
  sweep_uniform_simple_body<D, VMAX>(P);
}

// The same sweep with the survivors processed densely: three quarters of the edges a later round
// sweeps die, so the key / filter-word / atomic part of a batch ran with a quarter of its lanes.
// Survivors are queued per warp in shared memory (id + pins) and that part runs once 32 are
// waiting (and at the end of a region, because the candidate list is per region): the
// instructions of the survivor path are issued once per 32 survivors instead of once per batch
// (config 2: round 2 1.69 -> 1.58 ms, round 3 0.80 -> 0.75 ms).
template <int D>
__global__ void __launch_bounds__(kBlock, HLM_SIMPLE_MIN_BLOCKS) k_sweep_uniform_dense(const RoundParams P) {
  __shared__ uint32_t q_e[kWarpsPerBlock][64];
  __shared__ uint32_t q_v[kWarpsPerBlock][D][64];
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const bool in_ident = r <= 2;
  const bool out_ident = r == 1;
  const bool peek = r > 1 || P.ks.precheck;
  const bool dead_first = r > 1 && P.dead_first;
  const uint32_t* __restrict__ in = P.seg_ids[par];
  const uint32_t* __restrict__ in_cnt = P.seg_cnt[par];
  uint32_t* __restrict__ out = P.seg_ids[par ^ 1];
  uint32_t* __restrict__ out_cnt = P.seg_cnt[par ^ 1];
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t local_deact = 0, local_kept = 0;
  bool tie = false;
  const uint32_t gran = claim_granularity(P, c->active_prev);
  for (uint32_t seg = 0, seg_end = 0;; ++seg) {
    if (seg == seg_end) {
      seg = claim_region(&c->ticket_f, lane, false) * gran;
      seg_end = seg + gran;
    }
    if (seg >= P.nseg) break;
    const uint32_t cnt = region_count(P, in_ident, in_cnt, seg);
    const uint32_t seg_base = seg * P.seg_cap;
    uint32_t out_off = 0, cand_off = 0, qn = 0;
    if (r == 2 && cnt && span_all_dead(P, seg_base, cnt, lane)) {
      if (lane == 0) {
        out_cnt[seg] = 0;
        P.cand_cnt[seg] = 0;
        local_deact += cnt;
      }
      continue;
    }
    // key + vertex-max + candidate decision for the first `take` queued survivors
    auto drain = [&](uint32_t take) {
      bool cand = false;
      uint32_t e = 0;
      if (lane < take) {
        e = q_e[wib][lane];
        uint32_t v[D], cur[D];
#pragma unroll
        for (int i = 0; i < D; ++i) v[i] = q_v[wib][i][lane];
#pragma unroll
        for (int i = 0; i < D; ++i) cur[i] = peek ? ld_top(P, v[i]) : 0u;
        const unsigned long long key = priority_key(P.stream, P.ks, edge_gid(P, e), r, base_of(P, e), tag);
        const uint32_t hi = static_cast<uint32_t>(key >> 32);
        bool lost = false;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          tie |= deposit_key(P, v[i], key, cur[i]);
          lost |= cur[i] > hi;
        }
        cand = !lost;
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, cand);
      if (cand) P.cand_ids[seg_base + cand_off + __popc(ballot & lt_mask)] = e;
      cand_off += __popc(ballot);
      __syncwarp();
      // move what is left (fewer than 32 entries) to the front of the queue
      if (take == 32u && lane + 32u < qn) {
        q_e[wib][lane] = q_e[wib][lane + 32u];
#pragma unroll
        for (int i = 0; i < D; ++i) q_v[wib][i][lane] = q_v[wib][i][lane + 32u];
      }
      qn -= take;
      __syncwarp();
    };
    for (uint32_t t0 = 0; t0 < cnt; t0 += 32u) {
      const uint32_t idx = t0 + lane;
      bool survive = idx < cnt;
      uint32_t e = 0;
      PinVec<D> pv;
      if (survive) {
        e = in_ident ? seg_base + idx : __ldcs(in + seg_base + idx);
        pv = load_pins_stream<D>(P.csr.pins, e);
        if (r > 1) {
          bool dead_any = false;
          if (dead_first) {
#pragma unroll
            for (int i = 0; i < D; ++i) dead_any |= is_dead(P, pv.v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < D; ++i) dead_any |= (ld_top(P, pv.v[i]) == kTopDead);
          }
          if (dead_any) {
            survive = false;
            ++local_deact;
          }
        }
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, survive);
      const uint32_t rank = __popc(ballot & lt_mask);
      if (survive) {
        if (!out_ident) __stcs(out + seg_base + out_off + rank, e);
        q_e[wib][qn + rank] = e;
#pragma unroll
        for (int i = 0; i < D; ++i) q_v[wib][i][qn + rank] = pv.v[i];
      }
      out_off += __popc(ballot);
      qn += __popc(ballot);
      __syncwarp();
      if (qn >= 32u) drain(32u);
    }
    if (qn) drain(qn);
    if (lane == 0) {
      const uint32_t kept = out_ident ? cnt : out_off;
      out_cnt[seg] = kept;
      P.cand_cnt[seg] = cand_off;
      local_kept += kept;
    }
  }
  const uint32_t d = warp_sum(local_deact);
  if (lane == 0) {
    if (d) atomicAdd(P.deact_cnt + (r - 1), d);
    if (local_kept) atomicAdd(&c->active_small, local_kept);
  }
  if (tie) c->tie_flag = 1u;
}

// ---------------------------------------------------------------------------------------------
// Round sweep, runtime edge sizes (<= kLargeEdge pins per edge): one thread per short edge, the
// whole warp for a medium one.
// ---------------------------------------------------------------------------------------------
template <bool VMAX, bool STRIDED = false, bool MERGED = false>
__device__ __forceinline__ void filter_vmax_small_body(const RoundParams& P) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const bool in_ident = r <= 2;   // rounds 1 and 2 read the identity list
  const bool out_ident = r == 1;  // round 1 keeps every edge: nothing to write
  const uint32_t* __restrict__ in = P.seg_ids[par];
  const uint32_t* __restrict__ in_cnt = P.seg_cnt[par];
  uint32_t* __restrict__ out = P.seg_ids[par ^ 1];
  uint32_t* __restrict__ out_cnt = P.seg_cnt[par ^ 1];
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t local_deact = 0, local_kept = 0;
  unsigned long long local_pins = 0;  // pins of the edges this thread keeps (WorkCounters of work_optimal)
  bool tie = false;
  const bool dead_first = r > 1 && P.dead_first;

  const uint32_t gran = claim_granularity(P, c->active_prev);
  uint32_t next_claim = grid_warp();
  for (uint32_t seg = 0, seg_end = 0;; ++seg) {
    if (seg == seg_end) {
      if constexpr (STRIDED) {
        seg = next_claim * gran;
        next_claim += gridDim.x * kWarpsPerBlock;
      } else {
        seg = claim_region(&c->ticket_f, lane, false) * gran;
      }
      seg_end = seg + gran;
    }
    if (seg >= P.nseg) break;
    const uint32_t cnt = region_count(P, in_ident, in_cnt, seg);
    const uint32_t seg_base = seg * P.seg_cap;
    uint32_t out_off = 0, cand_off = 0;
    for (uint32_t t0 = 0; t0 < cnt; t0 += 32u) {
      const uint32_t idx = t0 + lane;
      bool survive = idx < cnt, cand = false;
      uint32_t e = 0;
      if (survive) e = in_ident ? seg_base + idx : __ldcg(in + seg_base + idx);
      bool is_long = false;
      uint64_t long_b = 0;
      uint32_t long_s = 0;
      uint32_t my_size = 0;
      if (survive) {
        uint64_t b;
        uint32_t s;
        P.csr.range(e, b, s);
        my_size = s;
        if (P.has_large && s > kLargeEdge) {
          survive = false;  // class-1 edge seen through the identity list
        } else {
          const uint32_t* __restrict__ pp = P.csr.pins + b;
          const bool peek = r > 1 || P.ks.precheck;
          if (s <= 8) {
            // short edge: every pin and its filter word in flight at once, one gather per pin
            uint32_t v[8], cur[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = static_cast<uint32_t>(i) < s ? __ldg(pp + i) : 0u;
            bool dead_any = false;
            if (dead_first) {
#pragma unroll
              for (int i = 0; i < 8; ++i) dead_any |= (static_cast<uint32_t>(i) < s && is_dead(P, v[i]));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
              cur[i] = (peek && !dead_any && static_cast<uint32_t>(i) < s) ? ld_top_x<MERGED>(P, v[i]) : 0u;
#pragma unroll
            for (int i = 0; i < 8; ++i) dead_any |= (static_cast<uint32_t>(i) < s && cur[i] == kTopDead);
            if (dead_any) {
              survive = false;
              ++local_deact;
            } else if constexpr (VMAX) {
              const unsigned long long key =
                  priority_key(P.stream, P.ks, edge_gid(P, e), r, base_of(P, e), tag);
              const uint32_t hi = static_cast<uint32_t>(key >> 32);
              bool lost = false;
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (static_cast<uint32_t>(i) < s) {
                  tie |= deposit_key_x<MERGED>(P, v[i], key, cur[i]);
                  lost |= cur[i] > hi;
                }
              cand = !lost;
            }
          } else {
            is_long = true;  // 9..32 pins: handled below by the whole warp, one pin per lane
            long_b = b;
            long_s = s;
          }
        }
      }
      // medium edges, one at a time, cooperatively: the 32 lanes take one pin each, so an edge
      // costs one gather round trip instead of one per pin
      uint32_t long_mask = __ballot_sync(0xffffffffu, is_long);
      while (long_mask) {
        const int src = __ffs(long_mask) - 1;
        long_mask &= long_mask - 1;
        const uint64_t eb = __shfl_sync(0xffffffffu, long_b, src);
        const uint32_t es = __shfl_sync(0xffffffffu, long_s, src);
        const uint32_t ee = __shfl_sync(0xffffffffu, e, src);
        const bool mine = lane < es;
        const uint32_t v = mine ? __ldg(P.csr.pins + eb + lane) : 0u;
        const bool peek = r > 1 || P.ks.precheck;
        bool dead_any = dead_first && __any_sync(0xffffffffu, mine && is_dead(P, v));
        const uint32_t cur = (mine && peek && !dead_any) ? ld_top_x<MERGED>(P, v) : 0u;
        dead_any = dead_any || __any_sync(0xffffffffu, mine && cur == kTopDead);
        bool lost = false;
        if (!dead_any) {
          if constexpr (VMAX) {
            const unsigned long long key = priority_key(P.stream, P.ks, edge_gid(P, ee), r, base_of(P, ee), tag);
            if (mine) tie |= deposit_key_x<MERGED>(P, v, key, cur);
            lost = __any_sync(0xffffffffu, mine && cur > static_cast<uint32_t>(key >> 32));
          }
        }
        if (static_cast<int>(lane) == src) {
          if (dead_any) {
            survive = false;
            ++local_deact;
          } else if (VMAX) {
            cand = !lost;
          }
        }
      }
      if (survive) local_pins += my_size;
      {
        // order-preserving warp compaction (round 1 keeps the identity list and only counts: the
        // large edges seen through it belong to class 1 and must not be counted here)
        const uint32_t ballot = __ballot_sync(0xffffffffu, survive);
        if (survive && !out_ident) out[seg_base + out_off + __popc(ballot & lt_mask)] = e;
        out_off += __popc(ballot);
      }
      if constexpr (VMAX) {
        // edges that may still win go to the (dense) candidate list of the check kernel
        const uint32_t ballot = __ballot_sync(0xffffffffu, cand);
        if (cand) P.cand_ids[seg_base + cand_off + __popc(ballot & lt_mask)] = e;
        cand_off += __popc(ballot);
      }
    }
    if (lane == 0) {
      out_cnt[seg] = out_ident ? cnt : out_off;  // list length (round 2 reads the identity list anyway)
      if (VMAX) P.cand_cnt[seg] = cand_off;
      local_kept += out_off;
    }
  }
  const uint32_t d = warp_sum(local_deact);
  for (int o = 16; o > 0; o >>= 1) local_pins += __shfl_xor_sync(0xffffffffu, local_pins, o);
  if (lane == 0) {
    if (d) atomicAdd(P.deact_cnt + (r - 1), d);
    if (local_kept) atomicAdd(&c->active_small, local_kept);
    if (local_pins) atomicAdd(&c->pins_round, local_pins);
  }
  if (tie) c->tie_flag = 1u;
}

// Check + commit over the candidate lists (local_max_par.hpp:202-224): a candidate is matched iff
// its key is the maximum at every pin; matched edges record their round and kill their pins.
// A warp claims P.check_claim (<= kCoarseClaim) regions and walks the concatenation of their (short)
// candidate lists, kCheckItems candidates per lane and step, so that several independent chains
// list id -> pins -> filter word are in flight per thread.
constexpr int kCheckItems = 4;

template <int D, bool STRIDED = false, bool MERGED = false>
__device__ __forceinline__ void check_commit_small_body(const RoundParams& P) {
  constexpr int ITEMS = D > 0 ? kCheckItems : 1;
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  if (c->tie_flag || r > c->max_rounds) return;
  const uint32_t* __restrict__ list = P.cand_ids;
  const uint32_t* __restrict__ list_cnt = P.cand_cnt;
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  uint32_t local_matched = 0, local_mpins = 0;

  // The regions of one claim are spread over the whole id space (ticket, ticket + stride, ...): on a
  // sorted, degree-renumbered instance the candidate density grows steadily along the id space (hub
  // regions hold almost none), and consecutive regions per claim left the last claims with all the work.
  const uint32_t stride = (P.nseg + P.check_claim - 1u) / P.check_claim;
  for (uint32_t ticket = grid_warp();;
       ticket = STRIDED ? ticket + gridDim.x * kWarpsPerBlock : claim_region(&c->ticket_c, lane, true)) {
    if (ticket >= stride) break;
    // end[j] = candidates in the first j+1 regions of the claim (inclusive prefix), the same in every lane
    uint32_t mine = (lane < P.check_claim && ticket + lane * stride < P.nseg) ? __ldcg(list_cnt + ticket + lane * stride) : 0u;
#pragma unroll
    for (int o = 1; o < static_cast<int>(kCoarseClaim); o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, mine, o);
      if (lane >= static_cast<uint32_t>(o)) mine += t;
    }
    uint32_t end[kCoarseClaim];
#pragma unroll
    for (int j = 0; j < static_cast<int>(kCoarseClaim); ++j) end[j] = __shfl_sync(0xffffffffu, mine, j);
    const uint32_t total = end[kCoarseClaim - 1];
    for (uint32_t t0 = 0; t0 < total; t0 += 32u * ITEMS) {
      uint32_t e[ITEMS];
      bool valid[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const uint32_t idx = t0 + k * 32u + lane;
        valid[k] = idx < total;
        uint32_t j = 0, begin = 0;
#pragma unroll
        for (int q = 0; q + 1 < static_cast<int>(kCoarseClaim); ++q)
          if (idx >= end[q]) {
            j = q + 1;
            begin = end[q];
          }
        e[k] = valid[k] ? __ldcg(list + static_cast<size_t>(ticket + j * stride) * P.seg_cap + (idx - begin)) : 0u;
      }
      if constexpr (D > 0) {
        PinVec<D> pv[ITEMS];
        uint32_t top0[ITEMS];
        unsigned long long key[ITEMS];
        bool win[ITEMS];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          if (valid[k]) pv[k] = load_pins<D>(P.csr.pins, e[k]);
        // 32-bit filter word of the first pin first: most candidates lose right here, and with
        // the edges sorted by first pin this load is nearly coalesced
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          if (valid[k]) top0[k] = MERGED ? __ldcg(top_half(P, pv[k].v[0])) : __ldcg(P.vtop + pv[k].v[0]);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          win[k] = false;
          if (valid[k]) {
            key[k] = priority_key(P.stream, P.ks, edge_gid(P, e[k]), r, base_of(P, e[k]), tag);
            win[k] = top0[k] == static_cast<uint32_t>(key[k] >> 32);
          }
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          if (win[k]) {
            uint32_t rest[D];
#pragma unroll
            for (int i = 1; i < D; ++i) rest[i] = MERGED ? __ldcg(top_half(P, pv[k].v[i])) : __ldcg(P.vtop + pv[k].v[i]);
#pragma unroll
            for (int i = 1; i < D; ++i) win[k] &= (rest[i] == static_cast<uint32_t>(key[k] >> 32));
          }
        // the few survivors of the 32-bit filter are confirmed against the full keys
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          if (win[k]) {
            unsigned long long full[D];
#pragma unroll
            for (int i = 0; i < D; ++i) full[i] = __ldcg(P.vkey + pv[k].v[i]);
#pragma unroll
            for (int i = 0; i < D; ++i) win[k] &= (full[i] == key[k]);
            if (win[k]) {
              mark_matched(P, e[k], r);
#pragma unroll
              for (int i = 0; i < D; ++i) mark_dead_x<MERGED>(P, pv[k].v[i]);
              ++local_matched;
            }
          }
      } else {
        if (valid[0]) {
          uint64_t b;
          uint32_t s;
          P.csr.range(e[0], b, s);
          if (!(P.has_large && s > kLargeEdge)) {
            const uint32_t* __restrict__ pp = P.csr.pins + b;
            const unsigned long long key =
                priority_key(P.stream, P.ks, edge_gid(P, e[0]), r, base_of(P, e[0]), tag);
            bool w = true;
            for (uint32_t i = 0; i < s && w; ++i)
              w = MERGED ? __ldcg(P.vkey + __ldg(pp + i)) == key : key_wins_at(P, __ldg(pp + i), key);
            if (w) {
              mark_matched(P, e[0], r);
              for (uint32_t i = 0; i < s; ++i) {
                const uint32_t v = __ldg(pp + i);
                mark_dead_x<MERGED>(P, v);
              }
              ++local_matched;
              local_mpins += s;
            }
          }
        }
      }
    }
  }
  const uint32_t t = warp_sum(local_matched);
  if (lane == 0 && t) atomicAdd(P.matched_cnt + r, t);
  if constexpr (D == 0) {
    const uint32_t mp = warp_sum(local_mpins);  // a warp matches far fewer than 2^32 pins per launch
    if (lane == 0 && mp) atomicAdd(&c->pins_matched, static_cast<unsigned long long>(mp));
  }
}

template <int D>
__global__ void __launch_bounds__(kBlock, 4) k_check_commit_small(const RoundParams P) {
  check_commit_small_body<D>(P);
}

// ---------------------------------------------------------------------------------------------
// Round kernels, class 1: one warp per large edge (ballot / shuffle reductions over its pins).
// ---------------------------------------------------------------------------------------------
// The large edges are few (a few percent at most), so their list is never compacted: a state
// byte per entry says whether the edge is still active and whether it can still win this round
// (an appended list costs one same-address atomic per surviving edge: 2.4 M of them took 7 ms on
// the power-law instance).
enum LargeState : uint8_t { LARGE_DROPPED = 0, LARGE_ACTIVE = 1, LARGE_CANDIDATE = 2 };

template <bool VMAX>
__global__ void __launch_bounds__(kBlock, HLM_MIN_BLOCKS) k_filter_vmax_small(const RoundParams P) {
  filter_vmax_small_body<VMAX>(P);
}
template <bool VMAX, bool MERGED = false>
__device__ __forceinline__ void filter_vmax_large_body(const RoundParams& P) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  uint32_t local_deact = 0, local_alive = 0;
  unsigned long long local_pins = 0;
  bool tie = false;
  // a warp takes 32 consecutive entries: one coalesced load of their state bytes, then the active
  // ones in turn, each with all 32 lanes
  const uint32_t ch = P.large_chunk;  // 1..32 entries per warp and step (fewer when the list is short)
  for (uint32_t chunk = warp; static_cast<uint64_t>(chunk) * ch < P.num_large; chunk += nwarps) {
   const uint32_t my_pos = chunk * ch + lane;
   uint32_t todo = __ballot_sync(0xffffffffu,
                                 lane < ch && my_pos < P.num_large && P.large_state[my_pos] != LARGE_DROPPED);
   while (todo) {
    const uint32_t pos = chunk * ch + (__ffs(todo) - 1u);
    todo &= todo - 1u;
    const uint32_t e = P.large_ids[pos];
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    const uint32_t* __restrict__ pp = P.csr.pins + b;
    unsigned long long key = 0ull;
    if constexpr (VMAX) key = priority_key(P.stream, P.ks, edge_gid(P, e), r, base_of(P, e), tag);
    const uint32_t hi = static_cast<uint32_t>(key >> 32);
    bool dead_any = false, lost = false;
    // pass 1: is a pin dead?  (32 gathers in flight per step; the bitmap when vtop is HBM-resident)
    if (r > 1) {
      const bool use_bits = P.dead_first != 0u;
      for (uint32_t i0 = 0; i0 < s && !dead_any; i0 += 32) {
        const uint32_t i = i0 + lane;
        bool d = false;
        if (i < s) {
          const uint32_t v = __ldg(pp + i);
          d = use_bits ? is_dead(P, v) : (ld_top_x<MERGED>(P, v) == kTopDead);
        }
        dead_any = __any_sync(0xffffffffu, d);
      }
    }
    if (dead_any) {
      if (lane == 0) {
        P.large_state[pos] = LARGE_DROPPED;
        ++local_deact;
      }
      continue;
    }
    if (lane == 0) {
      ++local_alive;
      local_pins += s;
    }
    if constexpr (VMAX) {
      for (uint32_t i = lane; i < s; i += 32) {
        const uint32_t v = __ldg(pp + i);
        const uint32_t cur = MERGED ? __ldcg(top_half(P, v)) : __ldcg(P.vtop + v);
        tie |= deposit_key_x<MERGED>(P, v, key, cur);
        lost |= cur > hi;
      }
      lost = __any_sync(0xffffffffu, lost);
      if (lane == 0) P.large_state[pos] = lost ? LARGE_ACTIVE : LARGE_CANDIDATE;
    }
   }
  }
  if (local_deact) atomicAdd(P.deact_cnt + (r - 1), local_deact);
  if (local_alive) atomicAdd(&c->count1[par ^ 1], local_alive);
  if (local_pins) atomicAdd(&c->pins_round, local_pins);
  if (tie) c->tie_flag = 1u;
}

template <bool VMAX>
__global__ void __launch_bounds__(kBlock) k_filter_vmax_large(const RoundParams P) {
  filter_vmax_large_body<VMAX>(P);
}

template <bool MERGED = false>
__device__ __forceinline__ void check_commit_large_body(const RoundParams& P) {
  const Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  if (c->tie_flag || r > c->max_rounds) return;
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  uint32_t local_matched = 0;
  unsigned long long local_mpins = 0;
  const uint32_t ch = P.large_chunk;
  for (uint32_t chunk = warp; static_cast<uint64_t>(chunk) * ch < P.num_large; chunk += nwarps) {
   const uint32_t my_pos = chunk * ch + lane;
   uint32_t todo = __ballot_sync(0xffffffffu,
                                 lane < ch && my_pos < P.num_large && P.large_state[my_pos] == LARGE_CANDIDATE);
   while (todo) {
    const uint32_t pos = chunk * ch + (__ffs(todo) - 1u);
    todo &= todo - 1u;
    const uint32_t e = P.large_ids[pos];
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    const uint32_t* __restrict__ pp = P.csr.pins + b;
    const unsigned long long key = priority_key(P.stream, P.ks, edge_gid(P, e), r, base_of(P, e), tag);
    bool win = true;
    for (uint32_t i0 = 0; i0 < s; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool ok = i < s ? (MERGED ? __ldcg(P.vkey + __ldg(pp + i)) == key : key_wins_at(P, __ldg(pp + i), key)) : true;
      win = __all_sync(0xffffffffu, ok);
      if (!win) break;  // first losing chunk ends the scan
    }
    if (win) {
      for (uint32_t i = lane; i < s; i += 32) {
        const uint32_t v = __ldg(pp + i);
        mark_dead_x<MERGED>(P, v);
      }
      if (lane == 0) {
        mark_matched(P, e, r);
        ++local_matched;
        local_mpins += s;
      }
    }
   }
  }
  if (local_matched) atomicAdd(P.matched_cnt + r, local_matched);
  if (local_mpins) atomicAdd(&P.ctrl->pins_matched, local_mpins);
}

__global__ void __launch_bounds__(kBlock) k_check_commit_large(const RoundParams P) { check_commit_large_body<>(P); }

// One thread.  Round bookkeeping between check/commit of round r and the filter of round r+1;
// sets the WHILE condition of the enclosing CUDA graph when there is one.
__device__ __forceinline__ uint32_t advance_round(const RoundParams& P, uint32_t active_elsewhere) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round, par = c->parity;
  const uint32_t active = c->active_small + c->count1[par ^ 1];
  uint32_t status = ST_RUNNING;
  c->ticket_f = 0;
  c->ticket_c = 0;
  if (c->tie_flag && r <= c->max_rounds) {  // beyond the cap nothing commits: a tie seen by that sweep is moot
    status = ST_TIE;
  } else if (active == 0 && active_elsewhere == 0) {  // edge shards: other ranks may still be busy
    status = ST_DONE;  // loop condition of run_soft_delete (local_max_par.hpp:117)
    c->rounds_done = r - 1;
  } else if (r > c->max_rounds) {
    status = ST_ROUND_LIMIT;  // local_max_par.hpp:119-124
    c->rounds_done = r - 1;
  } else {
    c->edges_swept += active;
    // uniform instances: kappa_r = d * m_r; ragged ones: counted by the sweeps of this round
    c->pins_swept += P.csr.uniform_d ? static_cast<unsigned long long>(active) * P.csr.uniform_d : c->pins_round;
    c->pins_round = 0;
    c->active_prev = c->active_small;
    c->active_small = 0;
    c->parity = par ^ 1;
    c->count1[par] = 0;
    c->round = r + 1;
    if (r % P.ks.tag_period == 0) status = ST_EPOCH;
  }
  c->status = status;
  return status;
}

__global__ void k_advance(const RoundParams P, cudaGraphConditionalHandle handle, int in_graph,
                          uint32_t active_elsewhere) {
  const uint32_t status = advance_round(P, active_elsewhere);
  if (in_graph) cudaGraphSetConditional(handle, status == ST_RUNNING ? 1u : 0u);
}

// ---------------------------------------------------------------------------------------------
// A whole matching of a small instance in ONE cooperative launch (which instances: fused_rounds_ok,
// hlm_engine.cu).  When the instance sits in L2 a round is a handful of dependent memory round trips,
// and three kernel launches per round (sweep, check, advance: ~85 us per round inside the CUDA graph
// on config 1) plus the per-call memsets, read-backs and assembly kernels cost several times the work
// itself.  Here the resident grid zeroes the per-call state, runs sweep -> grid barrier -> check (the
// CTA that finishes it last advances the round) -> grid barrier, round after round, until the status
// leaves ST_RUNNING (done, round cap; tie, tag wrap: the host handles those exactly as after a graph
// launch and relaunches), then assembles the result into the caller's page-locked arrays.  D = 2, 4, 8:
// uniform sizes; D = 0: any sizes (thread per edge, warp per edge above kLargeEdge pins).  The phases are
// the bodies of the stand-alone kernels, so the results are the same by construction; the lists and
// per-vertex words written in one phase are read in the next after the barrier's fence (the barrier of
// cooperative groups ends with MEMBAR.GPU + CCTL.IVALL in every CTA, so ld.ca lines of the hot windows do
// not survive a phase; the lists use ld.cg).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void grid_zero(void* p, size_t bytes) {  // bytes: a multiple of 4, p 16-byte aligned
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x, nth = static_cast<size_t>(gridDim.x) * blockDim.x;
  uint4* q = static_cast<uint4*>(p);
  const size_t vec = (reinterpret_cast<uintptr_t>(p) & 15u) ? 0 : bytes >> 4;
  for (size_t i = tid; i < vec; i += nth) q[i] = make_uint4(0u, 0u, 0u, 0u);
  uint32_t* t = static_cast<uint32_t*>(p) + (vec << 2);
  const size_t rest = (bytes >> 2) - (vec << 2);
  for (size_t i = tid; i < rest; i += nth) t[i] = 0u;
}

#ifndef HLM_FUSED_ITEMS
#define HLM_FUSED_ITEMS(D) ((D) == 2 ? 4 : ((D) == 4 ? 2 : 1))
#endif
// PIPE: the software-pipelined sweep (four batches in flight per warp, more registers) instead of the plain one
template <int D, bool PIPE>
__global__ void __launch_bounds__(kBlock, PIPE ? (D == 8 ? 2 : 3) : 4) k_rounds_fused(const RoundParams P, const FusedExtra X) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  __shared__ unsigned long long s_sum[kWarpsPerBlock];
#ifdef HLM_FUSED_TRACE
  uint32_t tr_n = 0;
#define FUSED_MARK()                                                                     \
  do {                                                                                   \
    if (X.sum && blockIdx.x == 0 && threadIdx.x == 0 && tr_n < 64u) {                    \
      unsigned long long t;                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                              \
      X.sum->trace[tr_n++] = t;                                                          \
    }                                                                                    \
  } while (0)
#else
#define FUSED_MARK() do {} while (0)
#endif
  constexpr bool MERGED = !PIPE;  // (the pipelined sweep of d = 8 keeps the separate filter array)
  FUSED_MARK();
  if (!X.init && MERGED) {
    // a run continued here (after the host's exact redo of a tied round, a tag wrap, or the vertex-owned
    // rounds of a handed-over run): covered vertices are known by the dead bitmap, which everyone maintains
    for (uint32_t v = blockIdx.x * kBlock + threadIdx.x; v < P.n; v += gridDim.x * kBlock)
      if ((__ldcg(P.dead + (v >> 5)) >> (v & 31u)) & 1u) P.vkey[v] = ~0ull;
    grid.sync();
  }
  if (X.init) {
    grid_zero(P.vkey, static_cast<size_t>(P.n) * 8);
    if (!MERGED) grid_zero(P.vtop, static_cast<size_t>(P.n) * 4);
    grid_zero(P.dead, ((static_cast<size_t>(P.n) + 31) / 32) * 4);
    grid_zero(P.mbits, static_cast<size_t>(X.mbits_words) * 4);
    grid_zero(P.matched_cnt, static_cast<size_t>(X.rounds_cap) * 4);
    grid_zero(P.deact_cnt, static_cast<size_t>(X.rounds_cap) * 4);
    for (uint32_t i = blockIdx.x * kBlock + threadIdx.x; i < P.num_large; i += gridDim.x * kBlock) P.large_state[i] = LARGE_ACTIVE;
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.ctrl = X.c0;
    grid.sync();
    FUSED_MARK();
  }
  uint32_t status;
  for (;;) {
    if constexpr (D == 0) {  // ragged sizes; the (few) edges above kLargeEdge pins by whole warps in the same phase
      filter_vmax_small_body<true, true, MERGED>(P);
      if (P.num_large) filter_vmax_large_body<true, MERGED>(P);
    }
    else if constexpr (PIPE) sweep_uniform_body<D, true, false, true>(P, nullptr);
    else sweep_uniform_ilp_body<D, HLM_FUSED_ITEMS(D), MERGED>(P);
    FUSED_MARK();
    grid.sync();
    FUSED_MARK();
    check_commit_small_body<D, true, MERGED>(P);
    if constexpr (D == 0) {
      if (P.num_large) check_commit_large_body<MERGED>(P);
    }
    FUSED_MARK();
    // the block that finishes the check last does the round bookkeeping: two grid barriers per round
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&P.ctrl->blocks_done, 1u) == gridDim.x - 1u) {
        __threadfence();
        P.ctrl->blocks_done = 0u;
        advance_round(P, 0u);
      }
    }
    grid.sync();
    FUSED_MARK();
    status = *reinterpret_cast<volatile uint32_t*>(&P.ctrl->status);
    if (status != ST_RUNNING) break;
  }
  if (MERGED && (status == ST_TIE || status == ST_EPOCH)) {
    // the host's kernels take the next step: give them the filter array they expect
    for (uint32_t v = blockIdx.x * kBlock + threadIdx.x; v < P.n; v += gridDim.x * kBlock) P.vtop[v] = __ldcg(top_half(P, v));
  }
  if (!X.sum) return;
  const Ctrl* c = P.ctrl;
  const uint32_t rounds = c->rounds_done;
  const bool finished = (status == ST_DONE || status == ST_ROUND_LIMIT) && rounds <= kFusedRounds;
  if (!finished) {  // tie / tag wrap: the host takes over and assembles the result the usual way
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      X.sum->ctrl = *c;
      X.sum->assembled = 0u;
    }
    return;
  }
  // ---- finish_matching (local_max_seq.hpp:74-83): matched ids in ascending order, straight into the
  // caller's page-locked arrays.  Every block owns a contiguous range of bitmap words, every thread a
  // contiguous piece of it: count, prefix over the blocks, write.
  const uint32_t per_block = (X.mbits_words + gridDim.x - 1u) / gridDim.x;
  const uint32_t per_thread = (per_block + kBlock - 1u) / kBlock;
  const uint32_t b1 = min(X.mbits_words, (blockIdx.x + 1u) * per_block);
  const uint32_t w0 = min(b1, blockIdx.x * per_block + threadIdx.x * per_thread);
  const uint32_t w1 = min(b1, w0 + per_thread);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t cnt = 0;
  unsigned long long wsum = 0;
  for (uint32_t w = w0; w < w1; ++w) {
    uint32_t b = __ldcg(P.mbits + w);
    cnt += __popc(b);
    if (X.base_int)
      while (b) {
        const uint32_t bit = __ffs(b) - 1u;
        b &= b - 1u;
        wsum += static_cast<unsigned long long>(__ldg(X.base_int + (w * 32u + bit)));
      }
  }
  uint32_t incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += t;
  }
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if (lane == 31) s_warp[warp] = incl;
  if (lane == 0) s_sum[warp] = wsum;
  __syncthreads();
  uint32_t before_warp = 0, block_total = 0;
#pragma unroll
  for (int w = 0; w < kWarpsPerBlock; ++w) {
    if (w < static_cast<int>(warp)) before_warp += s_warp[w];
    block_total += s_warp[w];
  }
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kWarpsPerBlock; ++w) t += s_sum[w];
    X.block_cnt[blockIdx.x] = block_total;
    X.block_isum[blockIdx.x] = t;
  }
  grid.sync();
  uint32_t mine = 0, every = 0;
  for (uint32_t i = threadIdx.x; i < gridDim.x; i += kBlock) {
    const uint32_t v = __ldcg(X.block_cnt + i);
    every += v;
    if (i < blockIdx.x) mine += v;
  }
  const uint32_t before_block = block_sum(mine, s_warp);
  const uint32_t total = block_sum(every, s_warp);
  const bool fits = total <= X.out_cap;  // (always: out_cap is an upper bound of any matching's size)
  uint32_t o = before_block + before_warp + incl - cnt;
  if (fits) {
    for (uint32_t w = w0; w < w1; ++w) {
      uint32_t b = __ldcg(P.mbits + w);
      while (b) {
        const uint32_t bit = __ffs(b) - 1u;
        b &= b - 1u;
        const uint32_t e = w * 32u + bit;
        X.dev_ids[o] = e + P.id_base;
        if (X.out_round) X.dev_round[o] = __ldcg(P.mround + e);
        ++o;
      }
    }
    // device staging -> the caller's page-locked arrays, 16 bytes per thread and store: scattered 4-byte
    // stores across the bus cost a transaction each (config 1: 0.25 ms for 144 K ids)
    grid.sync();
    const uint32_t tid = blockIdx.x * kBlock + threadIdx.x, nth = gridDim.x * kBlock;
    const uint4* src = reinterpret_cast<const uint4*>(X.dev_ids);
    uint4* dst = reinterpret_cast<uint4*>(X.out_ids);
    for (uint32_t i = tid; i < total / 4u; i += nth) dst[i] = __ldcg(src + i);
    if (tid < (total & 3u)) X.out_ids[(total & ~3u) + tid] = __ldcg(X.dev_ids + (total & ~3u) + tid);  // tail, by entry
    if (X.out_round) {
      src = reinterpret_cast<const uint4*>(X.dev_round);
      dst = reinterpret_cast<uint4*>(X.out_round);
      for (uint32_t i = tid; i < total / 8u; i += nth) dst[i] = __ldcg(src + i);
      if (tid < (total & 7u)) X.out_round[(total & ~7u) + tid] = __ldcg(X.dev_round + (total & ~7u) + tid);
    }
  }
  FUSED_MARK();
  if (blockIdx.x == gridDim.x - 1u) {  // the last block also writes the summary
    unsigned long long t = 0;
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += kBlock) t += __ldcg(X.block_isum + i);
    for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
    __syncthreads();
    if (lane == 0) s_sum[warp] = t;
    __syncthreads();
    for (uint32_t r = threadIdx.x; r <= rounds + 1u && r < kFusedRounds + 2u; r += kBlock) {
      X.sum->matched[r] = __ldcg(P.matched_cnt + r);
      X.sum->dropped[r] = __ldcg(P.deact_cnt + r);
    }
    if (threadIdx.x == 0) {
      unsigned long long all = 0;
      for (int w = 0; w < kWarpsPerBlock; ++w) all += s_sum[w];
      X.sum->ctrl = *c;
      X.sum->total = total;
      X.sum->isum = all;
      X.sum->assembled = fits ? 1u : 0u;
    }
  }
}

// Round tags wrapped: forget every running maximum but keep the dead marks.
__global__ void k_epoch_reset(unsigned long long* vkey, uint32_t* vtop, uint32_t n) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    vkey[v] = 0ull;
    if (vtop[v] != kTopDead) vtop[v] = 0u;
  }
}

// ---------------------------------------------------------------------------------------------
// Exact path: three max levels (weight bits, tie hash, id) -- the reference comparator
// weight_stream.hpp:105-113 verbatim.  One warp per edge, any edge size; host-driven.
// ---------------------------------------------------------------------------------------------
struct ExactParams {
  unsigned long long* va;  // n: max weight bits
  unsigned long long* vb;  // n: max tie hash among weight maxima
  uint32_t* vc;            // n: max (global id + 1) among (weight, hash) maxima
  uint32_t round;
  uint32_t cls;            // 0: segmented lists of buffer `buf`; 1: the large edges (state bytes)
  uint32_t buf;
  uint32_t ident;          // class 0 only: the list is the identity
};

template <int LEVEL>
__global__ void __launch_bounds__(kBlock) k_exact_level(const RoundParams P, const ExactParams X) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = blockIdx.x * static_cast<uint64_t>(kWarpsPerBlock) + (threadIdx.x >> 5);
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarpsPerBlock;
  const uint32_t r = X.round;
  const uint64_t slots = X.cls == 0 ? static_cast<uint64_t>(P.nseg) * P.seg_cap : P.num_large;
  uint32_t local_matched = 0;
  unsigned long long local_mpins = 0;
  for (uint64_t pos = warp; pos < slots; pos += nwarps) {
    uint32_t e;
    if (X.cls == 0) {
      const uint32_t seg = static_cast<uint32_t>(pos / P.seg_cap);
      const uint32_t idx = static_cast<uint32_t>(pos % P.seg_cap);
      if (idx >= region_count(P, X.ident, P.seg_cnt[X.buf], seg)) continue;
      e = X.ident ? static_cast<uint32_t>(pos) : P.seg_ids[X.buf][pos];
    } else {
      if (P.large_state[pos] == LARGE_DROPPED) continue;
      e = P.large_ids[pos];
    }
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    if (X.cls == 0 && P.has_large && s > kLargeEdge) {
      continue;
    }
    const uint32_t* __restrict__ pp = P.csr.pins + b;
    // (A, B, C) ascending = the reference comparator (weight, tie_hash, id); for the greedy variant
    // the static order of greedy_sorted: heavier first, then the LOWER id (local_max_seq.hpp:133-136)
    const unsigned long long A = static_cast<unsigned long long>(__double_as_longlong(
        P.greedy ? base_of(P, e) : edge_weight(P.stream, edge_gid(P, e), r, base_of(P, e))));
    const unsigned long long B = P.greedy ? 0ull : tie_hash(P.stream, edge_gid(P, e), r);
    const uint32_t C = P.greedy ? 0xFFFFFFFFu - edge_gid(P, e) : edge_gid(P, e) + 1u;
    bool win = true;
    for (uint32_t i = lane; i < s; i += 32) {
      const uint32_t v = __ldg(pp + i);
      if (LEVEL == 1) {
        atomicMax(X.va + v, A);
      } else if (LEVEL == 2) {
        if (X.va[v] == A) atomicMax(X.vb + v, B);
      } else if (LEVEL == 3) {
        if (X.va[v] == A && X.vb[v] == B) atomicMax(X.vc + v, C);
      } else {
        win &= (X.va[v] == A && X.vb[v] == B && X.vc[v] == C);
      }
    }
    if (LEVEL == 4) {
      win = __all_sync(0xffffffffu, win);
      if (win) {
        for (uint32_t i = lane; i < s; i += 32) {
          const uint32_t v = __ldg(pp + i);
          mark_dead(P, v);
        }
        if (lane == 0) {
          mark_matched(P, e, r);
          ++local_matched;
          local_mpins += s;
        }
      }
      }
  }
  if (LEVEL == 4 && local_matched) atomicAdd(P.matched_cnt + r, local_matched);
  if (LEVEL == 4 && local_mpins) atomicAdd(&P.ctrl->pins_matched, local_mpins);
}

// ---------------------------------------------------------------------------------------------
// Loader helpers
// ---------------------------------------------------------------------------------------------
struct EdgeStats {
  uint32_t min_size;
  uint32_t max_size;
  uint32_t num_large;
  uint32_t max_pin;        // largest vertex id seen
  uint32_t bad_offsets;    // offsets not monotone / first not 0
  uint32_t pad;
};

__global__ void k_edge_size_stats(const uint64_t* off64, uint32_t m, EdgeStats* st) {
  uint32_t mn = 0xffffffffu, mx = 0, large = 0, bad = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint64_t b = off64[e], en = off64[e + 1];
    if (en < b || en - b > 0xffffffffull) {
      bad = 1;
      continue;
    }
    const uint32_t s = static_cast<uint32_t>(en - b);
    mn = min(mn, s);
    mx = max(mx, s);
    large += s > kLargeEdge;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    large += __shfl_xor_sync(0xffffffffu, large, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->min_size, mn);
    atomicMax(&st->max_size, mx);
    if (large) atomicAdd(&st->num_large, large);
    if (bad) atomicOr(&st->bad_offsets, 1u);
  }
}

__global__ void k_max_pin(const uint32_t* pins, uint64_t kappa, EdgeStats* st) {
  uint32_t mx = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < kappa;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    mx = max(mx, pins[i]);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&st->max_pin, mx);
}

// the statistics k_weight_stats takes from the f64 weights, from the byte codes the host packed
// (integers 0..255, lo = 0): 1/8 of the bytes
__global__ void k_code_stats(const uint8_t* __restrict__ codes, uint32_t m, WeightStats* st) {
  uint32_t mn = 255u, mx = 0u;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint32_t c = codes[e];
    mn = min(mn, c);
    mx = max(mx, c);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->min_bits, static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(mn))));
    atomicMax(&st->max_bits, static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(mx))));
    if (mn == 0u) atomicOr(&st->non_positive, 1u);
  }
}

// edge sizes as shipped by the host-assisted loader (16 bits each) -> the 32-bit input of the offset scan
__global__ void k_widen_sizes(const uint16_t* __restrict__ s16, uint32_t* __restrict__ s32, uint64_t count) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    s32[i] = s16[i];
}

__global__ void k_narrow_offsets(const uint64_t* off64, uint32_t* off32, uint64_t count) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    off32[i] = static_cast<uint32_t>(off64[i]);
}

// first pin of the first edge of every 32-edge batch; the last entry repeats the largest first pin
__global__ void k_batch_first_pins(const uint32_t* pins, uint32_t m, uint32_t d, uint32_t entries, uint32_t* bat_pin0) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < entries; b += gridDim.x * blockDim.x) {
    const uint64_t e = min(static_cast<uint64_t>(b) * 32u, static_cast<uint64_t>(m) - 1);
    bat_pin0[b] = pins[e * d];
  }
}

// loader: integer weights 0..255 in resident order, one byte each (see RoundParams::base8)
__global__ void k_pack_u8(const double* __restrict__ base, uint32_t m, uint8_t* __restrict__ codes) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
    codes[e] = static_cast<uint8_t>(base[e]);
}

// loader: weights the host packed to one byte each (integers 1..255) back to the resident f64 form
__global__ void k_expand_u8(const uint8_t* __restrict__ codes, uint32_t m, double* __restrict__ base) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
    base[e] = static_cast<double>(codes[e]);
}

__global__ void k_collect_large(const EdgeCsr csr, uint32_t m, uint32_t* list, uint32_t* count) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    uint64_t b;
    uint32_t s;
    csr.range(e, b, s);
    if (s > kLargeEdge) list[atomicAdd(count, 1u)] = e;
  }
}


__global__ void k_weight_stats(const double* base, uint32_t m, double lo, WeightStats* st) {
  unsigned long long mn = ~0ull, mx = 0;
  uint32_t nonint = 0, nonpos = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double b = base[e];
    if (!(b > 0.0)) nonpos = 1;
    const double w = __dadd_rn(b, lo);
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(w));
    mn = min(mn, bits);
    mx = max(mx, bits);
    if (!(w < 4294967296.0) || w != floor(w)) nonint = 1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    nonint |= __shfl_xor_sync(0xffffffffu, nonint, o);
    nonpos |= __shfl_xor_sync(0xffffffffu, nonpos, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->min_bits, mn);
    atomicMax(&st->max_bits, mx);
    if (nonint) atomicOr(&st->non_integer, 1u);
    if (nonpos) atomicOr(&st->non_positive, 1u);
  }
}

__global__ void k_eval_stream(const StreamParams s, const uint32_t* edges, const uint32_t* rounds,
                              const double* base, size_t count, double* w_out,
                              unsigned long long* t_out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    w_out[i] = edge_weight(s, edges[i], rounds[i], base ? base[i] : 1.0);
    t_out[i] = tie_hash(s, edges[i], rounds[i]);
  }
}

// ---------------------------------------------------------------------------------------------
// Result assembly (finish_matching, local_max_seq.hpp:74-83): ordered compaction of the matched
// bitmap; ids come out ascending, with the round and (optionally) the base weight of each.
// ---------------------------------------------------------------------------------------------
constexpr int kAsmWords = 8;  // bitmap words per thread
constexpr uint32_t kAsmChunkWords = kBlock * kAsmWords;

__global__ void __launch_bounds__(kBlock) k_assemble_count(const uint32_t* mbits, uint32_t words,
                                                           uint32_t* chunk_cnt) {
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  const uint32_t w0 = blockIdx.x * kAsmChunkWords + threadIdx.x * kAsmWords;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kAsmWords; ++k)
    if (w0 + k < words) c += __popc(mbits[w0 + k]);
  const uint32_t t = block_sum(c, s_warp);
  if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = t;
}

// single block: exclusive scan of `cnt` values in place; total to *total
__global__ void __launch_bounds__(1024) k_scan_small(uint32_t* vals, uint32_t cnt,
                                                     unsigned long long* total) {
  __shared__ unsigned long long s_part[1024];
  const uint32_t per = (cnt + 1023) / 1024;
  const uint32_t b = min(cnt, threadIdx.x * per);
  const uint32_t e = min(cnt, b + per);
  unsigned long long acc = 0;
  for (uint32_t i = b; i < e; ++i) acc += vals[i];
  // inclusive scan of the 1024 partials (Hillis-Steele in shared memory)
  s_part[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned long long t = threadIdx.x >= static_cast<unsigned>(o) ? s_part[threadIdx.x - o] : 0ull;
    __syncthreads();
    s_part[threadIdx.x] += t;
    __syncthreads();
  }
  if (threadIdx.x == 1023) *total = s_part[1023];
  unsigned long long run = s_part[threadIdx.x] - acc;
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t v = vals[i];
    vals[i] = static_cast<uint32_t>(run);
    run += v;
  }
}

__global__ void __launch_bounds__(kBlock) k_assemble_write(const uint32_t* mbits, uint32_t words,
                                                           const uint32_t* chunk_off,
                                                           const uint16_t* mround, const double* base,
                                                           uint32_t id_base, uint32_t* out_ids,
                                                           uint16_t* out_round, double* out_w,
                                                           unsigned long long* int_weight_sum) {
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t w0 = blockIdx.x * kAsmChunkWords + threadIdx.x * kAsmWords;
  uint32_t bits[kAsmWords];
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kAsmWords; ++k) {
    bits[k] = w0 + k < words ? mbits[w0 + k] : 0u;
    c += __popc(bits[k]);
  }
  uint32_t incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t o = chunk_off[blockIdx.x] + incl - c;
  for (uint32_t w = 0; w < warp; ++w) o += s_warp[w];
  unsigned long long wsum = 0;
#pragma unroll
  for (int k = 0; k < kAsmWords; ++k) {
    uint32_t b = bits[k];
    while (b) {
      const uint32_t bit = __ffs(b) - 1;
      b &= b - 1;
      const uint32_t e = (w0 + k) * 32u + bit;
      out_ids[o] = e + id_base;
      if (out_round) out_round[o] = mround[e];
      if (out_w) out_w[o] = base[e];
      if (int_weight_sum) wsum += static_cast<unsigned long long>(base[e]);
      ++o;
    }
  }
  if (int_weight_sum) {
    for (int s = 16; s > 0; s >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, s);
    if (lane == 0 && wsum) atomicAdd(int_weight_sum, wsum);
  }
}

// ---------------------------------------------------------------------------------------------
// verify_matching (exact.hpp:115-140)
// ---------------------------------------------------------------------------------------------
struct VerifyOut {
  uint32_t overlap;      // some vertex covered twice
  uint32_t addable;      // some unmatched edge has no covered pin
  uint32_t out_of_range;
  uint32_t pad;
};

// pass 0: bitmap of the caller's matched ids (a repeated id covers its vertices twice)
__global__ void k_verify_mark(const uint32_t* matched, uint64_t count, uint32_t m, uint32_t id_base,
                              uint32_t* in_matching, VerifyOut* out) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t id = matched[k] - id_base;
    if (matched[k] < id_base || id >= m) {
      out->out_of_range = 1;
      continue;
    }
    const uint32_t bit = 1u << (id & 31);
    if (atomicOr(in_matching + (id >> 5), bit) & bit) out->overlap = 1;
  }
}

// pass 1: matched edges cover their pins; pass 2: every other edge must touch a covered vertex
template <int PASS>
__global__ void k_verify_sweep(const EdgeCsr csr, uint32_t m, const uint32_t* orig, uint32_t* covered,
                               const uint32_t* in_matching, VerifyOut* out) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint32_t id = orig ? orig[e] : e;
    const bool in_m = (in_matching[id >> 5] >> (id & 31)) & 1u;
    if (in_m != (PASS == 1)) continue;
    uint64_t b;
    uint32_t s;
    csr.range(e, b, s);
    if (PASS == 1) {
      for (uint32_t i = 0; i < s; ++i) {
        const uint32_t v = csr.pins[b + i];
        const uint32_t bit = 1u << (v & 31);
        if (atomicOr(covered + (v >> 5), bit) & bit) out->overlap = 1;
      }
    } else {
      bool any = false;
      for (uint32_t i = 0; i < s && !any; ++i) {
        const uint32_t v = csr.pins[b + i];
        any = (covered[v >> 5] >> (v & 31)) & 1u;
      }
      if (!any) out->addable = 1;
    }
  }
}

__global__ void k_gather_weights(const double* base, const uint32_t* ids, uint32_t id_base, uint64_t count,
                                 double* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = base[ids[i] - id_base];
}

}  // namespace hlmb
