// hlm_kernels.cuh -- sm_100a kernels of the local-max matching round (CRCW variant), the exact
// tie path, loader helpers, result assembly and verification.  Included by hlm_engine.cu only.
// Kernel roles and the reference phases they replace: see hlm_types.cuh and DESIGN.md.
#pragma once
#include "hlm_types.cuh"

namespace hlmb {

// ---------------------------------------------------------------------------------------------
// Round kernels, class 0: one thread per edge (size <= kLargeEdge).  D > 0: uniform edge size
// with one 64/128-bit pin load per thread; D == 0: runtime offsets.
// ---------------------------------------------------------------------------------------------
template <int D, bool VMAX>
__global__ void __launch_bounds__(kBlock) k_filter_vmax_small(const RoundParams P) {
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  __shared__ uint32_t s_base;
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const uint32_t cnt = c->count[par][0];
  const bool in_ident = P.ident0 && r <= 2;
  const bool out_ident = P.ident0 && r == 1;
  const uint32_t* __restrict__ in = P.list[0][par];
  uint32_t* __restrict__ out = P.list[0][par ^ 1];
  const uint8_t* __restrict__ mflag = P.mflag[0];
  const uint32_t tag = round_tag(P.ks, r);
  uint32_t local_deact = 0;
  bool tie = false;

  if (out_ident && blockIdx.x == 0 && threadIdx.x == 0) c->count[par ^ 1][0] = cnt;

  const uint32_t tiles = (cnt + kBlock - 1) / kBlock;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t pos = tile * kBlock + threadIdx.x;
    bool survive = false;
    uint32_t e = 0;
    if (pos < cnt) {
      e = in_ident ? pos : in[pos];
      const bool was_matched = r > 1 && mflag[pos];
      if (!was_matched) {
        if constexpr (D > 0) {
          const PinVec<D> pv = load_pins<D>(P.csr.pins, e);
          bool dead_any = false;
          if (r > 1) {
#pragma unroll
            for (int i = 0; i < D; ++i) dead_any |= vertex_dead(P.dead, pv.v[i]);
          }
          if (dead_any) {
            ++local_deact;
          } else {
            survive = true;
            if constexpr (VMAX) {
              const unsigned long long key = priority_key(P.stream, P.ks, e + P.id_base, r, base_of(P, e), tag);
              unsigned long long old[D];
#pragma unroll
              for (int i = 0; i < D; ++i) old[i] = atomicMax(P.vkey + pv.v[i], key);
#pragma unroll
              for (int i = 0; i < D; ++i) tie |= (old[i] == key);
            }
          }
        } else {
          uint64_t b;
          uint32_t s;
          P.csr.range(e, b, s);
          if (!(P.has_large && s > kLargeEdge)) {  // large edges belong to class 1
            const uint32_t* __restrict__ pp = P.csr.pins + b;
            bool dead_any = false;
            if (r > 1)
              for (uint32_t i = 0; i < s; ++i) dead_any |= vertex_dead(P.dead, __ldg(pp + i));
            if (dead_any) {
              ++local_deact;
            } else {
              survive = true;
              if constexpr (VMAX) {
                const unsigned long long key =
                    priority_key(P.stream, P.ks, e + P.id_base, r, base_of(P, e), tag);
                for (uint32_t i = 0; i < s; ++i)
                  tie |= (atomicMax(P.vkey + __ldg(pp + i), key) == key);
              }
            }
          }
        }
      }
    }
    if (!out_ident) {
      uint32_t total;
      const uint32_t rank = block_rank(survive, s_warp, total);
      if (threadIdx.x == 0) s_base = total ? atomicAdd(&c->count[par ^ 1][0], total) : 0u;
      __syncthreads();
      if (survive) out[s_base + rank] = e;
    }
  }
  const uint32_t d = block_sum(local_deact, s_warp);
  if (threadIdx.x == 0 && d) atomicAdd(P.deact_cnt + (r - 1), d);
  if (tie) c->tie_flag = 1u;
}

template <int D>
__global__ void __launch_bounds__(kBlock) k_check_commit_small(const RoundParams P) {
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  const Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  if (c->tie_flag || r > c->max_rounds) return;
  const uint32_t par = c->parity;
  const uint32_t cnt = c->count[par ^ 1][0];
  const bool ident = P.ident0 && r == 1;
  const uint32_t* __restrict__ list = P.list[0][par ^ 1];
  uint8_t* __restrict__ mflag = P.mflag[0];
  const uint32_t tag = round_tag(P.ks, r);
  uint32_t local_matched = 0;

  for (uint32_t pos = blockIdx.x * kBlock + threadIdx.x; pos < cnt; pos += gridDim.x * kBlock) {
    const uint32_t e = ident ? pos : list[pos];
    bool win = true;
    if constexpr (D > 0) {
      const PinVec<D> pv = load_pins<D>(P.csr.pins, e);
      const unsigned long long key = priority_key(P.stream, P.ks, e + P.id_base, r, base_of(P, e), tag);
      unsigned long long top[D];
#pragma unroll
      for (int i = 0; i < D; ++i) top[i] = __ldg(P.vkey + pv.v[i]);
#pragma unroll
      for (int i = 0; i < D; ++i) win &= (top[i] == key);
      if (win) {
        P.mround[e] = static_cast<uint16_t>(r);
#pragma unroll
        for (int i = 0; i < D; ++i) atomicOr(P.dead + (pv.v[i] >> 5), 1u << (pv.v[i] & 31));
      }
    } else {
      uint64_t b;
      uint32_t s;
      P.csr.range(e, b, s);
      if (P.has_large && s > kLargeEdge) {
        win = false;  // not this class's edge (identity list only)
      } else {
        const uint32_t* __restrict__ pp = P.csr.pins + b;
        const unsigned long long key = priority_key(P.stream, P.ks, e + P.id_base, r, base_of(P, e), tag);
        for (uint32_t i = 0; i < s && win; ++i) win = (__ldg(P.vkey + __ldg(pp + i)) == key);
        if (win) {
          P.mround[e] = static_cast<uint16_t>(r);
          for (uint32_t i = 0; i < s; ++i) {
            const uint32_t v = __ldg(pp + i);
            atomicOr(P.dead + (v >> 5), 1u << (v & 31));
          }
        }
      }
    }
    mflag[pos] = win ? 1 : 0;
    local_matched += win ? 1u : 0u;
  }
  const uint32_t t = block_sum(local_matched, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(P.matched_cnt + r, t);
}

// ---------------------------------------------------------------------------------------------
// Round kernels, class 1: one warp per large edge (ballot / shuffle reductions over its pins).
// ---------------------------------------------------------------------------------------------
template <bool VMAX>
__global__ void __launch_bounds__(kBlock) k_filter_vmax_large(const RoundParams P) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  const uint32_t par = c->parity;
  const uint32_t cnt = c->count[par][1];
  const uint32_t* __restrict__ in = P.list[1][par];
  uint32_t* __restrict__ out = P.list[1][par ^ 1];
  const uint8_t* __restrict__ mflag = P.mflag[1];
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  uint32_t local_deact = 0;
  bool tie = false;
  for (uint32_t pos = warp; pos < cnt; pos += nwarps) {
    const uint32_t e = in[pos];
    if (r > 1 && mflag[pos]) continue;
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    const uint32_t* __restrict__ pp = P.csr.pins + b;
    bool dead_any = false;
    if (r > 1)
      for (uint32_t i = lane; i < s; i += 32) dead_any |= vertex_dead(P.dead, __ldg(pp + i));
    dead_any = __any_sync(0xffffffffu, dead_any);
    if (dead_any) {
      local_deact += (lane == 0);
      continue;
    }
    if (lane == 0) out[atomicAdd(&c->count[par ^ 1][1], 1u)] = e;
    if constexpr (VMAX) {
      const unsigned long long key = priority_key(P.stream, P.ks, e + P.id_base, r, base_of(P, e), tag);
      for (uint32_t i = lane; i < s; i += 32) tie |= (atomicMax(P.vkey + __ldg(pp + i), key) == key);
    }
  }
  if (local_deact) atomicAdd(P.deact_cnt + (r - 1), local_deact);
  if (tie) c->tie_flag = 1u;
}

__global__ void __launch_bounds__(kBlock) k_check_commit_large(const RoundParams P) {
  const Ctrl* c = P.ctrl;
  const uint32_t r = c->round;
  if (c->tie_flag || r > c->max_rounds) return;
  const uint32_t par = c->parity;
  const uint32_t cnt = c->count[par ^ 1][1];
  const uint32_t* __restrict__ list = P.list[1][par ^ 1];
  uint8_t* __restrict__ mflag = P.mflag[1];
  const uint32_t tag = round_tag(P.ks, r);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  uint32_t local_matched = 0;
  for (uint32_t pos = warp; pos < cnt; pos += nwarps) {
    const uint32_t e = list[pos];
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    const uint32_t* __restrict__ pp = P.csr.pins + b;
    const unsigned long long key = priority_key(P.stream, P.ks, e + P.id_base, r, base_of(P, e), tag);
    bool win = true;
    for (uint32_t i0 = 0; i0 < s; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool ok = i < s ? (__ldg(P.vkey + __ldg(pp + i)) == key) : true;
      win = __all_sync(0xffffffffu, ok);
      if (!win) break;  // first losing chunk ends the scan
    }
    if (win) {
      for (uint32_t i = lane; i < s; i += 32) {
        const uint32_t v = __ldg(pp + i);
        atomicOr(P.dead + (v >> 5), 1u << (v & 31));
      }
      if (lane == 0) {
        P.mround[e] = static_cast<uint16_t>(r);
        ++local_matched;
      }
    }
    if (lane == 0) mflag[pos] = win ? 1 : 0;
  }
  if (local_matched) atomicAdd(P.matched_cnt + r, local_matched);
}

// One thread.  Round bookkeeping between check/commit of round r and the filter of round r+1;
// sets the WHILE condition of the enclosing CUDA graph when there is one.
__global__ void k_advance(const RoundParams P, cudaGraphConditionalHandle handle, int in_graph) {
  Ctrl* c = P.ctrl;
  const uint32_t r = c->round, par = c->parity;
  const uint32_t active = c->count[par ^ 1][0] + c->count[par ^ 1][1];
  uint32_t status = ST_RUNNING;
  if (c->tie_flag) {
    status = ST_TIE;
  } else if (active == 0) {
    status = ST_DONE;  // loop condition of run_soft_delete (local_max_par.hpp:117)
    c->rounds_done = r - 1;
  } else if (r > c->max_rounds) {
    status = ST_ROUND_LIMIT;  // local_max_par.hpp:119-124
    c->rounds_done = r - 1;
  } else {
    c->edges_swept += active;
    c->parity = par ^ 1;
    c->count[par][0] = 0;
    c->count[par][1] = 0;
    c->round = r + 1;
    if (r % P.ks.tag_period == 0) status = ST_EPOCH;
  }
  c->status = status;
  if (in_graph) cudaGraphSetConditional(handle, status == ST_RUNNING ? 1u : 0u);
}

// ---------------------------------------------------------------------------------------------
// Exact path: three max levels (weight bits, tie hash, id) -- the reference comparator
// weight_stream.hpp:105-113 verbatim.  One warp per edge, any edge size; host-driven.
// ---------------------------------------------------------------------------------------------
struct ExactParams {
  unsigned long long* va;  // n: max weight bits
  unsigned long long* vb;  // n: max tie hash among weight maxima
  uint32_t* vc;            // n: max (id + 1) among (weight, hash) maxima
  const uint32_t* list;    // null: identity
  uint32_t count;
  uint32_t round;
  uint32_t cls;            // 0: skip large edges of an identity list; 1: list of large edges
  uint8_t* mflag;
};

template <int LEVEL>
__global__ void __launch_bounds__(kBlock) k_exact_level(const RoundParams P, const ExactParams X) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  const uint32_t r = X.round;
  uint32_t local_matched = 0;
  for (uint32_t pos = warp; pos < X.count; pos += nwarps) {
    const uint32_t e = X.list ? X.list[pos] : pos;
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    if (X.cls == 0 && P.has_large && s > kLargeEdge) {
      if (LEVEL == 4 && lane == 0) X.mflag[pos] = 0;
      continue;
    }
    const uint32_t* __restrict__ pp = P.csr.pins + b;
    const unsigned long long A =
        static_cast<unsigned long long>(__double_as_longlong(edge_weight(P.stream, e + P.id_base, r, base_of(P, e))));
    const unsigned long long B = tie_hash(P.stream, e + P.id_base, r);
    const uint32_t C = e + P.id_base + 1u;
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
          atomicOr(P.dead + (v >> 5), 1u << (v & 31));
        }
        if (lane == 0) {
          P.mround[e] = static_cast<uint16_t>(r);
          ++local_matched;
        }
      }
      if (lane == 0) X.mflag[pos] = win ? 1 : 0;
    }
  }
  if (LEVEL == 4 && local_matched) atomicAdd(P.matched_cnt + r, local_matched);
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

__global__ void k_narrow_offsets(const uint64_t* off64, uint32_t* off32, uint64_t count) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    off32[i] = static_cast<uint32_t>(off64[i]);
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
// Result assembly (finish_matching, local_max_seq.hpp:74-83): ordered compaction of mround[].
// ---------------------------------------------------------------------------------------------
constexpr int kAsmItems = 16;  // entries per thread
constexpr uint32_t kAsmChunk = kBlock * kAsmItems;

__global__ void __launch_bounds__(kBlock) k_assemble_count(const uint16_t* mround, uint32_t m,
                                                           uint32_t* chunk_cnt) {
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  const uint32_t base = blockIdx.x * kAsmChunk;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kAsmItems; ++k) {
    const uint32_t e = base + k * kBlock + threadIdx.x;
    if (e < m) c += mround[e] != 0;
  }
  const uint32_t t = block_sum(c, s_warp);
  if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = t;
}

// single block: exclusive scan of `cnt` values in place; total to *total
__global__ void __launch_bounds__(1024) k_scan_small(uint32_t* vals, uint32_t cnt,
                                                     unsigned long long* total) {
  __shared__ unsigned long long s_part[1024];
  const uint32_t per = (cnt + 1023) / 1024;
  const uint32_t b = threadIdx.x * per;
  const uint32_t e = min(cnt, b + per);
  unsigned long long acc = 0;
  for (uint32_t i = b; i < e; ++i) acc += vals[i];
  s_part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int i = 0; i < 1024; ++i) {
      const unsigned long long v = s_part[i];
      s_part[i] = run;
      run += v;
    }
    *total = run;
  }
  __syncthreads();
  unsigned long long run = s_part[threadIdx.x];
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t v = vals[i];
    vals[i] = static_cast<uint32_t>(run);
    run += v;
  }
}

__global__ void __launch_bounds__(kBlock) k_assemble_write(const uint16_t* mround, uint32_t m,
                                                           const uint32_t* chunk_off,
                                                           const double* base, uint32_t id_base,
                                                           uint32_t* out_ids,
                                                           uint16_t* out_round, double* out_w) {
  __shared__ uint32_t s_warp[kWarpsPerBlock];
  const uint32_t base_e = blockIdx.x * kAsmChunk;
  uint32_t running = chunk_off[blockIdx.x];
  // entries are visited in id order: item k covers a contiguous run of kBlock ids
  for (int k = 0; k < kAsmItems; ++k) {
    const uint32_t e = base_e + k * kBlock + threadIdx.x;
    const uint16_t r = e < m ? mround[e] : 0;
    uint32_t total;
    const uint32_t rank = block_rank(r != 0, s_warp, total);
    if (r != 0) {
      const uint32_t o = running + rank;
      out_ids[o] = e + id_base;
      if (out_round) out_round[o] = r;
      if (out_w) out_w[o] = base[e];
    }
    running += total;
    __syncthreads();
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

__global__ void k_verify_cover(const EdgeCsr csr, uint32_t m, const uint32_t* matched, uint64_t count,
                               uint32_t* covered, uint32_t* in_matching, VerifyOut* out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = blockIdx.x * static_cast<uint64_t>(kWarpsPerBlock) + (threadIdx.x >> 5);
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarpsPerBlock;
  for (uint64_t k = warp; k < count; k += nwarps) {
    const uint32_t e = matched[k];
    if (e >= m) {
      if (lane == 0) out->out_of_range = 1;
      continue;
    }
    if (lane == 0) atomicOr(in_matching + (e >> 5), 1u << (e & 31));
    uint64_t b;
    uint32_t s;
    csr.range(e, b, s);
    for (uint32_t i = lane; i < s; i += 32) {
      const uint32_t v = csr.pins[b + i];
      const uint32_t bit = 1u << (v & 31);
      if (atomicOr(covered + (v >> 5), bit) & bit) out->overlap = 1;
    }
  }
}

__global__ void k_verify_maximal(const EdgeCsr csr, uint32_t m, const uint32_t* covered,
                                 const uint32_t* in_matching, VerifyOut* out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  // 32 edges per warp iteration; lanes walk their own edge (sizes are small on average)
  for (uint32_t e0 = warp * 32; e0 < m; e0 += nwarps * 32) {
    const uint32_t e = e0 + lane;
    if (e >= m) continue;
    if ((in_matching[e >> 5] >> (e & 31)) & 1u) continue;
    uint64_t b;
    uint32_t s;
    csr.range(e, b, s);
    bool any = false;
    for (uint32_t i = 0; i < s && !any; ++i) {
      const uint32_t v = csr.pins[b + i];
      any = (covered[v >> 5] >> (v & 31)) & 1u;
    }
    if (!any) out->addable = 1;
  }
}

__global__ void k_gather_weights(const double* base, const uint32_t* ids, uint64_t count, double* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = base[ids[i]];
}

}  // namespace hlmb
