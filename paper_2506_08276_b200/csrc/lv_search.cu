// lv_search.cu — batched two-level / best-first search kernels for sm_100a.
//
// One warp owns one query slot; thousands of slots run concurrently. All
// per-query state lives in HBM (per-slot SoA) and the warp keeps the scalar
// part in registers, uniform across its lanes. Semantics are the reference's
// (restated in oracle/search_port.py and pinned by golden vectors):
//   _descend                     search.py:257-285   (PH_ENTRY / PH_DESCENT)
//   best_first_search loop       search.py:308-323   (LV_MODE_EXACT_BESTFIRST)
//   two_level_search loop        search.py:376-419   (LV_MODE_TWO_LEVEL)
//   _ExactQueue try_insert/pop   search.py:217-241   (eq_insert / eq_pop)
//   k_best + delete filter       search.py:243-251   (finish_query)
//   _Recomputer counters/cache   search.py:155-188   (emit)
//   adc_build                    pq.py:153-178       (lut_kernel)
//   approx_distance_many         pq.py:186-189       (adc_one, lv_numerics.cuh)
//   distance_many                vectors.py:120-140  (resolve / dist_kernel)
#include <algorithm>
#include "lv_search.cuh"
#include "lv_numerics.cuh"

namespace lv {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }

__device__ __forceinline__ unsigned long long aq_key(float aw, int32_t w, bool elig) {
  return ((unsigned long long)ord_f32(aw) << 32) | ((unsigned long long)(uint32_t)w << 1) |
         (elig ? 1ull : 0ull);
}
__device__ __forceinline__ int32_t aq_id(unsigned long long key) {
  return (int32_t)(((uint32_t)key) >> 1);
}

// A per-query set of node ids: approx_known / exact_known of two_level_search
// (search.py:364-366). Dense bitmap over [0, n) or a bounded open-addressing
// hash set (linear probing, keys inserted with atomicCAS; all lanes of a warp
// may insert distinct ids concurrently).
struct VSet {
  uint32_t *bits;   // bitmap mode
  uint32_t *keys;   // hash mode (mask != 0)
  uint32_t mask;
  __device__ __forceinline__ bool test(int32_t w) const {
    if (!mask) return bit_test(bits, w);
    uint32_t h = hash_id((uint32_t)w) & mask;
    while (true) {
      const uint32_t k = keys[h];
      if (k == (uint32_t)w) return true;
      if (k == 0xffffffffu) return false;
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ void insert(int32_t w) const {
    if (!mask) {
      bit_set(bits, w);
      return;
    }
    uint32_t h = hash_id((uint32_t)w) & mask;
    while (true) {
      const uint32_t k = keys[h];
      if (k == (uint32_t)w) return;
      if (k == 0xffffffffu) {
        const uint32_t old = atomicCAS(keys + h, 0xffffffffu, (uint32_t)w);
        if (old == 0xffffffffu || old == (uint32_t)w) return;
      }
      h = (h + 1) & mask;
    }
  }
  __device__ static __forceinline__ uint32_t hash_id(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
  }
};

struct SlotPtrs {
  float *eq_d;
  uint32_t *eq_id;
  unsigned long long *aq;
  VSet aset;   // approx_known
  VSet xset;   // exact_known
  int32_t *xlist;
  int32_t *req;
};

struct WarpSmem {
  const float *lut;            // this query's LUT: shared memory (lut_smem) or global
  bool lut_shared;
  float *req_d;                // [req_cap] exact distances of the pending request
  int32_t *miss_idx;           // [req_cap] row index in the global request buffer (-1 = cached)
  int32_t *fresh;              // [max_degree]
  unsigned long long *tmpk;    // [max_degree]
  unsigned long long *newk;    // [max_degree]
};

__device__ __forceinline__ SlotPtrs slot_ptrs(const SearchCtx &c, int slot) {
  SlotPtrs p;
  p.eq_d = c.eq_d + (int64_t)slot * c.ef;
  p.eq_id = c.eq_id + (int64_t)slot * c.ef;
  p.aq = c.aq + (int64_t)slot * c.aq_cap;
  if (c.vmask) {
    const int64_t cap = (int64_t)c.vmask + 1;
    p.aset = VSet{nullptr, c.aset + (int64_t)slot * cap, c.vmask};
    p.xset = VSet{nullptr, c.xset + (int64_t)slot * cap, c.vmask};
  } else {
    p.aset = VSet{c.abits + (int64_t)slot * c.words, nullptr, 0u};
    p.xset = VSet{c.xbits + (int64_t)slot * c.words, nullptr, 0u};
  }
  p.xlist = c.xlist + (int64_t)slot * c.xl_cap;
  p.req = c.req + (int64_t)slot * c.req_cap;
  return p;
}

// ---------------------------------------------------------------- exact queue
// try_insert (search.py:217-232): keep the ef best by (d, id).
__device__ void eq_insert(const SearchCtx &c, const SlotPtrs &P, SlotState &S, float d,
                          int32_t id) {
  const int lane = lane_id();
  if (S.eq_size >= c.ef) {
    float wd = P.eq_d[S.eq_size - 1];
    int32_t wi = (int32_t)(P.eq_id[S.eq_size - 1] & ~kVisited);
    if (!pair_less(d, id, wd, wi)) return;
    S.eq_size -= 1;
  }
  int pos = 0;
  for (int base = 0; base < S.eq_size; base += 32) {
    int i = base + lane;
    bool lt = false;
    if (i < S.eq_size) lt = pair_less(P.eq_d[i], (int32_t)(P.eq_id[i] & ~kVisited), d, id);
    unsigned b = __ballot_sync(kFull, lt);
    pos += __popc(b);
    if (b != kFull) break;
  }
  for (int top = S.eq_size - 1; top >= pos; top -= 32) {
    int i = top - lane;
    bool act = i >= pos;
    float vd = 0.f;
    uint32_t vi = 0;
    if (act) {
      vd = P.eq_d[i];
      vi = P.eq_id[i];
    }
    __syncwarp();
    if (act) {
      P.eq_d[i + 1] = vd;
      P.eq_id[i + 1] = vi;
    }
    __syncwarp();
  }
  if (lane == 0) {
    P.eq_d[pos] = d;
    P.eq_id[pos] = (uint32_t)id;
  }
  __syncwarp();
  S.eq_size += 1;
  if (pos < S.eq_hint) S.eq_hint = pos;
}

// pop_closest_unvisited (search.py:234-241). Returns -1 when none is left.
__device__ int32_t eq_pop(const SlotPtrs &P, SlotState &S) {
  const int lane = lane_id();
  for (int base = S.eq_hint; base < S.eq_size; base += 32) {
    int i = base + lane;
    uint32_t v = 0;
    bool un = false;
    if (i < S.eq_size) {
      v = P.eq_id[i];
      un = !(v & kVisited);
    }
    unsigned b = __ballot_sync(kFull, un);
    if (b) {
      int src = __ffs(b) - 1;
      uint32_t id = __shfl_sync(kFull, v, src);
      int p = base + src;
      __syncwarp();
      if (lane == 0) P.eq_id[p] = id | kVisited;
      __syncwarp();
      S.eq_hint = p + 1;
      return (int32_t)id;
    }
  }
  S.eq_hint = S.eq_size;
  return -1;
}

// CSR row of v at `level` minus the nodes whose bit is set, in CSR order
// (graph.py:50-52 + search.py:269 / :314 / :385).
__device__ int filter_row(const SearchCtx &c, int32_t v, int level, const VSet &bits,
                          int32_t *out) {
  const int lane = lane_id();
  const uint64_t *off = c.offs[level];
  uint64_t a = off[v], b = off[v + 1];
  int deg = (int)(b - a);
  const uint32_t *row = c.nbrs[level] + a;
  int cnt = 0;
  for (int base = 0; base < deg; base += 32) {
    int i = base + lane;
    int32_t w = -1;
    bool keep = false;
    if (i < deg) {
      w = (int32_t)__ldg(row + i);
      keep = !bits.test(w);
    }
    unsigned bal = __ballot_sync(kFull, keep);
    if (keep) out[cnt + __popc(bal & lanemask_lt())] = w;
    cnt += __popc(bal);
  }
  __syncwarp();
  return cnt;
}

// Record ids whose exact bit is set outside the AQ (for cheap clearing).
__device__ void xlist_append(const SearchCtx &c, const SlotPtrs &P, SlotState &S,
                             const int32_t *ids, int cnt, bool set_bits) {
  const int lane = lane_id();
  for (int r = lane; r < cnt; r += 32) {
    int32_t w = ids[r];
    if (set_bits) P.xset.insert(w);
    int pos = S.xl_len + r;
    if (pos < c.xl_cap) P.xlist[pos] = w;
  }
  __syncwarp();
  S.xl_len += cnt;
}

// Publish the pending request: funnel counters (search.py:155-188) and, for
// the encoder source, the misses into the global request buffer.
__device__ void emit(const SearchCtx &c, const SlotPtrs &P, SlotState &S, const WarpSmem &W) {
  const int lane = lane_id();
  int misses = 0;
  for (int base = 0; base < S.req_n; base += 32) {
    int r = base + lane;
    bool miss = false;
    if (r < S.req_n) {
      int32_t w = P.req[r];
      miss = !(c.cached_bits && bit_test(c.cached_bits, w));
    }
    unsigned bal = __ballot_sync(kFull, miss);
    if (r < S.req_n) W.miss_idx[r] = miss ? misses + __popc(bal & lanemask_lt()) : -1;
    misses += __popc(bal);
  }
  __syncwarp();
  int hits = S.req_n - misses;
  S.hits += hits;
  if (misses > 0) {
    S.recomps += misses;
    if (lane == 0 && c.blog && S.blog_n < c.blog_cap)
      c.blog[(int64_t)S.qi * c.blog_cap + S.blog_n] = misses;
    S.blog_n += 1;
  }
  if (c.source == LV_SOURCE_ENCODER && misses > 0) {
    int off = 0;
    if (lane == 0) off = atomicAdd(c.greq_total, misses);
    off = __shfl_sync(kFull, off, 0);
    if (off + misses > c.greq_cap) {
      S.status = LV_Q_FAILED;  // cannot happen with greq_cap = slots * req_cap
      off = 0;
      misses = 0;
    }
    S.req_off = off;
    for (int r = lane; r < S.req_n; r += 32) {
      int mi = W.miss_idx[r];
      if (mi >= 0 && mi < misses) c.greq[off + mi] = P.req[r];
    }
    __syncwarp();
  }
}

// Exact distances of the pending request (distance_many, vectors.py:120-140),
// 4 lanes per row in the pinned einsum order; results into W.req_d.
__device__ void compute_request_distances(const SearchCtx &c, const SlotPtrs &P,
                                          const SlotState &S, const WarpSmem &W) {
  const int lane = lane_id();
  const int g = lane >> 2, l = lane & 3;
  const float *qv = c.q + (int64_t)S.qi * c.dim;
  const float qn = c.qn[S.qi];
  for (int base = 0; base < S.req_n; base += 8) {
    int r = base + g;
    bool act = r < S.req_n;
    float a_dot = 0.f, a_nrm = 0.f;
    if (act) {
      int32_t w = P.req[r];
      const float *row;
      if (c.source == LV_SOURCE_MATRIX) {
        row = c.matrix + (int64_t)w * c.dim;
      } else {
        int mi = W.miss_idx[r];
        row = (mi < 0) ? c.cache_rows + (int64_t)c.cache_slot[w] * c.dim
              : c.emb_buf + (int64_t)(c.emb_map ? c.emb_map[S.req_off + mi] : S.req_off + mi) * c.dim;
      }
      if (c.metric == LV_METRIC_L2) {
        a_dot = einsum_lane<true>(row, qv, c.dim, l);
      } else {
        a_dot = einsum_lane<false>(row, qv, c.dim, l);
        if (c.metric == LV_METRIC_COSINE) a_nrm = einsum_lane<false>(row, row, c.dim, l);
      }
    }
    float d0 = __shfl_sync(kFull, a_dot, g * 4 + 0), d1 = __shfl_sync(kFull, a_dot, g * 4 + 1);
    float d2 = __shfl_sync(kFull, a_dot, g * 4 + 2), d3 = __shfl_sync(kFull, a_dot, g * 4 + 3);
    float n0 = __shfl_sync(kFull, a_nrm, g * 4 + 0), n1 = __shfl_sync(kFull, a_nrm, g * 4 + 1);
    float n2 = __shfl_sync(kFull, a_nrm, g * 4 + 2), n3 = __shfl_sync(kFull, a_nrm, g * 4 + 3);
    if (act && l == 0) {
      float dot = einsum_combine(d0, d1, d2, d3);
      float nrm = einsum_combine(n0, n1, n2, n3);
      W.req_d[r] = finish_distance(c.metric, dot, nrm, qn);
    }
  }
  __syncwarp();
}

// Exact results of a request flow back into the traversal state.
__device__ void resolve(const SearchCtx &c, const SlotPtrs &P, SlotState &S, const WarpSmem &W) {
  compute_request_distances(c, P, S, W);
  S.bytes += 4 * (long long)c.dim * S.req_n;
  const int lane = lane_id();
  if (S.phase == PH_ENTRY) {
    float d0 = W.req_d[0];
    xlist_append(c, P, S, P.req, 1, true);
    eq_insert(c, P, S, d0, c.entry);
    S.cur = c.entry;
    S.cur_d = d0;
    S.phase = PH_DESCENT;
    S.level = c.level_count - 1;
  } else if (S.phase == PH_DESCENT) {
    xlist_append(c, P, S, P.req, S.req_n, true);
    float bd = S.cur_d;
    int32_t bi = S.cur;
    for (int r = 0; r < S.req_n; ++r) {
      float dw = W.req_d[r];
      int32_t w = P.req[r];
      eq_insert(c, P, S, dw, w);
      if (pair_less(dw, w, bd, bi)) {
        bd = dw;
        bi = w;
      }
    }
    if (bi == S.cur) {
      S.level -= 1;
    } else {
      S.cur = bi;
      S.cur_d = bd;
    }
  } else if (S.phase == PH_BASE) {
    for (int r = 0; r < S.req_n; ++r) eq_insert(c, P, S, W.req_d[r], P.req[r]);
  }
  (void)lane;
  S.req_n = 0;
}

// First k non-deleted EQ members (k_best, search.py:243-251), counters, and
// bitmap clean-up; the slot becomes idle.
__device__ void finish_query(const SearchCtx &c, const SlotPtrs &P, SlotState &S) {
  const int lane = lane_id();
  const int64_t qo = (int64_t)S.qi * c.k;
  int cnt = 0;
  for (int base = 0; base < S.eq_size && cnt < c.k; base += 32) {
    int i = base + lane;
    bool keep = false;
    int32_t id = -1;
    float d = 0.f;
    if (i < S.eq_size) {
      id = (int32_t)(P.eq_id[i] & ~kVisited);
      d = P.eq_d[i];
      keep = !(c.deleted_bits && bit_test(c.deleted_bits, id));
    }
    unsigned bal = __ballot_sync(kFull, keep);
    int pos = cnt + __popc(bal & lanemask_lt());
    if (keep && pos < c.k) {
      c.out_ids[qo + pos] = id;
      c.out_dist[qo + pos] = d;
    }
    cnt += __popc(bal);
  }
  if (cnt > c.k) cnt = c.k;
  for (int j = cnt + lane; j < c.k; j += 32) {
    c.out_ids[qo + j] = -1;
    c.out_dist[qo + j] = 0.f;
  }
  if (lane == 0) {
    if (c.bytes_total) atomicAdd(c.bytes_total, (unsigned long long)S.bytes);
    c.out_count[S.qi] = cnt;
    c.out_counters[(int64_t)S.qi * 4 + 0] = S.recomps;
    c.out_counters[(int64_t)S.qi * 4 + 1] = S.approx;
    c.out_counters[(int64_t)S.qi * 4 + 2] = S.hits;
    c.out_counters[(int64_t)S.qi * 4 + 3] = S.expansions;
    if (c.out_status) c.out_status[S.qi] = S.status;
  }
  if (c.vmask) {  // hash sets: reset both tables (16-byte stores, whole warp)
    const int64_t n4 = ((int64_t)c.vmask + 1) / 4;
    uint4 *a4 = reinterpret_cast<uint4 *>(P.aset.keys), *x4 = reinterpret_cast<uint4 *>(P.xset.keys);
    const uint4 e = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    for (int64_t i = lane; i < n4; i += 32) {
      a4[i] = e;
      x4[i] = e;
    }
  } else {  // clear the slot's bitmaps: every set bit belongs to an AQ or xlist id
    for (int i = lane; i < S.aq_len; i += 32) {
      int32_t w = aq_id(P.aq[i]);
      P.aset.bits[w >> 5] = 0u;
      P.xset.bits[w >> 5] = 0u;
    }
    if (S.xl_len <= c.xl_cap) {
      for (int i = lane; i < S.xl_len; i += 32) P.xset.bits[P.xlist[i] >> 5] = 0u;
    } else {
      for (int64_t i = lane; i < c.words; i += 32) P.xset.bits[i] = 0u;
    }
  }
  __syncwarp();
  if (lane == 0) atomicAdd(c.done_count, 1);
  S.phase = PH_IDLE;
  S.qi = -1;
}

// Approximate scores of the fresh neighbours and their AQ merge
// (search.py:385-394): ADC in fp64 pairwise order, keys sorted in-warp,
// then an in-place back-to-front merge into the sorted AQ.
__device__ void adc_insert(const SearchCtx &c, const SlotPtrs &P, SlotState &S,
                           const WarpSmem &W, int F) {
  const int lane = lane_id();
  const float *lut = W.lut;
  int n_el = 0;
  for (int base = 0; base < F; base += 32) {
    int j = base + lane;
    bool el = false;
    if (j < F) {
      int32_t w = W.fresh[j];
      float aw = W.lut_shared ? adc_one_shared(lut, c.codes + (int64_t)w * c.m, c.m)
                              : adc_one(lut, c.codes + (int64_t)w * c.m, c.m);
      el = !P.xset.test(w);
      P.aset.insert(w);
      W.tmpk[j] = aq_key(aw, w, el);
    }
    n_el += __popc(__ballot_sync(kFull, el));
  }
  __syncwarp();
  // rank sort of the F new keys (distinct)
  for (int j = lane; j < F; j += 32) {
    unsigned long long kj = W.tmpk[j];
    int rank = 0;
    for (int i = 0; i < F; ++i) rank += (W.tmpk[i] < kj) ? 1 : 0;
    W.newk[rank] = kj;
  }
  __syncwarp();
  const int L = S.aq_len;
  int carry = F;  // shift of the element just above the current chunk
  // the AQ chunks are read two ahead: a chunk's writes land at or above its own
  // positions, so the lower chunks still hold their original keys when prefetched
  auto ld = [&](int cb) -> unsigned long long {
    const int i = cb + lane;
    return (cb >= 0 && i < L) ? P.aq[i] : ~0ull;
  };
  int cbase = (L > 0) ? ((L - 1) & ~31) : -1;
  unsigned long long k0 = ld(cbase), k1 = ld(cbase - 32);
  for (; cbase >= 0; cbase -= 32) {
    const unsigned long long k2 = ld(cbase - 64);
    int i = cbase + lane;
    bool act = i < L;
    unsigned long long key = k0;
    k0 = k1;
    k1 = k2;
    int s = F;
    if (act) {  // number of new keys below `key`
      int lo = 0, hi = F;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (W.newk[mid] < key) lo = mid + 1; else hi = mid;
      }
      s = lo;
    }
    int s_next = __shfl_down_sync(kFull, s, 1);
    if (lane == 31) s_next = carry;
    __syncwarp();
    if (act) {
      P.aq[i + s] = key;
      for (int j = s; j < s_next; ++j) P.aq[j + i + 1] = W.newk[j];
    }
    carry = __shfl_sync(kFull, s, 0);
    __syncwarp();
  }
  const int s0 = (L > 0) ? carry : F;
  for (int j = lane; j < s0; j += 32) P.aq[j] = W.newk[j];
  __syncwarp();
  S.aq_len = L + F;
  S.bytes += (long long)c.m * F;
  S.n_elig += n_el;
  S.approx += F;
}

// cutoff = aq_sorted[min(L, max(1, ceil(alpha*L))) - 1]; promote every eligible
// entry <= cutoff in ascending order (search.py:395-405).
__device__ void select_step(const SearchCtx &c, const SlotPtrs &P, SlotState &S) {
  const int lane = lane_id();
  S.req_n = 0;
  if (S.aq_len == 0 || S.n_elig == 0) return;
  double prod = c.alpha * (double)S.aq_len;
  long long r = (long long)ceil(prod);
  if (r < 1) r = 1;
  if (r > S.aq_len) r = S.aq_len;
  int cnt = 0;
  for (int base = 0; base < r && cnt < S.n_elig; base += 32) {
    int i = base + lane;
    unsigned long long key = 0;
    bool e = false;
    if (i < r) {
      key = P.aq[i];
      e = key & 1ull;
    }
    unsigned bal = __ballot_sync(kFull, e);
    if (e) {
      P.req[cnt + __popc(bal & lanemask_lt())] = aq_id(key);
      P.aq[i] = key & ~1ull;
    }
    cnt += __popc(bal);
  }
  __syncwarp();
  S.n_elig -= cnt;
  S.req_n = cnt;
}

// Run one slot until it emits a recompute request (true) or its query ends (false).
__device__ bool advance(const SearchCtx &c, const SlotPtrs &P, SlotState &S, const WarpSmem &W) {
  const int lane = lane_id();
  while (true) {
    if (S.phase == PH_ENTRY) {
      if (lane == 0) P.req[0] = c.entry;
      __syncwarp();
      S.req_n = 1;
      emit(c, P, S, W);
      return true;
    }
    if (S.phase == PH_DESCENT) {
      if (S.level <= 0) {
        S.phase = PH_BASE;
        continue;
      }
      int cnt = filter_row(c, S.cur, S.level, P.xset, P.req);
      S.bytes += 16 + 4 * (long long)(c.offs[S.level][S.cur + 1] - c.offs[S.level][S.cur]);
      if (cnt == 0) {
        S.level -= 1;
        continue;
      }
      S.req_n = cnt;
      emit(c, P, S, W);
      return true;
    }
    // PH_BASE
    int32_t u = eq_pop(P, S);
    if (u < 0) {
      finish_query(c, P, S);
      return false;
    }
    if (lane == 0 && c.visits && S.visits_n < c.visits_cap)
      c.visits[(int64_t)S.qi * c.visits_cap + S.visits_n] = u;
    S.visits_n += 1;
    S.expansions += 1;
    S.bytes += 16 + 4 * (long long)(c.offs[0][u + 1] - c.offs[0][u]);
    if (c.mode == LV_MODE_EXACT_BESTFIRST) {
      int cnt = filter_row(c, u, 0, P.xset, P.req);
      if (cnt == 0) continue;
      xlist_append(c, P, S, P.req, cnt, true);  // claimed (search.py:317-318)
      S.req_n = cnt;
      emit(c, P, S, W);
      return true;
    }
    int F = filter_row(c, u, 0, P.aset, W.fresh);
    if (F > 0) {
      if (S.aq_len + F > c.aq_cap) {
        S.status = LV_Q_AQ_OVERFLOW;
        finish_query(c, P, S);
        return false;
      }
      adc_insert(c, P, S, W, F);
    }
    select_step(c, P, S);
    if (S.req_n > 0) {
      emit(c, P, S, W);
      return true;
    }
  }
}

__device__ bool claim(const SearchCtx &c, SlotState &S) {
  int pos = 0;
  if (lane_id() == 0) pos = atomicAdd(c.queue_head, 1);
  pos = __shfl_sync(kFull, pos, 0);
  if (pos >= c.B) return false;
  S = SlotState{};
  S.qi = pos;
  S.phase = PH_ENTRY;
  S.level = c.level_count - 1;
  S.status = LV_Q_OK;
  if (c.mode == LV_MODE_TWO_LEVEL) S.bytes = 4LL * c.m * kCentroids;  // the query's LUT
  return true;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
frontier_kernel(const __grid_constant__ SearchCtx c) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * (blockDim.x >> 5) + warp;
  if (slot >= c.slots) return;
  // carve this warp's scratch
  const size_t per_warp = frontier_smem_per_warp(c.max_degree, c.req_cap);
  unsigned char *base = smem_raw + per_warp * warp;
  WarpSmem W;
  W.newk = reinterpret_cast<unsigned long long *>(base);
  W.tmpk = W.newk + c.max_degree;
  W.req_d = reinterpret_cast<float *>(W.tmpk + c.max_degree);
  W.miss_idx = reinterpret_cast<int32_t *>(W.req_d + c.req_cap);
  W.fresh = W.miss_idx + c.req_cap;

  uint64_t *lut_bar = nullptr;
  uint32_t lut_phase = 0;
  W.lut_shared = c.lut_smem != 0;
  if (W.lut_shared) {  // [LUT][mbarrier][scratch] per warp
    float *lut = reinterpret_cast<float *>(smem_raw + frontier_smem_per_warp_lut(
                                                          c.max_degree, c.req_cap, c.m) * warp);
    lut_bar = reinterpret_cast<uint64_t *>(lut + (size_t)c.m * kCentroids);
    base = reinterpret_cast<unsigned char *>(lut_bar) + 16;
    W.newk = reinterpret_cast<unsigned long long *>(base);
    W.tmpk = W.newk + c.max_degree;
    W.req_d = reinterpret_cast<float *>(W.tmpk + c.max_degree);
    W.miss_idx = reinterpret_cast<int32_t *>(W.req_d + c.req_cap);
    W.fresh = W.miss_idx + c.req_cap;
    W.lut = lut;
    if (lane_id() == 0)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(lut_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  // this warp's query LUT -> shared memory: one cp.async.bulk (TMA engine)
  auto stage_lut = [&](int qi) {
    const uint32_t bytes = (uint32_t)c.m * kCentroids * 4;
    if (lane_id() == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_addr(lut_bar)),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(smem_addr(W.lut)),
          "l"(c.luts + (int64_t)qi * c.m * kCentroids), "r"(bytes), "r"(smem_addr(lut_bar))
          : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_addr(lut_bar)), "r"(lut_phase)
          : "memory");
    lut_phase ^= 1u;
    __syncwarp();
  };
  SlotState S = c.st[slot];
  const SlotPtrs P = slot_ptrs(c, slot);
  if (!W.lut_shared && S.qi >= 0) W.lut = c.luts + (int64_t)S.qi * c.m * kCentroids;
  if (c.source == LV_SOURCE_ENCODER && S.req_n > 0 &&
      (S.phase == PH_ENTRY || S.phase == PH_DESCENT || S.phase == PH_BASE)) {
    // misses were published by the previous launch; rebuild their indices
    const int lane = lane_id();
    int misses = 0;
    for (int b0 = 0; b0 < S.req_n; b0 += 32) {
      int r = b0 + lane;
      bool miss = false;
      if (r < S.req_n) miss = !(c.cached_bits && bit_test(c.cached_bits, P.req[r]));
      unsigned bal = __ballot_sync(kFull, miss);
      if (r < S.req_n) W.miss_idx[r] = miss ? misses + __popc(bal & lanemask_lt()) : -1;
      misses += __popc(bal);
    }
    __syncwarp();
    resolve(c, P, S, W);
  }
  while (S.phase != PH_FINISHED) {
    if (S.phase == PH_IDLE) {
      if (!claim(c, S)) {
        S.phase = PH_FINISHED;
        break;
      }
      if (c.mode == LV_MODE_TWO_LEVEL) {
        if (W.lut_shared)
          stage_lut(S.qi);
        else
          W.lut = c.luts + (int64_t)S.qi * c.m * kCentroids;
      }
    }
    bool emitted = advance(c, P, S, W);
    if (!emitted) continue;
    if (c.source == LV_SOURCE_MATRIX) {
      resolve(c, P, S, W);
      continue;
    }
    break;
  }
  if (lane_id() == 0) c.st[slot] = S;
}

// ------------------------------------------------------------------- LUT build
// adc_build (pq.py:153-178): cosine normalises q by the host qn, each table
// entry is an einsum over one sub-space (ip/cosine negated, l2 of cb - q_s).
__global__ void lut_kernel(const float *__restrict__ q, const float *__restrict__ qn, int dim,
                           int metric, const float *__restrict__ cb, int m, int padded,
                           float *__restrict__ luts) {
  extern __shared__ float qp[];
  const int qi = blockIdx.x;
  const float *qv = q + (int64_t)qi * dim;
  const float norm = (metric == LV_METRIC_COSINE) ? qn[qi] : 1.0f;
  for (int i = threadIdx.x; i < padded; i += blockDim.x) {
    float v = 0.0f;
    if (i < dim) v = (metric == LV_METRIC_COSINE) ? __fdiv_rn(qv[i], norm) : qv[i];
    qp[i] = v;
  }
  __syncthreads();
  const int sub = padded / m;
  float *out = luts + (int64_t)qi * m * kCentroids;
  for (int e = threadIdx.x; e < m * kCentroids; e += blockDim.x) {
    int s = e / kCentroids, cidx = e % kCentroids;
    const float *cv = cb + ((int64_t)s * kCentroids + cidx) * sub;
    const float *qs = qp + s * sub;
    float t;
    if (metric == LV_METRIC_L2) {
      t = einsum_dot_1t<true>(cv, qs, sub);
    } else {
      t = -einsum_dot_1t<false>(cv, qs, sub);
    }
    out[e] = t;
  }
}

__global__ void adc_score_kernel(const float *__restrict__ lut, int m,
                                 const uint8_t *__restrict__ codes,
                                 const int64_t *__restrict__ ids, int64_t count,
                                 float *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  out[i] = adc_one(lut, codes + ids[i] * m, m);
}

// Streaming ADC (approx_distance_many, pq.py:186-189) over many ids of one
// query: the query's LUT is staged in shared memory once per CTA (persistent
// grid), each thread reads its node's m code bytes with 16-byte loads (one
// 64-byte line at m = 64) and sums the LUT entries in numpy's fp64 pairwise
// order — bit-identical to adc_one.
template <int M>
__global__ void __launch_bounds__(256) adc_stream_kernel(const float *__restrict__ lut,
                                                         const uint8_t *__restrict__ codes,
                                                         const int64_t *__restrict__ ids,
                                                         int64_t count, float *__restrict__ out) {
  extern __shared__ float slut[];
  for (int i = threadIdx.x; i < M * 256; i += blockDim.x) slut[i] = lut[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 *cp = reinterpret_cast<const uint4 *>(codes + __ldg(ids + i) * M);
    uint8_t c[M];
#pragma unroll
    for (int v = 0; v < M / 16; ++v) *reinterpret_cast<uint4 *>(c + 16 * v) = __ldg(cp + v);
    auto get = [&](int s) -> double { return (double)slut[s * 256 + c[s]]; };
    out[i] = __double2float_rn(pairwise_sum(get, M));
  }
}

__global__ void dist_kernel(int metric, const float *__restrict__ rows, int64_t nrows, int dim,
                            const float *__restrict__ q, float qn, float *__restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t r = t >> 2;
  int l = (int)(t & 3);
  bool act = r < nrows;
  float a = 0.f, b = 0.f;
  if (act) {
    const float *row = rows + r * dim;
    if (metric == LV_METRIC_L2) {
      a = einsum_lane<true>(row, q, dim, l);
    } else {
      a = einsum_lane<false>(row, q, dim, l);
      if (metric == LV_METRIC_COSINE) b = einsum_lane<false>(row, row, dim, l);
    }
  }
  const int g = (threadIdx.x & 31) >> 2;
  float a0 = __shfl_sync(kFull, a, g * 4), a1 = __shfl_sync(kFull, a, g * 4 + 1);
  float a2 = __shfl_sync(kFull, a, g * 4 + 2), a3 = __shfl_sync(kFull, a, g * 4 + 3);
  float b0 = __shfl_sync(kFull, b, g * 4), b1 = __shfl_sync(kFull, b, g * 4 + 1);
  float b2 = __shfl_sync(kFull, b, g * 4 + 2), b3 = __shfl_sync(kFull, b, g * 4 + 3);
  if (act && l == 0)
    out[r] = finish_distance(metric, einsum_combine(a0, a1, a2, a3), einsum_combine(b0, b1, b2, b3), qn);
}

// distance_many (vectors.py:120-140) of query b against rows ids[b][0..C) of
// the matrix: 4 lanes per (b, c) in the einsum order; ids < 0 -> +inf.
__global__ void dist_gather_kernel(int metric, const float *__restrict__ rows, int dim,
                                   const int64_t *__restrict__ ids, int B, int C,
                                   const float *__restrict__ q, const float *__restrict__ qn,
                                   float *__restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t pair = t >> 2;
  const int l = (int)(t & 3);
  const bool act = pair < (int64_t)B * C;
  const int b = act ? (int)(pair / C) : 0;
  const int64_t id = act ? ids[pair] : -1;
  float a = 0.f, nr = 0.f;
  if (act && id >= 0) {
    const float *row = rows + id * dim;
    const float *qv = q + (int64_t)b * dim;
    if (metric == LV_METRIC_L2) {
      a = einsum_lane<true>(row, qv, dim, l);
    } else {
      a = einsum_lane<false>(row, qv, dim, l);
      if (metric == LV_METRIC_COSINE) nr = einsum_lane<false>(row, row, dim, l);
    }
  }
  const int g = (threadIdx.x & 31) >> 2;
  float a0 = __shfl_sync(kFull, a, g * 4), a1 = __shfl_sync(kFull, a, g * 4 + 1);
  float a2 = __shfl_sync(kFull, a, g * 4 + 2), a3 = __shfl_sync(kFull, a, g * 4 + 3);
  float n0 = __shfl_sync(kFull, nr, g * 4), n1 = __shfl_sync(kFull, nr, g * 4 + 1);
  float n2 = __shfl_sync(kFull, nr, g * 4 + 2), n3 = __shfl_sync(kFull, nr, g * 4 + 3);
  if (act && l == 0)
    out[pair] = id < 0 ? __int_as_float(0x7f800000)
                       : finish_distance(metric, einsum_combine(a0, a1, a2, a3),
                                         einsum_combine(n0, n1, n2, n3), qn[b]);
}

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void dedup_kernel(const int32_t *__restrict__ greq, int total, int32_t *keys,
                             int32_t *vals, uint32_t mask, int32_t *row_count, int32_t base,
                             int32_t *__restrict__ new_ids, int32_t *__restrict__ map) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= total) return;
  const int32_t w = greq[r];
  uint32_t slot = mix32((uint32_t)w) & mask;
  while (true) {
    const int32_t k = atomicCAS(keys + slot, -1, w);
    if (k == -1) {  // first request of w in this step: claim a row, schedule its encode
      const int32_t row = atomicAdd(row_count, 1);
      new_ids[row - base] = w;
      atomicExch(vals + slot, row);
      map[r] = row;
      return;
    }
    if (k == w) {  // shared: wait for the claimer to publish the row
      int32_t row;
      do {
        row = atomicAdd(vals + slot, 0);
      } while (row < 0);
      map[r] = row;
      return;
    }
    slot = (slot + 1) & mask;
  }
}

// qn = np.float32(np.sqrt(np.dot(q, q))) (vectors.py:138, pq.py:163) in the
// OpenBLAS sdot order (lv_numerics.cuh); one thread per query.
__global__ void qnorm_kernel(const float *__restrict__ q, int B, int dim, float *__restrict__ qn) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const float *v = q + (int64_t)i * dim;
  qn[i] = __fsqrt_rn(sdot_openblas<false>(v, v, dim));
}

// buffer_scan (update.py:483-488): distance(q, vec) (vectors.py:94-116) of
// every query to every pending vector; one thread per (query, pending) pair.
// Cosine: -np.dot(q, v) / np.float32(float(sqrt(q.q)) * float(sqrt(v.v))),
// the denominator multiplied in float64. A zero denominator sets *bad.
__global__ void pending_dist_kernel(int metric, const float *__restrict__ pend, int64_t np_,
                                    int dim, const float *__restrict__ q,
                                    const float *__restrict__ qn, int B,
                                    float *__restrict__ out, int *bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * np_) return;
  const int b = (int)(t / np_);
  const int64_t p = t % np_;
  const float *qv = q + (int64_t)b * dim;
  const float *pv = pend + p * dim;
  float d;
  if (metric == LV_METRIC_L2) {
    d = sdot_openblas<true>(qv, pv, dim);
  } else if (metric == LV_METRIC_IP) {
    d = -sdot_openblas<false>(qv, pv, dim);
  } else {
    const float pn = __fsqrt_rn(sdot_openblas<false>(pv, pv, dim));
    const double denom = __dmul_rn((double)qn[b], (double)pn);
    if (denom == 0.0) atomicExch(bad, 1);
    d = __fdiv_rn(-sdot_openblas<false>(qv, pv, dim), __double2float_rn(denom));
  }
  out[t] = d;
}

// Engine.search merge (index.py:320-327): the graph's k results plus every
// pending item, sorted by (distance, id); the first k are kept. One warp per
// query, k rounds of a warp-wide (d, id) minimum.
__global__ void pending_merge_kernel(const float *__restrict__ pdist,
                                     const int64_t *__restrict__ pids, int64_t np_, int B, int k,
                                     int64_t *ids, float *dist, int32_t *count) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= B) return;
  const int b = warp;
  const int cnt0 = count[b];
  const int64_t total = cnt0 + np_;
  const float *pd = pdist + (int64_t)b * np_;
  int64_t *oid = ids + (int64_t)b * k;
  float *od = dist + (int64_t)b * k;
  // candidates: [0, cnt0) the graph results (staged in shared memory: the
  // output rows are overwritten), then the pending items
  extern __shared__ __align__(8) unsigned char merge_smem[];
  const int wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t *ci = reinterpret_cast<int64_t *>(merge_smem) + (int64_t)wib * k;
  float *cd = reinterpret_cast<float *>(reinterpret_cast<int64_t *>(merge_smem) + (int64_t)nw * k) +
              (int64_t)wib * k;
  for (int j = lane; j < cnt0; j += 32) {
    cd[j] = od[j];
    ci[j] = oid[j];
  }
  __syncwarp();
  // candidates are taken in strictly increasing (d, id) order (ids are unique
  // across the two lists: pending ids are >= the graph's n)
  float last_d = 0.f;
  int64_t last_i = INT64_MIN;
  bool have_last = false;
  int out_n = 0;
  for (int r = 0; r < k && r < total; ++r) {
    float best_d = 0.f;
    int64_t best_i = INT64_MAX;
    bool have = false;
    for (int64_t j = lane; j < total; j += 32) {
      float d;
      int64_t id;
      if (j < cnt0) {
        d = cd[j];
        id = ci[j];
      } else {
        d = pd[j - cnt0];
        id = pids[j - cnt0];
      }
      const uint32_t od_ = ord_f32(d);
      if (have_last) {
        const uint32_t ol = ord_f32(last_d);
        if (od_ < ol || (od_ == ol && id <= last_i)) continue;  // already taken
      }
      const uint32_t ob = ord_f32(best_d);
      if (!have || od_ < ob || (od_ == ob && id < best_i)) {
        best_d = d;
        best_i = id;
        have = true;
      }
    }
    // warp argmin over (have, d, id)
    for (int off = 16; off > 0; off >>= 1) {
      const float d2 = __shfl_xor_sync(0xffffffffu, best_d, off);
      const long long i2 = __shfl_xor_sync(0xffffffffu, (long long)best_i, off);
      const int h2 = __shfl_xor_sync(0xffffffffu, (int)have, off);
      const uint32_t a = ord_f32(best_d), c = ord_f32(d2);
      if (h2 && (!have || c < a || (c == a && i2 < best_i))) {
        best_d = d2;
        best_i = i2;
        have = true;
      }
    }
    if (!have) break;
    if (lane == 0) {
      od[r] = best_d;
      oid[r] = best_i;
    }
    last_d = best_d;
    last_i = best_i;
    have_last = true;
    out_n = r + 1;
  }
  __syncwarp();
  if (lane == 0) count[b] = out_n;
  for (int j = out_n + lane; j < k; j += 32) {
    oid[j] = -1;
    od[j] = 0.f;
  }
}

__global__ void count_zero_kernel(const float *__restrict__ v, int n, int32_t *count) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && v[i] == 0.0f) atomicAdd(count, 1);
}

__global__ void slot_reset_kernel(SlotState *st, int slots) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= slots) return;
  SlotState s{};
  s.qi = -1;
  s.phase = PH_IDLE;
  st[i] = s;
}

}  // namespace

size_t frontier_smem_bytes(const SearchCtx &c) {
  return (c.lut_smem ? frontier_smem_per_warp_lut(c.max_degree, c.req_cap, c.m)
                     : frontier_smem_per_warp(c.max_degree, c.req_cap)) *
         c.warps_per_block;
}

cudaError_t launch_frontier(SearchCtx &ctx, cudaStream_t s) {
  if (ctx.warps_per_block <= 0) ctx.warps_per_block = kWarpsPerBlock;
  if (ctx.lut_smem) {  // as many warps per block as their LUTs fit (<= 227 KB)
    const size_t per = frontier_smem_per_warp_lut(ctx.max_degree, ctx.req_cap, ctx.m);
    ctx.warps_per_block = (int)std::max<size_t>(1, std::min<size_t>(kWarpsPerBlock,
                                                                   (227 * 1024) / per));
  }
  size_t smem = frontier_smem_bytes(ctx);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(frontier_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int wpb = ctx.warps_per_block;
  int blocks = (ctx.slots + wpb - 1) / wpb;
  frontier_kernel<<<blocks, wpb * 32, smem, s>>>(ctx);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_dedup(const int32_t *greq, int total, int32_t *keys, int32_t *vals,
                         uint32_t mask, int32_t *row_count, int32_t base, int32_t *new_ids,
                         int32_t *map, cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  dedup_kernel<<<(total + 255) / 256, 256, 0, s>>>(greq, total, keys, vals, mask, row_count, base,
                                                   new_ids, map);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_qnorm(const float *q, int B, int dim, float *qn, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  qnorm_kernel<<<(B + 127) / 128, 128, 0, s>>>(q, B, dim, qn);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pending_merge(int metric, const float *pend, const int64_t *pids, int64_t np_,
                                 int dim, const float *q, const float *qn, int B, int k,
                                 int64_t *ids, float *dist, int32_t *count, float *scratch,
                                 int *bad, cudaStream_t s) {
  if (B <= 0 || np_ <= 0) return cudaSuccess;
  const int64_t pairs = (int64_t)B * np_;
  pending_dist_kernel<<<(unsigned)((pairs + 127) / 128), 128, 0, s>>>(metric, pend, np_, dim, q,
                                                                       qn, B, scratch, bad);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int warps = 4;
  const size_t smem = (size_t)warps * k * (sizeof(float) + sizeof(int64_t));
  pending_merge_kernel<<<(B + warps - 1) / warps, warps * 32, smem, s>>>(scratch, pids, np_, B, k,
                                                                        ids, dist, count);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_count_zero(const float *v, int n, int32_t *count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_zero_kernel<<<(n + 255) / 256, 256, 0, s>>>(v, n, count);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_slot_reset(SlotState *st, int slots, cudaStream_t s) {
  slot_reset_kernel<<<(slots + 255) / 256, 256, 0, s>>>(st, slots);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_lut(const float *q, const float *qn, int B, int dim, int metric,
                       const float *codebooks, int m, int padded, float *luts, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  lut_kernel<<<B, 256, padded * sizeof(float), s>>>(q, qn, dim, metric, codebooks, m, padded, luts);
  note_launch();
  return cudaGetLastError();
}

template <int M>
cudaError_t launch_adc_stream(const float *lut, const uint8_t *codes, const int64_t *ids,
                              int64_t count, float *out, cudaStream_t s) {
  const int smem = M * 256 * 4;
  cudaError_t e =
      cudaFuncSetAttribute(adc_stream_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)sms * (M <= 64 ? 3 : 2));
  adc_stream_kernel<M><<<(unsigned)blocks, 256, smem, s>>>(lut, codes, ids, count, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_adc_score(const float *lut, int m, const uint8_t *codes, const int64_t *ids,
                             int64_t count, float *out, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const bool aligned = ((uintptr_t)codes & 15) == 0;
  if (aligned && m == 32) return launch_adc_stream<32>(lut, codes, ids, count, out, s);
  if (aligned && m == 64) return launch_adc_stream<64>(lut, codes, ids, count, out, s);
  if (aligned && m == 96) return launch_adc_stream<96>(lut, codes, ids, count, out, s);
  adc_score_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(lut, m, codes, ids, count, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_distance_gather(int metric, const float *rows, int dim, const int64_t *ids,
                                   int B, int C, const float *q, const float *qn, float *out,
                                   cudaStream_t s) {
  const int64_t threads = (int64_t)B * C * 4;
  if (threads <= 0) return cudaSuccess;
  dist_gather_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(metric, rows, dim, ids, B,
                                                                       C, q, qn, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_distance_many(int metric, const float *rows, int64_t nrows, int dim,
                                 const float *q, float qn, float *out, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  int64_t threads = nrows * 4;
  dist_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(metric, rows, nrows, dim, q, qn, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace lv
