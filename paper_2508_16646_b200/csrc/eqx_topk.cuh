// eqx_topk.cuh -- the admission loop of admit_requests (engine.cpp:207-271) as rounds of a
// block-radix top-K selection over per-client key streams (included by eqx_kernels.cu).
//
// Why a round is exact.  select_next (scheduler.cpp:131-156) takes the argmin of
// (selection_key, head arrival, client_id) over the non-empty, non-skipped queues.  Under fixed
// maxima (scheduler.cpp:40-48) a client's key only depends on its own ledger, and on_admit only
// adds non-negative increments (scheduler.cpp:158-183), so along one client's FIFO the tuples
// (key, arrival) never decrease: the greedy argmin sequence is the merge of the per-client
// streams, i.e. their sorted order.  A round therefore
//   0. (rosters larger than the block) radix-selects the K clients with the smallest heads: the
//      K smallest tuples of all streams come from them;
//   1. generates those clients' next D tuples under the current maxima: the head entries are
//      gathered in parallel, the ledger chain of on_admit runs in the reference's FP64 order by
//      one thread per client, the keys of all items in parallel;
//   2. selects the K smallest tuples with an MSB-first radix select over the composite
//      (key, arrival, client_id rank, stream index) -- the stream index keeps equal tuples of one
//      client in FIFO order;
//   3. ranks them (pairwise counting) into admission order;
//   4. applies the exact loop body (reject / break / backfill skip / admit) to the ranked items:
//      slot and KV budgets are prefix sums, so the walk is a block scan up to the first item that
//      does not fit or that ends the round (an admission raising a maximum, a max holder leaving
//      the backlog, a client whose generated stream ran out); backfill skips continue one item at
//      a time.  The next round regenerates from there.
// Every round makes at least one pick (its first item is the true argmin of the current heads),
// so the result is the reference's sequence, for every policy and norm mode.  A stream also ends
// early at a negative increment or an arrival going backwards (inputs outside the engine's
// invariants), which keeps the merge argument valid.

struct TopkScratch {
  // items: slot-major runs, stream item d of slot s at x = off[s] + d (capacity `cap`)
  uint64_t* k;    // ordered key bits
  uint64_t* a;    // ordered head-arrival bits
  double* u;      // gathered: ufc increment -> ufc before the item
  double* r;      // gathered: rfc increment -> rfc before the item
  double* cn;     // gathered: VTC charge -> counter before the item
  uint8_t* fl;    // kTkValid | kFlAlone | kFlExh
  uint8_t* st;    // radix state: 0 out, 1 in play, 2 selected, 3 consumed
  uint32_t* sd;   // slot << 8 | d
  int32_t cap;
  // slots (clients whose streams a round generates)
  int32_t* sc;    // [max(C, Kcap)] client of slot s
  int32_t* snd;   // items generated for slot s
  int32_t* spos;  // FIFO position of slot s's head
  int32_t* sk0;   // its head-window index (pos - pos0)
  int32_t* off;   // first item of slot s
  int32_t* cut;   // stream length after the order / sign checks
  // ranked list
  uint64_t* gk;   // [Kcap] composites of the selected items
  uint64_t* ga;
  uint64_t* go;
  int32_t* gx;    // [Kcap] selected item
  int32_t* rank;  // [Kcap]
  int32_t* srt;   // [Kcap] items in admission order
  WinEntry* ent;  // [Kcap] their head entries
  // heads (rosters beyond Kcap): one tuple per client
  uint64_t* hk;   // [C]
  uint64_t* ha;   // [C]
  uint8_t* hst;   // [C]
  uint32_t* hist; // [256]
  uint64_t* stage;  // [warps][160] coalesced head-window words in flight
  int32_t Kcap, dsh_max;
};

enum : uint32_t { kTkValid = 16 };
constexpr uint64_t kZeroKey = 0x8000000000000000ull;  // ordered_bits(0.0)

// One event of the step's log with its payload, written by the selection itself from the item's
// head entry (the window kernel scored it with the same function the whole-queue scoring uses):
// the request id, and for an admission the PendingContribution (scheduler.hpp:131-138) --
// ufc / rfc increments, the VTC charge (scheduler.cpp:169-181) and wait_s = now - arrival
// (engine.cpp:257).
__device__ __forceinline__ void topk_event(const SelectArgs& a, int64_t ev, const WinEntry& e, int32_t kind, int32_t c,
                                           double w) {
  if (ev >= a.ev_cap) return;
  const bool adm = kind == 1;
  a.ev_row[ev] = e.row;
  a.ev_kind[ev] = kind;
  a.ev_client[ev] = c;
  a.ev_pred[ev] = e.pred;
  a.ev_ufc[ev] = adm ? e.ufc_inc : 0.0;
  a.ev_rfc[ev] = adm ? e.rfc_inc : 0.0;
  a.ev_vtc[ev] = adm ? vtc_inc(a.pol, e, w) : 0.0;
  a.ev_wait[ev] = adm ? __dsub_rn(a.now, from_ordered_bits(e.abits)) : 0.0;
  a.ev_id[ev] = e.row < 0 ? -1 : (a.id ? a.id[e.row] : a.id_base + e.row);
}

struct TopkShared {
  unsigned long long orv[3], andv[3];
  int32_t nvalid, nsel, nslot, bin, below, inbin, stop, fn, fs, fb, bad, nlist;
  int32_t passes;  // EQX_PROF: radix passes
  unsigned long long bk, ba, bo;                 // the boundary tuple (continuation rounds)
  unsigned long long wbk[32], wba[32], wbo[32];  // its per-warp minima
  int32_t wm[32];
  long long wr[32], wp[32];
  double wu[32], wv[32];
};

// Head entry j of client c: the head windows of window_kernel (L2), or scored on demand beyond
// them (deep_entry; a client-sharded step reads the gathered windows and flags underflow).
__device__ __forceinline__ WinEntry topk_entry(const SelectArgs& a, const ModelTables& M, const ClientWork& cw,
                                               int32_t c, int32_t j) {
  const int32_t k = j - cw.pos0[c];
  const int32_t depth = a.gW > 0 ? a.gW : a.W;
  if (k < depth) {
    // 40-byte entries are 8-byte aligned: five 64-bit L2 loads
    const unsigned long long* p =
        reinterpret_cast<const unsigned long long*>(a.win_g + static_cast<int64_t>(c) * depth + k);
    const uint64_t v0 = __ldcg(p), v1 = __ldcg(p + 1), v2 = __ldcg(p + 2), v3 = __ldcg(p + 3), v4 = __ldcg(p + 4);
    WinEntry e;
    e.ufc_inc = __longlong_as_double(static_cast<long long>(v0));
    e.rfc_inc = __longlong_as_double(static_cast<long long>(v1));
    e.abits = v2;
    e.in = static_cast<int32_t>(v3);
    e.pred = static_cast<int32_t>(v3 >> 32);
    e.row = static_cast<int32_t>(v4);
    e.alone = static_cast<int32_t>(v4 >> 32);
    return e;
  }
  return deep_entry(a, M, c, j, k, cw.w[c]);
}

// Radix-select views: the composite of entry x is (field 0, field 1, field 2).
struct ItemView {
  const TopkScratch& T;
  const ClientWork& cw;
  int64_t n;
  __device__ __forceinline__ uint8_t* st() const { return T.st; }
  __device__ __forceinline__ uint64_t field(int64_t x, int f) const {
    if (f == 0) return T.k[x];
    if (f == 1) return T.a[x];
    const uint32_t sd = T.sd[x];
    return (static_cast<uint64_t>(cw.order[T.sc[sd >> 8]]) << 32) | (sd & 255u);
  }
};
struct HeadView {
  const TopkScratch& T;
  const ClientWork& cw;
  int64_t n;
  __device__ __forceinline__ uint8_t* st() const { return T.hst; }
  __device__ __forceinline__ uint64_t field(int64_t x, int f) const {
    if (f == 0) return T.hk[x];
    if (f == 1) return T.ha[x];
    return static_cast<uint64_t>(cw.order[x]) << 32;
  }
};

// The in-play heads after a first pass over a large roster, compacted into shared memory: list
// entry i is client idx[i], with its own radix state lst[i].
struct HeadListView {
  const TopkScratch& T;
  const ClientWork& cw;
  const uint32_t* idx;
  uint8_t* lst;
  int64_t n;
  __device__ __forceinline__ uint8_t* st() const { return lst; }
  __device__ __forceinline__ uint64_t field(int64_t x, int f) const {
    const uint32_t c = idx[x];
    if (f == 0) return T.hk[c];
    if (f == 1) return T.ha[c];
    return static_cast<uint64_t>(cw.order[c]) << 32;
  }
};

__device__ __forceinline__ void topk_or_and_commit(uint64_t o, uint64_t an, TopkShared& X, int b) {
  const uint32_t ohi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(o >> 32));
  const uint32_t olo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(o));
  const uint32_t ahi = __reduce_and_sync(0xffffffffu, static_cast<uint32_t>(an >> 32));
  const uint32_t alo = __reduce_and_sync(0xffffffffu, static_cast<uint32_t>(an));
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&X.orv[b], (static_cast<unsigned long long>(ohi) << 32) | olo);
    atomicAnd(&X.andv[b], (static_cast<unsigned long long>(ahi) << 32) | alo);
  }
}

// OR and AND of field f over the in-play entries (st == 1), optionally below bit `lo` only.
template <class V>
__device__ __forceinline__ uint64_t topk_diff(const V& v, int f, TopkShared& X) {
  const int tid = threadIdx.x, NT = blockDim.x;
  if (tid == 0) {
    X.orv[2] = 0;
    X.andv[2] = ~0ull;
  }
  __syncthreads();
  uint64_t o = 0, an = ~0ull;
  for (int64_t x = tid; x < v.n; x += NT) {
    if (v.st()[x] != 1) continue;
    const uint64_t w = v.field(x, f);
    o |= w;
    an &= w;
  }
  topk_or_and_commit(o, an, X, 2);
  __syncthreads();
  const uint64_t d = X.orv[2] ^ X.andv[2];
  __syncthreads();  // X.orv[2] / X.andv[2] are reset by the next call
  return d;
}

// Warp 0: the histogram bin where the running count reaches need, into X.bin / below / inbin.
__device__ __forceinline__ void topk_find_bin(const uint32_t* hist, int32_t need, TopkShared& X) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 32) {  // the bin where the running count reaches need
    uint32_t h[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      h[i] = hist[lane * 8 + i];
      sum += h[i];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - sum;
    const unsigned hit =
        __ballot_sync(0xffffffffu, excl < static_cast<uint32_t>(need) && static_cast<uint32_t>(need) <= incl);
    if (lane == __ffs(hit) - 1) {
      uint32_t cum = excl;
      int b = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (cum + h[i] >= static_cast<uint32_t>(need)) {
          b = i;
          break;
        }
        cum += h[i];
      }
      X.bin = lane * 8 + b;
      X.below = static_cast<int32_t>(cum);
      X.inbin = static_cast<int32_t>(h[b]);
    }
  }
}

// MSB-first radix select of the `need` smallest composites among the in-play entries (st == 1):
// they end with st == 2, the others with st == 0.  Composites are unique (client rank, stream
// index), so exactly `need` are selected.  Each pass histograms the next (up to) 8 bits below
// the leading bits every in-play entry shares: the pass that keeps a bin also reduces the OR /
// AND of that bin's remaining bits, so runs of common bits (and whole common fields, e.g. the
// zero keys of a cold ledger) cost no pass.
template <class V>
__device__ void topk_radix_select(const V& v, int32_t need, uint32_t* hist, TopkShared& X) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
  uint8_t* st = v.st();
  const int64_t n = v.n;
  int f = 0;
  uint64_t diff = topk_diff(v, 0, X);
  int hi = diff ? 63 - __clzll(static_cast<long long>(diff)) : -1;
  int par = 0;
#pragma unroll 1
  for (;;) {
    while (hi < 0) {  // every in-play entry agrees on the rest of this field
      if (++f == 3) return;
      diff = topk_diff(v, f, X);
      hi = diff ? 63 - __clzll(static_cast<long long>(diff)) : -1;
    }
    const int lo = hi >= 7 ? hi - 7 : 0;
    const uint32_t mask = (1u << (hi - lo + 1)) - 1u;
#ifdef EQX_PROF
    if (tid == 0) ++X.passes;
#endif
    for (int i = tid; i < 256; i += NT) hist[i] = 0;
    if (tid == 0) {
      X.orv[par] = 0;
      X.andv[par] = ~0ull;
    }
    __syncthreads();
    // warp-uniform trip count so the peer-mask ballots see all 32 lanes
    for (int64_t base = tid - lane; base < n; base += NT) {
      const int64_t x = base + lane;
      uint32_t dg = 256;
      if (x < n && st[x] == 1) dg = static_cast<uint32_t>(v.field(x, f) >> lo) & mask;
      if (!__ballot_sync(0xffffffffu, dg != 256)) continue;
      const unsigned m = peer_mask(dg, 9);
      if (dg != 256 && lane == __ffs(m) - 1) atomicAdd(&hist[dg], static_cast<uint32_t>(__popc(m)));
    }
    __syncthreads();
    topk_find_bin(hist, need, X);
    __syncthreads();
    const uint32_t bin = static_cast<uint32_t>(X.bin);
    need -= X.below;
    const bool all_in = X.inbin == need;
    const uint64_t low = lo > 0 ? (1ull << lo) - 1 : 0;
    uint64_t o = 0, an = ~0ull;
    for (int64_t x = tid; x < n; x += NT) {
      if (st[x] != 1) continue;
      const uint64_t w = v.field(x, f);
      const uint32_t dg = static_cast<uint32_t>(w >> lo) & mask;
      if (dg < bin || (dg == bin && all_in)) {
        st[x] = 2;
      } else if (dg > bin) {
        st[x] = 0;
      } else {
        o |= w & low;
        an &= w | ~low;
      }
    }
    if (all_in) {
      __syncthreads();
      return;
    }
    topk_or_and_commit(o, an, X, par);
    __syncthreads();
    diff = (X.orv[par] ^ X.andv[par]) & low;
    hi = diff ? 63 - __clzll(static_cast<long long>(diff)) : -1;
    par ^= 1;
  }
}

// Block-wide exclusive scan of (count, tokens, prefill) over list positions (one per thread).
__device__ __forceinline__ void topk_scan(int32_t m, long long rv, long long pv, int32_t& mx, long long& rx,
                                          long long& px, TopkShared& X) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t mi = m;
  long long ri = rv, pi = pv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t a = __shfl_up_sync(0xffffffffu, mi, o);
    const long long b = __shfl_up_sync(0xffffffffu, ri, o), c = __shfl_up_sync(0xffffffffu, pi, o);
    if (lane >= o) {
      mi += a;
      ri += b;
      pi += c;
    }
  }
  if (lane == 31) {
    X.wm[warp] = mi;
    X.wr[warp] = ri;
    X.wp[warp] = pi;
  }
  __syncthreads();
  int32_t mb = 0;
  long long rb = 0, pb = 0;
  for (int w = 0; w < warp; ++w) {
    mb += X.wm[w];
    rb += X.wr[w];
    pb += X.wp[w];
  }
  mx = mb + mi - m;
  rx = rb + ri - rv;
  px = pb + pi - pv;
}

// topk_scan plus the running maxima of two doubles: exclusive (before this position) and
// inclusive maxima of (cu, cr) over list positions (-inf where an item contributes nothing).
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ void topk_scan_mx(int32_t m, long long rv, long long pv, double cu, double cr, int32_t& mx,
                                             long long& rx, long long& px, double& xu, double& xr, double& iu_out,
                                             double& ir_out, TopkShared& X) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t mi = m;
  long long ri = rv, pi = pv;
  double iu = cu, ir = cr;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t a = __shfl_up_sync(0xffffffffu, mi, o);
    const long long b = __shfl_up_sync(0xffffffffu, ri, o), c = __shfl_up_sync(0xffffffffu, pi, o);
    const double du = __shfl_up_sync(0xffffffffu, iu, o), dr = __shfl_up_sync(0xffffffffu, ir, o);
    if (lane >= o) {
      mi += a;
      ri += b;
      pi += c;
      iu = dmax(iu, du);
      ir = dmax(ir, dr);
    }
  }
  double pu = __shfl_up_sync(0xffffffffu, iu, 1), pr = __shfl_up_sync(0xffffffffu, ir, 1);
  if (lane == 0) pu = pr = -INFINITY;
  if (lane == 31) {
    X.wm[warp] = mi;
    X.wr[warp] = ri;
    X.wp[warp] = pi;
    X.wu[warp] = iu;
    X.wv[warp] = ir;
  }
  __syncthreads();
  int32_t mb = 0;
  long long rb = 0, pb = 0;
  double bu = -INFINITY, br = -INFINITY;
  for (int w = 0; w < warp; ++w) {
    mb += X.wm[w];
    rb += X.wr[w];
    pb += X.wp[w];
    bu = dmax(bu, X.wu[w]);
    br = dmax(br, X.wv[w]);
  }
  mx = mb + mi - m;
  rx = rb + ri - rv;
  px = pb + pi - pv;
  xu = dmax(bu, pu);
  xr = dmax(br, pr);
  iu_out = dmax(bu, iu);
  ir_out = dmax(br, ir);
}

// tuple order of select_next: key, head arrival, client_id rank (and stream index for items)
__device__ __forceinline__ bool tuple_lt(uint64_t k1, uint64_t a1, uint64_t o1, uint64_t k2, uint64_t a2, uint64_t o2) {
  return k1 < k2 || (k1 == k2 && (a1 < a2 || (a1 == a2 && o1 < o2)));
}

// The boundary of a continuation: the smallest head tuple (key under maxima mu / mr, head
// arrival, client rank) among the candidate clients outside the slots, into X.bk / ba / bo.
// Whole CTA; the caller synchronises before reading X.b*.
__device__ __noinline__ void topk_boundary(const Policy& P, const ClientWork& cw, const TopkScratch& T, TopkShared& X,
                                           int32_t C, double mu, double mr) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
  uint64_t bk = ~0ull, ba = ~0ull, bo = ~0ull;
  for (int32_t c = tid; c < C; c += NT) {
    if (T.hst[c] == 2 || cw.pos[c] >= cw.end[c] || (cw.flags[c] & kSkipped)) continue;
    const uint64_t k = ordered_bits(hf_key(P, cw.ufc[c], cw.rfc[c], mu, mr, cw.cnt[c]));
    const uint64_t av = T.ha[c], o = static_cast<uint64_t>(cw.order[c]) << 32;
    if (tuple_lt(k, av, o, bk, ba, bo)) {
      bk = k;
      ba = av;
      bo = o;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o), a2 = __shfl_xor_sync(0xffffffffu, ba, o),
                   o2 = __shfl_xor_sync(0xffffffffu, bo, o);
    if (tuple_lt(k2, a2, o2, bk, ba, bo)) {
      bk = k2;
      ba = a2;
      bo = o2;
    }
  }
  if (lane == 0) {
    X.wbk[tid >> 5] = bk;
    X.wba[tid >> 5] = ba;
    X.wbo[tid >> 5] = bo;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (NT >> 5); ++w) {
      const uint64_t k2 = X.wbk[w], a2 = X.wba[w], o2 = X.wbo[w];
      if (tuple_lt(k2, a2, o2, bk, ba, bo)) {
        bk = k2;
        ba = a2;
        bo = o2;
      }
    }
    X.bk = bk;
    X.ba = ba;
    X.bo = bo;
  }
}

// The K smallest head tuples of a large roster (entries with T.hst == 1; X.orv / andv hold each
// field's OR / AND over them): they end with hst == 2, the others with 0.  The first radix pass
// runs over the whole roster in global scratch and compacts the entries left in play (the bin
// that holds the K-th tuple) into shared memory; the remaining passes run over that list.
__device__ __forceinline__ void topk_head_select(const TopkScratch& T, const ClientWork& cw, int32_t C, int32_t K,
                                                 TopkShared& X) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
  int f = 0;
  uint64_t diff = X.orv[0] ^ X.andv[0];
  if (!diff) {
    f = 1;
    diff = X.orv[1] ^ X.andv[1];
  }
  if (!diff) {
    f = 2;
    diff = X.orv[2] ^ X.andv[2];  // client ranks are distinct: nonzero with two candidates
  }
  const int hi = 63 - __clzll(static_cast<long long>(diff));
  const int lo = hi >= 7 ? hi - 7 : 0;
  const uint32_t mask = (1u << (hi - lo + 1)) - 1u;
  const HeadView hv{T, cw, C};
  uint32_t* hist = T.hist;
  for (int i = tid; i < 256; i += NT) hist[i] = 0;
  if (tid == 0) X.nlist = 0;
  __syncthreads();
  // the scans load kB entries' state and field together (one L2 round trip per batch; the field
  // of a non-candidate is a stale but readable word)
  constexpr int kB = 4;
  for (int64_t base = tid - lane; base < C; base += kB * NT) {
    uint32_t dg[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int64_t x = base + lane + j * NT;
      const bool in = x < C;
      const uint8_t h = in ? T.hst[x] : 0;
      const uint64_t w = in ? hv.field(x, f) : 0;
      dg[j] = h == 1 ? static_cast<uint32_t>(w >> lo) & mask : 256u;
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      if (!__ballot_sync(0xffffffffu, dg[j] != 256)) continue;
      const unsigned m = peer_mask(dg[j], 9);
      if (dg[j] != 256 && lane == __ffs(m) - 1) atomicAdd(&hist[dg[j]], static_cast<uint32_t>(__popc(m)));
    }
  }
  __syncthreads();
  topk_find_bin(hist, K, X);
  __syncthreads();
  const uint32_t bin = static_cast<uint32_t>(X.bin);
  const int32_t need = K - X.below;
  const bool all_in = X.inbin == need;
  uint32_t* idx = T.sd;  // item arrays are free before a round's streams are generated
  uint8_t* lst = T.st;
  for (int64_t base = tid - lane; base < C; base += kB * NT) {
    uint32_t dg[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int64_t x = base + lane + j * NT;
      const bool in = x < C;
      const uint8_t h = in ? T.hst[x] : 0;
      const uint64_t w = in ? hv.field(x, f) : 0;
      dg[j] = h == 1 ? static_cast<uint32_t>(w >> lo) & mask : 256u;
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int64_t x = base + lane + j * NT;
      const bool keep = dg[j] == bin && !all_in;
      if (dg[j] != 256 && !keep) T.hst[x] = dg[j] < bin || dg[j] == bin ? 2 : 0;
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (!km) continue;
      int32_t b0 = 0;
      if (lane == __ffs(km) - 1) b0 = atomicAdd(&X.nlist, __popc(km));
      b0 = __shfl_sync(0xffffffffu, b0, __ffs(km) - 1);
      const int32_t i = b0 + __popc(km & ((1u << lane) - 1u));
      if (keep && i < T.cap) {
        idx[i] = static_cast<uint32_t>(x);
        lst[i] = 1;
      }
    }
  }
  __syncthreads();
  if (all_in) return;
  const int32_t nl = X.nlist;
  if (nl > T.cap) {  // the bin overflows the list: the remaining passes over the whole roster
    topk_radix_select(hv, need, hist, X);
    return;
  }
  topk_radix_select(HeadListView{T, cw, idx, lst, nl}, need, hist, X);
  for (int32_t i = tid; i < nl; i += NT) T.hst[idx[i]] = lst[i];
  __syncthreads();
}

// The rounds (see the file comment).  Runs on the whole CTA after select_body's prologue.
template <bool kHugeRoster>
__device__ __forceinline__ void topk_select(const SelectArgs& a, const ModelTables& M, const ClientWork& cw, SelShared& S,
                            const TopkScratch& T) {
  __shared__ TopkShared X;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
  const int32_t C = a.C;
  const Policy P = a.pol;
  const bool maxmode = P.kind == kEquinox && P.norm_mode == 0;
  const int64_t tmax = a.tmax;
  const bool big = C > T.Kcap;  // rosters beyond one slot per thread: pre-select the K best heads
  if (!big)
    for (int32_t s = tid; s < C; s += NT) T.sc[s] = s;
  // K of a round: the free slots (+ a margin for rejections), grown while lists run out
  const int32_t want = P.backfill ? T.Kcap : max(32, min(T.Kcap, P.max_batch - S.members + 8));
  int32_t K = min(want, a.tk_k0);
#ifdef EQX_PROF
  unsigned long long n_total_items = 0;
  unsigned long long rounds = 0, cy[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64(), t1, tk_t1;
#define TK_STAMP(i) \
  t1 = clock64();   \
  cy[i] += t1 - t0; \
  t0 = t1;
#else
#define TK_STAMP(i)
#endif
  __syncthreads();
  // A round either regenerates the key streams (regen) or continues over the items generated
  // earlier: those stay valid -- a client's ledger chain depends only on its own admissions --
  // and only their keys, which move with the maxima, are recomputed.  A continuation stops at
  // the smallest head of a client outside the slot set (the boundary B), at a stream that ran
  // out, or when no item is left; the next round then regenerates.
  // every ledger non-negative (then so is every generated item's: streams end at a negative
  // increment) -- a condition of the zero-key fast path below
  bool nonneg = true;
  for (int32_t c = tid; c < C; c += NT) nonneg &= cw.ufc[c] >= 0.0 && cw.rfc[c] >= 0.0;
  nonneg = __syncthreads_and(nonneg) != 0;
  bool regen = true;      // block-uniform
  bool all_slots = true;  // the slots hold every candidate client (no boundary)
  int64_t n = 0;          // items of the current streams
  int32_t nslot = 0;
  for (;;) {
    const double mu = S.max_u, mr = S.max_r;
    if (tid == 0) {
      X.nvalid = 0;
      X.nsel = 0;
      X.nslot = 0;
      X.stop = 0;
      X.fn = 0x7fffffff;
      X.fs = 0x7fffffff;
      X.fb = 0x7fffffff;
    }
    __syncthreads();
    if (regen) {
    // ---- 0. slots: every client, or the K clients with the smallest heads ----
    nslot = C;
    all_slots = true;
    if (big) {
      // Heads in global scratch (huge rosters): every candidate's head tuple with the OR / AND of
      // each field, then topk_head_select (first pass over the roster, the rest over a shared-
      // memory list).  Heads in shared memory: the tuples, then the generic radix select.
      constexpr bool gheads = kHugeRoster;  // == (a.tk_heads != nullptr)
      int32_t nc = 0;
      uint64_t o0 = 0, a0 = ~0ull, o1 = 0, a1 = ~0ull, o2 = 0, a2 = ~0ull;
      if (gheads) {
        if (tid == 0)
          for (int i = 0; i < 3; ++i) {
            X.orv[i] = 0;
            X.andv[i] = ~0ull;
          }
        const int32_t depth = a.gW > 0 ? a.gW : a.W;
        for (int32_t c0 = tid; c0 < C; c0 += 2 * NT) {  // two clients' loads in flight together
          int32_t pos[2], k0[2];
          bool cnd[2];
          double u[2], r[2], n[2];
          uint32_t ord[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int32_t c = min(c0 + j * NT, C - 1);
            pos[j] = cw.pos[c];
            k0[j] = pos[j] - cw.pos0[c];
            cnd[j] = c0 + j * NT < C && pos[j] < cw.end[c] && !(cw.flags[c] & kSkipped);
            u[j] = cw.ufc[c];
            r[j] = cw.rfc[c];
            n[j] = cw.cnt[c];
            ord[j] = cw.order[c];
          }
          uint64_t hab[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int32_t c = min(c0 + j * NT, C - 1);
            hab[j] = cnd[j] && k0[j] < depth
                         ? __ldcg(reinterpret_cast<const unsigned long long*>(
                                      a.win_g + static_cast<int64_t>(c) * depth + k0[j]) + 2)
                         : 0;
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int32_t c = c0 + j * NT;
            if (c >= C) continue;
            const bool cand = cnd[j];
            if (cand) {
              const uint64_t hav = k0[j] < depth ? hab[j] : topk_entry(a, M, cw, c, pos[j]).abits;
              const uint64_t hkv = ordered_bits(hf_key(P, u[j], r[j], mu, mr, n[j]));
              const uint64_t hov = static_cast<uint64_t>(ord[j]) << 32;
              T.ha[c] = hav;
              T.hk[c] = hkv;
              o0 |= hkv;
              a0 &= hkv;
              o1 |= hav;
              a1 &= hav;
              o2 |= hov;
              a2 &= hov;
            }
            T.hst[c] = cand ? 1 : 0;
            nc += cand;
          }
        }
      } else {
        for (int32_t c = tid; c < C; c += NT) {
          const bool cand = cw.pos[c] < cw.end[c] && !(cw.flags[c] & kSkipped);
          if (cand) {
            T.ha[c] = topk_entry(a, M, cw, c, cw.pos[c]).abits;
            T.hk[c] = ordered_bits(hf_key(P, cw.ufc[c], cw.rfc[c], mu, mr, cw.cnt[c]));
          }
          T.hst[c] = cand ? 1 : 0;
          nc += cand;
        }
      }
      nc = __reduce_add_sync(0xffffffffu, nc);
      if ((tid & 31) == 0 && nc) atomicAdd(&X.nvalid, nc);
      __syncthreads();  // X.orv / andv reset before the commits
      if constexpr (gheads) {
        topk_or_and_commit(o0, a0, X, 0);
        topk_or_and_commit(o1, a1, X, 1);
        topk_or_and_commit(o2, a2, X, 2);
        __syncthreads();
      }
      const int32_t ncand = X.nvalid;
      if (ncand == 0) break;  // no candidates (engine.cpp:217)
#ifdef EQX_PROF
      if (tid == 0) X.passes = 0;
      tk_t1 = clock64();
      tk[0] += tk_t1 - t0;
#endif
      if (ncand > K) {
        if (gheads) topk_head_select(T, cw, C, K, X);
        else topk_radix_select(HeadView{T, cw, C}, K, T.hist, X);
      }
      all_slots = ncand <= K;
#ifdef EQX_PROF
      tk[1] += clock64() - tk_t1;
      tk[2] += X.passes;
#endif
      for (int32_t c = tid; c < C; c += NT)
        if (T.hst[c] == (ncand > K ? 2 : 1)) T.sc[atomicAdd(&X.nslot, 1)] = c;
      __syncthreads();
      nslot = X.nslot;
      if (tid == 0) X.nvalid = 0;
    }
    TK_STAMP(0)
    // ---- 1. key streams ----
    // 1a. per slot: FIFO position, window index, head tuple, longest useful stream
    for (int32_t s = tid; s < nslot; s += NT) {
      const int32_t c = T.sc[s], pos = cw.pos[c], end = cw.end[c], k0 = pos - cw.pos0[c];
      int32_t lim = 0;
      uint64_t hkv = ~0ull, hav = ~0ull, hov = ~0ull;
      if (pos < end && !(cw.flags[c] & kSkipped)) {
        lim = min(64, end - pos);
        if (a.gW > 0) lim = min(lim, max(a.gW - k0, 1));  // stay inside the gathered windows
        hkv = big ? T.hk[c] : ordered_bits(hf_key(P, cw.ufc[c], cw.rfc[c], mu, mr, cw.cnt[c]));
        hav = big ? T.ha[c] : topk_entry(a, M, cw, c, pos).abits;
        hov = static_cast<uint64_t>(cw.order[c]) << 32;
      }
      T.spos[s] = pos;
      T.sk0[s] = k0;
      T.snd[s] = lim;
      T.gk[s] = hkv;
      T.ga[s] = hav;
      T.go[s] = hov;
      T.rank[s] = 0;
    }
    __syncthreads();
    // 1b. depth budget: the client with the r-th smallest head gets about K / (r + 1) items
    //     (a client's items sit below the K-th smallest tuple only while its key climbs past
    //     the others'), large slot sets one to a few each
    const bool harmonic = nslot <= 128;
    if (harmonic) {
      const int parts = max(1, NT / nslot);
      if (tid < nslot * parts) {
        const int32_t i = tid % nslot, part = tid / nslot;
        const uint64_t k = T.gk[i], av = T.ga[i], o = T.go[i];
        int32_t rk = 0;
        for (int32_t j = part; j < nslot; j += parts) {
          const uint64_t kj = T.gk[j], aj = T.ga[j], oj = T.go[j];
          rk += (kj < k) | ((kj == k) & ((aj < av) | ((aj == av) & (oj < o))));
        }
        if (rk) atomicAdd(&T.rank[i], rk);
      }
      __syncthreads();
    }
    {
      const int32_t room = T.cap - nslot;  // one item per slot, the rest shared out
      int32_t extra = 0;
      if (tid < nslot && T.snd[tid] > 0) {
        const int32_t w = harmonic ? (K + T.rank[tid]) / (T.rank[tid] + 1) : max(1, room / max(nslot, 1));
        extra = min(w, T.snd[tid]) - 1;
      }
      int32_t ex;
      long long e1, e2;
      topk_scan(extra, 0, 0, ex, e1, e2, X);
      if (tid < nslot) {
        const int32_t take = max(0, min(extra, room - ex));
        const int32_t o = tid + min(ex, room);
        T.off[tid] = o;
        const int32_t len = T.snd[tid] > 0 ? 1 + take : 0;
        T.snd[tid] = len;
        T.cut[tid] = len;
        for (int32_t d = 0; d < max(len, 1); ++d) T.sd[o + d] = (static_cast<uint32_t>(tid) << 8) | d;
        if (tid == nslot - 1) X.nvalid = o + max(len, 1);  // items this round
      }
      __syncthreads();
      n = X.nvalid;
      __syncthreads();
      if (tid == 0) X.nvalid = 0;
#ifdef EQX_PROF
      n_total_items += n;
#endif
    }
    {  // 1c. head entries: a warp moves 32 consecutive items (mostly one client's contiguous
       //     window run) as 160 coalesced 64-bit words through shared memory
      const int32_t depth = a.gW > 0 ? a.gW : a.W;
      const int lane = tid & 31;
      uint64_t* stg = T.stage + (tid >> 5) * 160;
      for (int64_t base = tid - lane; base < n; base += NT) {
        const int64_t li = base + lane;
        const uint32_t sdv = li < n ? T.sd[li] : 0u;
        const int32_t s = static_cast<int32_t>(sdv >> 8), d = static_cast<int32_t>(sdv & 255u);
        const bool valid = li < n && d < T.snd[s];
        int32_t c = 0, k = 0;
        unsigned long long p = 0;
        if (valid) {
          c = T.sc[s];
          k = T.sk0[s] + d;
          if (k < depth) p = reinterpret_cast<unsigned long long>(a.win_g + static_cast<int64_t>(c) * depth + k);
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const int w = j * 32 + lane, e = w / 5;
          const unsigned long long pe = __shfl_sync(0xffffffffu, p, e);
          if (pe) stg[w] = __ldcg(reinterpret_cast<const unsigned long long*>(pe) + (w - 5 * e));
        }
        __syncwarp();
        if (li < n) {
          uint8_t f = 0;
          if (valid) {
            WinEntry e;
            if (p) {
              e.ufc_inc = __longlong_as_double(static_cast<long long>(stg[5 * lane]));
              e.rfc_inc = __longlong_as_double(static_cast<long long>(stg[5 * lane + 1]));
              e.abits = stg[5 * lane + 2];
              const uint64_t ip = stg[5 * lane + 3];
              e.in = static_cast<int32_t>(ip);
              e.pred = static_cast<int32_t>(ip >> 32);
              e.alone = static_cast<int32_t>(stg[5 * lane + 4] >> 32);
            } else {
              e = deep_entry(a, M, c, T.spos[s] + d, k, cw.w[c]);  // beyond the head window
            }
            T.a[li] = e.abits;
            T.u[li] = e.ufc_inc;
            T.r[li] = e.rfc_inc;
            T.cn[li] = vtc_inc(P, e, cw.w[c]);
            f = kTkValid | (e.alone ? kFlAlone : 0);
          }
          T.fl[li] = f;
          T.st[li] = 0;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // 1d. stream ends: an arrival going backwards (the stream stops before it) or a negative
    //     increment (the stream stops after it)
    for (int64_t x = tid; x < n; x += NT) {
      const uint8_t f = T.fl[x];
      if (!(f & kTkValid)) continue;
      const uint32_t sdv = T.sd[x];
      const int32_t s = static_cast<int32_t>(sdv >> 8), d = static_cast<int32_t>(sdv & 255u);
      if (d > 0 && T.a[x] < T.a[x - 1]) atomicMin(&T.cut[s], d);
      if ((f & kFlAlone) && d + 1 < T.snd[s] &&
          (!(T.u[x] >= 0.0) || !(T.r[x] >= 0.0) || (P.kind == kVtc && !(T.cn[x] >= 0.0))))
        atomicMin(&T.cut[s], d + 1);
    }
    __syncthreads();
    TK_STAMP(1)
    // 1e. ledger chains (on_admit's adds in FIFO order): a warp per slot, 32 items at a time in
    //     the lanes; the increments are broadcast by shuffles, so only the adds are serial
    {
      const int lane = tid & 31, nw = NT >> 5;
      for (int32_t s = tid >> 5; s < nslot; s += nw) {
        const int32_t c = T.sc[s], pos = T.spos[s], end = cw.end[c], x0 = T.off[s];
        const int32_t nd = T.cut[s];
        double u = cw.ufc[c], r = cw.rfc[c], cn = cw.cnt[c];
        for (int32_t base = 0; base < nd; base += 32) {
          const int32_t d = base + lane, x = x0 + d;
          const bool in = d < nd;
          uint8_t f = in ? T.fl[x] : 0;
          const double iu = in ? T.u[x] : 0.0, ir = in ? T.r[x] : 0.0, ic = in ? T.cn[x] : 0.0;
          double ub = 0.0, rb = 0.0, cb = 0.0;
          const int32_t m = min(32, nd - base);
          if (P.kind == kVtc) {
#pragma unroll 4
            for (int32_t j = 0; j < m; ++j) {
              if (lane == j) {
                ub = u;
                rb = r;
                cb = cn;
              }
              const bool al = __shfl_sync(0xffffffffu, f, j) & kFlAlone;
              const double iuj = __shfl_sync(0xffffffffu, iu, j), irj = __shfl_sync(0xffffffffu, ir, j),
                           icj = __shfl_sync(0xffffffffu, ic, j);
              const double nu = __dadd_rn(u, iuj), nr = __dadd_rn(r, irj), nc = __dadd_rn(cn, icj);
              u = al ? nu : u;
              r = al ? nr : r;
              cn = al ? nc : cn;
            }
          } else {
#pragma unroll 4
            for (int32_t j = 0; j < m; ++j) {
              if (lane == j) {
                ub = u;
                rb = r;
              }
              const bool al = __shfl_sync(0xffffffffu, f, j) & kFlAlone;
              const double iuj = __shfl_sync(0xffffffffu, iu, j), irj = __shfl_sync(0xffffffffu, ir, j);
              const double nu = __dadd_rn(u, iuj), nr = __dadd_rn(r, irj);
              u = al ? nu : u;
              r = al ? nr : r;
            }
            cb = cn;
          }
          if (in) {
            T.u[x] = ub;
            T.r[x] = rb;
            T.cn[x] = cb;
            if (d + 1 == nd && pos + nd < end) f |= kFlExh;  // later items were not generated
            T.fl[x] = f;
          }
        }
        for (int32_t d = nd + lane; d < T.snd[s]; d += 32) T.fl[x0 + d] = 0;
        __syncwarp();
        if (lane == 0) T.snd[s] = nd;
      }
    }
    __syncthreads();
    TK_STAMP(2)
    }  // regen
    // ---- keys of the items still in play (unconsumed, client not skipped) under the maxima ----
    {
      int32_t nv = 0;
      for (int64_t x = tid; x < n; x += NT) {
        const uint8_t st = T.st[x];
        bool v = (T.fl[x] & kTkValid) && st != 3;
        if (v && P.backfill) v = !(cw.flags[T.sc[T.sd[x] >> 8]] & kSkipped);
        if (v) T.k[x] = ordered_bits(hf_key(P, T.u[x], T.r[x], mu, mr, T.cn[x]));
        T.st[x] = v ? 1 : (st == 3 ? 3 : 0);
        nv += v;
      }
      nv = __reduce_add_sync(0xffffffffu, nv);
      if ((tid & 31) == 0 && nv) atomicAdd(&X.nvalid, nv);
    }
    // ---- continuation with clients outside the slots: their smallest head is the boundary ----
    const bool bounded = !regen && !all_slots;
    if (bounded) topk_boundary(P, cw, T, X, C, mu, mr);
    __syncthreads();
    const int32_t nvalid = X.nvalid;
    TK_STAMP(3)
    if (nvalid == 0) {  // no candidates (engine.cpp:217) -- or none left in the generated streams
      if (regen) break;
      regen = true;
      __syncthreads();
      continue;
    }
    // ---- 2. the K smallest tuples ----
    const int32_t ks = min(nvalid, K);
    const ItemView iv{T, cw, n};
    if (ks < nvalid) {
#ifdef EQX_PROF
      if (tid == 0) X.passes = 0;
#endif
      topk_radix_select(iv, ks, T.hist, X);
#ifdef EQX_PROF
      tk[3] += X.passes;
      tk[4] += 1;
#endif
    } else {
      for (int64_t x = tid; x < n; x += NT)
        if (T.st[x] == 1) T.st[x] = 2;
      __syncthreads();
    }
    TK_STAMP(4)
    // ---- 3. admission order: gather, rank by pairwise counting ----
    for (int64_t x = tid; x < n; x += NT) {
      if (T.st[x] != 2) continue;
      const int32_t i = atomicAdd(&X.nsel, 1);
      T.gx[i] = static_cast<int32_t>(x);
      T.gk[i] = T.k[x];
      T.ga[i] = T.a[x];
      T.go[i] = iv.field(x, 2);
      T.rank[i] = 0;
    }
    __syncthreads();
    const int32_t ns = X.nsel;
    {
      const int parts = max(1, NT / ns);
      if (tid < ns * parts) {
        const int32_t i = tid % ns, part = tid / ns;
        const uint64_t k = T.gk[i], av = T.ga[i], o = T.go[i];
        int32_t rk = 0;
        for (int32_t j = part; j < ns; j += parts) {
          const uint64_t kj = T.gk[j], aj = T.ga[j], oj = T.go[j];
          rk += (kj < k) | ((kj == k) & ((aj < av) | ((aj == av) & (oj < o))));
        }
        if (rk) atomicAdd(&T.rank[i], rk);
      }
      __syncthreads();
      const uint64_t bk = X.bk, ba = X.ba, bo = X.bo;
      for (int32_t i = tid; i < ns; i += NT) {
        const int32_t x = T.gx[i], rk = T.rank[i];
        T.srt[rk] = x;
        const uint32_t sdv = T.sd[x];
        const int32_t s = static_cast<int32_t>(sdv >> 8);
        T.ent[rk] = topk_entry(a, M, cw, T.sc[s], T.spos[s] + static_cast<int32_t>(sdv & 255u));
        if (bounded) {  // items past the boundary wait for a regenerating round
          const uint64_t k = T.gk[i], av = T.ga[i], o = T.go[i];
          if (!(k < bk || (k == bk && (av < ba || (av == ba && o < bo))))) atomicMin(&X.fb, rk);
        }
      }
      __syncthreads();
    }
    TK_STAMP(5)
    // ---- 4. the loop body over the ranked items (engine.cpp:216-268) ----
    // The ranked list is walked in segments: a segment ends at the first item that does not
    // fit or that ends the sorted order's validity (an admission raising a maximum, a max
    // holder leaving the backlog, the last generated item of a stream).  After a moved maximum
    // the rest of the list stays usable when, under the new maxima, it is still sorted and its
    // last item is still below every other unconsumed item and the boundary: the keys are
    // recomputed and checked in place, and the next segment continues the walk.
    const int32_t nse = min(ns, X.fb);  // the ranked items below the boundary
    int32_t base = 0;                   // first ranked position of the segment
    for (;;) {
      // 4a. block scan: slot / KV budgets as prefix sums, up to the first item that does not
      //     fit or ends the segment
      const int32_t members0 = S.members;
      const int64_t reserved0 = S.reserved;
      const double smu = S.max_u, smr = S.max_r;
      const int32_t q = base + tid;  // this thread's ranked position
      // zero-key regime: the rest of the list keys 0 under positive maxima and non-negative
      // ledgers -- rising maxima leave its order and its place below every other item as they
      // are, so the walk goes on through them (their running maxima are a prefix max)
      const bool zfast = maxmode && nonneg && smu > 0.0 && smr > 0.0 && T.k[T.srt[base]] == kZeroKey &&
                         T.k[T.srt[nse - 1]] == kZeroKey;
      int32_t m = 0;
      long long rv = 0, pv = 0;
      bool alone = false, last = false;
      double ub = 0.0, rb = 0.0, cu = -INFINITY, cr = -INFINITY;
      uint8_t f = 0;
      if (q < nse) {
        const int32_t x = T.srt[q];
        const int32_t s = static_cast<int32_t>(T.sd[x] >> 8), c = T.sc[s], d = static_cast<int32_t>(T.sd[x] & 255u);
        const WinEntry& e = T.ent[q];
        f = T.fl[x];
        last = T.spos[s] + d + 1 == cw.end[c];
        alone = e.alone;
        ub = T.u[x];
        rb = T.r[x];
        if (alone && !last) {  // an admission that keeps its client backlogged: a max candidate
          cu = __dadd_rn(ub, e.ufc_inc);
          cr = __dadd_rn(rb, e.rfc_inc);
        }
        m = alone ? 1 : 0;
        rv = alone ? static_cast<long long>(e.in) + e.pred : 0;
        pv = alone ? e.in : 0;
      }
      int32_t mx;
      long long rx, px;
      double xu = -INFINITY, xr = -INFINITY, iu = cu, ir = cr;
      // running maxima only in the zero-key regime; otherwise the segment ends at its first
      // raise, so the segment-start maxima hold up to it (and its own values raise them)
      if (zfast) topk_scan_mx(m, rv, pv, cu, cr, mx, rx, px, xu, xr, iu, ir, X);
      else topk_scan(m, rv, pv, mx, rx, px, X);
      bool flag = false;
      if (q < nse) {
        // the maxima-dependent outcomes under the maxima in force at this position: a max
        // holder leaving the backlog with its last request, an admission raising a maximum
        const double cmu = dmax(smu, xu), cmr = dmax(smr, xr);
        const bool holder = maxmode && last && (ub == cmu || rb == cmr);
        const bool raise = maxmode && alone && !last && (cmu < cu || cmr < cr);
        flag = last ? holder : ((f & kFlExh) || (raise && !zfast));
      }
      if (q < nse) {
        const bool nofit = alone && !((members0 + mx + 1 <= P.max_batch) && (reserved0 + rx + rv <= tmax));
        if (nofit) atomicMin(&X.fn, q);
        if (flag) atomicMin(&X.fs, q);
      }
      __syncthreads();
      const int32_t fn = X.fn, fs = X.fs;
      const int32_t cend = fn <= fs ? min(fn, nse) : fs + 1;  // positions [base, cend) are consumed
      // 4b. commit: events, admissions, per-client ledgers after the client's last consumed item
      if (q < cend) {
        const int32_t x = T.srt[q];
        const int32_t c = T.sc[T.sd[x] >> 8];
        topk_event(a, S.n_ev + tid, T.ent[q], alone ? 1 : 2, c, cw.w[c]);
        if (alone) atomicAdd(&cw.adm[c], 1);
        T.st[x] = 3;
      }
      __syncthreads();
      if (q == cend - 1) {  // segment totals; the maxima after its admissions
        S.max_u = dmax(smu, iu);
        S.max_r = dmax(smr, ir);
        S.members = members0 + mx + m;
        S.reserved = reserved0 + rx + rv;
        S.prefill += px + pv;
        S.n_adm += mx + m;
        S.n_rej += (cend - base) - (mx + m);
        S.n_ev += cend - base;
      }
      if (q < cend) {
        const int32_t x = T.srt[q];
        const int32_t s = static_cast<int32_t>(T.sd[x] >> 8), c = T.sc[s], d = static_cast<int32_t>(T.sd[x] & 255u);
        if (d + 1 >= T.snd[s] || T.st[x + 1] != 3) {  // the client's last consumed item
          const WinEntry& e = T.ent[q];
          double nu = T.u[x], nr = T.r[x], ncn = T.cn[x];
          if (alone) {
            nu = __dadd_rn(nu, e.ufc_inc);
            nr = __dadd_rn(nr, e.rfc_inc);
            if (P.kind == kVtc) ncn = __dadd_rn(ncn, vtc_inc(P, e, cw.w[c]));
          }
          cw.ufc[c] = nu;
          cw.rfc[c] = nr;
          cw.cnt[c] = ncn;
          const int32_t np = T.spos[s] + d + 1;
          if (np == cw.end[c]) cw.flags[c] &= ~kBacklogged;  // pop_head emptied the queue
          cw.pos[c] = np;
          if (q == fs && fs < fn) {  // the item that ends the segment
            if (np == cw.end[c]) X.stop = 4;             // a holder left: maxima need a rescan
            else if (T.fl[x] & kFlExh) X.stop = 16;      // the client's stream ran out: regenerate
          }
        }
      }
      if (tid == 0 && fn < nse && fn <= fs) {
        if (!P.backfill) X.stop = 2;  // engine.cpp:239: the head does not fit, the step is over
        else X.stop = 8;              // backfill: skip its client, continue item by item
      }
      __syncthreads();
      // 4c'. continue the walk after a moved maximum when the rest of the list is still valid
      const int32_t sstop = X.stop;
      if (!(fs < fn && fs < nse) || (sstop & 16) || cend >= nse) break;
      // Fast path: a maximum rose (no holder left) and the rest of the list has key 0 from its
      // first to its last item.  With non-negative ledgers and both maxima positive before the
      // rise, a key is 0 exactly when its weighted numerators are, which a rising maximum keeps
      // (a positive key stays positive, a zero key stays zero), so those items keep their order
      // and stay below every other item -- nothing to recompute.
      if (sstop == 0 && nonneg && smu > 0.0 && smr > 0.0 && T.k[T.srt[cend]] == kZeroKey &&
          T.k[T.srt[nse - 1]] == kZeroKey) {
        if (tid == 0) {
          X.fn = 0x7fffffff;
          X.fs = 0x7fffffff;
        }
        base = cend;
        __syncthreads();
        continue;
      }
#ifdef EQX_PROF
      const long long tv0 = clock64();
#endif
      if (sstop & 4) cta_maxima(cw, C, S);  // a holder left: the maxima over the backlog
      const double nmu = S.max_u, nmr = S.max_r;
      if (tid == 0) X.bad = 0;
      for (int64_t x = tid; x < n; x += NT) {  // the unconsumed items' keys under the new maxima
        if (T.st[x] == 3 || !(T.fl[x] & kTkValid)) continue;
        T.k[x] = ordered_bits(hf_key(P, T.u[x], T.r[x], nmu, nmr, T.cn[x]));
      }
      if (bounded) topk_boundary(P, cw, T, X, C, nmu, nmr);
      __syncthreads();
      auto item_tuple = [&](int64_t x, uint64_t& k, uint64_t& av, uint64_t& o) {
        const uint32_t sdv = T.sd[x];
        k = T.k[x];
        av = T.a[x];
        o = (static_cast<uint64_t>(cw.order[T.sc[sdv >> 8]]) << 32) | (sdv & 255u);
      };
      uint64_t lk, la, lo;
      item_tuple(T.srt[nse - 1], lk, la, lo);
      bool bad = bounded && !tuple_lt(lk, la, lo, X.bk, X.ba, X.bo);
      for (int32_t r = cend + tid; r + 1 < nse && !bad; r += NT) {  // still sorted
        uint64_t k1, a1, o1, k2, a2, o2;
        item_tuple(T.srt[r], k1, a1, o1);
        item_tuple(T.srt[r + 1], k2, a2, o2);
        bad = !tuple_lt(k1, a1, o1, k2, a2, o2);
      }
      for (int64_t x = tid; x < n && !bad; x += NT) {  // below every other unconsumed item:
        if (T.st[x] != 0 || !(T.fl[x] & kTkValid)) continue;  // the ones not selected
        uint64_t k2, a2, o2;
        item_tuple(x, k2, a2, o2);
        bad = !tuple_lt(lk, la, lo, k2, a2, o2);
      }
      for (int32_t r = nse + tid; r < ns && !bad; r += NT) {  // and the selected ones past the boundary
        uint64_t k2, a2, o2;
        item_tuple(T.srt[r], k2, a2, o2);
        bad = !tuple_lt(lk, la, lo, k2, a2, o2);
      }
      if (bad) X.bad = 1;
      __syncthreads();
      const bool valid = X.bad == 0;

#ifdef EQX_PROF
      tk[6] += clock64() - tv0;
      tk[7] += 1;
#endif
      if (!valid) {  // end the round; the next one re-selects under the new maxima
        if (tid == 0) X.stop = sstop & ~4;  // the maxima were rescanned here already
        __syncthreads();
        break;
      }
      if (tid == 0) {
        X.stop = 0;
        X.fn = 0x7fffffff;
        X.fs = 0x7fffffff;
      }
      base = cend;
      __syncthreads();
    }
    TK_STAMP(6)
    // 4c. backfill after a head that did not fit: the exact loop body, one item at a time
    // (a volatile read inside the thread-0 branch: the flag is rewritten by that thread below)
    if (tid == 0 && *reinterpret_cast<volatile int32_t*>(&X.stop) == 8) {
      int32_t stop = 0;
      int32_t members = S.members;
      int64_t reserved = S.reserved, n_ev = S.n_ev, n_adm = S.n_adm, n_rej = S.n_rej, prefill = S.prefill;
      double max_u = S.max_u, max_r = S.max_r;
      for (int32_t i = X.fn; i < nse && !stop; ++i) {
        const int32_t x = T.srt[i];
        const int32_t c = T.sc[T.sd[x] >> 8];
        const int32_t fc = cw.flags[c];
        if (fc & kSkipped) continue;  // skipped earlier in the round
        const WinEntry& e = T.ent[i];
        const uint8_t fl = T.fl[x];
        const int32_t j = cw.pos[c];
        const bool last = j + 1 == cw.end[c];
        // a max holder leaving the backlog, under the maxima in force now
        const bool holder = maxmode && last && (cw.ufc[c] == max_u || cw.rfc[c] == max_r);
        if (!e.alone) {  // engine.cpp:223-234: Rejected, pop_head, no counter change
          topk_event(a, n_ev, e, 2, c, cw.w[c]);
          ++n_ev;
          ++n_rej;
          T.st[x] = 3;
          cw.pos[c] = j + 1;
          if (last) {
            cw.flags[c] = fc & ~kBacklogged;
            if (holder) stop = 4;
          } else if (fl & kFlExh) {
            stop = 16;
          }
          continue;
        }
        if (!((members + 1 <= P.max_batch) && (reserved + e.in + e.pred <= tmax))) {
          cw.flags[c] = fc | kSkipped;  // engine.cpp:236-238
          continue;
        }
        members += 1;
        reserved += static_cast<int64_t>(e.in) + e.pred;
        prefill += e.in;
        const double nu = __dadd_rn(cw.ufc[c], e.ufc_inc), nr = __dadd_rn(cw.rfc[c], e.rfc_inc);
        cw.ufc[c] = nu;
        cw.rfc[c] = nr;
        if (P.kind == kVtc) cw.cnt[c] = __dadd_rn(cw.cnt[c], vtc_inc(P, e, cw.w[c]));
        cw.adm[c] += 1;
        topk_event(a, n_ev, e, 1, c, cw.w[c]);
        ++n_ev;
        ++n_adm;
        T.st[x] = 3;
        cw.pos[c] = j + 1;
        if (last) {
          cw.flags[c] = fc & ~kBacklogged;
          if (holder) stop = 4;
        } else {
          if (maxmode && (max_u < nu || max_r < nr)) {  // the admission raises a maximum
            if (max_u < nu) max_u = nu;
            if (max_r < nr) max_r = nr;
            stop = 1;
          }
          if (fl & kFlExh) stop = 16;
        }
      }
      S.members = members;
      S.reserved = reserved;
      S.n_ev = n_ev;
      S.n_adm = n_adm;
      S.n_rej = n_rej;
      S.prefill = prefill;
      S.max_u = max_u;
      S.max_r = max_r;
      X.stop = stop | (stop ? 0 : 32);  // 32: the walk reached the end of the list
    }
    __syncthreads();
    TK_STAMP(7)
#ifdef EQX_PROF
    ++rounds;
#endif
    const int32_t stop = X.stop, consumed = X.fn <= X.fs ? min(X.fn, nse) : X.fs + 1;
    if (stop == 2) break;
    if (stop & 4) cta_maxima(cw, C, S);  // max over the backlogged clients (scheduler.cpp:40-48)
    const bool ran_out = (stop & 32) || (X.fn >= nse && X.fs >= nse);
    // regenerate when a stream ran out, or when the walk reached the boundary
    regen = (stop & 16) || (ran_out && nse < ns);
    // next K: double it when the list ran out, else about twice what this round consumed
    K = (ran_out && nse == ns) ? min(want, 2 * K) : min(want, max(32, 2 * consumed));
    __syncthreads();
  }
#ifdef EQX_PROF
  if (tid == 0) {
    a.st->t[7] = rounds;
    for (int i = 0; i < 8; ++i) a.st->t[8 + i] = cy[i];
    tk[5] = n_total_items;  // tk[6] / tk[7]: in-round verification cycles / segments
    for (int i = 0; i < 8; ++i) a.st->tk[i] = tk[i];
  }
#endif
#undef TK_STAMP
  if (tid == 0) S.flags = kDone;
}
