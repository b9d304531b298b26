// Fused elementwise round kernels for the Beaver / SPK-adder protocols.
//
// Every secure round is "combine the previous open, build the next payload" in ONE
// pass over the elements, with the dealer's triple shares regenerated in registers
// (no triple ever touches HBM). A round kernel serves all local party slots in one
// launch; a slot reads only its own state, its own outbox and the peer payload.
#pragma once

#include "core.hpp"

namespace mpcg {

struct Pid2 {
  int v[2];
};

// Slot and party at position k of a step<NS>(slot0, ...) loop. Pair evaluation (NS == 2, both
// parties local, so the two slots play parties 0 and 1): position k is PARTY k, which makes
// every party-dependent branch of the share algebra a compile-time constant.
template <int NS>
__device__ __forceinline__ int pair_slot(const Pid2& pid, int slot0, int k) {
  if constexpr (NS == 2) return pid.v[0] == k ? 0 : 1;
  else return slot0 + k;
}
template <int NS>
__device__ __forceinline__ int pair_party(const Pid2& pid, int slot, int k) {
  if constexpr (NS == 2) return k;
  else return pid.v[slot];
}

struct Ptr2 {
  u64* p[2];
};
struct CPtr2 {
  const u64* p[2];
};
// Slot pointer / party of a runtime slot by selection: indexing a kernel-parameter array with a
// runtime index makes the compiler copy the array to local memory (STL/LDL in the hot loops).
__host__ __device__ __forceinline__ u64* sel(const Ptr2& x, int slot) { return slot ? x.p[1] : x.p[0]; }
__host__ __device__ __forceinline__ const u64* sel(const CPtr2& x, int slot) { return slot ? x.p[1] : x.p[0]; }

inline Pid2 pids(const Session& s) { return Pid2{{s.party_of[0], s.party_of[1]}}; }
// Opened wire (AdderRound, MulBuild/MulCombine, the compare chain's b2a and multiply): exactly
// when the pair kernel evaluates every kernel of the exchange (both slots local, pair
// evaluation on); MPCG_PAIR_EVAL=0 = per-slot evaluation with two payloads.
inline bool adder_opened_wire(const Session& s) { return s.n_local == 2 && pair_eval_enabled(); }
// Element-by-element Beaver chains (beaver_chain_pair_kernel) and one-pass multiplies
// (MulFused): pair evaluation with the opened wire, no link, seeded dealer (queue-sourced
// triples keep the per-round kernels), not forced to per-round kernels. MPCG_FUSED_BCHAIN=0
// disables.
inline bool pair_chain_ok(const Session& s) {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_FUSED_BCHAIN");
    return !(e && e[0] == '0');
  }();
  return on && adder_opened_wire(s) && !(s.cfg.link_bandwidth > 0) && !s.source_q && s.persistent_mode != 0;
}

inline Ptr2 ptrs(const DT& t) { return Ptr2{{t.s[0], t.s[1]}}; }
inline CPtr2 cptrs(const DT& t) { return CPtr2{{t.s[0], t.s[1]}}; }
inline Ptr2 own_ptrs(const Open& o) {
  return Ptr2{{o.own(0), o.n_local == 2 ? o.own(1) : nullptr}};
}
inline CPtr2 peer_ptrs(const Open& o) {
  return CPtr2{{o.peer(0), o.n_local == 2 ? o.peer(1) : nullptr}};
}

// ---------------------------------------------------------------- value sources
struct SrcMem {  // x[g]
  CPtr2 x;
  // select, not index: a runtime slot index into the parameter array spills it to local memory
  __device__ u64 operator()(int slot, u64 g) const { return (slot ? x.p[1] : x.p[0])[g]; }
};
struct SrcZero {
  __device__ u64 operator()(int, u64) const { return 0; }
};
struct SrcSub {  // x[g] - y[g]
  CPtr2 x, y;
  __device__ u64 operator()(int slot, u64 g) const { return sel(x, slot)[g] - sel(y, slot)[g]; }
};
struct SrcSar {  // sar(x[g], k)
  CPtr2 x;
  int k;
  __device__ u64 operator()(int slot, u64 g) const { return sar64(sel(x, slot)[g], k); }
};

// ---------------------------------------------------------------- sinks (post-combine)
struct SinkStore {  // out[g] = z
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64 z) const { sel(out, slot)[g] = z; }
};
struct SinkTrunc {  // out[g] = sar(z, k)
  Ptr2 out;
  int k;
  __device__ void operator()(int slot, int, u64 g, u64 z) const { sel(out, slot)[g] = sar64(z, k); }
};

// ---------------------------------------------------------------- Beaver multiply
// payload of a chunk of width w: [eps(w) | delta(w)]   (H/protocols/beaver.hpp:53,68-69)
template <class XF, class YF>
struct MulBuild {
  EwTriple T;
  Pid2 pid;
  Ptr2 own;
  u64 lo, w;
  XF xf;
  YF yf;
  bool opened = false;  // pair evaluation: write the opened (eps, delta) once (see MulCombine)
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j); }
  __device__ void both(u64 j) const { step<2>(0, j); }
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j) const {
    const u64 g = lo + j;
    if (NS == 2 && opened) {  // eps0 + eps1 = x0 + x1 - (a0 + a1), a0 + a1 = A: masks cancel
      const Dw d = ew_secrets(T, T.off + g);
      own.p[0][j] = xf(0, g) + xf(1, g) - d.A;
      own.p[0][w + j] = yf(0, g) + yf(1, g) - d.B;
      return;
    }
    const Dw d = ew_draw<false>(T, T.off + g, NS == 2 || pid.v[slot0] == 0);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int slot = pair_slot<NS>(pid, slot0, k);
      u64 a, b, c;
      ew_share<false>(T, pid.v[slot], d, a, b, c);
      sel(own, slot)[j] = xf(slot, g) - a;
      sel(own, slot)[w + j] = yf(slot, g) - b;
    }
  }
};

// Functors that can take both party slots' values at once (pair evaluation): FF::pair(q0, g,
// j, v0, v1) / PF::pair(q0, g, z0, z1), v_k / z_k being party k's, q0 the slot of party 0.
template <class F, class = void>
struct has_pair_pf : std::false_type {};
template <class F>
struct has_pair_pf<F, std::void_t<decltype(std::declval<const F&>().pair(0, u64(0), u64(0), u64(0)))>>
    : std::true_type {};
template <class F, class = void>
struct has_pair_ff : std::false_type {};
template <class F>
struct has_pair_ff<F, std::void_t<decltype(std::declval<const F&>().pair(0, u64(0), u64(0), u64(0), u64(0)))>>
    : std::true_type {};

template <class PF>
struct MulCombine {
  EwTriple T;
  Pid2 pid;
  CPtr2 own, peer;
  u64 lo, w;
  PF pf;
  // Pair evaluation only, and only if the payload's builder wrote it the same way: the opened
  // (eps, delta) = own0 + own1 sits once in slot 0's outbox (8 B each per element pair
  // instead of both payloads read by both slots).
  bool opened = false;
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j); }
  __device__ void both(u64 j) const { step<2>(0, j); }
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j) const {
    const u64 g = lo + j;
    const Dw dr = ew_draw<true>(T, T.off + g, NS == 2 || pid.v[slot0] == 0);
    const bool op = NS == 2 && opened;
    u64 oe = 0, od = 0;
    if (op) oe = own.p[0][j], od = own.p[0][w + j];
    u64 zs[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
      u64 e = oe, d = od;
      if (!op) {
        const u64* o = sel(own, slot);
        const u64* q = sel(peer, slot);
        e = o[j] + q[j];
        d = o[w + j] + q[w + j];
      }
      u64 a, b, c;
      ew_share<true>(T, party, dr, a, b, c);
      u64 z = c + (e * b + d * a);
      if (party == 0) z += e * d;
      zs[k] = z;
      if constexpr (!(NS == 2 && has_pair_pf<PF>::value)) pf(slot, party, g, z);
    }
    if constexpr (NS == 2 && has_pair_pf<PF>::value) pf.pair(pair_slot<2>(pid, 0, 0), g, zs[0], zs[1]);
  }
};

inline CPtr2 as_const(Ptr2 p) { return CPtr2{{p.p[0], p.p[1]}}; }

// Pair evaluation with in-device opens (pair_chain_ok): the Beaver multiply of element g in one
// pass — the opened (eps, delta) of MulBuild's opened wire kept in registers and combined at
// once (MulCombine's algebra), A and B drawn once for both. Arithmetic triples only.
template <class XF, class YF, class PF>
struct MulFused {
  EwTriple T;
  Pid2 pid;
  XF xf;
  YF yf;
  PF pf;
  __device__ void operator()(int, u64) const {}  // pair evaluation only (launch_ew's both())
  __device__ void both(u64 g) const {
    const int q0 = pid.v[0] == 0 ? 0 : 1, q1 = 1 - q0;
    const Dw d = ew_draw<true>(T, T.off + g, true);
    const u64 e = xf(q0, g) + xf(q1, g) - d.A, dd = yf(q0, g) + yf(q1, g) - d.B;
    const u64 z0 = (d.A * d.B - d.rc) + (e * (d.B - d.rb) + dd * (d.A - d.ra)) + e * dd;
    const u64 z1 = d.rc + (e * d.rb + dd * d.ra);
    if constexpr (has_pair_pf<PF>::value) {
      pf.pair(q0, g, z0, z1);
    } else {
      pf(q0, 0, g, z0);
      pf(q1, 1, g, z1);
    }
  }
};

// z = x*y with sources/sink functors; `chunks` reveals as in beaver_mul.
template <class XF, class YF, class PF>
void mul_op(Session& s, const EwTriple& T, size_t m, int chunks, const std::string& tag, XF xf, YF yf,
            PF pf) {
  chunks = clamp_chunks(chunks, m);
  const int acct = chunks;                                // lanes as the reference accounts them
  const int xl = acct > 1 && s.fuse_lanes() ? 1 : acct;  // lanes launched (Session::fuse_lanes)
  auto ltag = [&](int k) { return acct == 1 ? tag : tag + ".chunk" + std::to_string(k); };
  if (m > 0 && !T.bin && pair_chain_ok(s)) {  // build + open + combine in one pass (MulFused)
    {
      ClassScope cs(kClsOther, 0);
      launch_ew(s.stream, s.n_local, m, MulFused<XF, YF, PF>{T, pids(s), xf, yf, pf});
    }
    for (int k = 0; k < acct; ++k) {  // the opens, as post / post_lanes account them
      const auto r = chunk_range(m, acct, k);
      s.account(2 * (r.second - r.first), Reduce::Sum, ltag(k));
    }
    s.check();
    return;
  }
  std::vector<Open> opens(static_cast<size_t>(xl));
  const Pid2 pid = pids(s);
  // SURVEY 8(d) algorithmic bytes: beaver_mul = 2 x 16 B wire + 8 x (2 in + 1 out) = 56 B/elem/
  // party over build + combine (28 per launch). The opened wire (pair evaluation) moves less — the
  // 16 B opened pair is written and read once per element pair — but the roofline counts 8(d)'s.
  const bool opened = adder_opened_wire(s);
  ClassScope cs(kClsBeaver, 28.0 * double(m / xl) * s.n_local);
  for (int k = 0; k < xl; ++k) {
    const auto rng_ = chunk_range(m, xl, k); const size_t lo = rng_.first, hi = rng_.second;
    opens[k] = s.begin_open(2 * (hi - lo), Reduce::Sum);
    MulBuild<XF, YF> mb{T, pid, own_ptrs(opens[k]), lo, hi - lo, xf, yf};
    mb.opened = opened;
    launch_ew(s.stream, s.n_local, hi - lo, mb);
    if (xl == acct) s.post(opens[k], ltag(k));
    else s.post_lanes(opens[k], m, acct, 2, ltag);
  }
  for (int k = 0; k < xl; ++k) {
    const auto rng_ = chunk_range(m, xl, k); const size_t lo = rng_.first, hi = rng_.second;
    s.wait(opens[k]);
    MulCombine<PF> mc{T, pid, as_const(own_ptrs(opens[k])), peer_ptrs(opens[k]), lo, hi - lo, pf};
    mc.opened = opened;
    launch_ew(s.stream, s.n_local, hi - lo, mc);
    s.check();
  }
}

// One warp per row: of(slot, row, sum_j vf(slot, row*L + j)) with wrapping u64 adds (exact
// and order-independent mod 2^64). Rows are contiguous, so lanes read coalesced 256 B runs.
template <class VF, class OF>
__global__ void __launch_bounds__(256) row_reduce_kernel(u64 rows, u32 L, VF vf, OF of) {
  pdl_enter();
  const int slot = blockIdx.y;
  const unsigned lane = threadIdx.x & 31;
  const u64 nw = u64(gridDim.x) * (blockDim.x / 32);
  for (u64 r = (blockIdx.x * u64(blockDim.x) + threadIdx.x) / 32; r < rows; r += nw) {
    u64 acc = 0;
    for (u32 j = lane; j < L; j += 32) acc += vf(slot, r * L + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) of(slot, r, acc);
  }
}

template <class VF, class OF>
void row_reduce(Session& s, u64 rows, u32 L, VF vf, OF of) {
  if (rows == 0) return;
  u64 blocks = (rows * 32 + 255) / 256;
  const u64 cap = u64(num_sms()) * 8;
  blocks = blocks > cap ? cap : blocks;
  cudaEvent_t pe;
  probe_begin(s.stream, &pe);
  launch_pdl(row_reduce_kernel<VF, OF>, dim3(unsigned(blocks), s.n_local), dim3(256), 0, s.stream, rows, L, vf, of);
  probe_end(s.stream, pe);
  s.check();
}


// Square-triple draws of element g: A (party 0 only), r_A, r_C (H/sharing/triple.hpp:96-114).
struct Sw {
  u64 A, ra, rc;
};
__device__ __forceinline__ Sw sq_draw(const EwTriple& t, u64 g, bool p0, bool with_c) {
  const u64 key = tkey(t.key, t.kp);
  const u64 gp = g * kPhi;
  return by_source(t.pool, [&](auto src) {
    constexpr bool P = decltype(src)::value;
    Sw d;
    d.ra = drawp<P>(key + t.pra + gp, key, t.pool);
    d.rc = with_c ? drawp<P>(key + t.prc + gp, key, t.pool) : 0;
    d.A = p0 ? drawp<P>(key + t.pA + gp, key, t.pool) : 0;
    return d;
  });
}
__device__ __forceinline__ u64 sq_share_a(int party, const Sw& d) { return party ? d.ra : d.A - d.ra; }
// the square triple's secret A alone (a0 + a1 = A: all an opened-wire build needs)
__device__ __forceinline__ u64 sq_secret(const EwTriple& t, u64 g) {
  const u64 key = tkey(t.key, t.kp);
  return dmix(key + t.pA + g * kPhi, key, t.pool);
}
__device__ __forceinline__ u64 sq_share_c(int party, const Sw& d) { return party ? d.rc : d.A * d.A - d.rc; }

// ---------------------------------------------------------------- Beaver square
template <class XF>
struct SqBuild {
  EwTriple T;
  Pid2 pid;
  Ptr2 own;
  u64 lo;
  XF xf;
  bool opened = false;  // pair evaluation: the opened eps once (slot 0's outbox)
  __device__ void operator()(int slot, u64 j) const {
    const u64 g = lo + j;
    sel(own, slot)[j] = xf(slot, g) - sq_a(T, pid.v[slot], T.off + g);
  }
  __device__ void both(u64 j) const {
    const u64 g = lo + j;
    if (opened) {  // eps0 + eps1 = x0 + x1 - A
      own.p[0][j] = xf(0, g) + xf(1, g) - sq_secret(T, T.off + g);
      return;
    }
    (*this)(0, j);
    (*this)(1, j);
  }
};
template <class PF>
struct SqCombine {
  EwTriple T;
  Pid2 pid;
  CPtr2 own, peer;
  u64 lo;
  PF pf;
  bool opened = false;  // pair evaluation: read the opened eps once
  __device__ void operator()(int slot, u64 j) const {
    const int party = pid.v[slot];
    const u64 g = lo + j;
    const u64 e = sel(own, slot)[j] + sel(peer, slot)[j];
    u64 a, c;
    sq_ac(T, party, T.off + g, a, c);
    u64 z = c + (e * a) * 2;
    if (party == 0) z += e * e;
    pf(slot, party, g, z);
  }
  __device__ void both(u64 j) const {
    if (!opened) {
      (*this)(0, j);
      (*this)(1, j);
      return;
    }
    const u64 g = lo + j;
    const u64 e = own.p[0][j];
    const Sw d = sq_draw(T, T.off + g, true, true);  // one draw set for both parties
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int slot = pair_slot<2>(pid, 0, k);
      u64 z = sq_share_c(k, d) + (e * sq_share_a(k, d)) * 2;
      if (k == 0) z += e * e;
      pf(slot, k, g, z);
    }
  }
};

// Pair evaluation with in-device opens (pair_chain_ok): the Beaver square of element g in one
// pass (SqBuild's opened eps kept in a register, SqCombine's algebra), one draw set.
template <class XF, class PF>
struct SqFused {
  EwTriple T;
  Pid2 pid;
  XF xf;
  PF pf;
  __device__ void operator()(int, u64) const {}  // pair evaluation only (launch_ew's both())
  __device__ void both(u64 g) const {
    const Sw d = sq_draw(T, T.off + g, true, true);
    const u64 e = xf(0, g) + xf(1, g) - d.A;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int slot = pair_slot<2>(pid, 0, k);
      u64 z = sq_share_c(k, d) + (e * sq_share_a(k, d)) * 2;
      if (k == 0) z += e * e;
      pf(slot, k, g, z);
    }
  }
};

template <class XF, class PF>
void square_op(Session& s, const EwTriple& T, size_t m, int chunks, const std::string& tag, XF xf, PF pf) {
  chunks = clamp_chunks(chunks, m);
  const int acct = chunks;
  const int xl = acct > 1 && s.fuse_lanes() ? 1 : acct;  // lanes launched (Session::fuse_lanes)
  auto ltag = [&](int k) { return acct == 1 ? tag : tag + ".chunk" + std::to_string(k); };
  if (m > 0 && pair_chain_ok(s)) {  // build + open + combine in one pass (SqFused)
    {
      ClassScope cs(kClsOther, 0);
      launch_ew(s.stream, s.n_local, m, SqFused<XF, PF>{T, pids(s), xf, pf});
    }
    for (int k = 0; k < acct; ++k) {  // the opens, as post / post_lanes account them
      const auto r = chunk_range(m, acct, k);
      s.account(r.second - r.first, Reduce::Sum, ltag(k));
    }
    s.check();
    return;
  }
  std::vector<Open> opens(static_cast<size_t>(xl));
  const Pid2 pid = pids(s);
  // beaver_square = 2 x 8 B wire + 8 x (1 in + 1 out) = 32 B/elem/party over build + combine
  // (the opened wire moves 24 B, the roofline counts 8(d)'s 32)
  const bool opened = adder_opened_wire(s);
  ClassScope cs(kClsBeaver, 16.0 * double(m / xl) * s.n_local);
  for (int k = 0; k < xl; ++k) {
    const auto rng_ = chunk_range(m, xl, k); const size_t lo = rng_.first, hi = rng_.second;
    opens[k] = s.begin_open(hi - lo, Reduce::Sum);
    SqBuild<XF> b{T, pid, own_ptrs(opens[k]), lo, xf};
    b.opened = opened;
    launch_ew(s.stream, s.n_local, hi - lo, b);
    if (xl == acct) s.post(opens[k], ltag(k));
    else s.post_lanes(opens[k], m, acct, 1, ltag);
  }
  for (int k = 0; k < xl; ++k) {
    const auto rng_ = chunk_range(m, xl, k); const size_t lo = rng_.first, hi = rng_.second;
    s.wait(opens[k]);
    SqCombine<PF> c{T, pid, as_const(own_ptrs(opens[k])), peer_ptrs(opens[k]), lo, pf};
    c.opened = opened;
    launch_ew(s.stream, s.n_local, hi - lo, c);
    s.check();
  }
}

// ---------------------------------------------------------------- fused Beaver chains
// A chain of dependent Beaver rounds (exp's repeated squaring, the reciprocal's Newton
// steps) runs as "combine round r, build round r+1" in ONE pass per element, exactly like
// the SPK adder rounds: the intermediate value never round-trips through HBM and the kernel
// count halves. Posts keep the reference's collective order: every lane of round r is
// posted before any lane of round r+1 (lane k of r+1 is posted right after lane k of r is
// combined), and the sequence numbers are assigned at post time.

// Build of the first square of a chain: payload eps = x - a (pair-evaluated).
template <class XF>
struct SqBuild2 {
  EwTriple T;
  Pid2 pid;
  Ptr2 own;
  u64 lo;
  XF xf;
  bool opened = false;  // pair evaluation: write the opened eps once (slot 0's outbox)
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j); }
  __device__ void both(u64 j) const { step<2>(0, j); }
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j) const {
    const u64 g = lo + j;
    if (NS == 2 && opened) {  // eps0 + eps1 = x0 + x1 - A
      own.p[0][j] = xf(0, g) + xf(1, g) - sq_secret(T, T.off + g);
      return;
    }
    const Sw d = sq_draw(T, T.off + g, NS == 2 || pid.v[slot0] == 0, false);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int slot = pair_slot<NS>(pid, slot0, k);
      sel(own, slot)[j] = xf(slot, g) - sq_share_a(pid.v[slot], d);
    }
  }
};

// Combine square Tp, y = yf(slot, party, g, z); unless last, build square Tn on y.
template <class YF>
struct SqChainStep {
  EwTriple Tp, Tn;
  Pid2 pid;
  CPtr2 ownp, peerp;
  Ptr2 ownn;
  u64 lo;
  int last;
  YF yf;
  bool opened = false;  // pair evaluation: read / write the opened eps once (slot 0's outbox)
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j); }
  __device__ void both(u64 j) const { step<2>(0, j); }
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j) const {
    const u64 g = lo + j;
    const bool p0 = NS == 2 || pid.v[slot0] == 0;
    const bool op = NS == 2 && opened;
    const Sw dp = sq_draw(Tp, Tp.off + g, p0, true);
    Sw dn{0, 0, 0};
    if (!last && !op) dn = sq_draw(Tn, Tn.off + g, p0, false);
    const u64 oe = op ? ownp.p[0][j] : 0;
    u64 ysum = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
      const u64 e = op ? oe : sel(ownp, slot)[j] + sel(peerp, slot)[j];
      u64 z = sq_share_c(party, dp) + (e * sq_share_a(party, dp)) * 2;
      if (party == 0) z += e * e;
      const u64 y = yf(slot, party, g, z);
      if (op) ysum += y;
      else if (!last) sel(ownn, slot)[j] = y - sq_share_a(party, dn);
    }
    if (op && !last) ownn.p[0][j] = ysum - sq_secret(Tn, Tn.off + g);  // masks cancel in the open
  }
};

// Small chains in 1-GPU mode run as ONE cooperative kernel (grid barriers instead of kernel
// boundaries, as the compare chains do); defined after grid_barrier below.
template <class B0, class ST>
void persistent_beaver_chain(Session& s, u64 n, const B0& build, const std::vector<ST>& steps);
// the reference's collective order of a chain of R lane-chunked rounds: round by round, lanes
// in order within a round (what post_lanes accounts)
template <class TagOf>
void account_chain(Session& s, size_t n, int R, int lanes, TagOf words_tag) {
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < lanes; ++k) {
      const size_t lo = n * size_t(k) / size_t(lanes), hi = n * size_t(k + 1) / size_t(lanes);
      const auto wt = words_tag(r, k);
      s.account(wt.first * (hi - lo), Reduce::Sum, wt.second);
    }
}

// Rounds tr[0..R) of squares: round 0 squares x0(slot, g); round r squares the value
// yf_for(r-1) produced from round r-1's product; yf_for(R-1) sees the chain's last product.
template <class XF, class YFF>
void square_chain(Session& s, size_t n, int chunks, const std::vector<Triple>& tr,
                  const std::vector<std::string>& tags, XF x0, YFF yf_for) {
  const bool opened = adder_opened_wire(s);  // pair evaluation: opened wire between the rounds
  chunks = clamp_chunks(chunks, n);
  const int R = int(tr.size());
  const Pid2 pid = pids(s);
  const int acct_ = chunks;  // lanes as the reference accounts them (tags)
  auto ctag = [&](int r, int k) { return acct_ == 1 ? tags[r] : tags[r] + ".chunk" + std::to_string(k); };
  using YF0 = decltype(yf_for(0));
  if (R <= 24 && n > 0 && ((chunks == 1 && s.persistent_ok(n)) || pair_chain_ok(s))) {
    std::vector<Open> op(static_cast<size_t>(R));
    for (int r = 0; r < R; ++r) op[r] = s.begin_open(n, Reduce::Sum);
    std::vector<SqChainStep<YF0>> st;
    for (int r = 1; r <= R; ++r)
      st.push_back(SqChainStep<YF0>{tr[r - 1].ew, r < R ? tr[r].ew : tr[r - 1].ew, pid, as_const(own_ptrs(op[r - 1])),
                                    peer_ptrs(op[r - 1]), r < R ? own_ptrs(op[r]) : Ptr2{{nullptr, nullptr}}, 0,
                                    r == R ? 1 : 0, yf_for(r - 1)});
    SqBuild2<XF> b0{tr[0].ew, pid, own_ptrs(op[0]), 0, x0};
    b0.opened = opened;
    for (auto& x : st) x.opened = opened;
    persistent_beaver_chain(s, n, b0, st);
    account_chain(s, n, R, chunks, [&](int r, int k) { return std::make_pair(size_t(1), ctag(r, k)); });
    s.check();
    return;
  }
  const int acct = acct_;
  if (chunks > 1 && s.fuse_lanes()) chunks = 1;  // lanes launched (Session::fuse_lanes)
  auto post_r = [&](Open& o, int r, int k) {
    if (chunks == acct) s.post(o, ctag(r, k));
    else s.post_lanes(o, n, acct, 1, [&](int kk) { return ctag(r, kk); });
  };
  std::vector<Open> hs(static_cast<size_t>(chunks));
  // R squares x 32 B/elem/party spread over the R+1 fused launches of a lane
  ClassScope cs(kClsBeaver, 32.0 * R / (R + 1) * double(n / chunks) * s.n_local);
  for (int k = 0; k < chunks; ++k) {
    const auto rg = chunk_range(n, chunks, k);
    hs[k] = s.begin_open(rg.second - rg.first, Reduce::Sum);
    SqBuild2<XF> b0{tr[0].ew, pid, own_ptrs(hs[k]), rg.first, x0};
    b0.opened = opened;
    launch_ew(s.stream, s.n_local, rg.second - rg.first, b0);
    post_r(hs[k], 0, k);
  }
  using YF = decltype(yf_for(0));
  for (int r = 1; r <= R; ++r) {
    for (int k = 0; k < chunks; ++k) {
      const auto rg = chunk_range(n, chunks, k);
      const size_t w = rg.second - rg.first;
      Open next;
      if (r < R) next = s.begin_open(w, Reduce::Sum);
      s.wait(hs[k]);
      SqChainStep<YF> st{tr[r - 1].ew, r < R ? tr[r].ew : tr[r - 1].ew, pid, as_const(own_ptrs(hs[k])),
                         peer_ptrs(hs[k]), r < R ? own_ptrs(next) : Ptr2{{nullptr, nullptr}}, rg.first,
                         r == R ? 1 : 0, yf_for(r - 1)};
      st.opened = opened;
      launch_ew(s.stream, s.n_local, w, st);
      if (r < R) {
        hs[k] = std::move(next);
        post_r(hs[k], r, k);
      }
    }
  }
  s.check();
}

// Combine mul Tp, v = P.val(slot, party, g, z); unless last, build mul Tn with
// eps = P.nx(slot, g, v), delta = P.ny(slot, g, v). Payload of a lane: [eps(w) | delta(w)].
template <class PV>
struct MulChainStep {
  EwTriple Tp, Tn;
  Pid2 pid;
  CPtr2 ownp, peerp;
  Ptr2 ownn;
  u64 lo, w;
  int last;
  PV pv;
  bool opened = false;  // pair evaluation: read / write the opened (eps, delta) once
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j); }
  __device__ void both(u64 j) const { step<2>(0, j); }
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j) const {
    const u64 g = lo + j;
    const bool p0 = NS == 2 || pid.v[slot0] == 0;
    const bool op = NS == 2 && opened;
    const Dw dp = ew_draw<true>(Tp, Tp.off + g, p0);
    Dw dn{0, 0, 0, 0, 0};
    if (!last) dn = op ? ew_secrets(Tn, Tn.off + g) : ew_draw<false>(Tn, Tn.off + g, p0);
    u64 oe = 0, od = 0, sx = 0, sy = 0;
    if (op) oe = ownp.p[0][j], od = ownp.p[0][w + j];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
      u64 e = oe, d = od;
      if (!op) {
        const u64* o = sel(ownp, slot);
        const u64* q = sel(peerp, slot);
        e = o[j] + q[j], d = o[w + j] + q[w + j];
      }
      u64 a, b, c;
      ew_share<true>(Tp, party, dp, a, b, c);
      u64 z = c + (e * b + d * a);
      if (party == 0) z += e * d;
      const u64 v = pv.val(slot, party, g, z);
      if (!last) {
        if (op) {
          sx += pv.nx(slot, g, v), sy += pv.ny(slot, g, v);
        } else {
          u64 an, bn, cn;
          ew_share<false>(Tn, party, dn, an, bn, cn);
          sel(ownn, slot)[j] = pv.nx(slot, g, v) - an;
          sel(ownn, slot)[w + j] = pv.ny(slot, g, v) - bn;
        }
      }
    }
    if (op && !last) {  // a0 + a1 = A, b0 + b1 = B
      ownn.p[0][j] = sx - dn.A;
      ownn.p[0][w + j] = sy - dn.B;
    }
  }
};

// Rounds tr[0..R) of multiplies: round 0 multiplies x0 * y0; round r's operands come from
// pv_for(r-1) (applied to round r-1's product); pv_for(R-1).val sees the last product.
template <class XF, class YF, class PVF>
void mul_chain(Session& s, size_t n, int chunks, const std::vector<Triple>& tr, const std::vector<std::string>& tags,
               XF x0, YF y0, PVF pv_for) {
  const bool opened = adder_opened_wire(s);  // pair evaluation: opened wire between the rounds
  chunks = clamp_chunks(chunks, n);
  const int R = int(tr.size());
  const Pid2 pid = pids(s);
  const int acct_ = chunks;  // lanes as the reference accounts them (tags)
  auto ctag = [&](int r, int k) { return acct_ == 1 ? tags[r] : tags[r] + ".chunk" + std::to_string(k); };
  using PV0 = decltype(pv_for(0));
  if (R <= 24 && n > 0 && ((chunks == 1 && s.persistent_ok(n)) || pair_chain_ok(s))) {
    std::vector<Open> op(static_cast<size_t>(R));
    for (int r = 0; r < R; ++r) op[r] = s.begin_open(2 * n, Reduce::Sum);
    std::vector<MulChainStep<PV0>> st;
    for (int r = 1; r <= R; ++r)
      st.push_back(MulChainStep<PV0>{tr[r - 1].ew, r < R ? tr[r].ew : tr[r - 1].ew, pid,
                                     as_const(own_ptrs(op[r - 1])), peer_ptrs(op[r - 1]),
                                     r < R ? own_ptrs(op[r]) : Ptr2{{nullptr, nullptr}}, 0, n, r == R ? 1 : 0,
                                     pv_for(r - 1)});
    MulBuild<XF, YF> b0{tr[0].ew, pid, own_ptrs(op[0]), 0, n, x0, y0};
    b0.opened = opened;
    for (auto& x : st) x.opened = opened;
    persistent_beaver_chain(s, n, b0, st);
    account_chain(s, n, R, chunks, [&](int r, int k) { return std::make_pair(size_t(2), ctag(r, k)); });
    s.check();
    return;
  }
  const int acct = acct_;
  if (chunks > 1 && s.fuse_lanes()) chunks = 1;  // lanes launched (Session::fuse_lanes)
  auto post_r = [&](Open& o, int r, int k) {
    if (chunks == acct) s.post(o, ctag(r, k));
    else s.post_lanes(o, n, acct, 2, [&](int kk) { return ctag(r, kk); });
  };
  std::vector<Open> hs(static_cast<size_t>(chunks));
  // R multiplies x 56 B/elem/party spread over the R+1 fused launches of a lane
  ClassScope cs(kClsBeaver, 56.0 * R / (R + 1) * double(n / chunks) * s.n_local);
  for (int k = 0; k < chunks; ++k) {
    const auto rg = chunk_range(n, chunks, k);
    const size_t w = rg.second - rg.first;
    hs[k] = s.begin_open(2 * w, Reduce::Sum);
    MulBuild<XF, YF> b0{tr[0].ew, pid, own_ptrs(hs[k]), rg.first, w, x0, y0};
    b0.opened = opened;
    launch_ew(s.stream, s.n_local, w, b0);
    post_r(hs[k], 0, k);
  }
  using PV = decltype(pv_for(0));
  for (int r = 1; r <= R; ++r) {
    for (int k = 0; k < chunks; ++k) {
      const auto rg = chunk_range(n, chunks, k);
      const size_t w = rg.second - rg.first;
      Open next;
      if (r < R) next = s.begin_open(2 * w, Reduce::Sum);
      s.wait(hs[k]);
      MulChainStep<PV> st{tr[r - 1].ew, r < R ? tr[r].ew : tr[r - 1].ew, pid, as_const(own_ptrs(hs[k])),
                          peer_ptrs(hs[k]), r < R ? own_ptrs(next) : Ptr2{{nullptr, nullptr}}, rg.first, w,
                          r == R ? 1 : 0, pv_for(r - 1)};
      st.opened = opened;
      launch_ew(s.stream, s.n_local, w, st);
      if (r < R) {
        hs[k] = std::move(next);
        post_r(hs[k], r, k);
      }
    }
  }
  s.check();
}

// Mixed chain: any sequence of Beaver squares and multiplies, each "combine round r, build
// round r+1" in one pass (LayerNorm's inverse-sqrt Newton step is square, mul, mul). The
// policy PV maps round r's product to the value v (val) and the next round's operands
// (nx, ny; a square uses nx only). Payload of a lane: square [eps(w)], multiply [eps(w) | delta(w)].
template <class PV>
struct MixedChainStep {
  EwTriple Tp, Tn;
  int psq, nsq;  // round r / r+1 is a square
  Pid2 pid;
  CPtr2 ownp, peerp;
  Ptr2 ownn;
  u64 lo, w;
  int last;
  PV pv;
  bool opened = false;  // pair evaluation: read / write the opened payload once
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j); }
  __device__ void both(u64 j) const { step<2>(0, j); }
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j) const {
    const u64 g = lo + j;
    const bool p0 = NS == 2 || pid.v[slot0] == 0;
    const bool op = NS == 2 && opened;
    Sw sp{0, 0, 0}, sn{0, 0, 0};
    Dw dp{0, 0, 0, 0, 0}, dn{0, 0, 0, 0, 0};
    if (psq) sp = sq_draw(Tp, Tp.off + g, p0, true);
    else dp = ew_draw<true>(Tp, Tp.off + g, p0);
    if (!last) {
      if (op) {  // the secrets only: the masks cancel in the open
        if (nsq) sn.A = sq_secret(Tn, Tn.off + g);
        else dn = ew_secrets(Tn, Tn.off + g);
      } else if (nsq) {
        sn = sq_draw(Tn, Tn.off + g, p0, false);
      } else {
        dn = ew_draw<false>(Tn, Tn.off + g, p0);
      }
    }
    u64 oe = 0, od = 0, sx = 0, sy = 0;
    if (op) {
      oe = ownp.p[0][j];
      if (!psq) od = ownp.p[0][w + j];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
      const u64* o = sel(ownp, slot);
      const u64* q = sel(peerp, slot);
      u64 z;
      if (psq) {
        const u64 e = op ? oe : o[j] + q[j];
        z = sq_share_c(party, sp) + (e * sq_share_a(party, sp)) * 2;
        if (party == 0) z += e * e;
      } else {
        const u64 e = op ? oe : o[j] + q[j], d = op ? od : o[w + j] + q[w + j];
        u64 a, b, c;
        ew_share<true>(Tp, party, dp, a, b, c);
        z = c + (e * b + d * a);
        if (party == 0) z += e * d;
      }
      const u64 v = pv.val(slot, party, g, z);
      if (!last) {
        if (op) {
          sx += pv.nx(slot, g, v);
          if (!nsq) sy += pv.ny(slot, g, v);
        } else if (nsq) {
          sel(ownn, slot)[j] = pv.nx(slot, g, v) - sq_share_a(party, sn);
        } else {
          u64 an, bn, cn;
          ew_share<false>(Tn, party, dn, an, bn, cn);
          sel(ownn, slot)[j] = pv.nx(slot, g, v) - an;
          sel(ownn, slot)[w + j] = pv.ny(slot, g, v) - bn;
        }
      }
    }
    if (op && !last) {
      if (nsq) {
        ownn.p[0][j] = sx - sn.A;
      } else {
        ownn.p[0][j] = sx - dn.A;
        ownn.p[0][w + j] = sy - dn.B;
      }
    }
  }
};

// Rounds tr[0..R) (sq[r] says square or multiply): round 0 on (x0, y0) (square: x0 only),
// round r on pv_for(r-1)'s operands; pv_for(R-1).val sees the last product.
template <class XF, class YF, class PVF>
void mixed_chain(Session& s, size_t n, int chunks, const std::vector<Triple>& tr, const std::vector<int>& sq,
                 const std::vector<std::string>& tags, XF x0, YF y0, PVF pv_for) {
  const bool opened = adder_opened_wire(s);  // pair evaluation: opened wire between the rounds
  chunks = clamp_chunks(chunks, n);
  const int R = int(tr.size());
  const Pid2 pid = pids(s);
  const int acct_ = chunks;  // lanes as the reference accounts them (tags)
  auto ctag = [&](int r, int k) { return acct_ == 1 ? tags[r] : tags[r] + ".chunk" + std::to_string(k); };
  auto words = [&](int r, size_t w) { return sq[r] ? w : 2 * w; };
  using PV0 = decltype(pv_for(0));
  if (R <= 24 && n > 0 && ((chunks == 1 && s.persistent_ok(n)) || pair_chain_ok(s))) {  // one kernel
    std::vector<Open> op(static_cast<size_t>(R));
    for (int r = 0; r < R; ++r) op[r] = s.begin_open(words(r, n), Reduce::Sum);
    std::vector<MixedChainStep<PV0>> st;
    for (int r = 1; r <= R; ++r)
      st.push_back(MixedChainStep<PV0>{tr[r - 1].ew, r < R ? tr[r].ew : tr[r - 1].ew, sq[r - 1], r < R ? sq[r] : 0,
                                       pid, as_const(own_ptrs(op[r - 1])), peer_ptrs(op[r - 1]),
                                       r < R ? own_ptrs(op[r]) : Ptr2{{nullptr, nullptr}}, 0, n, r == R ? 1 : 0,
                                       pv_for(r - 1)});
    for (auto& x : st) x.opened = opened;
    if (sq[0]) {
      SqBuild2<XF> b0{tr[0].ew, pid, own_ptrs(op[0]), 0, x0};
      b0.opened = opened;
      persistent_beaver_chain(s, n, b0, st);
    } else {
      MulBuild<XF, YF> b0{tr[0].ew, pid, own_ptrs(op[0]), 0, n, x0, y0};
      b0.opened = opened;
      persistent_beaver_chain(s, n, b0, st);
    }
    account_chain(s, n, R, chunks, [&](int r, int k) { return std::make_pair(words(r, 1), ctag(r, k)); });
    s.check();
    return;
  }
  const int acct = acct_;
  if (chunks > 1 && s.fuse_lanes()) chunks = 1;  // lanes launched (Session::fuse_lanes)
  auto post_r = [&](Open& o, int r, int k) {
    if (chunks == acct) s.post(o, ctag(r, k));
    else s.post_lanes(o, n, acct, words(r, 1), [&](int kk) { return ctag(r, kk); });
  };
  std::vector<Open> hs(static_cast<size_t>(chunks));
  for (int k = 0; k < chunks; ++k) {
    const auto rg = chunk_range(n, chunks, k);
    const size_t w = rg.second - rg.first;
    hs[k] = s.begin_open(words(0, w), Reduce::Sum);
    if (sq[0]) {
      SqBuild2<XF> b0{tr[0].ew, pid, own_ptrs(hs[k]), rg.first, x0};
      b0.opened = opened;
      launch_ew(s.stream, s.n_local, w, b0);
    } else {
      MulBuild<XF, YF> b0{tr[0].ew, pid, own_ptrs(hs[k]), rg.first, w, x0, y0};
      b0.opened = opened;
      launch_ew(s.stream, s.n_local, w, b0);
    }
    post_r(hs[k], 0, k);
  }
  using PV = decltype(pv_for(0));
  for (int r = 1; r <= R; ++r) {
    for (int k = 0; k < chunks; ++k) {
      const auto rg = chunk_range(n, chunks, k);
      const size_t w = rg.second - rg.first;
      Open next;
      if (r < R) next = s.begin_open(words(r, w), Reduce::Sum);
      s.wait(hs[k]);
      MixedChainStep<PV> st{tr[r - 1].ew, r < R ? tr[r].ew : tr[r - 1].ew, sq[r - 1], r < R ? sq[r] : 0, pid,
                            as_const(own_ptrs(hs[k])), peer_ptrs(hs[k]),
                            r < R ? own_ptrs(next) : Ptr2{{nullptr, nullptr}}, rg.first, w, r == R ? 1 : 0,
                            pv_for(r - 1)};
      st.opened = opened;
      launch_ew(s.stream, s.n_local, w, st);
      if (r < R) {
        hs[k] = std::move(next);
        post_r(hs[k], r, k);
      }
    }
  }
  s.check();
}

// ---------------------------------------------------------------- SPK adder rounds
// H/protocols/adder.hpp:122-223. Round 0 is the generate AND on (x, y); rounds 1..L are
// the prefix levels on the stacked (S, P) pair. One kernel settles round rp and issues
// round rn for a lane [lo, lo+w); rn == L+1 finalises sum = p_orig ^ (s << 1).
struct SpkLevel {
  u64 in, out, mult;
};


// Issue-to-settle draw cache (L2-sized rounds): the issue of round r draws A, B, r_A, r_B of
// triple r for the payload; the settle of round r (next kernel) needs them again plus r_C.
// When the cache is on, the issue kernel keeps the four draws of each half in a small
// SoA buffer ([half][4][n], coalesced) that stays L2-resident, and the settle draws only
// r_C: 10 instead of 18 splitmix64 per element and level round. Values are unchanged.
__device__ __forceinline__ void dw_store(u64* c, u64 n, u64 g, int half, const Dw& d) {
  u64* b = c + u64(half) * 4 * n + g;
  b[0] = d.A;
  b[n] = d.B;
  b[2 * n] = d.ra;
  b[3 * n] = d.rb;
}
__device__ __forceinline__ Dw dw_load(const u64* c, u64 n, u64 g, int half, const EwTriple& t, u64 gidx) {
  const u64* b = c + u64(half) * 4 * n + g;
  Dw d;
  d.A = b[0];
  d.B = b[n];
  d.ra = b[2 * n];
  d.rb = b[3 * n];
  const u64 key = tkey(t.key, t.kp);
  d.rc = dmix(key + t.prc + gidx * kPhi, key, t.pool);
  return d;
}

template <class XF, class YF, class FF, bool Pool = false>
struct AdderRound {
  int rp, rn, levels;
  EwTriple Tp, Tn;
  SpkLevel lp, ln;
  Pid2 pid;
  CPtr2 ownp, peerp;
  Ptr2 ownn;
  Ptr2 S, P, P0;
  u64 lo, w, wmask;
  XF xf;
  YF yf;
  FF ff;
  const u64* cwp = nullptr;  // draw cache written by the previous round's issue (or null)
  u64* cwn = nullptr;        // draw cache for the next round's settle (or null)
  u64 cwN = 0;               // elements per cache plane
  struct Keys {
    u64 p, n;
  };
  __device__ Keys keys() const { return {tkey(Tp.key, Tp.kp), tkey(Tn.key, Tn.kp)}; }
  __device__ void operator()(int slot, u64 j) const { step<1>(slot, j, keys()); }
  __device__ void both(u64 j) const { step<2>(0, j, keys()); }
  // ew_pair_kernel: the two triples' keys (device key slots under graph replay) read once
  __device__ Keys prep() const { return keys(); }
  __device__ void both_p(u64 j, const Keys& k) const { step<2>(0, j, k); }

  // NS party slots (slot0, slot0+1, ...) of element j; dealer draws are shared by the slots.
  template <int NS>
  __device__ __forceinline__ void step(int slot0, u64 j, const Keys& ks) const {
    const u64 g = lo + j;
    const bool p0 = NS == 2 || pid.v[slot0] == 0;  // does any evaluated slot play party 0
    u64 dummy;
    // Pair evaluation (NS == 2; the launchers use it for every round of an adder or none): the
    // wire holds the opened value (payload0 ^ payload1, what the XOR open reveals to both
    // parties) once, in slot 0's outbox, instead of the two payloads — a settle reads 32 B per
    // element instead of 2 x 32, an issue writes 32 instead of 2 x 32.
    constexpr bool op = NS == 2;
    if (rn == 0) {  // issue the generate AND: payload [x^a | y^b]
      // opened wire: payload0 ^ payload1 = (x0 ^ x1) ^ (a0 ^ a1) with a0 ^ a1 = A (the masks
      // r_A cancel), so only the dealer's A, B are drawn
      const Dw dn = op && !cwn ? ew_secrets_t<Pool>(Tn, Tn.off + g) : ew_draw_t<false, Pool>(Tn, Tn.off + g, p0);
      if (cwn) dw_store(cwn, cwN, g, 0, dn);
      u64 o0 = 0, o1 = 0;
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int slot = pair_slot<NS>(pid, slot0, k);
        const u64 x = xf(slot, g), y = yf(slot, g);
        sel(P0, slot)[g] = x ^ y;
        u64 a, b;
        ew_share<false>(Tn, pid.v[slot], dn, a, b, dummy);
        if (op) {
          o0 ^= x;
          o1 ^= y;
        } else {
          sel(ownn, slot)[j] = x ^ a;
          sel(ownn, slot)[w + j] = y ^ b;
        }
      }
      if (op) {
        ownn.p[0][j] = o0 ^ dn.A;
        ownn.p[0][w + j] = o1 ^ dn.B;
      }
      return;
    }
    u64 s[NS], p[NS];
    if (rp == 0) {  // settle the generate AND (H/protocols/adder.hpp:209-223)
      const Dw dp = cwp ? dw_load(cwp, cwN, g, 0, Tp, Tp.off + g) : ew_draw_t<true, Pool>(Tp, Tp.off + g, p0);
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
        const u64* o = ownp.p[op ? 0 : slot];
        const u64* q = sel(peerp, slot);
        const u64 e = op ? o[j] : o[j] ^ q[j], d = op ? o[w + j] : o[w + j] ^ q[w + j];
        u64 a, b, c;
        ew_share<true>(Tp, party, dp, a, b, c);
        s[k] = c ^ (e & b) ^ (d & a);
        if (party == 0) s[k] ^= e & d;
        p[k] = sel(P0, slot)[g];
      }
    } else {  // settle a prefix level (H/protocols/adder.hpp:142-165)
      // Own payload is recomputed from the pre-round state instead of re-read from HBM:
      // it is a function of (s, p) and the triple, all of which this thread holds.
      const u64 kp = ks.p, gp0 = (Tp.off + g) * kPhi;  // one multiply for both triples
      const Dw d0 = cwp ? dw_load(cwp, cwN, g, 0, Tp, Tp.off + g) : ew_draw_kg<true, Pool>(Tp, kp, gp0, p0);
      const Dw d1 = cwp ? dw_load(cwp, cwN, g, 1, Tp, Tp.ghalf + Tp.off + g)
                        : ew_draw_kg<true, Pool>(Tp, kp, gp0 + Tp.ghalf * kPhi, p0);
      u64 oe0 = 0, oe1 = 0, od0 = 0, od1 = 0;  // the opened wire (pair evaluation)
      if (op) {
        const u64* o = ownp.p[0];
        oe0 = o[j], oe1 = o[w + j], od0 = o[2 * w + j], od1 = o[3 * w + j];
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
        const u64* q = sel(peerp, slot);
        u64 a0, b0, c0, a1, b1, c1;
        ew_share<true>(Tp, party, d0, a0, b0, c0);
        ew_share<true>(Tp, party, d1, a1, b1, c1);
        const u64 s0 = sel(S, slot)[g], p0s = sel(P, slot)[g];
        const u64 po = p0s & lp.out;
        const u64 e0 = op ? oe0 : (po ^ a0) ^ q[j], e1 = op ? oe1 : (po ^ a1) ^ q[w + j];
        const u64 dd0 = op ? od0 : (((s0 & lp.in) * lp.mult) ^ b0) ^ q[2 * w + j];
        const u64 dd1 = op ? od1 : (((p0s & lp.in) * lp.mult) ^ b1) ^ q[3 * w + j];
        u64 z0 = c0 ^ (e0 & b0) ^ (dd0 & a0);
        u64 z1 = c1 ^ (e1 & b1) ^ (dd1 & a1);
        if (party == 0) {
          z0 ^= e0 & dd0;
          z1 ^= e1 & dd1;
        }
        s[k] = s0 ^ z0;
        p[k] = (p0s & ~lp.out) ^ z1;
      }
    }
    if (rn <= levels) {  // issue level rn-1 (H/protocols/adder.hpp:122-140)
      // opened wire: the masks r_A, r_B cancel between the two payloads (see rn == 0)
      const bool sec = op && !cwn;
      const u64 kn = ks.n, gn0 = (Tn.off + g) * kPhi, gn1 = gn0 + Tn.ghalf * kPhi;
      const Dw d0 = sec ? ew_secrets_kg<Pool>(Tn, kn, gn0) : ew_draw_kg<false, Pool>(Tn, kn, gn0, p0);
      const Dw d1 = sec ? ew_secrets_kg<Pool>(Tn, kn, gn1) : ew_draw_kg<false, Pool>(Tn, kn, gn1, p0);
      if (cwn) {
        dw_store(cwn, cwN, g, 0, d0);
        dw_store(cwn, cwN, g, 1, d1);
      }
      u64 o[4] = {0, 0, 0, 0};  // o[1] unused: words 0 and 1 share the unmasked half po
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int slot = pair_slot<NS>(pid, slot0, k), party = pair_party<NS>(pid, slot, k);
        u64 a0, b0, a1, b1;
        ew_share<false>(Tn, party, d0, a0, b0, dummy);
        ew_share<false>(Tn, party, d1, a1, b1, dummy);
        const u64 po = p[k] & ln.out, ms = (s[k] & ln.in) * ln.mult, mp = (p[k] & ln.in) * ln.mult;
        if (op) {  // the unmasked halves; the XOR of the two parties' masks is added below
          o[0] ^= po, o[2] ^= ms, o[3] ^= mp;
        } else {
          const u64 v0 = po ^ a0, v1 = po ^ a1, v2 = ms ^ b0, v3 = mp ^ b1;
          u64* nn = sel(ownn, slot);
          nn[j] = v0;
          nn[w + j] = v1;
          nn[2 * w + j] = v2;
          nn[3 * w + j] = v3;
        }
        sel(S, slot)[g] = s[k];
        sel(P, slot)[g] = p[k];
      }
      if (op) {  // a0 ^ a1 = A, b0 ^ b1 = B for each of the two triples
        u64* nn = ownn.p[0];
        nn[j] = o[0] ^ d0.A;
        nn[w + j] = o[0] ^ d1.A;
        nn[2 * w + j] = o[2] ^ d0.B;
        nn[3 * w + j] = o[3] ^ d1.B;
      }
    } else if constexpr (NS == 2 && has_pair_ff<FF>::value) {
      const int q0 = pair_slot<2>(pid, 0, 0);
      ff.pair(q0, g, j, (sel(P0, q0)[g] ^ (s[0] << 1)) & wmask, (sel(P0, 1 - q0)[g] ^ (s[1] << 1)) & wmask);
    } else {
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int slot = pair_slot<NS>(pid, slot0, k);
        ff(slot, pid.v[slot], g, j, (sel(P0, slot)[g] ^ (s[k] << 1)) & wmask);
      }
    }
  }
};

struct SpkConsts {
  int levels;
  u64 wmask;
  SpkLevel lv[6];
};
SpkConsts make_spk_constants(int width);

struct NoPost {
  void operator()(int) const {}
};

// The issue-to-settle draw cache is used when one thread evaluates every local slot of an
// element (pair evaluation, or one party per process) and the two buffers stay L2-resident.
inline bool adder_draw_cache_ok(const Session& s, size_t n) {
  static const bool on = [] {  // measured slower on LeNet-size rounds (extra L2 traffic): opt-in
    const char* e = std::getenv("MPCG_DRAW_CACHE");
    return e && e[0] == '1';
  }();
  const bool one_thread = s.n_local == 1 || pair_eval_enabled();
  return on && one_thread && n > 0 && n * 2 * 64 <= (size_t(48) << 20);
}


// Secure binary addition of XOR-shared operands given by sources. The last kernel of each
// lane hands the sum to ff_for_lane(lane, lo, w) — a functor (slot, party, g, j, sum) that
// may already build the next protocol's payload for the same lane — and post_lane(lane)
// runs right after it (to post that payload), so a protocol tail costs no extra kernel.
template <bool Pool, class XF, class YF, class FFL, class POST>
void adder_op_t(Session& s, size_t n, const AdderOptions& opt, const std::string& tag, XF xf, YF yf,
                FFL ff_for_lane, POST post_lane) {
  using FF = decltype(ff_for_lane(0, size_t(0), size_t(0)));
  const SpkConsts c = make_spk_constants(opt.width);
  const int chunks = clamp_chunks(opt.chunks, n);  // lanes as the reference accounts them
  const int xl = chunks > 1 && s.fuse_lanes() ? 1 : chunks;  // lanes launched (Session::fuse_lanes)
  const Pid2 pid = pids(s);
  DT S = s.alloc(Shape{n}), P = s.alloc(Shape{n}), P0 = s.alloc(Shape{n});
  const int rounds = 1 + c.levels;
  DT cw[2];
  if (adder_draw_cache_ok(s, n))
    for (auto& b : cw) b = s.alloc(Shape{8 * n});
  Triple tr[7];
  auto fetch_round = [&](int r) {
    tr[r] = r == 0 ? s.fetch(TripleSpec::elementwise(TripleKind::Bin, Shape{n}), tag + ".g")
                   : s.fetch(TripleSpec::elementwise(TripleKind::Bin, Shape{2, n}),
                             tag + ".l" + std::to_string(r - 1), /*stacked=*/true);
    tr[r].mark_consumed();
  };
  auto round_tag = [&](int r, int lane) {
    std::string t = r == 0 ? tag + ".g" : tag + ".l" + std::to_string(r - 1);
    return chunks > 1 && !opt.merged ? t + ".chunk" + std::to_string(lane) : t;
  };
  std::vector<Open> hs(static_cast<size_t>(xl));
  auto post_round = [&](int r, int lane) {
    if (xl == chunks) s.post(hs[lane], round_tag(r, lane));
    else s.post_lanes(hs[lane], n, chunks, r == 0 ? 2 : 4, [&](int k) { return round_tag(r, k); });
  };
  auto kernel = [&](int rp, int rn, int lane, Open* prev, Open* next) {
    const auto rng_ = chunk_range(n, xl, lane);
    const size_t lo = rng_.first, hi = rng_.second;
    AdderRound<XF, YF, FF, Pool> k{};
    k.rp = rp;
    k.rn = rn;
    k.levels = c.levels;
    if (rp >= 0) k.Tp = tr[rp].ew;
    if (rn <= c.levels) k.Tn = tr[rn].ew;
    if (rp >= 1) k.lp = c.lv[rp - 1];
    if (rn >= 1 && rn <= c.levels) k.ln = c.lv[rn - 1];
    k.pid = pid;
    if (prev) {
      k.ownp = as_const(own_ptrs(*prev));
      k.peerp = peer_ptrs(*prev);
    }
    if (next) k.ownn = own_ptrs(*next);
    k.S = ptrs(S);
    k.P = ptrs(P);
    k.P0 = ptrs(P0);
    k.lo = lo;
    k.w = hi - lo;
    k.wmask = c.wmask;
    k.xf = xf;
    k.yf = yf;
    if (cw[0]) {
      k.cwN = n;
      if (rp >= 0) k.cwp = cw[rp & 1].s[0];
      if (rn <= c.levels) k.cwn = cw[rn & 1].s[0];
    }
    if (rn > c.levels) k.ff = ff_for_lane(lane, lo, hi - lo);
    // algorithmic bytes per element per party (2 x wire + 8 x (in + out)):
    // level round = 2x32 wire + 8x(2 state in + 2 state out) = 96 B. With the opened wire (pair
    // evaluation) the 32-byte opened value is written once and read once per element pair, so
    // the form needs 64 B per element per party; the roofline counts the bytes of the form run.
    const double bpe = s.n_local == 2 && pair_eval_enabled() ? 64.0 : 96.0;
    ClassScope cs(rn >= 1 && rn <= c.levels ? kClsAdderRound : kClsOther, bpe * double(hi - lo) * s.n_local);
    launch_ew(s.stream, s.n_local, hi - lo, k);
  };
  fetch_round(0);
  for (int lane = 0; lane < xl; ++lane) {
    const auto rng_ = chunk_range(n, xl, lane);
    hs[lane] = s.begin_open(2 * (rng_.second - rng_.first), Reduce::Xor);
    kernel(-1, 0, lane, nullptr, &hs[lane]);
    post_round(0, lane);
  }
  for (int r = 1; r < rounds; ++r) {
    fetch_round(r);
    for (int lane = 0; lane < xl; ++lane) {
      const auto rng_ = chunk_range(n, xl, lane);
      Open next = s.begin_open(4 * (rng_.second - rng_.first), Reduce::Xor);
      s.wait(hs[lane]);
      kernel(r - 1, r, lane, &hs[lane], &next);
      hs[lane] = std::move(next);
      post_round(r, lane);
    }
  }
  for (int lane = 0; lane < xl; ++lane) {
    s.wait(hs[lane]);
    kernel(rounds - 1, rounds, lane, &hs[lane], nullptr);
    post_lane(lane);
  }
  s.check();
}

// The SPK adder rounds are the hottest kernels: they are instantiated per triple source so the
// seeded-dealer build keeps its straight-line code (queue mode: triples read from HBM).
template <class XF, class YF, class FFL, class POST = NoPost>
void adder_op(Session& s, size_t n, const AdderOptions& opt, const std::string& tag, XF xf, YF yf,
              FFL ff_for_lane, POST post_lane = NoPost{}) {
  if (s.source_q)
    adder_op_t<true>(s, n, opt, tag, xf, yf, ff_for_lane, post_lane);
  else
    adder_op_t<false>(s, n, opt, tag, xf, yf, ff_for_lane, post_lane);
}

// ---------------------------------------------------------------- persistent round chain
// Launch geometry of a persistent chain over n elements: one element per thread per round, in
// CTAs of 256 threads, or smaller CTAs when n is small so the chain spreads over more SMs (a
// round's cost is one element's dealer-draw latency on a lightly loaded sub-partition, plus the
// grid barrier). MPCG_CHAIN_TPB forces a CTA size.
inline unsigned chain_tpb(u64 n) {
  static const int forced = [] {
    const char* e = std::getenv("MPCG_CHAIN_TPB");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 64 || forced == 128 || forced == 256) return unsigned(forced);
  const u64 sms = u64(num_sms());
  return n <= sms * 64 ? 64u : n <= sms * 128 ? 128u : 256u;
}
// In 1-GPU mode an open is only an ordering point between the two party slots, so a whole
// chain of secure rounds can run as ONE cooperative kernel: each round is a grid-stride
// pass over the elements, and a grid-wide barrier (release/acquire at gpu scope) takes the
// place of the kernel boundary. Round logic is the same functors as the multi-kernel path.
#ifndef MPCG_BARRIER_SLEEP
#define MPCG_BARRIER_SLEEP 20
#endif
constexpr unsigned kBarrierSleep = MPCG_BARRIER_SLEEP;  // ns between polls of the grid barrier
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      if (kBarrierSleep) __nanosleep(kBarrierSleep);
    }
  }
  __syncthreads();
}

template <class MR, class AR, class BR, class CR>
struct ChainParams {
  MR mask;       // a2b mask + p2p payload
  AR adder[8];   // round 0 issue, 6 x (settle, issue), final (+ b2a build)
  int nadder;
  BR b2a;        // b2a combine + select build
  CR fin;        // select combine -> output sink
  u64 n;
  unsigned* bar;
  int pair;       // one thread evaluates both local slots (grid y == 1)
  int skip_mask;  // the mask is folded into the adder's generate round (pair evaluation)
};

template <class MR, class AR, class BR, class CR>
__global__ void __launch_bounds__(256) chain_kernel(const __grid_constant__ ChainParams<MR, AR, BR, CR> p) {
  const int slot = blockIdx.y;
  const bool pr = p.pair != 0;
  const unsigned nb = gridDim.x * gridDim.y;
  const u64 t0 = blockIdx.x * u64(blockDim.x) + threadIdx.x, st = u64(gridDim.x) * blockDim.x;
  unsigned ep = 0;
  if (!p.skip_mask) {
    for (u64 g = t0; g < p.n; g += st) eval_slots(p.mask, pr, slot, g);
    grid_barrier(p.bar, ++ep * nb);
  }
  for (int r = 0; r < p.nadder; ++r) {
    for (u64 g = t0; g < p.n; g += st) eval_slots(p.adder[r], pr, slot, g);
    grid_barrier(p.bar, ++ep * nb);
  }
  for (u64 g = t0; g < p.n; g += st) eval_slots(p.b2a, pr, slot, g);
  grid_barrier(p.bar, ++ep * nb);
  for (u64 g = t0; g < p.n; g += st) eval_slots(p.fin, pr, slot, g);
}

// Pair evaluation with in-device opens: round r+1 of element g reads only element g's adder
// state and opened wire, which the same thread wrote in round r (the SPK levels shift inside
// the 64-bit word; the b2a and the multiply are elementwise), so the whole chain runs element
// by element in one ordinary kernel — no grid barrier, and the round-to-round state is re-read
// from L1/L2 while it is hot instead of from HBM a whole pass later. Same functors and values
// as chain_kernel; the opens are still posted / accounted by the launcher.
template <class MR, class AR, class BR, class CR>
__global__ void __launch_bounds__(256) chain_pair_kernel(const __grid_constant__ ChainParams<MR, AR, BR, CR> p) {
  const u64 t0 = blockIdx.x * u64(blockDim.x) + threadIdx.x, st = u64(gridDim.x) * blockDim.x;
  for (u64 g = t0; g < p.n; g += st) {
    if (!p.skip_mask) eval_slots(p.mask, true, 0, g);
    for (int r = 0; r < p.nadder; ++r) eval_slots(p.adder[r], true, 0, g);
    eval_slots(p.b2a, true, 0, g);
    eval_slots(p.fin, true, 0, g);
  }
}

constexpr int kMaxChainSteps = 24;
template <class B0, class ST>
struct BeaverChainParams {
  B0 build;
  ST steps[kMaxChainSteps];
  int nsteps;
  u64 n;
  unsigned* bar;
  int pair;
};

template <class B0, class ST>
__global__ void __launch_bounds__(256) beaver_chain_kernel(const __grid_constant__ BeaverChainParams<B0, ST> p) {
  const int slot = blockIdx.y;
  const bool pr = p.pair != 0;
  const unsigned nb = gridDim.x * gridDim.y;
  const u64 t0 = blockIdx.x * u64(blockDim.x) + threadIdx.x, stride = u64(gridDim.x) * blockDim.x;
  unsigned ep = 0;
  for (u64 g = t0; g < p.n; g += stride) eval_slots(p.build, pr, slot, g);
  for (int r = 0; r < p.nsteps; ++r) {
    grid_barrier(p.bar, ++ep * nb);
    for (u64 g = t0; g < p.n; g += stride) eval_slots(p.steps[r], pr, slot, g);
  }
}

// Pair evaluation with in-device opens: each round of a Beaver chain (exp squares, Newton
// steps) is elementwise and its opened wire for element g is written and read by the same
// thread, so the chain runs element by element with no grid barrier (as chain_pair_kernel).
template <class B0, class ST>
__global__ void __launch_bounds__(256) beaver_chain_pair_kernel(const __grid_constant__ BeaverChainParams<B0, ST> p) {
  const u64 t0 = blockIdx.x * u64(blockDim.x) + threadIdx.x, stride = u64(gridDim.x) * blockDim.x;
  for (u64 g = t0; g < p.n; g += stride) {
    eval_slots(p.build, true, 0, g);
    for (int r = 0; r < p.nsteps; ++r) eval_slots(p.steps[r], true, 0, g);
  }
}

template <class B0, class ST>
void persistent_beaver_chain(Session& s, u64 n, const B0& build, const std::vector<ST>& steps) {
  if (steps.size() > size_t(kMaxChainSteps)) throw Error(kInternalError, "beaver chain too long");
  if (pair_chain_ok(s)) {  // element by element (beaver_chain_pair_kernel), any size
    BeaverChainParams<B0, ST> p{};
    p.build = build;
    for (size_t i = 0; i < steps.size(); ++i) p.steps[i] = steps[i];
    p.nsteps = int(steps.size());
    p.n = n;
    p.pair = 1;
    ClassScope cs(kClsOther, 0);
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    const u64 blocks = std::min<u64>((n + 255) / 256, u64(num_sms()) * 16);
    beaver_chain_pair_kernel<B0, ST><<<unsigned(blocks), 256, 0, s.stream>>>(p);
    MPCG_CUDA(cudaGetLastError());
    probe_end(s.stream, pe);
    return;
  }
  BeaverChainParams<B0, ST> p{};
  p.build = build;
  for (size_t i = 0; i < steps.size(); ++i) p.steps[i] = steps[i];
  p.nsteps = int(steps.size());
  p.n = n;
  p.pair = s.n_local == 2 && pair_eval_enabled();
  DT bar = s.alloc(Shape{1});
  MPCG_CUDA(cudaMemsetAsync(bar.s[0], 0, 8, s.stream));
  p.bar = reinterpret_cast<unsigned*>(bar.s[0]);
  const unsigned gy = p.pair ? 1u : unsigned(s.n_local);
  auto kern = beaver_chain_kernel<B0, ST>;
  static int per_sm = -1;
  if (per_sm < 0) {
    MPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    if (per_sm < 1) throw Error(kInternalError, "beaver chain kernel cannot be resident");
  }
  const unsigned tpb = chain_tpb(n);
  const u64 cap = u64(per_sm) * (256 / tpb) * num_sms() / gy;  // residency measured at 256 threads
  u64 blocks = (n + tpb - 1) / tpb;
  blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(unsigned(blocks), gy);
  lc.blockDim = dim3(tpb);
  lc.stream = s.stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  lc.attrs = &attr;
  lc.numAttrs = 1;
  cudaEvent_t pe;
  probe_begin(s.stream, &pe);
  MPCG_CUDA(cudaLaunchKernelEx(&lc, kern, p));
  probe_end(s.stream, pe);
}

// Plain final sinks for adder_op (same functor for every lane).
struct SumSink {  // binary share of the sum
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64, u64 sum) const { sel(out, slot)[g] = sum; }
};
struct MsbSink {  // sign bit in position 0 (H/protocols/compare.hpp:57-62)
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64, u64 sum) const { sel(out, slot)[g] = sum >> 63; }
};
template <class FF>
struct SameFF {
  FF f;
  FF operator()(int, size_t, size_t) const { return f; }
};
template <class FF>
SameFF<FF> same(FF f) {
  return SameFF<FF>{f};
}

}  // namespace mpcg
