// Secure protocols on device shares: Beaver mul/square/AND, SPK adder, conversions,
// comparison-based activations and the exp/reciprocal/softmax chain.
// Reference: H/protocols/{beaver,adder,compare,trunc}.hpp, H/nonlinear/{approx,activations}.hpp.
#include <cmath>

#include "ew.cuh"

namespace mpcg {

void require_same_shape(const DT& a, const DT& b, const char* op) {
  if (a.shape != b.shape)
    throw Error(kShapeError, std::string(op) + ": shape mismatch " + shape_str(a.shape) + " vs " +
                                 shape_str(b.shape));
}

int clamp_chunks(int chunks, size_t numel) {
  if (chunks < 1) chunks = 1;
  return int(std::min<size_t>(size_t(chunks), numel ? numel : 1));
}

int chunks_for(const Session& s, size_t numel) {
  if (s.cfg.chunks <= 1) return 1;
  if (s.cfg.chunk_threshold != 0 && numel * sizeof(u64) < s.cfg.chunk_threshold) return 1;
  return s.cfg.chunks;
}

static AdderOptions adder_for(const Session& s, size_t numel) {
  AdderOptions o;
  o.merged = s.cfg.merged_adder;
  o.chunks = chunks_for(s, numel);
  return o;
}

SpkConsts make_spk_constants(int width) {
  // H/protocols/adder.hpp:37-57
  if (width < 2 || width > 64 || (width & (width - 1)))
    throw Error(kConfigError, "adder width must be a power of two in [2, 64]");
  SpkConsts c{};
  int m = 0;
  while ((1 << m) < width) ++m;
  c.levels = m;
  c.wmask = width == 64 ? ~u64(0) : ((u64(1) << width) - 1);
  for (int i = 0; i < m; ++i) {
    u64 in = 0, out = 0;
    const u64 half = u64(1) << i;
    for (int p = 0; p < width; ++p) {
      const u64 r = u64(p) & (2 * half - 1);
      if (r == half - 1) in |= u64(1) << p;
      if (r >= half) out |= u64(1) << p;
    }
    c.lv[i] = SpkLevel{in, out, ((u64(1) << half) - 1) << 1};
  }
  return c;
}

// ---------------------------------------------------------------- local helpers
DT reshape(const DT& a, Shape shape) {
  if (shape_numel(shape) != a.numel())
    throw Error(kShapeError, "reshape: numel mismatch " + shape_str(a.shape) + " -> " + shape_str(shape));
  DT t = a;
  t.shape = std::move(shape);
  return t;
}

DT add_public(Session& s, const DT& x, u64 v) {
  DT z = s.alloc(x.shape, x.scale);
  const Pid2 pid = pids(s);
  const CPtr2 xp = cptrs(x);
  const Ptr2 zp = ptrs(z);
  launch_ew(s.stream, s.n_local, x.numel(), [=] __device__(int slot, u64 i) {
    sel(zp, slot)[i] = sel(xp, slot)[i] + (pid.v[slot] == 0 ? v : 0);
  });
  return z;
}

DT scale_public(Session& s, const DT& x, u64 k) {
  DT z = s.alloc(x.shape, x.scale);
  const CPtr2 xp = cptrs(x);
  const Ptr2 zp = ptrs(z);
  launch_ew(s.stream, s.n_local, x.numel(), [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sel(xp, slot)[i] * k; });
  return z;
}

DT sub_t(Session& s, const DT& a, const DT& b) {
  require_same_shape(a, b, "sub");
  DT z = s.alloc(a.shape, a.scale);
  const CPtr2 ap = cptrs(a), bp = cptrs(b);
  const Ptr2 zp = ptrs(z);
  launch_ew(s.stream, s.n_local, a.numel(),
            [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sel(ap, slot)[i] - sel(bp, slot)[i]; });
  return z;
}

DT add_t(Session& s, const DT& a, const DT& b) {
  require_same_shape(a, b, "add");
  DT z = s.alloc(a.shape, a.scale);
  const CPtr2 ap = cptrs(a), bp = cptrs(b);
  const Ptr2 zp = ptrs(z);
  launch_ew(s.stream, s.n_local, a.numel(),
            [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sel(ap, slot)[i] + sel(bp, slot)[i]; });
  return z;
}

// 2PC truncation: local arithmetic shift of each share (H/protocols/trunc.hpp:25-42).
DT truncate_shares(Session& s, const DT& x, int bits) {
  DT z = s.alloc(x.shape, x.scale);
  const CPtr2 xp = cptrs(x);
  const Ptr2 zp = ptrs(z);
  launch_ew(s.stream, s.n_local, x.numel(),
            [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sar64(sel(xp, slot)[i], bits); });
  return z;
}

// Reveal: every slot receives the reconstructed value (Communicator::reveal).
DT open_value(Session& s, const DT& x, Reduce kind, const std::string& tag) {
  const size_t n = x.numel();
  DT z = s.alloc(x.shape, x.scale);
  Open o = s.begin_open(n, kind);
  const Ptr2 own = own_ptrs(o);
  const CPtr2 xp = cptrs(x);
  launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) { sel(own, slot)[i] = sel(xp, slot)[i]; });
  s.post(o, tag);
  s.wait(o);
  const CPtr2 ow = as_const(own_ptrs(o)), pe = peer_ptrs(o);
  const Ptr2 zp = ptrs(z);
  const int xr = kind == Reduce::Xor;
  launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) {
    const u64 a = sel(ow, slot)[i], b = sel(pe, slot)[i];
    sel(zp, slot)[i] = xr ? (a ^ b) : (a + b);
  });
  s.check();
  return z;
}

// ---------------------------------------------------------------- Beaver ops
DT beaver_mul(Session& s, const DT& x, const DT& y, const std::string& tag, int chunks) {
  require_same_shape(x, y, "beaver_mul");
  Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, x.shape), tag);
  t.mark_consumed();
  DT z = s.alloc(x.shape, x.scale);
  mul_op(s, t.ew, x.numel(), chunks, tag, SrcMem{cptrs(x)}, SrcMem{cptrs(y)}, SinkStore{ptrs(z)});
  return z;
}

DT beaver_square(Session& s, const DT& x, const std::string& tag, int chunks) {
  Triple t = s.fetch(TripleSpec::square_of(x.shape), tag);
  t.mark_consumed();
  DT z = s.alloc(x.shape, x.scale);
  square_op(s, t.ew, x.numel(), chunks, tag, SrcMem{cptrs(x)}, SinkStore{ptrs(z)});
  return z;
}

namespace {
template <class XF, class YF>
struct AndBuild {
  EwTriple T;
  Pid2 pid;
  Ptr2 own;
  u64 lo, w;
  XF xf;
  YF yf;
  __device__ void operator()(int slot, u64 j) const {
    const u64 g = lo + j;
    u64 a, b;
    ew_ab(T, pid.v[slot], T.off + g, a, b);
    sel(own, slot)[j] = xf(slot, g) ^ a;
    sel(own, slot)[w + j] = yf(slot, g) ^ b;
  }
};
struct AndCombine {
  EwTriple T;
  Pid2 pid;
  CPtr2 own, peer;
  Ptr2 out;
  u64 lo, w;
  __device__ void operator()(int slot, u64 j) const {
    const int party = pid.v[slot];
    const u64 g = lo + j;
    const u64 e = sel(own, slot)[j] ^ sel(peer, slot)[j];
    const u64 d = sel(own, slot)[w + j] ^ sel(peer, slot)[w + j];
    u64 a, b, c;
    ew_abc(T, party, T.off + g, a, b, c);
    u64 z = c ^ (e & b) ^ (d & a);
    if (party == 0) z ^= e & d;
    sel(out, slot)[g] = z;
  }
};
}  // namespace

DT beaver_and(Session& s, const DT& x, const DT& y, const std::string& tag, int chunks) {
  require_same_shape(x, y, "beaver_and");
  Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Bin, x.shape), tag);
  t.mark_consumed();
  const size_t m = x.numel();
  chunks = clamp_chunks(chunks, m);
  const int acct = chunks;
  const int xl = acct > 1 && s.fuse_lanes() ? 1 : acct;  // lanes launched (Session::fuse_lanes)
  auto ltag = [&](int k) { return acct == 1 ? tag : tag + ".chunk" + std::to_string(k); };
  DT z = s.alloc(x.shape, x.scale);
  const Pid2 pid = pids(s);
  std::vector<Open> opens(static_cast<size_t>(xl));
  for (int k = 0; k < xl; ++k) {
    const auto rng_ = chunk_range(m, xl, k); const size_t lo = rng_.first, hi = rng_.second;
    opens[k] = s.begin_open(2 * (hi - lo), Reduce::Xor);
    launch_ew(s.stream, s.n_local, hi - lo,
              AndBuild<SrcMem, SrcMem>{t.ew, pid, own_ptrs(opens[k]), lo, hi - lo, SrcMem{cptrs(x)}, SrcMem{cptrs(y)}});
    if (xl == acct) s.post(opens[k], ltag(k));
    else s.post_lanes(opens[k], m, acct, 2, ltag);
  }
  for (int k = 0; k < xl; ++k) {
    const auto rng_ = chunk_range(m, xl, k); const size_t lo = rng_.first, hi = rng_.second;
    s.wait(opens[k]);
    launch_ew(s.stream, s.n_local, hi - lo,
              AndCombine{t.ew, pid, as_const(own_ptrs(opens[k])), peer_ptrs(opens[k]), ptrs(z), lo, hi - lo});
  }
  s.check();
  return z;
}

// ---------------------------------------------------------------- adder / conversions
DT binary_add(Session& s, const DT& x, const DT& y, const AdderOptions& opt, const std::string& tag) {
  require_same_shape(x, y, "binary_add");
  DT z = s.alloc(x.shape, x.scale);
  adder_op(s, x.numel(), opt, tag, SrcMem{cptrs(x)}, SrcMem{cptrs(y)}, same(SumSink{ptrs(z)}));
  return z;
}

namespace {
// a2b parts in 2PC (H/protocols/compare.hpp:31-53): party 0 adds (keep0, r1), party 1 (r0, keep1).
struct PartX {
  Pid2 pid;
  CPtr2 keep, peer;
  __device__ u64 operator()(int slot, u64 g) const {
    return pid.v[slot] == 0 ? sel(keep, slot)[g] : sel(peer, slot)[g];
  }
};
struct PartY {
  Pid2 pid;
  CPtr2 keep, peer;
  __device__ u64 operator()(int slot, u64 g) const {
    return pid.v[slot] == 0 ? sel(peer, slot)[g] : sel(keep, slot)[g];
  }
};

// Mask draw + p2p send of r, keep = x ^ r (H/protocols/compare.hpp:31-46).
template <class XF>
DT a2b_mask(Session& s, size_t n, XF xf, Open& o) {
  DT keep = s.alloc(Shape{n});
  const Session::MaskRef mr = s.take_mask(n);
  o = s.begin_open(n, Reduce::Sum);
  const Ptr2 own = own_ptrs(o), kp = ptrs(keep);
  const u64 k0 = s.mask_key[0], k1 = s.mask_key[1];
  launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) {
    const u64 r = drw(slot == 0 ? k0 : k1, tkey(mr.base, mr.bp) + 1 + i);
    sel(own, slot)[i] = r;
    sel(kp, slot)[i] = xf(slot, i) ^ r;
  });
  s.post(o, "", /*p2p=*/true);
  s.wait(o);
  return keep;
}

// The a2b mask folded into the adder's generate round (pair evaluation): the adder operands
// PartX / PartY computed from x and the two parties' mask draws directly instead of read back
// from keep = x ^ r and the peer's mask outbox. Operand y = 0 (X): party 0 holds x ^ r and
// party 1 the peer's r; y = 1 (Y): the other way round.
template <class XF>
struct MaskedPart {
  Pid2 pid;
  u64 k0, k1;
  Session::MaskRef mr;
  XF xf;
  int y;
  __device__ u64 operator()(int slot, u64 g) const {
    const u64 c = tkey(mr.base, mr.bp) + 1 + g;
    const int party = slot ? pid.v[1] : pid.v[0];  // select: no local copy of pid
    if ((party == 0) == (y == 0)) return xf(slot, g) ^ drw(slot == 0 ? k0 : k1, c);  // keep
    return drw(slot == 0 ? k1 : k0, c);  // the peer slot's mask r
  }
};

// Adder operand of the a2b: from keep = x ^ r and the peer's mask outbox (PartX / PartY), or,
// when `fused` (pair evaluation), straight from x and the two mask draws (MaskedPart).
template <class XF>
struct A2bPart {
  Pid2 pid;
  CPtr2 keep, peer;
  u64 k0, k1;
  Session::MaskRef mr;
  XF xf;
  int y;  // 0 = X operand, 1 = Y operand
  int fused;
  __device__ u64 operator()(int slot, u64 g) const {
    if (fused) return MaskedPart<XF>{pid, k0, k1, mr, xf, y}(slot, g);
    return (pid.v[slot] == 0) == (y == 0) ? sel(keep, slot)[g] : sel(peer, slot)[g];
  }
};

template <class XF, class FFL, class POST = NoPost>
void a2b_op(Session& s, size_t n, const AdderOptions& opt, const std::string& tag, XF xf, FFL ffl,
            POST post = NoPost{}) {
  const Pid2 pid = pids(s);
  if (adder_opened_wire(s)) {  // one thread plays both parties: no mask kernel, no keep tensor
    const Session::MaskRef mr = s.take_mask(n);
    Open o = s.begin_open(n, Reduce::Sum);
    s.post(o, "", /*p2p=*/true);  // the mask exchange, accounted as the reference sends it
    s.wait(o);
    adder_op(s, n, opt, tag + ".add1", MaskedPart<XF>{pid, s.mask_key[0], s.mask_key[1], mr, xf, 0},
             MaskedPart<XF>{pid, s.mask_key[0], s.mask_key[1], mr, xf, 1}, ffl, post);
    return;
  }
  Open o;
  DT keep = a2b_mask(s, n, xf, o);
  adder_op(s, n, opt, tag + ".add1", PartX{pid, cptrs(keep), peer_ptrs(o)}, PartY{pid, cptrs(keep), peer_ptrs(o)},
           ffl, post);
}

// b2a_bit (H/protocols/compare.hpp:67-83, n=2): acc = b0 on party 0, bq = b1 on party 1;
// result acc + bq - 2*acc*bq.
struct BitAcc {
  Pid2 pid;
  CPtr2 b;
  __device__ u64 operator()(int slot, u64 g) const { return pid.v[slot] == 0 ? (sel(b, slot)[g] & 1) : 0; }
};
struct BitBq {
  Pid2 pid;
  CPtr2 b;
  __device__ u64 operator()(int slot, u64 g) const { return pid.v[slot] == 1 ? (sel(b, slot)[g] & 1) : 0; }
};
struct B2aSink {
  CPtr2 b;
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64 prod) const {
    sel(out, slot)[g] = (sel(b, slot)[g] & 1) - (prod + prod);
  }
};

// ---- fused comparison tail ----------------------------------------------------------
// adder final (lane k) -> msb bit -> b2a ".m1" payload of chunk k, in the same kernel.
struct B2aBuildFF {
  EwTriple T;
  Ptr2 own, bits;
  u64 lo, w;
  bool opened = false;  // pair evaluation: the opened (eps, delta) once in slot 0's outbox
  __device__ void operator()(int slot, int party, u64 g, u64 j, u64 sum) const {
    const u64 bit = sum >> 63;
    sel(bits, slot)[g] = bit;
    u64 a, b;
    ew_ab(T, party, T.off + g, a, b);
    sel(own, slot)[j] = (party == 0 ? bit : 0) - a;      // eps = acc - a
    sel(own, slot)[w + j] = (party == 1 ? bit : 0) - b;  // delta = bq - b
  }
  // both parties (sum_k = party k's, q0 = slot of party 0)
  __device__ void pair(int q0, u64 g, u64 j, u64 sum0, u64 sum1) const {
    if (!opened) {
      (*this)(q0, 0, g, j, sum0);
      (*this)(1 - q0, 1, g, j, sum1);
      return;
    }
    const u64 bit0 = sum0 >> 63, bit1 = sum1 >> 63;
    sel(bits, q0)[g] = bit0;
    sel(bits, 1 - q0)[g] = bit1;
    const Dw d = ew_secrets(T, T.off + g);  // eps0 + eps1 = bit0 - A, delta0 + delta1 = bit1 - B
    own.p[0][j] = bit0 - d.A;
    own.p[0][w + j] = bit1 - d.B;
  }
};
// b2a combine (c = bit - 2*prod) -> payload of the multiply by c, chunk k, same kernel.
template <class UF>
struct MulByBitBuild {
  EwTriple T;
  Ptr2 own;
  CPtr2 bits;
  u64 lo, w;
  UF uf;
  Ptr2 cout;  // optional: keep the arithmetic bit c (sigmoid's select reuses it)
  bool opened = false;  // pair evaluation: the opened (eps, delta) once in slot 0's outbox
  __device__ void operator()(int slot, int party, u64 g, u64 prod) const {
    const u64 c = (sel(bits, slot)[g] & 1) - (prod + prod);
    if (sel(cout, slot)) sel(cout, slot)[g] = c;
    const u64 j = g - lo;
    u64 a, b;
    ew_ab(T, party, T.off + g, a, b);
    sel(own, slot)[j] = uf(slot, g) - a;
    sel(own, slot)[w + j] = c - b;
  }
  __device__ void pair(int q0, u64 g, u64 prod0, u64 prod1) const {
    if (!opened) {
      (*this)(q0, 0, g, prod0);
      (*this)(1 - q0, 1, g, prod1);
      return;
    }
    const int q1 = 1 - q0;
    const u64 c0 = (sel(bits, q0)[g] & 1) - (prod0 + prod0), c1 = (sel(bits, q1)[g] & 1) - (prod1 + prod1);
    if (sel(cout, q0)) sel(cout, q0)[g] = c0;
    if (sel(cout, q1)) sel(cout, q1)[g] = c1;
    const u64 j = g - lo;
    const Dw d = ew_secrets(T, T.off + g);  // the masks cancel in the open
    own.p[0][j] = uf(q0, g) + uf(q1, g) - d.A;
    own.p[0][w + j] = c0 + c1 - d.B;
  }
};

// z = u * b2a(msb(d)) with every round one kernel: the 2PC compare-and-select behind ReLU
// (H/nonlinear/activations.hpp:39-47) and the tournament pick (activations.hpp:62-70).
// Tags and collective order are the reference's; chunk lanes must align (they do for every
// caller in the reference: adder, b2a and the multiply all use chunks_for(numel)).
// a2b mask round as a functor (persistent chain form of a2b_mask).
template <class XF>
struct MaskRound {
  u64 k0, k1;
  Session::MaskRef mr;
  Ptr2 own, keep;
  XF xf;
  __device__ void operator()(int slot, u64 i) const {
    const u64 r = drw(slot == 0 ? k0 : k1, tkey(mr.base, mr.bp) + 1 + i);
    sel(own, slot)[i] = r;
    sel(keep, slot)[i] = xf(slot, i) ^ r;
  }
};

// Register form of the element-by-element chain (pair evaluation, seeded dealer, 64-bit
// adder): the round algebra of AdderRound::step<2> (opened wire), B2aBuildFF::pair,
// MulCombine and MulByBitBuild::pair, with the adder state (s, p, P0), the opened wires and
// the bits held in registers instead of memory, and each triple's secrets A, B drawn once for
// its issue and reused by its settle (the per-round kernels redraw them a launch later). Only
// the input x (through the sources) and the sink's output touch HBM.
template <class DF, class UF, class PF>
using ChainP = ChainParams<MaskRound<DF>, AdderRound<A2bPart<DF>, A2bPart<DF>, B2aBuildFF>,
                           MulCombine<MulByBitBuild<UF>>, MulCombine<PF>>;

// the masks r_A, r_B, r_C of element gp (= global index * phi) with the secrets A, B given
__device__ __forceinline__ Dw masks_with(const EwTriple& t, u64 key, u64 gp, const Dw& sec) {
  Dw d;
  d.A = sec.A;
  d.B = sec.B;
  d.ra = mix64(key + t.pra + gp);
  d.rb = mix64(key + t.prb + gp);
  d.rc = mix64(key + t.prc + gp);
  return d;
}

template <class DF, class UF, class PF>
__global__ void __launch_bounds__(256) chain_reg_kernel(const __grid_constant__ ChainP<DF, UF, PF> p) {
  const Pid2 pid = p.adder[0].pid;
  const int q0 = pid.v[0] == 0 ? 0 : 1, q1 = 1 - q0;  // slots of party 0 and party 1
  constexpr int L = 6;                               // SPK levels of the 64-bit adder
  const u64 t0 = blockIdx.x * u64(blockDim.x) + threadIdx.x, st = u64(gridDim.x) * blockDim.x;
  for (u64 g = t0; g < p.n; g += st) {
    // round 0: issue the generate AND (x ^ a | y ^ b), opened
    const auto& R0 = p.adder[0];
    const u64 x0 = R0.xf(q0, g), x1 = R0.xf(q1, g), y0 = R0.yf(q0, g), y1 = R0.yf(q1, g);
    const u64 P0a = x0 ^ y0, P0b = x1 ^ y1;
    u64 s0, s1, pa, pb;
    {
      const EwTriple& T = R0.Tn;
      const u64 key = tkey(T.key, T.kp), gp = (T.off + g) * kPhi;
      const Dw dn = ew_secrets_kg<false>(T, key, gp);
      const u64 e = (x0 ^ x1) ^ dn.A, d = (y0 ^ y1) ^ dn.B;
      // round 1 settles it (adder.hpp:209-223)
      const Dw dp = masks_with(T, key, gp, dn);
      const u64 a0 = dp.A ^ dp.ra, b0 = dp.B ^ dp.rb, c0 = (dp.A & dp.B) ^ dp.rc;
      s0 = c0 ^ (e & b0) ^ (d & a0) ^ (e & d);
      s1 = dp.rc ^ (e & dp.rb) ^ (d & dp.ra);
      pa = P0a;
      pb = P0b;
    }
#pragma unroll  // constant parameter offsets: the triples' fields fold into the instructions
    for (int r = 1; r <= L; ++r) {  // issue level r-1 (adder.hpp:122-140), settle it (142-165)
      const auto& R = p.adder[r];
      const EwTriple& T = R.Tn;
      const SpkLevel lv = R.ln;
      const u64 key = tkey(T.key, T.kp), gp0 = (T.off + g) * kPhi, gp1 = gp0 + T.ghalf * kPhi;
      const Dw d0 = ew_secrets_kg<false>(T, key, gp0), d1 = ew_secrets_kg<false>(T, key, gp1);
      const u64 po = (pa & lv.out) ^ (pb & lv.out);
      const u64 w0 = po ^ d0.A, w1 = po ^ d1.A;
      const u64 w2 = (((s0 & lv.in) * lv.mult) ^ ((s1 & lv.in) * lv.mult)) ^ d0.B;
      const u64 w3 = (((pa & lv.in) * lv.mult) ^ ((pb & lv.in) * lv.mult)) ^ d1.B;
      const Dw e0 = masks_with(T, key, gp0, d0), e1 = masks_with(T, key, gp1, d1);
      // party 0 (absorbs the secrets) and party 1 (the masks)
      const u64 a00 = e0.A ^ e0.ra, b00 = e0.B ^ e0.rb, c00 = (e0.A & e0.B) ^ e0.rc;
      const u64 a01 = e1.A ^ e1.ra, b01 = e1.B ^ e1.rb, c01 = (e1.A & e1.B) ^ e1.rc;
      const u64 z0a = c00 ^ (w0 & b00) ^ (w2 & a00) ^ (w0 & w2);
      const u64 z1a = c01 ^ (w1 & b01) ^ (w3 & a01) ^ (w1 & w3);
      const u64 z0b = e0.rc ^ (w0 & e0.rb) ^ (w2 & e0.ra);
      const u64 z1b = e1.rc ^ (w1 & e1.rb) ^ (w3 & e1.ra);
      s0 ^= z0a;
      s1 ^= z0b;
      pa = (pa & ~lv.out) ^ z1a;
      pb = (pb & ~lv.out) ^ z1b;
    }
    // final round: sums -> msb bits -> b2a ".m1" open (B2aBuildFF::pair)
    const auto& RF = p.adder[L + 1];
    const u64 bit0 = ((P0a ^ (s0 << 1)) & RF.wmask) >> 63, bit1 = ((P0b ^ (s1 << 1)) & RF.wmask) >> 63;
    const EwTriple& T1 = RF.ff.T;
    const u64 k1 = tkey(T1.key, T1.kp), g1 = (T1.off + g) * kPhi;
    const Dw t1 = ew_secrets_kg<false>(T1, k1, g1);
    const u64 eB = bit0 - t1.A, dB = bit1 - t1.B;
    // b2a combine (MulCombine over T1): prod_k, then MulByBitBuild::pair
    const Dw m1 = masks_with(T1, k1, g1, t1);
    const u64 prod0 = (m1.A * m1.B - m1.rc) + (eB * (m1.B - m1.rb) + dB * (m1.A - m1.ra)) + eB * dB;
    const u64 prod1 = m1.rc + (eB * m1.rb + dB * m1.ra);
    const auto& MB = p.b2a.pf;
    const u64 c0 = (bit0 & 1) - (prod0 + prod0), c1 = (bit1 & 1) - (prod1 + prod1);
    u64* const co0 = q0 ? MB.cout.p[1] : MB.cout.p[0];
    u64* const co1 = q0 ? MB.cout.p[0] : MB.cout.p[1];
    if (co0) co0[g] = c0;
    if (co1) co1[g] = c1;
    const EwTriple& T2 = MB.T;
    const u64 k2 = tkey(T2.key, T2.kp), g2 = (T2.off + g) * kPhi;
    const Dw t2 = ew_secrets_kg<false>(T2, k2, g2);
    const u64 eM = MB.uf(q0, g) + MB.uf(q1, g) - t2.A, dM = c0 + c1 - t2.B;
    // the multiply's combine (MulCombine over T2) -> sink
    const Dw m2 = masks_with(T2, k2, g2, t2);
    const u64 z0 = (m2.A * m2.B - m2.rc) + (eM * (m2.B - m2.rb) + dM * (m2.A - m2.ra)) + eM * dM;
    const u64 z1 = m2.rc + (eM * m2.rb + dM * m2.ra);
    if constexpr (has_pair_pf<PF>::value) {
      p.fin.pf.pair(q0, g, z0, z1);
    } else {
      p.fin.pf(q0, 0, g, z0);
      p.fin.pf(q1, 1, g, z1);
    }
  }
}

// The element-by-element chain: pair evaluation with the opened wire, no link, seeded dealer
// (queue-sourced triples run the per-round kernels), not forced to per-round kernels
// (mpcg_session_set_persistent(0)). The register form (chain_reg_kernel, MPCG_CHAIN_REG=0
// disables) takes every size: ResNet-18 27.6 -> 20.7 ms, BERT-base 46.2 -> 40.9 ms, LeNet-5
// 0.51 -> 0.41 ms against the per-round kernels (A/B on one box). The memory form
// (chain_pair_kernel) only up to MPCG_FUSED_CHAIN_MAX elements (default 4M): at 8.4M it was 8%
// slower than the per-round kernels (each thread's round-to-round state round-trips through
// L2 with every round's latency exposed), at <= 2M 10-45% faster.
bool chain_reg_on() {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_CHAIN_REG");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool fused_chain_ok(const Session& s, size_t n) {
  static const size_t max_n = [] {
    const char* e = std::getenv("MPCG_FUSED_CHAIN_MAX");
    return e ? size_t(std::strtoull(e, nullptr, 10)) : size_t(4000000);
  }();
  return (chain_reg_on() || n <= max_n) && adder_opened_wire(s) && !(s.cfg.link_bandwidth > 0) && !s.source_q &&
         s.persistent_mode != 0;
}

// One persistent cooperative kernel for the whole compare-and-select chain (1-GPU mode):
// 10 exchanges become 10 grid barriers. Values, tags and collective accounting are those
// of the per-round path (chunk lanes only change where an open may start; with in-device
// opens there is nothing to overlap, so the lanes are accounted but not split).
template <class DF, class UF, class PF>
void compare_mul_persistent(Session& s, size_t n, const AdderOptions& opt, const std::string& tag_msb,
                            const std::string& tag_b2a, const std::string& tag_mul, DF df, UF uf, PF pf,
                            Ptr2 cout, bool fused = false) {
  const bool opened = adder_opened_wire(s);  // pair evaluation: opened wire for b2a and the multiply
  const int ch = clamp_chunks(opt.chunks, n);
  const Pid2 pid = pids(s);
  const SpkConsts c = make_spk_constants(opt.width);
  const std::string at = tag_msb + ".add1";
  // dealer fetches in reference order: adder .g, .l0..l5, then b2a .m1, then the select
  Triple tr[7];
  for (int r = 0; r < 7; ++r) {
    tr[r] = r == 0 ? s.fetch(TripleSpec::elementwise(TripleKind::Bin, Shape{n}), at + ".g")
                   : s.fetch(TripleSpec::elementwise(TripleKind::Bin, Shape{2, n}), at + ".l" + std::to_string(r - 1),
                             /*stacked=*/true);
    tr[r].mark_consumed();
  }
  Triple t1 = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{n}), tag_b2a + ".m1");
  t1.mark_consumed();
  Triple t2 = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{n}), tag_mul);
  t2.mark_consumed();
  const Session::MaskRef mr = s.take_mask(n);
  DT keep = s.alloc(Shape{n}), S = s.alloc(Shape{n}), P = s.alloc(Shape{n}), P0 = s.alloc(Shape{n}),
     bits = s.alloc(Shape{n});
  DT cw[2];  // issue-to-settle draw cache (ew.cuh)
  if (adder_draw_cache_ok(s, n) && (s.n_local == 1 || pair_eval_enabled()))
    for (auto& b : cw) b = s.alloc(Shape{8 * n});
  Open om = s.begin_open(n, Reduce::Sum);
  Open oa[7];
  for (int r = 0; r < 7; ++r) oa[r] = s.begin_open((r == 0 ? 2 : 4) * n, Reduce::Xor);
  Open ob = s.begin_open(2 * n, Reduce::Sum), og = s.begin_open(2 * n, Reduce::Sum);

  using XF = A2bPart<DF>;
  using AR = AdderRound<XF, XF, B2aBuildFF>;
  using BR = MulCombine<MulByBitBuild<UF>>;
  using CR = MulCombine<PF>;
  ChainParams<MaskRound<DF>, AR, BR, CR> p{};
  p.mask = MaskRound<DF>{s.mask_key[0], s.mask_key[1], mr, own_ptrs(om), ptrs(keep), df};
  const XF xf{pid, cptrs(keep), peer_ptrs(om), s.mask_key[0], s.mask_key[1], mr, df, 0, opened ? 1 : 0};
  const XF yf{pid, cptrs(keep), peer_ptrs(om), s.mask_key[0], s.mask_key[1], mr, df, 1, opened ? 1 : 0};
  for (int r = 0; r <= 7; ++r) {
    AR& k = p.adder[r];
    k.rp = r - 1;
    k.rn = r;
    k.levels = c.levels;
    if (r >= 1) k.Tp = tr[r - 1].ew;
    if (r <= 6) k.Tn = tr[r].ew;
    if (r >= 2) k.lp = c.lv[r - 2];
    if (r >= 1 && r <= 6) k.ln = c.lv[r - 1];
    k.pid = pid;
    if (r >= 1) {
      k.ownp = as_const(own_ptrs(oa[r - 1]));
      k.peerp = peer_ptrs(oa[r - 1]);
    }
    if (r <= 6) k.ownn = own_ptrs(oa[r]);
    k.S = ptrs(S);
    k.P = ptrs(P);
    k.P0 = ptrs(P0);
    k.lo = 0;
    k.w = n;
    k.wmask = c.wmask;
    k.xf = xf;
    k.yf = yf;
    if (cw[0]) {
      k.cwN = n;
      if (r >= 1) k.cwp = cw[(r - 1) & 1].s[0];
      if (r <= 6) k.cwn = cw[r & 1].s[0];
    }
    if (r == 7) {
      k.ff = B2aBuildFF{t1.ew, own_ptrs(ob), ptrs(bits), 0, n};
      k.ff.opened = opened;
    }
  }
  p.nadder = 8;
  p.b2a = BR{t1.ew, pid, as_const(own_ptrs(ob)), peer_ptrs(ob), 0, n,
             MulByBitBuild<UF>{t2.ew, own_ptrs(og), cptrs(bits), 0, n, uf, cout}};
  p.b2a.opened = p.b2a.pf.opened = opened;
  p.fin = CR{t2.ew, pid, as_const(own_ptrs(og)), peer_ptrs(og), 0, n, pf};
  p.fin.opened = opened;
  DT bar = s.alloc(Shape{1});
  MPCG_CUDA(cudaMemsetAsync(bar.s[0], 0, 8, s.stream));
  p.n = n;
  p.bar = reinterpret_cast<unsigned*>(bar.s[0]);
  p.pair = s.n_local == 2 && pair_eval_enabled();
  p.skip_mask = opened ? 1 : 0;
  const unsigned gy = p.pair ? 1u : unsigned(s.n_local);

  if (fused) {  // element by element, no grid barrier (chain_reg_kernel / chain_pair_kernel)
    const u64 blocks = std::min<u64>((n + 255) / 256, u64(num_sms()) * 16);
    const bool reg = chain_reg_on();
    bool seeded = t1.ew.pool == nullptr && t2.ew.pool == nullptr;
    for (int r = 0; r < 7; ++r) seeded = seeded && tr[r].ew.pool == nullptr;
    const bool use_reg = reg && seeded && c.levels == 6 && !cw[0];
    // register form: ALU-bound on the dealer, so its unit is the draw — 2 mask + 65 adder
    // (generate AND + 12 level ANDs, 5 each: A, B once for issue and settle, r_A, r_B, r_C)
    // + 5 b2a + 5 multiply = 77 splitmix64 draws per element pair
    ClassScope cs(use_reg ? kClsChainReg : kClsChain, use_reg ? 77.0 * double(n) : 512.0 * double(n) * s.n_local);
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    if (use_reg)
      chain_reg_kernel<DF, UF, PF><<<unsigned(blocks), 256, 0, s.stream>>>(p);
    else
      chain_pair_kernel<MaskRound<DF>, AR, BR, CR><<<unsigned(blocks), 256, 0, s.stream>>>(p);
    MPCG_CUDA(cudaGetLastError());
    probe_end(s.stream, pe);
  } else {
  auto kern = chain_kernel<MaskRound<DF>, AR, BR, CR>;
  static int per_sm = -1;  // resident 256-thread CTAs per SM for this instantiation
  if (per_sm < 0) {
    MPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    if (per_sm < 1) throw Error(kInternalError, "chain kernel cannot be resident");
  }
  const unsigned tpb = chain_tpb(n);  // one element per thread per round (PRG-latency bound)
  const u64 cap = u64(per_sm) * (256 / tpb) * num_sms() / gy;  // residency measured at 256 threads
  u64 blocks = (n + tpb - 1) / tpb;
  blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(unsigned(blocks), gy);
  lc.blockDim = dim3(tpb);
  lc.stream = s.stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barrier)
  attr.val.cooperative = 1;
  lc.attrs = &attr;
  lc.numAttrs = 1;
  {
    // ReLU / compared pair = 2 x 248 B wire + 8 x (in + out) ~ 512 B/elem/party
    ClassScope cs(kClsChain, 512.0 * double(n) * s.n_local);
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    MPCG_CUDA(cudaLaunchKernelEx(&lc, kern, p));
    probe_end(s.stream, pe);
  }
  }
  // bookkeeping in the reference's collective order (H/protocols/compare.hpp:37-52,
  // adder.hpp:312-322, beaver.hpp:63-71)
  auto ctag = [&](const std::string& t, int k) { return ch == 1 ? t : t + ".chunk" + std::to_string(k); };
  s.account(n, Reduce::Sum, "", /*p2p=*/true);
  for (int r = 0; r < 7; ++r)
    for (int k = 0; k < ch; ++k) {
      const auto rg = chunk_range(n, ch, k);
      const std::string t = r == 0 ? at + ".g" : at + ".l" + std::to_string(r - 1);
      s.account((r == 0 ? 2 : 4) * (rg.second - rg.first), Reduce::Xor,
                ch > 1 && !opt.merged ? t + ".chunk" + std::to_string(k) : t);
    }
  for (int k = 0; k < ch; ++k) {
    const auto rg = chunk_range(n, ch, k);
    s.account(2 * (rg.second - rg.first), Reduce::Sum, ctag(tag_b2a + ".m1", k));
  }
  for (int k = 0; k < ch; ++k) {
    const auto rg = chunk_range(n, ch, k);
    s.account(2 * (rg.second - rg.first), Reduce::Sum, ctag(tag_mul, k));
  }
  s.check();
}

template <class DF, class UF, class PF>
void compare_mul(Session& s, size_t n, const AdderOptions& opt, const std::string& tag_msb,
                 const std::string& tag_b2a, int chunks_b2a, const std::string& tag_mul, int chunks_mul, DF df,
                 UF uf, PF pf, Ptr2 cout = Ptr2{{nullptr, nullptr}}) {
  const bool opened = adder_opened_wire(s);  // pair evaluation: opened wire for b2a and the multiply
  const int ch = clamp_chunks(opt.chunks, n);
  if (clamp_chunks(chunks_b2a, n) != ch || clamp_chunks(chunks_mul, n) != ch)
    throw Error(kUsageError, "compare_mul: misaligned chunk lanes");
  if (n > 0 && fused_chain_ok(s, n)) {
    compare_mul_persistent(s, n, opt, tag_msb, tag_b2a, tag_mul, df, uf, pf, cout, /*fused=*/true);
    return;
  }
  if (n > 0 && s.persistent_ok(n)) {
    compare_mul_persistent(s, n, opt, tag_msb, tag_b2a, tag_mul, df, uf, pf, cout);
    return;
  }
  const Pid2 pid = pids(s);
  const int xl = ch > 1 && s.fuse_lanes() ? 1 : ch;  // lanes launched (Session::fuse_lanes)
  DT bits = s.alloc(Shape{n});
  std::vector<Open> ob(static_cast<size_t>(xl)), og(static_cast<size_t>(xl));
  for (int k = 0; k < xl; ++k) {
    const auto r = chunk_range(n, xl, k);
    ob[k] = s.begin_open(2 * (r.second - r.first), Reduce::Sum);
    og[k] = s.begin_open(2 * (r.second - r.first), Reduce::Sum);
  }
  auto ctag = [&](const std::string& t, int k) { return ch == 1 ? t : t + ".chunk" + std::to_string(k); };
  auto post_lane = [&](Open& o, const std::string& t, int k) {
    if (xl == ch) s.post(o, ctag(t, k));
    else s.post_lanes(o, n, ch, 2, [&](int kk) { return ctag(t, kk); });
  };
  Triple t1, t2;
  bool fetched = false;
  auto fetch_tail = [&] {  // after the adder's fetches, in reference order
    if (fetched) return;
    t1 = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{n}), tag_b2a + ".m1");
    t1.mark_consumed();
    t2 = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{n}), tag_mul);
    t2.mark_consumed();
    fetched = true;
  };
  a2b_op(
      s, n, opt, tag_msb, df,
      [&](int lane, size_t lo, size_t w) {
        fetch_tail();
        B2aBuildFF f{t1.ew, own_ptrs(ob[lane]), ptrs(bits), lo, w};
        f.opened = opened;
        return f;
      },
      [&](int lane) { post_lane(ob[lane], tag_b2a + ".m1", lane); });
  for (int k = 0; k < xl; ++k) {
    const auto r = chunk_range(n, xl, k);
    const size_t lo = r.first, w = r.second - r.first;
    s.wait(ob[k]);
    MulByBitBuild<UF> gb{t2.ew, own_ptrs(og[k]), cptrs(bits), lo, w, uf, cout};
    gb.opened = opened;
    MulCombine<MulByBitBuild<UF>> bc{t1.ew, pid, as_const(own_ptrs(ob[k])), peer_ptrs(ob[k]), lo, w, gb};
    bc.opened = opened;
    launch_ew(s.stream, s.n_local, w, bc);
    post_lane(og[k], tag_mul, k);
  }
  for (int k = 0; k < xl; ++k) {
    const auto r = chunk_range(n, xl, k);
    s.wait(og[k]);
    MulCombine<PF> fc{t2.ew, pid, as_const(own_ptrs(og[k])), peer_ptrs(og[k]), r.first, r.second - r.first, pf};
    fc.opened = opened;
    launch_ew(s.stream, s.n_local, r.second - r.first, fc);
  }
  s.check();
}
}  // namespace

DT a2b(Session& s, const DT& x, const AdderOptions& opt, const std::string& tag) {
  DT z = s.alloc(x.shape, x.scale);
  a2b_op(s, x.numel(), opt, tag, SrcMem{cptrs(x)}, same(SumSink{ptrs(z)}));
  return z;
}

DT msb(Session& s, const DT& x, const AdderOptions& opt, const std::string& tag) {
  DT z = s.alloc(x.shape, x.scale);
  a2b_op(s, x.numel(), opt, tag, SrcMem{cptrs(x)}, same(MsbSink{ptrs(z)}));
  return z;
}

DT b2a_bit(Session& s, const DT& b, const std::string& tag, int chunks) {
  Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, b.shape), tag + ".m1");
  t.mark_consumed();
  DT z = s.alloc(b.shape, b.scale);
  const Pid2 pid = pids(s);
  mul_op(s, t.ew, b.numel(), chunks, tag + ".m1", BitAcc{pid, cptrs(b)}, BitBq{pid, cptrs(b)},
         B2aSink{cptrs(b), ptrs(z)});
  return z;
}

DT less_than(Session& s, const DT& x, const DT& y, const AdderOptions& opt, const std::string& tag) {
  require_same_shape(x, y, "less_than");
  DT m = s.alloc(x.shape, 0);
  a2b_op(s, x.numel(), opt, tag + ".msb", SrcSub{cptrs(x), cptrs(y)}, same(MsbSink{ptrs(m)}));
  return b2a_bit(s, m, tag + ".b2a", opt.chunks);
}

// ---------------------------------------------------------------- activations
namespace {
struct SinkXMinus {  // out = x - z  (relu gate, H/nonlinear/activations.hpp:46)
  CPtr2 x;
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64 z) const {
    (slot ? out.p[1] : out.p[0])[g] = (slot ? x.p[1] : x.p[0])[g] - z;
  }
};
}  // namespace

DT relu_shares(Session& s, const DT& x, const std::string& tag) {
  // x - x*b2a(msb(x)): tags "<l>.msb.add1.*", "<l>.b2a.m1", "<l>.gate" (activations.hpp:39-47)
  const size_t n = x.numel();
  const int ch = chunks_for(s, n);
  DT out = s.alloc(x.shape, x.scale);
  compare_mul(s, n, adder_for(s, n), tag + ".msb", tag + ".b2a", ch, tag + ".gate", ch, SrcMem{cptrs(x)},
              SrcMem{cptrs(x)}, SinkXMinus{cptrs(x), ptrs(out)});
  return out;
}

namespace {
// Tournament halves of cur [outer, len]: a = cur[:, :h], b = cur[:, h:2h] read in place
// (H/nonlinear/activations.hpp:20-33,62-63). sign > 0 gives a - b, else b - a.
struct SrcHalfDiff {
  CPtr2 cur;
  u32 h, len;
  int sign;
  __device__ u64 operator()(int slot, u64 g) const {
    const u32 o = u32(g) / h, j = u32(g) - o * h;
    const u64* row = (slot ? cur.p[1] : cur.p[0]) + u64(o) * len;
    return sign > 0 ? row[j] - row[h + j] : row[h + j] - row[j];
  }
};
struct SinkPick {  // m = a + step, written into the next [outer, nw] row layout
  CPtr2 cur;
  Ptr2 next;
  u32 h, len, nw;
  __device__ void operator()(int slot, int, u64 g, u64 z) const {
    const u32 o = u32(g) / h, j = u32(g) - o * h;
    (slot ? next.p[1] : next.p[0])[u64(o) * nw + j] = (slot ? cur.p[1] : cur.p[0])[u64(o) * len + j] + z;
  }
};
}  // namespace

DT max_last_dim(Session& s, const DT& x, size_t L, const std::string& tag) {
  if (L == 0 || x.numel() % L != 0) throw Error(kShapeError, "max_last_dim: bad row length");
  const size_t outer = x.numel() / L;
  DT cur = reshape(x, Shape{outer, L});
  size_t len = L;
  int round = 0;
  while (len > 1) {
    const size_t h = len / 2;
    const bool odd = len & 1;
    const std::string rt = tag + ".r" + std::to_string(round++);
    const size_t n = outer * h;
    const AdderOptions opt = adder_for(s, n);
    const size_t nw = odd ? h + 1 : h;
    DT next = s.alloc(Shape{outer, nw}, cur.scale);
    if (odd) {  // carry the odd tail (H/nonlinear/activations.hpp:71-82)
      const CPtr2 cp = cptrs(cur);
      const Ptr2 np = ptrs(next);
      const u32 LEN = u32(len), NW = u32(nw), HH = u32(h);
      launch_ew(s.stream, s.n_local, outer, [=] __device__(int slot, u64 o) {
        sel(np, slot)[o * NW + HH] = sel(cp, slot)[o * LEN + LEN - 1];
      });
    }
    // gate = less_than(a, b) (tags rt.msb.add1.*, rt.b2a.m1); pick = (b - a) * gate (rt.pick)
    const CPtr2 cp = cptrs(cur);
    compare_mul(s, n, opt, rt + ".msb", rt + ".b2a", opt.chunks, rt + ".pick", chunks_for(s, n),
                SrcHalfDiff{cp, u32(h), u32(len), +1}, SrcHalfDiff{cp, u32(h), u32(len), -1},
                SinkPick{cp, ptrs(next), u32(h), u32(len), u32(nw)});
    cur = next;
    len = nw;
  }
  return reshape(cur, Shape{outer, 1});
}

namespace {
// exp chain (H/nonlinear/approx.hpp:22-39) as ONE fused square chain: round 0 squares
// w = trunc(x, it) and forms y = w + trunc(w^2, f+1) + [p0] 2^f; rounds 1..it square y with
// truncation by f; the last y goes to of(slot, party, g, y).
template <class XF, class OF>
struct ExpY {
  XF xsrc;
  OF of;
  int it, f, first, last;
  __device__ u64 operator()(int slot, int party, u64 g, u64 z) const {
    const u64 y = first ? sar64(xsrc(slot, g), it) + sar64(z, f + 1) + (party == 0 ? (u64(1) << f) : 0)
                        : sar64(z, f);
    if (last) of(slot, party, g, y);
    return y;
  }
};
template <class XF>
struct SarOf {  // w = trunc(x, it), the first squared value
  XF x;
  int it;
  __device__ u64 operator()(int slot, u64 g) const { return sar64(x(slot, g), it); }
};
struct OutStore {  // out[g] = y
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64 y) const { sel(out, slot)[g] = y; }
};
struct OutAffine {  // out[g] = k*y + [p0] c   (reciprocal seed 3 exp + 0.003; sigmoid's 1 + exp)
  Ptr2 out;
  u64 k, c;
  __device__ void operator()(int slot, int party, u64 g, u64 y) const {
    sel(out, slot)[g] = y * k + (party == 0 ? c : 0);
  }
};
struct OutRecipSeed {  // d = y + [p0] 1; seed = [p0] c0 - trunc(d * c1, f)
  Ptr2 d, seed;
  u64 one, c1, c0;
  int f;
  __device__ void operator()(int slot, int party, u64 g, u64 y) const {
    const u64 dv = y + (party == 0 ? one : 0);
    sel(d, slot)[g] = dv;
    sel(seed, slot)[g] = (party == 0 ? c0 : 0) - sar64(dv * c1, f);
  }
};
struct SrcConstMinus {  // [p0] c - x[g]   (reciprocal seed argument 0.5 - x)
  Pid2 pid;
  CPtr2 x;
  u64 c;
  __device__ u64 operator()(int slot, u64 g) const { return (pid.v[slot] == 0 ? c : 0) - sel(x, slot)[g]; }
};

template <class XF, class OF>
void exp_chain(Session& s, const Shape& shape, const std::string& tag, int square_iters, XF xsrc, OF of) {
  const int f = s.cfg.frac_bits;
  const size_t n = shape_numel(shape);
  std::vector<Triple> tr;
  std::vector<std::string> tags;
  tags.push_back(tag + ".w2");
  for (int i = 0; i < square_iters; ++i) tags.push_back(tag + ".sq" + std::to_string(i));
  for (auto& t : tags) {
    tr.push_back(s.fetch(TripleSpec::square_of(shape), t));
    tr.back().mark_consumed();
  }
  const int R = int(tr.size());
  square_chain(s, n, chunks_for(s, n), tr, tags, SarOf<XF>{xsrc, square_iters}, [&](int r) {
    return ExpY<XF, OF>{xsrc, of, square_iters, f, r == 0 ? 1 : 0, r == R - 1 ? 1 : 0};
  });
}
}  // namespace

DT exp_shares(Session& s, const DT& x, const std::string& tag, int square_iters) {
  DT y = s.alloc(x.shape, x.scale);
  exp_chain(s, x.shape, tag, square_iters, SrcMem{cptrs(x)}, OutStore{ptrs(y)});
  return y;
}

namespace {
// Newton steps of reciprocal_shares (H/nonlinear/approx.hpp:52-60) as one fused mul chain:
// after xy_i: u = [p0] 2^(f+1) - trunc(x*y, f), next eps/delta = (y, u);
// after yu_i: y = trunc(y*u, f) (stored), next eps/delta = (x, y).
struct RecipPV {
  CPtr2 x;
  Ptr2 y;
  int f, odd;
  __device__ u64 val(int slot, int party, u64 g, u64 z) const {
    if (!odd) return (party == 0 ? (u64(2) << f) : 0) - sar64(z, f);
    const u64 v = sar64(z, f);
    sel(y, slot)[g] = v;
    return v;
  }
  __device__ u64 nx(int slot, u64 g, u64) const { return odd ? sel(x, slot)[g] : sel(y, slot)[g]; }
  __device__ u64 ny(int, u64, u64 v) const { return v; }
};
}  // namespace

// Newton steps for 1/d on [1, 2] from the 1/17-accurate linear seed: error (1/17)^(2^k) drops
// below 2^-f once 2^k log2(17) > f (oracle recip_unit_iters).
int recip_unit_iters(int f) {
  int k = 1;
  while (double(1 << k) * std::log2(17.0) <= double(f)) ++k;
  return k;
}

// Newton steps y <- trunc(y (2 - trunc(x y))) on y in place (approx.hpp:52-60), one fused chain.
static void recip_newton(Session& s, const DT& x, DT& y, const std::string& tag, int newton_iters) {
  const int f = s.cfg.frac_bits;
  const size_t n = x.numel();
  if (newton_iters <= 0) return;
  std::vector<Triple> tr;
  std::vector<std::string> tags;
  for (int i = 0; i < newton_iters; ++i) {
    tags.push_back(tag + ".xy" + std::to_string(i));
    tags.push_back(tag + ".yu" + std::to_string(i));
  }
  for (auto& t : tags) {
    tr.push_back(s.fetch(TripleSpec::elementwise(TripleKind::Arith, x.shape), t));
    tr.back().mark_consumed();
  }
  mul_chain(s, n, chunks_for(s, n), tr, tags, SrcMem{cptrs(x)}, SrcMem{cptrs(y)},
            [&](int r) { return RecipPV{cptrs(x), ptrs(y), f, r & 1}; });
}

DT reciprocal_shares(Session& s, const DT& x, const std::string& tag, int newton_iters) {
  const int f = s.cfg.frac_bits;
  // y0 = 3 exp(0.5 - x) + 0.003  (H/nonlinear/approx.hpp:49-51), the seed exp fused in
  DT y = s.alloc(x.shape, x.scale);
  exp_chain(s, x.shape, tag + ".seed", 7, SrcConstMinus{pids(s), cptrs(x), encode_fixed(0.5, f)},
            OutAffine{ptrs(y), 3, encode_fixed(0.003, f)});
  recip_newton(s, x, y, tag, newton_iters);
  return y;
}

namespace {
struct SrcSubRowMax {  // x[g] - m[g / L]
  CPtr2 x, m;
  u32 L;
  __device__ u64 operator()(int slot, u64 g) const { return sel(x, slot)[g] - sel(m, slot)[u32(g) / L]; }
};
struct SrcBcast {  // r[g / L]
  CPtr2 r;
  u32 L;
  __device__ u64 operator()(int slot, u64 g) const { return sel(r, slot)[u32(g) / L]; }
};
}  // namespace

struct OutRowStore {  // out[r] = acc
  Ptr2 out;
  __device__ void operator()(int slot, u64 r, u64 acc) const { sel(out, slot)[r] = acc; }
};

DT softmax_shares(Session& s, const DT& x, size_t L, const std::string& tag) {
  const size_t outer = x.numel() / L;
  const size_t n = x.numel();
  const int ch = chunks_for(s, n);
  DT mx = max_last_dim(s, x, L, tag + ".max");
  DT e = s.alloc(Shape{outer, L}, x.scale);  // exp(x - max), the centring fused into the exp chain
  exp_chain(s, Shape{outer, L}, tag + ".exp", 7, SrcSubRowMax{cptrs(x), cptrs(mx), u32(L)}, OutStore{ptrs(e)});
  DT rowsum = s.alloc(Shape{outer, 1}, x.scale);
  row_reduce(s, outer, u32(L), SrcMem{cptrs(e)}, OutRowStore{ptrs(rowsum)});  // warp per row
  DT r = reciprocal_shares(s, rowsum, tag + ".recip");
  Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{outer, L}), tag + ".scale");
  t.mark_consumed();
  DT out = s.alloc(x.shape, x.scale);
  mul_op(s, t.ew, n, ch, tag + ".scale", SrcMem{cptrs(e)}, SrcBcast{cptrs(r), u32(L)},
         SinkTrunc{ptrs(out), s.cfg.frac_bits});
  return out;
}

DT maxpool2d_shares(Session& s, const DT& x, size_t N, size_t C, size_t H, size_t W, size_t k,
                    size_t stride, const std::string& tag) {
  if (H < k || W < k) throw Error(kShapeError, "maxpool2d: window larger than input");
  const size_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
  const size_t rows = N * C * OH * OW;
  DT win = s.alloc(Shape{rows, k * k}, x.scale);
  {
    const CPtr2 xp = cptrs(x);
    const Ptr2 wp = ptrs(win);
    const u32 KK = u32(k * k), K = u32(k), S = u32(stride), OWw = u32(OW), OHh = u32(OH), HH = u32(H),
              WW = u32(W);
    launch_ew(s.stream, s.n_local, rows * k * k, [=] __device__(int slot, u64 i) {
      const u32 r = u32(i) / KK, t = u32(i) - r * KK;
      const u32 ki = t / K, kj = t - ki * K;
      const u32 ow = r % OWw, oh = (r / OWw) % OHh, nc = r / (OWw * OHh);
      const u64 src = (u64(nc) * HH + oh * S + ki) * WW + ow * S + kj;
      sel(wp, slot)[i] = sel(xp, slot)[src];
    });
  }
  DT mx = max_last_dim(s, win, k * k, tag);
  return reshape(mx, Shape{N, C, OH, OW});
}

// ---------------------------------------------------------------- extension: sigmoid
// NOT in the reference (needed by GeLU for BERT-base; SURVEY 8(a*)). Built only from the
// reference's blocks in its tag style; restated in oracle/mpc_oracle.py:sigmoid_shares.
//   b = b2a(msb(x)), -|x| = 2 x b - x  (one fused compare-and-multiply chain, as relu_shares)
//   r = 1 / (1 + exp(-|x|))  (exp sees only x <= 0, the reciprocal only (1, 2])
//   sigma(x) = r + b (1 - 2 r)
namespace {
struct SinkNegAbs {  // -|x| = 2 x b - x
  CPtr2 x;
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64 z) const {
    (slot ? out.p[1] : out.p[0])[g] = (z + z) - (slot ? x.p[1] : x.p[0])[g];
  }
};
struct SrcOneMinus2 {  // [p0] 2^f - 2 r
  Pid2 pid;
  CPtr2 r;
  u64 one;
  __device__ u64 operator()(int slot, u64 g) const {
    return (pid.v[slot] == 0 ? one : 0) - (sel(r, slot)[g] + sel(r, slot)[g]);
  }
};
struct SinkAddTo {  // out = r + z
  CPtr2 r;
  Ptr2 out;
  __device__ void operator()(int slot, int, u64 g, u64 z) const { sel(out, slot)[g] = sel(r, slot)[g] + z; }
};
}  // namespace

DT sigmoid_shares(Session& s, const DT& x, const std::string& tag) {
  const int f = s.cfg.frac_bits;
  const size_t n = x.numel();
  const int ch = chunks_for(s, n);
  DT b = s.alloc(x.shape, 0), nabs = s.alloc(x.shape, x.scale);
  compare_mul(s, n, adder_for(s, n), tag + ".msb", tag + ".b2a", ch, tag + ".abs", ch, SrcMem{cptrs(x)},
              SrcMem{cptrs(x)}, SinkNegAbs{cptrs(x), ptrs(nabs)}, ptrs(b));
  // d = 1 + exp(-|x|) in (1, 2] and the reciprocal's linear seed y0 = 24/17 - 8/17 d, both
  // formed in the exp chain's last round; then three Newton steps (oracle recip_unit_shares)
  DT d = s.alloc(x.shape, x.scale), r = s.alloc(x.shape, x.scale);
  exp_chain(s, x.shape, tag + ".exp", 7, SrcMem{cptrs(nabs)},
            OutRecipSeed{ptrs(d), ptrs(r), u64(1) << f, encode_fixed(8.0 / 17.0, f), encode_fixed(24.0 / 17.0, f), f});
  recip_newton(s, d, r, tag + ".recip", recip_unit_iters(f));
  Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, x.shape), tag + ".sel");
  t.mark_consumed();
  DT out = s.alloc(x.shape, x.scale);
  mul_op(s, t.ew, n, ch, tag + ".sel", SrcMem{cptrs(b)}, SrcOneMinus2{pids(s), cptrs(r), u64(1) << f},
         SinkAddTo{cptrs(r), ptrs(out)});
  return out;
}

}  // namespace mpcg
