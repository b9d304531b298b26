// Config-enabling layers the reference lacks (SURVEY.md 0, 8(a*), 8f row 1): GeLU and
// LayerNorm (BERT-base), global average pooling (ResNet-18; residual adds are local share
// additions and BatchNorm is folded into conv weights by the weight owner).
//
// NOT in the reference. Each op is composed from the reference's own building blocks
// (Beaver mul/square rounds, the fused compare chain, exp_shares / reciprocal_shares,
// local truncation) with tags "<layer>.<step>" in the style of relu_shares/softmax_shares,
// and is restated step for step in oracle/mpc_oracle.py (sigmoid_shares, gelu_shares,
// inv_sqrt_shares, layernorm_shares, global_avg_pool) — parity is against that restatement.
#include "ew.cuh"

namespace mpcg {

namespace {

struct SrcSubRow {  // x[g] - mu[g / d]
  CPtr2 x, mu;
  u32 d;
  __device__ u64 operator()(int slot, u64 g) const { return sel(x, slot)[g] - sel(mu, slot)[g / d]; }
};
struct SrcRowB {  // y[g / d]
  CPtr2 y;
  u32 d;
  __device__ u64 operator()(int slot, u64 g) const { return sel(y, slot)[g / d]; }
};
struct SrcColB {  // v[g % d]
  CPtr2 v;
  u32 d;
  __device__ u64 operator()(int slot, u64 g) const { return sel(v, slot)[g % d]; }
};
struct OutScaleRescale {  // out[r] = sar(acc * k, f) (+ [p0] add)
  Pid2 pid;
  Ptr2 out;
  u64 k, add;
  int f;
  __device__ void operator()(int slot, u64 r, u64 acc) const {
    sel(out, slot)[r] = sar64(acc * k, f) + (pid.v[slot] == 0 ? add : 0);
  }
};
// Round policy of the fused inverse-sqrt Newton chain (oracle inv_sqrt_shares):
//   after square y2_i: y2 = trunc(z, f)            -> next mul (v, y2)
//   after mul vy_i:    u = [p0] 3 - trunc(z, f)    -> next mul (y, u)
//   after mul yu_i:    y = trunc(z, f+1), stored   -> next square (y)
struct IsqrtPV {
  Pid2 pid;
  CPtr2 v;
  Ptr2 y;
  int f;
  u64 three;
  int phase;
  __device__ u64 val(int slot, int party, u64 g, u64 z) const {
    if (phase == 0) return sar64(z, f);
    if (phase == 1) return (party == 0 ? three : 0) - sar64(z, f);
    const u64 yy = sar64(z, f + 1);
    sel(y, slot)[g] = yy;
    return yy;
  }
  __device__ u64 nx(int slot, u64 g, u64 val) const {
    return phase == 0 ? sel(v, slot)[g] : (phase == 1 ? sel(y, slot)[g] : val);
  }
  __device__ u64 ny(int, u64, u64 val) const { return val; }
};
struct SinkTruncAddCol {  // out = sar(z, f) + beta[g % d]
  Ptr2 out;
  CPtr2 beta;
  int f;
  u32 d;
  __device__ void operator()(int slot, int, u64 g, u64 z) const {
    sel(out, slot)[g] = sar64(z, f) + sel(beta, slot)[g % d];
  }
};

}  // namespace

DT gelu_shares(Session& s, const DT& x, const std::string& tag) {
  // x * sigmoid(1.702 x)  (oracle gelu_shares)
  const int f = s.cfg.frac_bits;
  const size_t n = x.numel();
  const int ch = chunks_for(s, n);
  const u64 k = encode_fixed(1.702, f);
  DT z = s.alloc(x.shape, x.scale);
  {
    const CPtr2 xp = cptrs(x);
    const Ptr2 zp = ptrs(z);
    launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sar64(sel(xp, slot)[i] * k, f); });
  }
  DT sg = sigmoid_shares(s, z, tag + ".sig");
  Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, x.shape), tag + ".out");
  t.mark_consumed();
  DT out = s.alloc(x.shape, x.scale);
  mul_op(s, t.ew, n, ch, tag + ".out", SrcMem{cptrs(x)}, SrcMem{cptrs(sg)}, SinkTrunc{ptrs(out), f});
  return out;
}

DT inv_sqrt_shares(Session& s, const DT& v, const std::string& tag, int newton_iters) {
  // y0 = 2.2 exp(-(v/2 + 0.2)) + 0.2 - v/1024; y <- y (3 - v y^2) / 2  (oracle inv_sqrt_shares)
  const int f = s.cfg.frac_bits;
  const size_t n = v.numel();
  const int ch = chunks_for(s, n);
  const u64 c02 = encode_fixed(0.2, f), c22 = encode_fixed(2.2, f), three = encode_fixed(3.0, f);
  const Pid2 pid = pids(s);
  DT t0 = s.alloc(v.shape, v.scale);
  {
    const CPtr2 vp = cptrs(v);
    const Ptr2 tp = ptrs(t0);
    launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) {
      sel(tp, slot)[i] = (pid.v[slot] == 0 ? u64(0) - c02 : 0) - sar64(sel(vp, slot)[i], 1);
    });
  }
  DT e = exp_shares(s, t0, tag + ".seed");
  DT y = s.alloc(v.shape, v.scale);
  {
    const CPtr2 ep = cptrs(e), vp = cptrs(v);
    const Ptr2 yp = ptrs(y);
    launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) {
      sel(yp, slot)[i] = (sar64(sel(ep, slot)[i] * c22, f) - sar64(sel(vp, slot)[i], 10)) + (pid.v[slot] == 0 ? c02 : 0);
    });
  }
  if (newton_iters <= 0) return y;
  // Newton steps as ONE fused chain of 3*iters rounds: square y -> y2, mul v*y2 -> u, mul y*u -> y
  std::vector<Triple> tr;
  std::vector<int> sq;
  std::vector<std::string> tags;
  for (int i = 0; i < newton_iters; ++i) {
    const std::string it = std::to_string(i);
    tags.push_back(tag + ".y2" + it);
    tr.push_back(s.fetch(TripleSpec::square_of(v.shape), tags.back()));
    sq.push_back(1);
    tags.push_back(tag + ".vy" + it);
    tr.push_back(s.fetch(TripleSpec::elementwise(TripleKind::Arith, v.shape), tags.back()));
    sq.push_back(0);
    tags.push_back(tag + ".yu" + it);
    tr.push_back(s.fetch(TripleSpec::elementwise(TripleKind::Arith, v.shape), tags.back()));
    sq.push_back(0);
  }
  for (auto& t : tr) t.mark_consumed();
  mixed_chain(s, n, ch, tr, sq, tags, SrcMem{cptrs(y)}, SrcZero{},
              [&](int r) { return IsqrtPV{pids(s), cptrs(v), ptrs(y), f, three, r % 3}; });
  return y;
}

DT layernorm_shares(Session& s, const DT& x, size_t d, const DT& gamma, const DT& beta, bool public_weights,
                    const std::string& tag) {
  if (d == 0 || x.numel() % d != 0) throw Error(kShapeError, "layernorm: bad row length");
  if (gamma.numel() != d || beta.numel() != d) throw Error(kShapeError, "layernorm: gamma/beta must be [d]");
  const int f = s.cfg.frac_bits;
  const size_t n = x.numel(), rows = n / d;
  const int ch = chunks_for(s, n);
  const Pid2 pid = pids(s);
  const u64 kd = encode_fixed(1.0 / double(d), f), eps = encode_fixed(kLnEps, f);
  const u32 D = u32(d);
  // mean = scale_and_rescale(rowsum(x), 1/d)
  DT mu = s.alloc(Shape{rows, 1}, x.scale);
  row_reduce(s, rows, D, SrcMem{cptrs(x)}, OutScaleRescale{pid, ptrs(mu), kd, 0, f});
  // var = scale_and_rescale(rowsum(trunc((x - mean)^2)), 1/d) + eps
  DT sq = s.alloc(x.shape, x.scale);
  {
    Triple t = s.fetch(TripleSpec::square_of(Shape{rows, d}), tag + ".sq");
    t.mark_consumed();
    square_op(s, t.ew, n, ch, tag + ".sq", SrcSubRow{cptrs(x), cptrs(mu), D}, SinkTrunc{ptrs(sq), f});
  }
  DT var = s.alloc(Shape{rows, 1}, x.scale);
  row_reduce(s, rows, D, SrcMem{cptrs(sq)}, OutScaleRescale{pid, ptrs(var), kd, eps, f});
  DT y = inv_sqrt_shares(s, var, tag + ".isqrt", kIsqrtIters);
  // norm = trunc((x - mean) * y, f)
  DT nrm = s.alloc(x.shape, x.scale);
  {
    Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{rows, d}), tag + ".norm");
    t.mark_consumed();
    mul_op(s, t.ew, n, ch, tag + ".norm", SrcSubRow{cptrs(x), cptrs(mu), D}, SrcRowB{cptrs(y), D},
           SinkTrunc{ptrs(nrm), f});
  }
  DT out = s.alloc(x.shape, x.scale);
  if (public_weights) {  // local scale by the plaintext gamma column, party 0 adds beta
    const CPtr2 np = cptrs(nrm), gp = cptrs(gamma), bp = cptrs(beta);
    const Ptr2 op = ptrs(out);
    launch_ew(s.stream, s.n_local, n, [=] __device__(int slot, u64 i) {
      const u32 c = u32(i % D);
      sel(op, slot)[i] = sar64(sel(np, slot)[i] * sel(gp, slot)[c], f) + (pid.v[slot] == 0 ? sel(bp, slot)[c] : 0);
    });
  } else {
    Triple t = s.fetch(TripleSpec::elementwise(TripleKind::Arith, Shape{rows, d}), tag + ".gamma");
    t.mark_consumed();
    mul_op(s, t.ew, n, ch, tag + ".gamma", SrcMem{cptrs(nrm)}, SrcColB{cptrs(gamma), D},
           SinkTruncAddCol{ptrs(out), cptrs(beta), f, D});
  }
  return out;
}

DT global_avg_pool(Session& s, const DT& x, size_t N, size_t C, size_t HW) {
  // NCHW -> [N, C]: rowsum over H*W, scale_and_rescale(1/(H*W))  (as MeanPool, executor.hpp:399-410)
  if (N * C * HW != x.numel()) throw Error(kShapeError, "global_avg_pool: shape mismatch");
  const int f = s.cfg.frac_bits;
  DT out = s.alloc(Shape{N, C}, x.scale);
  row_reduce(s, N * C, u32(HW), SrcMem{cptrs(x)},
             OutScaleRescale{pids(s), ptrs(out), encode_fixed(1.0 / double(HW), f), 0, f});
  return out;
}

}  // namespace mpcg
