// Secure executor: per-layer dispatch, Beaver linear layers with the inter-linear-layer
// delta pipeline, attention. Mirrors H/engine/executor.hpp:173-422 (values, tags and
// collective order), on device shares.
#include <algorithm>
#include <cmath>

#include "ew.cuh"
#include "executor.hpp"
#include "gemm.cuh"

namespace mpcg {

LayerWiring layer_wiring(const ModelGraph& g) {
  // The reference's graphs are chains (H/engine/model.hpp:18-20); the extension lets a layer
  // read an earlier output ("from") and an Add combine two ("with").
  LayerWiring w;
  std::map<std::string, long> names;
  for (size_t i = 0; i < g.layers.size(); ++i) {
    const LayerSpec& l = g.layers[i];
    auto look = [&](const std::string& n) -> long {
      if (n == "input") return -1;
      auto it = names.find(n);
      if (it == names.end()) throw Error(kConfigError, l.name + ": unknown or later layer '" + n + "'");
      return it->second;
    };
    w.src.push_back(l.from.empty() ? long(i) - 1 : look(l.from));
    if (l.kind == LayerKind::Add) {
      if (l.with.empty()) throw Error(kConfigError, l.name + ": add needs 'with'");
      w.other.push_back(look(l.with));
    } else {
      w.other.push_back(-2);
    }
    if (!names.emplace(l.name, long(i)).second) throw Error(kConfigError, "duplicate layer name: " + l.name);
  }
  return w;
}

std::vector<Shape> infer_shapes(const ModelGraph& g) {
  // H/engine/model.hpp:69-122 (+ the extension layers)
  std::vector<Shape> out;
  const LayerWiring wr = layer_wiring(g);
  for (size_t li = 0; li < g.layers.size(); ++li) {
    const LayerSpec& l = g.layers[li];
    Shape cur = wr.src[li] < 0 ? g.input : out[size_t(wr.src[li])];
    switch (l.kind) {
      case LayerKind::Add: {
        const Shape& o = wr.other[li] < 0 ? g.input : out[size_t(wr.other[li])];
        if (o != cur) throw Error(kConfigError, l.name + ": add operand shapes differ");
        break;
      }
      case LayerKind::GlobalAvgPool:
        if (cur.size() != 4) throw Error(kConfigError, l.name + ": global_avg_pool expects NCHW input");
        cur = {cur[0], cur[1]};
        break;
      case LayerKind::Gelu:
        break;
      case LayerKind::LayerNorm:
        if (cur.empty()) throw Error(kConfigError, l.name + ": layernorm needs a trailing feature dim");
        break;
      case LayerKind::Dense:
        if (cur.empty()) throw Error(kConfigError, l.name + ": dense needs a trailing feature dim");
        cur.back() = l.out;
        break;
      case LayerKind::Conv2d: {
        if (cur.size() != 4) throw Error(kConfigError, l.name + ": conv2d expects NCHW input");
        const size_t h = cur[2], w = cur[3];
        if (h + 2 * l.pad < l.kernel || w + 2 * l.pad < l.kernel)
          throw Error(kConfigError, l.name + ": kernel larger than padded input");
        if (l.stride == 0) throw Error(kConfigError, l.name + ": stride must be >= 1");
        cur = {cur[0], l.out, (h + 2 * l.pad - l.kernel) / l.stride + 1, (w + 2 * l.pad - l.kernel) / l.stride + 1};
        break;
      }
      case LayerKind::Maxpool2d:
        if (cur.size() != 4) throw Error(kConfigError, l.name + ": maxpool2d expects NCHW input");
        if (cur[2] < l.kernel || cur[3] < l.kernel) throw Error(kConfigError, l.name + ": pool window larger than input");
        if (l.stride == 0) throw Error(kConfigError, l.name + ": stride must be >= 1");
        cur = {cur[0], cur[1], (cur[2] - l.kernel) / l.stride + 1, (cur[3] - l.kernel) / l.stride + 1};
        break;
      case LayerKind::Flatten: {
        if (cur.empty()) throw Error(kConfigError, l.name + ": flatten on scalar");
        size_t rest = 1;
        for (size_t i = 1; i < cur.size(); ++i) rest *= cur[i];
        cur = {cur[0], rest};
        break;
      }
      case LayerKind::Attention:
        if (cur.size() != 3) throw Error(kConfigError, l.name + ": attention expects [B, T, d]");
        if (l.heads == 0 || cur[2] % l.heads != 0)
          throw Error(kConfigError, l.name + ": head count must divide the model dim");
        break;
      case LayerKind::Relu:
      case LayerKind::Softmax:
        break;
      case LayerKind::MeanPool:
        if (cur.size() != 3) throw Error(kConfigError, l.name + ": mean_pool expects [B, T, d]");
        cur = {cur[0], cur[2]};
        break;
    }
    out.push_back(cur);
  }
  return out;
}

std::vector<std::pair<std::string, Shape>> model_weight_shapes(const ModelGraph& g) {
  // H/engine/model.hpp:213-252
  std::vector<std::pair<std::string, Shape>> out;
  const auto shapes = infer_shapes(g);
  const LayerWiring wr = layer_wiring(g);
  for (size_t i = 0; i < g.layers.size(); ++i) {
    const LayerSpec& l = g.layers[i];
    const Shape& cur = wr.src[i] < 0 ? g.input : shapes[size_t(wr.src[i])];
    if (l.kind == LayerKind::LayerNorm) {  // extension
      out.push_back({l.name + ".gamma", Shape{cur.back()}});
      out.push_back({l.name + ".beta", Shape{cur.back()}});
    } else if (l.kind == LayerKind::Dense) {
      out.push_back({l.name + ".W", Shape{cur.back(), l.out}});
      if (l.bias) out.push_back({l.name + ".b", Shape{l.out}});
    } else if (l.kind == LayerKind::Conv2d) {
      out.push_back({l.name + ".W", Shape{cur[1] * l.kernel * l.kernel, l.out}});
      if (l.bias) out.push_back({l.name + ".b", Shape{l.out}});
    } else if (l.kind == LayerKind::Attention) {
      const size_t d = cur[2];
      out.push_back({l.name + ".Wqkv", Shape{d, 3 * d}});
      if (l.bias) out.push_back({l.name + ".bqkv", Shape{3 * d}});
      out.push_back({l.name + ".Wo", Shape{d, d}});
      if (l.bias) out.push_back({l.name + ".bo", Shape{d}});
    }
  }
  return out;
}

SecureExecutor::SecureExecutor(Session& s, ModelGraph g, bool public_weights, ExecOptions opt)
    : s_(s), g_(std::move(g)), public_(public_weights), opt_(opt) {
  shapes_ = infer_shapes(g_);
  s_.cfg.frac_bits = g_.frac_bits;
  s_.cfg.merged_adder = opt_.merged_adder;
  if (opt_.pipelined) {
    s_.cfg.chunks = opt_.chunks;
    s_.cfg.chunk_threshold = opt_.chunk_threshold;
  } else {
    s_.cfg.chunks = 1;
    s_.cfg.chunk_threshold = 0;
  }
  build_weight_ops();
}

SecureExecutor::~SecureExecutor() {
  if (captured_) {  // the session's dealer streams return to eager use
    try {
      s_.sync();
      s_.release_graph();
    } catch (...) {
    }
  }
  for (auto e : ev_) cudaEventDestroy(e);
}

void SecureExecutor::add_weight_op(const std::string& tag, const std::string& wkey, const std::string& bkey,
                                   Shape x_shape) {
  Shape wshape;
  for (auto& [k, sh] : model_weight_shapes(g_))
    if (k == wkey) wshape = sh;
  WeightOp op;
  op.tag = tag;
  op.wkey = wkey;
  op.bkey = bkey;
  op.spec = TripleSpec::matmul_of(x_shape, wshape);
  op.x_shape = std::move(x_shape);
  wop_index_.emplace(op.tag, wops_.size());
  wops_.push_back(std::move(op));
}

void SecureExecutor::build_weight_ops() {
  // H/engine/executor.hpp:244-273
  const LayerWiring wr = layer_wiring(g_);
  for (size_t i = 0; i < g_.layers.size(); ++i) {
    const LayerSpec& l = g_.layers[i];
    const Shape& cur = wr.src[i] < 0 ? g_.input : shapes_[size_t(wr.src[i])];
    switch (l.kind) {
      case LayerKind::Dense: {
        const size_t in = cur.back();
        add_weight_op(l.name + ".mm", l.name + ".W", l.bias ? l.name + ".b" : "", Shape{shape_numel(cur) / in, in});
        break;
      }
      case LayerKind::Conv2d: {
        const size_t rows = cur[0] * ((cur[2] + 2 * l.pad - l.kernel) / l.stride + 1) *
                            ((cur[3] + 2 * l.pad - l.kernel) / l.stride + 1);
        add_weight_op(l.name + ".mm", l.name + ".W", l.bias ? l.name + ".b" : "",
                      Shape{rows, cur[1] * l.kernel * l.kernel});
        break;
      }
      case LayerKind::Attention: {
        const Shape x2{cur[0] * cur[1], cur[2]};
        add_weight_op(l.name + ".qkv", l.name + ".Wqkv", l.bias ? l.name + ".bqkv" : "", x2);
        add_weight_op(l.name + ".proj", l.name + ".Wo", l.bias ? l.name + ".bo" : "", x2);
        break;
      }
      default:
        break;
    }
  }
}

void SecureExecutor::deal_weights(const std::vector<std::string>& names, const std::vector<const double*>& values,
                                  const std::vector<size_t>& counts, u64 seed) {
  // check_weights (H/engine/model.hpp:366-376): same entries, same shapes, before any read
  const auto expected = model_weight_shapes(g_);
  if (names.size() != expected.size()) throw Error(kConfigError, "weights entry count mismatch for model " + g_.name);
  if (values.size() != names.size() || counts.size() != names.size())
    throw Error(kUsageError, "deal_weights: names, values and counts differ in length");
  std::map<std::string, const double*> byname;
  std::map<std::string, size_t> given;
  for (size_t i = 0; i < names.size(); ++i) {
    byname[names[i]] = values[i];
    given[names[i]] = counts[i];
  }
  std::map<std::string, Shape> shapes;
  for (auto& [k, sh] : expected) {
    if (!byname.count(k)) throw Error(kConfigError, "missing weight tensor: " + k);
    if (given.at(k) != shape_numel(sh)) throw Error(kConfigError, "wrong shape for weight tensor: " + k);
    if (!byname.at(k) && given.at(k)) throw Error(kUsageError, "null values for weight tensor: " + k);
    shapes[k] = sh;
  }
  HostRng rng(seed, 0x3e1f);  // one stream over sorted names (H/engine/executor.hpp:49-59)
  for (auto& [key, vals] : byname) {
    const Shape& sh = shapes.at(key);
    const size_t n = shape_numel(sh);
    std::vector<u64> enc(n), host(n * s_.n_local);
    for (size_t i = 0; i < n; ++i) enc[i] = encode_fixed(vals[i], g_.frac_bits);
    if (public_) {
      for (int sl = 0; sl < s_.n_local; ++sl) std::copy(enc.begin(), enc.end(), host.begin() + sl * n);
    } else {
      std::vector<u64> r(n);
      for (size_t i = 0; i < n; ++i) r[i] = rng();
      for (int sl = 0; sl < s_.n_local; ++sl)
        for (size_t i = 0; i < n; ++i) host[sl * n + i] = s_.party_of[sl] == 0 ? enc[i] - r[i] : r[i];
    }
    w_[key] = s_.upload(sh, g_.frac_bits, host.data());
  }
}

void SecureExecutor::set_weight(const std::string& name, const u64* host_words) {
  for (auto& [k, sh] : model_weight_shapes(g_))
    if (k == name) {
      w_[k] = s_.upload(sh, g_.frac_bits, host_words);
      return;
    }
  throw Error(kConfigError, "unknown weight tensor: " + name);
}

std::vector<std::string> SecureExecutor::linear_tags() const {
  std::vector<std::string> t;
  for (auto& op : wops_) t.push_back(op.tag);
  return t;
}

// Fetch the op's triple and put its weight-side opening W - B on the wire
// (H/engine/executor.hpp:279-286).
void SecureExecutor::prepare(size_t i) {
  WeightOp& op = wops_[i];
  Triple t = s_.fetch(op.spec, op.tag);
  t.mark_consumed();
  const DT& W = w_.at(op.wkey);
  const size_t nb = W.numel();
  if (!op.dbuf_out) {  // fixed address: the wrap-around prefetch crosses graph replays
    op.dbuf_out = Block::persistent(nb * s_.n_local + Session::kTrailer);
    if (s_.n_local == 1) op.dbuf_in = Block::persistent(nb + Session::kTrailer);
  }
  Open d = s_.begin_open(nb, Reduce::Sum, op.dbuf_out, op.dbuf_in);
  // fused in-device open of delta, on the same condition as eps's (weight_matmul)
  const size_t M = op.x_shape[0], K = op.x_shape[1];
  d.summed = beaver_combine_fuses_eps(s_, 1, u32(M), u32(nb / K), u32(K));
  if (!delta_defer(s_, d, W.s, u32(M), u32(nb / K), u32(K))) delta_build_mem(s_, t, W.s, nb, d);
  s_.post(d, op.tag + ".delta");
  op.triple = t;
  op.delta = std::move(d);
}

DT SecureExecutor::weight_matmul(size_t i, const DT& x, const ConvGeom* geom, bool col2im_out, Shape out_shape,
                                 const DT* addend) {
  WeightOp& op = wops_[i];
  const u32 M = u32(op.x_shape[0]), K = u32(op.x_shape[1]);
  const DT& W = w_.at(op.wkey);
  const u32 N = u32(W.shape[1]);
  const int f = g_.frac_bits;
  Epi ep{};
  ep.trunc_bits = f;  // finish_linear: truncate then add bias (H/engine/executor.hpp:319-324)
  if (!op.bkey.empty()) {
    const DT& b = w_.at(op.bkey);
    for (int sl = 0; sl < s_.n_local; ++sl)
      ep.bias[sl] = (!public_ || s_.party_of[sl] == 0) ? b.s[sl] : nullptr;
  }
  if (col2im_out) {
    ep.col2im = 1;
    ep.OHW = geom->OH * geom->OW;
  }
  if (addend)  // a following residual add fused into the epilogue (run())
    for (int sl = 0; sl < s_.n_local; ++sl) ep.addend[sl] = addend->s[sl];
  DT z = s_.alloc(out_shape, g_.frac_bits);
  if (public_) {  // local product, no triple, no opening (H/engine/executor.hpp:294-298)
    DT cols = x;
    if (geom) {
      cols = s_.alloc(Shape{M, K}, x.scale);
      const ConvGeom g = *geom;
      const CPtr2 xp = cptrs(x);
      const Ptr2 cp = ptrs(cols);
      launch_ew(s_.stream, s_.n_local, u64(M) * K, [=] __device__(int slot, u64 idx) {
        const u32 KK = g.C * g.k * g.k;
        const u32 r = u32(idx / KK), c = u32(idx - u64(r) * KK);
        const u32 ow = r % g.OW, oh = (r / g.OW) % g.OH, n = r / (g.OW * g.OH);
        const u32 kj = c % g.k, ki = (c / g.k) % g.k, ci = c / (g.k * g.k);
        const int ih = int(oh * g.stride + ki) - int(g.pad), iw = int(ow * g.stride + kj) - int(g.pad);
        u64 v = 0;
        if (ih >= 0 && iw >= 0 && ih < int(g.H) && iw < int(g.W))
          v = sel(xp, slot)[((u64(n) * g.C + ci) * g.H + u32(ih)) * g.W + u32(iw)];
        sel(cp, slot)[idx] = v;
      });
    }
    public_gemm(s_, cols.s, W.s[0], z.s, M, N, K, ep);
    return z;
  }
  if (!op.triple) prepare(i);
  Triple t = *op.triple;
  Open d = std::move(*op.delta);
  op.triple.reset();
  op.delta.reset();
  const size_t na = size_t(M) * K;
  // Inner-layer pipeline on the linear layer (extension, ExecOptions::linear_chunks; the
  // reference's weight_matmul opens eps whole, H/engine/executor.hpp:305): the activation-side
  // opening leaves in n row blocks "<tag>.eps.chunk<k>" and the combine GEMM of block k runs as
  // soon as it lands, while blocks k+1.. are still in flight — the chunk unit and labels of
  // beaver_matmul (H/protocols/beaver.hpp:197-250). Triples, values and bytes are unchanged; a
  // conv chunk is a block of whole output rows (n, oh) so the im2col build stays tiled.
  int nch = opt_.pipelined && opt_.linear_chunks ? chunks_for(s_, na) : 1;
  const size_t unit = geom ? size_t(geom->OW) : 1;  // rows per chunk granule
  nch = clamp_chunks(nch, M / unit);
  std::vector<Open> es(static_cast<size_t>(nch));
  std::vector<DT> aops(static_cast<size_t>(nch));  // A-side combine operands (memory-operand combines only)
  std::vector<std::pair<size_t, size_t>> rows(static_cast<size_t>(nch));
  for (int k = 0; k < nch; ++k) {
    const auto r = chunk_range(M / unit, nch, k);
    rows[k] = {r.first * unit, k + 1 == nch ? size_t(M) : r.second * unit};
    const u32 mk = u32(rows[k].second - rows[k].first);
    const size_t nak = size_t(mk) * K;
    es[k] = s_.begin_open(nak, Reduce::Sum);
    if (beaver_combine_wants_aops(s_, 1, mk, N, K)) aops[k] = s_.alloc(Shape{2, nak});
    else if (!geom || nak < (size_t(1) << 32)) es[k].summed = beaver_combine_fuses_eps(s_, 1, mk, N, K);
    if (aops[k] || !eps_defer(s_, es[k], x.s, geom, rows[k].first * K, mk, N, K)) {
      if (geom)
        eps_build_im2col(s_, t, x.s, *geom, rows[k].first * K, nak, es[k], aops[k] ? &aops[k] : nullptr);
      else
        eps_build_mem(s_, t, x.s, rows[k].first * K, nak, es[k], aops[k] ? &aops[k] : nullptr);
    }
    s_.post(es[k], nch == 1 ? op.tag + ".eps" : op.tag + ".eps.chunk" + std::to_string(k));
  }
  if (opt_.pipelined && wops_.size() > 1) {  // next op's delta leaves while this eps travels
    const size_t next = (i + 1) % wops_.size();
    if (!wops_[next].triple) prepare(next);
  }
  s_.wait(d);
  DT rcache;
  for (int k = 0; k < nch; ++k) {
    const u32 mk = u32(rows[k].second - rows[k].first);
    s_.wait(es[k]);
    beaver_combine(s_, t, es[k], rows[k].first * K, size_t(mk) * K, d, W.numel(), &rcache, z.s,
                   rows[k].first * N, 1, mk, N, K, false, false, 0, ep, aops[k] ? &aops[k] : nullptr);
  }
  return z;
}

DT SecureExecutor::scale_and_rescale(const DT& x, double c) {
  // H/engine/executor.hpp:326-330: multiply by encode(c), then truncate by f.
  const u64 k = encode_fixed(c, g_.frac_bits);
  const int f = g_.frac_bits;
  DT z = s_.alloc(x.shape, x.scale);
  const CPtr2 xp = cptrs(x);
  const Ptr2 zp = ptrs(z);
  launch_ew(s_.stream, s_.n_local, x.numel(),
            [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sar64(sel(xp, slot)[i] * k, f); });
  return z;
}

DT SecureExecutor::attention(const LayerSpec& l, const DT& x, const Shape& in_shape, const DT* addend) {
  // H/engine/executor.hpp:332-362
  const size_t B = in_shape[0], T = in_shape[1], d = in_shape[2];
  const size_t heads = l.heads, dh = d / heads;
  const size_t qkv_op = wop_index_.at(l.name + ".qkv");
  const size_t proj_op = wop_index_.at(l.name + ".proj");
  DT x2 = reshape(x, Shape{B * T, d});
  DT qkv = weight_matmul(qkv_op, x2, nullptr, false, Shape{B * T, 3 * d});
  DT qkvh = s_.alloc(Shape{3, B * heads, T, dh}, qkv.scale);  // split_heads x3 in one gather
  {
    const CPtr2 src = cptrs(qkv);
    const Ptr2 dst = ptrs(qkvh);
    const u32 Tt = u32(T), D = u32(d), H = u32(heads), DH = u32(dh);
    const u64 per = B * heads * T * dh;
    if (3 * per >= (u64(1) << 32)) throw Error(kShapeError, "attention: activation too large");
    const u32 per32 = u32(per);
    launch_ew(s_.stream, s_.n_local, 3 * per, [=] __device__(int slot, u64 i64) {  // 32-bit index math
      const u32 i = u32(i64), part = i / per32, r = i - part * per32;
      const u32 rj = r / DH, j = r - rj * DH, rt = rj / Tt, t = rj - rt * Tt, b = rt / H, h = rt - b * H;
      sel(dst, slot)[i] = sel(src, slot)[(u64(b) * Tt + t) * 3 * D + part * D + h * DH + j];
    });
  }
  const size_t per = B * heads * T * dh;
  DT q, k, v;
  q = qkvh;
  q.shape = Shape{B * heads, T, dh};
  k = q;
  v = q;
  k.s[0] = qkvh.s[0] + per;
  v.s[0] = qkvh.s[0] + 2 * per;
  if (s_.n_local == 2) {
    q.s[1] = qkvh.s[1];
    k.s[1] = qkvh.s[1] + per;
    v.s[1] = qkvh.s[1] + 2 * per;
  }
  DT scores = beaver_matmul(s_, q, k, true, l.name + ".qk", chunks_for(s_, B * heads * T * T));
  {  // truncate, then scale_and_rescale by 1/sqrt(dh), in one local pass (same values as two)
    const u64 kc = encode_fixed(1.0 / std::sqrt(static_cast<double>(dh)), g_.frac_bits);
    const int f = g_.frac_bits;
    DT z = s_.alloc(scores.shape, scores.scale);
    const CPtr2 xp = cptrs(scores);
    const Ptr2 zp = ptrs(z);
    launch_ew(s_.stream, s_.n_local, scores.numel(),
              [=] __device__(int slot, u64 i) { sel(zp, slot)[i] = sar64(sar64(sel(xp, slot)[i], f) * kc, f); });
    scores = z;
  }
  DT probs = softmax_shares(s_, scores, T, l.name + ".softmax");
  DT mixed = beaver_matmul(s_, probs, v, false, l.name + ".av", chunks_for(s_, B * heads * T * dh));
  DT merged = s_.alloc(Shape{B * T, d}, mixed.scale);  // truncate + merge_heads in one local pass
  {
    const CPtr2 src = cptrs(mixed);
    const Ptr2 dst = ptrs(merged);
    const u32 Tt = u32(T), D = u32(d), H = u32(heads), DH = u32(dh);
    const int f = g_.frac_bits;
    if (B * T * d >= (u64(1) << 32)) throw Error(kShapeError, "attention: activation too large");
    launch_ew(s_.stream, s_.n_local, B * T * d, [=] __device__(int slot, u64 i64) {
      const u32 i = u32(i64), q1 = i / DH, j = i - q1 * DH, q2 = q1 / H, h = q1 - q2 * H, b = q2 / Tt, t = q2 - b * Tt;
      sel(dst, slot)[i] = sar64(sel(src, slot)[((u64(b) * H + h) * Tt + t) * DH + j], f);
    });
  }
  DT out = weight_matmul(proj_op, merged, nullptr, false, Shape{B * T, d}, addend);
  return reshape(out, Shape{B, T, d});
}

DT SecureExecutor::run_layer(const LayerSpec& l, const DT& x, const Shape& in_shape, const DT* addend) {
  switch (l.kind) {
    case LayerKind::Dense: {
      const size_t op = wop_index_.at(l.name + ".mm");
      Shape out_shape = in_shape;
      out_shape.back() = l.out;
      DT x2 = reshape(x, wops_[op].x_shape);
      return reshape(weight_matmul(op, x2, nullptr, false, Shape{wops_[op].x_shape[0], l.out}, addend), out_shape);
    }
    case LayerKind::Conv2d: {
      const size_t N = in_shape[0], C = in_shape[1], H = in_shape[2], W = in_shape[3];
      const size_t OH = (H + 2 * l.pad - l.kernel) / l.stride + 1;
      const size_t OW = (W + 2 * l.pad - l.kernel) / l.stride + 1;
      const size_t op = wop_index_.at(l.name + ".mm");
      ConvGeom g{u32(N), u32(C), u32(H), u32(W), u32(l.kernel), u32(l.stride), u32(l.pad), u32(OH), u32(OW)};
      return weight_matmul(op, x, &g, true, Shape{N, l.out, OH, OW}, addend);
    }
    case LayerKind::Relu:
      return relu_shares(s_, x, l.name);
    case LayerKind::Maxpool2d:
      return maxpool2d_shares(s_, x, in_shape[0], in_shape[1], in_shape[2], in_shape[3], l.kernel, l.stride, l.name);
    case LayerKind::Flatten: {
      size_t rest = 1;
      for (size_t i = 1; i < in_shape.size(); ++i) rest *= in_shape[i];
      return reshape(x, Shape{in_shape[0], rest});
    }
    case LayerKind::Attention:
      return attention(l, x, in_shape, addend);
    case LayerKind::Softmax:
      return softmax_shares(s_, x, in_shape.back(), l.name);
    case LayerKind::MeanPool: {
      const size_t B = in_shape[0], T = in_shape[1], d = in_shape[2];
      const u64 k = encode_fixed(1.0 / static_cast<double>(T), g_.frac_bits);
      const int f = g_.frac_bits;
      DT out = s_.alloc(Shape{B, d}, x.scale);
      const CPtr2 xp = cptrs(x);
      const Ptr2 op = ptrs(out);
      const u64 Tt = T, D = d;
      launch_ew(s_.stream, s_.n_local, B * d, [=] __device__(int slot, u64 i) {
        const u64 b = i / D, j = i - b * D;
        u64 acc = 0;
        for (u64 t = 0; t < Tt; ++t) acc += sel(xp, slot)[(b * Tt + t) * D + j];
        sel(op, slot)[i] = sar64(acc * k, f);
      });
      return out;
    }
    case LayerKind::GlobalAvgPool:
      return global_avg_pool(s_, x, in_shape[0], in_shape[1], in_shape[2] * in_shape[3]);
    case LayerKind::Gelu:
      return gelu_shares(s_, x, l.name);
    case LayerKind::LayerNorm:
      return layernorm_shares(s_, x, in_shape.back(), w_.at(l.name + ".gamma"), w_.at(l.name + ".beta"), public_,
                              l.name);
    case LayerKind::Add:
      break;  // needs both operands: handled in run()
  }
  throw Error(kProtocolError, "unhandled layer kind");
}

void SecureExecutor::capture(const DT& input) {
  if (opt_.pipelined && !public_ && !wops_.empty() && !wops_[0].triple)
    throw Error(kUsageError, "capture needs one eager run first (pipelined prologue)");
  // An open posted before the capture (the wrap-around delta on an emulated link / NCCL) must
  // be waited outside it; inside the graph its data is then already in place, and each replay
  // joins its own comm-stream work before it ends (Session::end_capture).
  for (auto& op : wops_)
    if (op.delta && op.delta->ready) {
      MPCG_CUDA(cudaStreamWaitEvent(s_.stream, op.delta->ready, 0));
      op.delta->ready = nullptr;
    }
  s_.begin_capture();
  try {
    for (auto& op : wops_)  // prefetched before the capture, consumed inside it
      if (op.triple) s_.capture_adopt(*op.triple);
    graph_out_ = run(input);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s_.stream, &g);
    if (g) cudaGraphDestroy(g);
    s_.cap.active = false;
    throw;
  }
  s_.end_capture();
  captured_ = true;
}

DT SecureExecutor::replay() {
  if (!captured_) throw Error(kUsageError, "replay before capture");
  s_.replay();
  return graph_out_;
}

// Hand the dealer streams back to eager calls. A triple prefetched inside the graph (the
// pipelined wrap-around) reads its key from the device key table, which holds the key of the
// last replay's prefetch; it is pinned to that key so the next eager run() consumes exactly
// the triple whose delta the last replay left in the persistent payload buffer.
void SecureExecutor::release_graph() {
  if (!captured_) return;
  s_.sync();
  for (auto& op : wops_)
    if (op.triple && (op.triple->ew.kp || op.triple->mm.kp)) {
      const u64* kp = op.triple->mm.kp ? op.triple->mm.kp : op.triple->ew.kp;
      u64 key = 0;
      MPCG_CUDA(cudaMemcpy(&key, kp, sizeof key, cudaMemcpyDeviceToHost));
      op.triple->key = op.triple->ew.key = op.triple->mm.key = key;
      op.triple->ew.kp = op.triple->mm.kp = nullptr;
    }
  s_.release_graph();
  captured_ = false;
  graph_out_ = DT{};
}

DT SecureExecutor::run(const DT& input) {
  if (!s_.cap.active) s_.require_eager_streams("run");  // before any prefetched state is consumed
  if (input.shape != g_.input) throw Error(kConfigError, "run: input shape mismatch");
  for (auto& [k, sh] : model_weight_shapes(g_))
    if (!w_.count(k)) throw Error(kConfigError, "missing weight tensor: " + k);
  if (opt_.pipelined && !public_ && !wops_.empty() && !wops_[0].triple) prepare(0);
  if (time_layers && ev_.size() < g_.layers.size() + 1) {
    for (auto e : ev_) cudaEventDestroy(e);
    ev_.assign(g_.layers.size() + 1, nullptr);
    for (auto& e : ev_) MPCG_CUDA(cudaEventCreate(&e));
  }
  const unsigned rec_flags = s_.cap.active ? cudaEventRecordExternal : cudaEventRecordDefault;  // graph event nodes
  if (time_layers) MPCG_CUDA(cudaEventRecordWithFlags(ev_[0], s_.stream, rec_flags));
  // Layers run in list order (the reference's chain order, executor.hpp:193-205); an output
  // is kept only until its last reader ("from"/"with" of a later layer) has run.
  const LayerWiring wr = layer_wiring(g_);
  const size_t nl = g_.layers.size();
  std::vector<size_t> last(nl, 0);
  for (size_t i = 0; i < nl; ++i) {
    last[i] = i + 1 < nl ? i + 1 : i;
    if (wr.src[i] >= 0) last[size_t(wr.src[i])] = std::max(last[size_t(wr.src[i])], i);
    if (wr.other[i] >= 0) last[size_t(wr.other[i])] = std::max(last[size_t(wr.other[i])], i);
  }
  // A conv / dense / attention layer (its output projection) whose only reader is the residual add right after it takes the add's
  // other operand as an epilogue addend (one pass over the output instead of a separate add
  // kernel re-reading it; values identical, the add has no collective). MPCG_FUSE_RESIDUAL=0
  // keeps the separate add.
  static const bool fuse_res = [] {
    const char* e = std::getenv("MPCG_FUSE_RESIDUAL");
    return !(e && e[0] == '0');
  }();
  std::vector<int> fused_into(nl, -1);  // add layer j -> the linear layer that produced it
  if (fuse_res)
    for (size_t j = 1; j < nl; ++j) {
      const LayerSpec& l = g_.layers[j];
      const size_t i = j - 1;
      const LayerKind k = g_.layers[i].kind;
      if (l.kind != LayerKind::Add || (k != LayerKind::Conv2d && k != LayerKind::Dense && k != LayerKind::Attention))
        continue;
      if (!(wr.src[j] == int(i)) == !(wr.other[j] == int(i))) continue;  // exactly one operand is layer i
      bool only = true;
      for (size_t q = 0; q < nl; ++q)
        if (q != j && (wr.src[q] == int(i) || wr.other[q] == int(i))) only = false;
      if (only && shape_numel(shapes_[i]) == shape_numel(shapes_[j])) fused_into[j] = int(i);
    }
  std::vector<DT> outs(nl);
  for (size_t i = 0; i < nl; ++i) {
    const LayerSpec& l = g_.layers[i];
    const DT& x = wr.src[i] < 0 ? input : outs[size_t(wr.src[i])];
    const Shape& xs = wr.src[i] < 0 ? g_.input : shapes_[size_t(wr.src[i])];
    if (l.kind == LayerKind::Add && fused_into[i] >= 0) {  // already added in the GEMM epilogue
      outs[i] = outs[size_t(fused_into[i])];
    } else if (l.kind == LayerKind::Add) {  // residual: local share addition
      outs[i] = add_t(s_, x, wr.other[i] < 0 ? input : outs[size_t(wr.other[i])]);
    } else if (i + 1 < nl && fused_into[i + 1] == int(i)) {
      const long o = wr.src[i + 1] == long(i) ? wr.other[i + 1] : wr.src[i + 1];
      outs[i] = run_layer(l, x, xs, o < 0 ? &input : &outs[size_t(o)]);
    } else {
      outs[i] = run_layer(l, x, xs);
    }
    if (time_layers) MPCG_CUDA(cudaEventRecordWithFlags(ev_[i + 1], s_.stream, rec_flags));
    for (size_t j = 0; j < i; ++j)
      if (outs[j] && last[j] <= i) outs[j] = DT{};
  }
  if (time_layers && !s_.cap.active) collect_timings();  // captured: event nodes, read after replay
  return outs[nl - 1];
}

void SecureExecutor::collect_timings() {
  if (ev_.size() < g_.layers.size() + 1) return;
  MPCG_CUDA(cudaEventSynchronize(ev_.back()));
  timings.clear();
  for (size_t i = 0; i < g_.layers.size(); ++i) {
    float ms = 0;
    MPCG_CUDA(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]));
    timings.push_back({g_.layers[i].name, ms});
  }
}

}  // namespace mpcg
