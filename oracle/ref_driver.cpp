// Oracle driver over the UNMODIFIED reference headers (test infrastructure only).
//
// Built by oracle/Makefile into oracle/_ref/ref_driver from /root/reference/proj/include
// (read in place, never copied). Two subcommands:
//
//   ref_driver golden <out.bin>
//       Runs each hot-path op of the reference (H/protocols, H/nonlinear, H/engine)
//       on seeded inputs with 2 parties over the deterministic SimNet and dumps
//       inputs and per-party output shares. tests/golden/make_golden.py turns the
//       dump into tests/golden/*.npz fixtures.
//
//   ref_driver mpcw <model.json> <seed> <out.mpcw> [<in.mpcw>]
//       The reference's init_weights written with its save_weights, or a file read back by
//       its load_weights/check_weights and re-saved (MPCW interchange pin).
//
//   ref_driver model_pin <model.json> <mode> <iters> <private|public> <seed> <out.bin>
//       As `model` (the per-party output shares of SecureExecutor::run), pinned by FNV-1a
//       hash + head/tail words: single-layer models at BASELINE layer shapes.
//
//   ref_driver scale <case|all> <out.bin>
//       Reference ops at BASELINE shapes (ResNet-18 ReLU, VGG-16 pool1, BERT-base softmax /
//       QK^T / AV, full-word GEMMs at ResNet-18 layer4 and VGG-16 fc6), pinned the same way.
//
//   ref_driver triples <out.bin>
//       Two dealer triples written by the reference's save_triples (triple-file pin).
//
//   ref_driver opsum <model.json> <private|public> <div> <pairs> <seed>
//       Op-sum CPU estimate of one inference (configs the reference cannot express): the
//       reference's ops timed at every layer's shape on 1/div of its rows, scaled; `pairs`
//       concurrent pairs (2 threads each). Prints one JSON line.
//
//   ref_driver bench <model.json> <blocking|pipelined> <iters> <private|public> <seed>
//                    [<chunks> <threshold_bytes>]
//       Times bench_party (H/engine/bench.hpp:36-79) with the two parties as threads
//       over SocketComm on loopback (real wall clock, 1 thread per party) and prints
//       one JSON line: per-iteration wall seconds, bytes, collectives, logits hash.
//
// H/ = /root/reference/proj/include/mpcpipe.
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "mpcpipe/engine/bench.hpp"
#include "mpcpipe/engine/executor.hpp"
#include "mpcpipe/engine/reference.hpp"
#include "mpcpipe/nonlinear/activations.hpp"
#include "mpcpipe/protocols/adder.hpp"
#include "mpcpipe/protocols/beaver.hpp"
#include "mpcpipe/protocols/compare.hpp"
#include "mpcpipe/protocols/trunc.hpp"
#include "mpcpipe/transport/harness.hpp"

using namespace mpcpipe;

namespace {

std::FILE* g_out = nullptr;

void put(const std::string& name, const Shape& shape, std::span<const u64> data) {
  uint32_t nl = static_cast<uint32_t>(name.size());
  std::fwrite(&nl, 4, 1, g_out);
  std::fwrite(name.data(), 1, nl, g_out);
  uint32_t nd = static_cast<uint32_t>(shape.size());
  std::fwrite(&nd, 4, 1, g_out);
  for (auto d : shape) {
    u64 dd = d;
    std::fwrite(&dd, 8, 1, g_out);
  }
  std::fwrite(data.data(), 8, data.size(), g_out);
}

void put(const std::string& name, const RingTensor& t) { put(name, t.shape(), t.data()); }

SessionConfig sim2() {
  SessionConfig cfg;
  cfg.n_parties = 2;
  cfg.backend = Backend::Sim;
  cfg.latency_s = 0;
  cfg.sec_per_message = 0;
  cfg.sec_per_unit = 0;
  cfg.sec_per_dispatch = 0;
  return cfg;
}

RingTensor rand_t(const Shape& s, CounterRng& r, int scale = 0) {
  RingTensor t(s, scale);
  for (auto& w : t.data()) w = r();
  return t;
}

// Small signed fixed-point values in [-range, range) at scale f.
RingTensor rand_fixed(const Shape& s, CounterRng& r, double range, int f) {
  RingTensor t(s, f);
  for (auto& w : t.data()) {
    double u = static_cast<double>(r() >> 11) * 0x1.0p-53;
    w = encode_fixed((2 * u - 1) * range, f);
  }
  return t;
}

// One op case: `fn(ctx, party, share_x, share_y)` -> output share tensor.
template <class Fn>
void run_case(const std::string& name, const RingTensor& x, const RingTensor& y, u64 seed, int f,
              int chunks, Fn fn) {
  CounterRng share_rng(seed);
  auto xs = share_additive(x, 2, share_rng);
  auto ys = share_additive(y, 2, share_rng);
  put(name + "/x0", xs[0].tensor);
  put(name + "/x1", xs[1].tensor);
  put(name + "/y0", ys[0].tensor);
  put(name + "/y1", ys[1].tensor);
  std::vector<RingTensor> outs(2);
  std::vector<CommStats> stats(2);
  auto comms = make_sim_comms(sim2());
  run_parties(2, [&](int p) {
    SeededDealer dealer(seed + 1, p, 2);
    CounterRng mask(seed + 2, static_cast<u64>(p));
    ProtoCtx ctx{dealer, *comms[p], mask, f};
    ctx.chunks = chunks;
    ctx.chunk_threshold = 0;
    outs[p] = fn(ctx, p, xs[p], ys[p]);
    stats[p] = comms[p]->stats();
  });
  put(name + "/z0", outs[0]);
  put(name + "/z1", outs[1]);
  std::vector<u64> st{stats[0].bytes_sent, stats[0].collectives, stats[0].p2p_sends};
  put(name + "/stats", Shape{3}, st);
}

int cmd_golden(const char* path) {
  g_out = std::fopen(path, "wb");
  if (!g_out) return 2;
  // PRG known answers (H/sharing/rng.hpp:10-32).
  {
    CounterRng r(123, 7);
    std::vector<u64> v;
    for (int i = 0; i < 16; ++i) v.push_back(r());
    put("prg/123_7", Shape{16}, v);
  }
  // Dealer triples (H/sharing/triple.hpp:85-151): fetch twice per tag + untagged.
  {
    struct D {
      std::string name;
      TripleSpec spec;
      std::string tag;
    };
    std::vector<D> ds{
        {"mul0", TripleSpec::elementwise(TripleKind::Arith, {3, 4}), "t.mul"},
        {"mul1", TripleSpec::elementwise(TripleKind::Arith, {3, 4}), "t.mul"},
        {"and", TripleSpec::elementwise(TripleKind::Bin, {2, 5}), "t.and"},
        {"sq", TripleSpec::square_of({7}), "t.sq"},
        {"mm", TripleSpec::matmul_of({3, 4}, {4, 5}), "t.mm"},
        {"qk", TripleSpec::matmul_of({2, 3, 4}, {2, 5, 4}, true), "t.qk"},
        {"av", TripleSpec::matmul_of({2, 3, 5}, {2, 5, 4}, false), "t.av"},
        {"untag0", TripleSpec::elementwise(TripleKind::Arith, {6}), ""},
        {"untag1", TripleSpec::elementwise(TripleKind::Arith, {6}), ""},
    };
    for (int p = 0; p < 2; ++p) {
      SeededDealer dealer(5, p, 2);
      for (auto& d : ds) {
        BeaverTriple t = dealer.fetch(d.spec, d.tag);
        std::string b = "dealer/" + d.name + "/p" + std::to_string(p);
        put(b + "/a", t.a);
        put(b + "/b", t.b);
        put(b + "/c", t.c);
      }
    }
  }
  // Protocol ops on seeded inputs.
  CounterRng gen(2024);
  const int f = 16;
  {
    RingTensor x = rand_t({5, 7}, gen), y = rand_t({5, 7}, gen);
    for (int ch : {1, 3}) {
      run_case("mul_c" + std::to_string(ch), x, y, 11, f, ch, [&](ProtoCtx& c, int, auto& a, auto& b) {
        return beaver_mul(a, b, c.triples, c.comm, "mul", ch).tensor;
      });
      run_case("square_c" + std::to_string(ch), x, y, 12, f, ch, [&](ProtoCtx& c, int, auto& a, auto&) {
        return beaver_square(a, c.triples, c.comm, "square", ch).tensor;
      });
      run_case("and_c" + std::to_string(ch), x, y, 13, f, ch, [&](ProtoCtx& c, int p, auto& a, auto& b) {
        return beaver_and(BinaryShare{p, a.tensor}, BinaryShare{p, b.tensor}, c.triples, c.comm, "and", ch)
            .tensor;
      });
      run_case("badd_c" + std::to_string(ch), x, y, 14, f, ch, [&](ProtoCtx& c, int p, auto& a, auto& b) {
        AdderOptions o;
        o.chunks = ch;
        return binary_add(BinaryShare{p, a.tensor}, BinaryShare{p, b.tensor}, c.triples, c.comm, o, "badd")
            .tensor;
      });
    }
    RingTensor xf = rand_fixed({6, 9}, gen, 50.0, f), yf = rand_fixed({6, 9}, gen, 50.0, f);
    run_case("a2b", xf, yf, 15, f, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return a2b(a, c.triples, c.comm, c.rng, c.adder, "a2b").tensor;
    });
    run_case("msb", xf, yf, 16, f, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return msb(a, c.triples, c.comm, c.rng, c.adder, "msb").tensor;
    });
    run_case("lt", xf, yf, 17, f, 1, [&](ProtoCtx& c, int, auto& a, auto& b) {
      return less_than(a, b, c.triples, c.comm, c.rng, c.adder, "lt").tensor;
    });
    run_case("relu", xf, yf, 18, f, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return relu_shares(a, c, "relu").tensor;
    });
    run_case("relu_c4", xf, yf, 18, f, 4, [&](ProtoCtx& c, int, auto& a, auto&) {
      return relu_shares(a, c, "relu").tensor;
    });
    run_case("trunc", xf, yf, 19, f, 1, [&](ProtoCtx& c, int, auto& a, auto& b) {
      AdditiveShare z = beaver_mul(a, b, c.triples, c.comm, "tm");
      return truncate_shares(z, f, c.comm, c.rng).tensor;
    });
    for (std::size_t L : {5u, 8u, 9u}) {
      RingTensor m = rand_fixed({4, L}, gen, 20.0, f);
      run_case("max_L" + std::to_string(L), m, m, 20, f, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
        return max_last_dim(a, L, c, "max").tensor;
      });
    }
    RingTensor e = rand_fixed({3, 6}, gen, 4.0, 20);
    for (auto& w : e.data()) w = w - encode_fixed(4.0, 20);  // exp domain x <= 0
    run_case("exp", e, e, 21, 20, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return exp_shares(a, c, "exp").tensor;
    });
    RingTensor rr(Shape{8}, 20);
    double rv[8] = {0.25, 0.5, 1.0, 3.0, 7.5, 30.0, 100.0, 1000.0};
    for (int i = 0; i < 8; ++i) rr.at(i) = encode_fixed(rv[i], 20);
    run_case("recip", rr, rr, 22, 20, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return reciprocal_shares(a, c, "recip").tensor;
    });
    RingTensor sm = rand_fixed({4, 6}, gen, 3.0, 20);
    run_case("softmax", sm, sm, 23, 20, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return softmax_shares(a, 6, c, "softmax").tensor;
    });
    run_case("softmax_c2", sm, sm, 23, 20, 2, [&](ProtoCtx& c, int, auto& a, auto&) {
      return softmax_shares(a, 6, c, "softmax").tensor;
    });
    RingTensor mp = rand_fixed({2, 3, 5, 4}, gen, 10.0, f);
    run_case("maxpool", mp, mp, 24, f, 1, [&](ProtoCtx& c, int, auto& a, auto&) {
      return maxpool2d_shares(a, 2, 3, 5, 4, 2, 2, c, "pool").tensor;
    });
    RingTensor ma = rand_t({3, 4}, gen), mb = rand_t({4, 5}, gen);
    run_case("matmul", ma, mb, 25, f, 1, [&](ProtoCtx& c, int, auto& a, auto& b) {
      return beaver_matmul(a, b, false, c.triples, c.comm, "mm").tensor;
    });
    RingTensor qa = rand_t({2, 3, 4}, gen), qb = rand_t({2, 5, 4}, gen);
    run_case("matmul_t", qa, qb, 26, f, 2, [&](ProtoCtx& c, int, auto& a, auto& b) {
      return beaver_matmul(a, b, true, c.triples, c.comm, "qk", 2).tensor;
    });
  }
  std::fclose(g_out);
  return 0;
}

// ---------------------------------------------------------------- BASELINE-scale pins
// Inputs are pure functions of (seed, stream) so the GPU tests regenerate them in numpy:
// a value word v_i = (i64)draw_i >> (64 - bits) of CounterRng(seed, 0), party 1's share
// draw_i of CounterRng(seed, 1), party 0's share v_i - that. Full-word operands (GEMMs) are
// the two draw streams themselves. Outputs are too large for fixtures, so each party's
// share is pinned by its FNV-1a word hash (H/engine/report.hpp:18-23) plus head/tail words.
RingTensor draws_t(const Shape& s, u64 seed, u64 stream) {
  CounterRng r(seed, stream);
  RingTensor t(s, 0);
  for (auto& w : t.data()) w = r();
  return t;
}

std::array<RingTensor, 2> small_shares(const Shape& s, u64 seed, int bits, int f) {
  CounterRng v(seed, 0);
  RingTensor x1 = draws_t(s, seed, 1), x0(s, f);
  x1.set_scale_bits(f);
  for (std::size_t i = 0; i < x0.numel(); ++i)
    x0.at(i) = static_cast<u64>(static_cast<std::int64_t>(v()) >> (64 - bits)) - x1.at(i);
  return {x0, x1};
}

void put_pin(const std::string& name, const RingTensor& t) {
  const auto d = t.data();
  const std::size_t k = std::min<std::size_t>(16, d.size());
  std::vector<u64> meta{fnv1a_words(d), d.size()};
  put(name + "/hash", Shape{2}, meta);
  put(name + "/head", Shape{k}, std::span<const u64>(d.data(), k));
  put(name + "/tail", Shape{k}, std::span<const u64>(d.data() + d.size() - k, k));
}

template <class Fn>
void run_scale(const std::string& name, const std::array<RingTensor, 2>& xs, const std::array<RingTensor, 2>& ys,
               u64 seed, int f, int chunks, std::size_t threshold, Fn fn) {
  std::vector<RingTensor> outs(2);
  std::vector<CommStats> stats(2);
  auto comms = make_sim_comms(sim2());
  const auto t0 = std::chrono::steady_clock::now();
  run_parties(2, [&](int p) {
    SeededDealer dealer(seed + 1, p, 2);
    CounterRng mask(seed + 2, static_cast<u64>(p));
    ProtoCtx ctx{dealer, *comms[p], mask, f};
    ctx.chunks = chunks;
    ctx.chunk_threshold = threshold;
    outs[p] = fn(ctx, p, AdditiveShare{p, xs[p]}, AdditiveShare{p, ys[p]});
    stats[p] = comms[p]->stats();
  });
  const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  put_pin(name + "/z0", outs[0]);
  put_pin(name + "/z1", outs[1]);
  put_pin(name + "/open", add(outs[0], outs[1]));
  std::vector<u64> st{stats[0].bytes_sent, stats[0].collectives, stats[0].p2p_sends};
  put(name + "/stats", Shape{3}, st);
  std::fprintf(stderr, "%s: %.1f s\n", name.c_str(), dt);
}

int cmd_scale(const std::string& which, const char* path) {
  g_out = std::fopen(path, "wb");
  if (!g_out) return 2;
  const std::size_t thr = std::size_t(2) << 20;  // ExecOptions default (H/engine/executor.hpp:28-36)
  const std::array<RingTensor, 2> none{RingTensor{}, RingTensor{}};
  auto want = [&](const char* n) { return which == "all" || which == n; };
  if (want("relu_r18")) {  // ResNet-18 conv1 output, 8.4M elements (H/nonlinear/activations.hpp:39-47)
    auto xs = small_shares({128, 64, 32, 32}, 31, 24, 20);
    run_scale("relu_r18", xs, none, 31, 20, 4, thr,
              [](ProtoCtx& c, int, const AdditiveShare& x, const AdditiveShare&) {
                return relu_shares(x, c, "relu").tensor;
              });
  }
  if (want("pool_vgg1")) {  // VGG-16 pool1 (activations.hpp:114-137)
    auto xs = small_shares({1, 64, 224, 224}, 32, 24, 20);
    run_scale("pool_vgg1", xs, none, 32, 20, 4, thr,
              [](ProtoCtx& c, int, const AdditiveShare& x, const AdditiveShare&) {
                return maxpool2d_shares(x, 1, 64, 224, 224, 2, 2, c, "pool1").tensor;
              });
  }
  if (want("softmax_bert")) {  // BERT-base attention scores [B*H*T, T] (activations.hpp:93-110)
    auto xs = small_shares({12288, 128}, 33, 18, 16);
    run_scale("softmax_bert", xs, none, 33, 16, 4, thr,
              [](ProtoCtx& c, int, const AdditiveShare& x, const AdditiveShare&) {
                return softmax_shares(x, 128, c, "softmax").tensor;
              });
  }
  if (want("qk_bert")) {  // Q K^T of BERT-base, chunked (beaver.hpp:186-250)
    std::array<RingTensor, 2> q{draws_t({96, 128, 64}, 34, 0), draws_t({96, 128, 64}, 34, 1)};
    std::array<RingTensor, 2> k{draws_t({96, 128, 64}, 34, 2), draws_t({96, 128, 64}, 34, 3)};
    run_scale("qk_bert", q, k, 34, 16, 4, thr, [](ProtoCtx& c, int, const AdditiveShare& a, const AdditiveShare& b) {
      return beaver_matmul(a, b, true, c.triples, c.comm, "attn.qk", c.chunks_for(96 * 128 * 128)).tensor;
    });
  }
  if (want("av_bert")) {  // P V of BERT-base
    std::array<RingTensor, 2> p{draws_t({96, 128, 128}, 35, 0), draws_t({96, 128, 128}, 35, 1)};
    std::array<RingTensor, 2> v{draws_t({96, 128, 64}, 35, 2), draws_t({96, 128, 64}, 35, 3)};
    run_scale("av_bert", p, v, 35, 16, 4, thr, [](ProtoCtx& c, int, const AdditiveShare& a, const AdditiveShare& b) {
      return beaver_matmul(a, b, false, c.triples, c.comm, "attn.av", c.chunks_for(96 * 128 * 64)).tensor;
    });
  }
  if (want("gemm_r18l4")) {  // full-word operands at ResNet-18 layer4's im2col shape: K' = 3*4608
    std::array<RingTensor, 2> x{draws_t({2048, 4608}, 36, 0), draws_t({2048, 4608}, 36, 1)};
    std::array<RingTensor, 2> w{draws_t({4608, 512}, 36, 2), draws_t({4608, 512}, 36, 3)};
    run_scale("gemm_r18l4", x, w, 36, 20, 1, thr, [](ProtoCtx& c, int, const AdditiveShare& a, const AdditiveShare& b) {
      return beaver_matmul(a, b, false, c.triples, c.comm, "l4.mm").tensor;
    });
  }
  if (want("gemm_fc6")) {  // full-word operands at VGG-16 fc6's shape (1, 25088, 4096)
    std::array<RingTensor, 2> x{draws_t({1, 25088}, 37, 0), draws_t({1, 25088}, 37, 1)};
    std::array<RingTensor, 2> w{draws_t({25088, 4096}, 37, 2), draws_t({25088, 4096}, 37, 3)};
    run_scale("gemm_fc6", x, w, 37, 20, 1, thr, [](ProtoCtx& c, int, const AdditiveShare& a, const AdditiveShare& b) {
      return beaver_matmul(a, b, false, c.triples, c.comm, "fc6.mm").tensor;
    });
  }
  std::fclose(g_out);
  return 0;
}

// Model-level golden: per-party logits shares after `iters` runs plus the hash. With
// pin_only the shares are pinned by hash + head/tail words (outputs of BASELINE-scale layers).
int cmd_model_golden(const char* model_path, const char* mode, int iters, const char* weights,
                     u64 seed, const char* out_path, bool pin_only = false) {
  BenchSpec spec;
  spec.model = load_model(model_path);
  spec.weights = init_weights(spec.model, seed + 11);
  spec.input = demo_input(spec.model, seed + 12);
  spec.public_weights = std::string(weights) == "public";
  spec.iterations = iters;
  spec.session = sim2();
  spec.session.seed = seed;
  spec.exec.mode = std::string(mode) == "pipelined" ? ExecMode::Pipelined : ExecMode::Blocking;
  auto comms = make_sim_comms(spec.session);
  std::vector<RingTensor> outs(2);
  std::vector<PartyResult> res(2);
  // Capture the logits share of each party by re-running the body: bench_party opens the
  // logits, so we replicate its share-producing part here (H/engine/bench.hpp:36-60).
  run_parties(2, [&](int p) {
    Communicator& comm = *comms[p];
    SeededDealer dealer(seed, p, 2);
    CounterRng mask_rng(seed ^ 0x9e3779b97f4a7c15ull, static_cast<u64>(p));
    WeightSet wset = spec.public_weights ? public_weight_set(spec.model, spec.weights)
                                         : deal_weight_shares(spec.model, spec.weights, 2, p, seed);
    SecureExecutor exec(spec.model, std::move(wset), dealer, comm, mask_rng, spec.exec);
    AdditiveShare input = deal_input_share(spec.input, spec.model.frac_bits, 2, p, seed + 1);
    AdditiveShare out{p, RingTensor{}};
    for (int it = 0; it < iters; ++it) out = exec.run(input);
    outs[p] = out.tensor;
    RingTensor logits = comm.reveal(out.tensor, Reduce::Sum, "logits.open");
    res[p].logits = logits;
    res[p].report.bytes_sent = comm.stats().bytes_sent;
    res[p].report.collectives = comm.stats().collectives;
    res[p].report.p2p_sends = comm.stats().p2p_sends;
  });
  g_out = std::fopen(out_path, "wb");
  if (!g_out) return 2;
  std::vector<u64> meta{fnv1a_words(res[0].logits.data()), res[0].report.bytes_sent,
                        res[0].report.collectives, res[0].report.p2p_sends};
  put("meta", Shape{4}, meta);
  if (pin_only) {
    put_pin("z0", outs[0]);
    put_pin("z1", outs[1]);
    std::fclose(g_out);
    std::printf("hash 0x%016llx\n", static_cast<unsigned long long>(meta[0]));
    return 0;
  }
  put("z0", outs[0]);
  put("z1", outs[1]);
  put("logits", res[0].logits);
  DoubleTensor ref = reference_forward(spec.model, spec.weights, spec.input);
  std::vector<u64> refbits(ref.v.size());
  std::memcpy(refbits.data(), ref.v.data(), 8 * ref.v.size());
  put("reference_forward", ref.shape, refbits);
  std::fclose(g_out);
  std::printf("hash 0x%016llx\n", static_cast<unsigned long long>(meta[0]));
  return 0;
}

int cmd_bench(int argc, char** argv) {
  if (argc < 7) return 2;
  BenchSpec spec;
  spec.model = load_model(argv[2]);
  const u64 seed = std::strtoull(argv[6], nullptr, 10);
  spec.weights = init_weights(spec.model, seed + 11);
  spec.input = demo_input(spec.model, seed + 12);
  spec.public_weights = std::string(argv[5]) == "public";
  spec.iterations = std::atoi(argv[4]);
  spec.session.n_parties = 2;
  spec.session.backend = Backend::Socket;
  spec.session.seed = seed;
  if (const char* env = std::getenv("MPCPIPE_PORT_BASE")) spec.session.port_base = std::atoi(env);
  spec.exec.mode = std::string(argv[3]) == "pipelined" ? ExecMode::Pipelined : ExecMode::Blocking;
  if (argc >= 9) {
    spec.exec.chunks = std::atoi(argv[7]);
    spec.exec.chunk_threshold = std::strtoull(argv[8], nullptr, 10);
  }
  std::vector<RunReport> reps(2);
  run_parties(2, [&](int p) { reps[p] = run_socket_bench_party(spec, p); });
  std::printf("{\"model\": \"%s\", \"mode\": \"%s\", \"iterations\": %d, \"iter_wall_s\": [",
              spec.model.name.c_str(), argv[3], spec.iterations);
  const auto& p0 = reps[0].parties[0];
  const auto& p1 = reps[1].parties[0];
  for (std::size_t i = 0; i < p0.iter_wall_s.size(); ++i)
    std::printf("%s%.6f", i ? ", " : "", std::max(p0.iter_wall_s[i], p1.iter_wall_s[i]));
  std::printf("], \"bytes_sent\": %llu, \"collectives\": %llu, \"p2p_sends\": %llu, "
              "\"logits_hash\": \"0x%016llx\"}\n",
              static_cast<unsigned long long>(p0.bytes_sent),
              static_cast<unsigned long long>(p0.collectives),
              static_cast<unsigned long long>(p0.p2p_sends),
              static_cast<unsigned long long>(reps[0].logits_hash));
  return 0;
}

// ---------------------------------------------------------------- op-sum estimate
// ResNet-18 and BERT-base are not expressible in the reference (no residual add, GeLU,
// LayerNorm; H/engine/model.hpp:21), so its CPU cost for them is estimated the way SURVEY
// 8(d) prescribes: the reference's own ops (beaver_matmul + truncate_shares for a private
// linear layer, matmul for a public one, relu_shares, max_last_dim, softmax_shares, ...) timed
// at each layer's shape on a row sample (1/div of the rows, at least one), scaled linearly.
// Each pair runs both parties as threads over the in-memory SimComm (no link cost: the
// estimate is compute only, i.e. a lower bound on the reference's latency), and `pairs`
// independent pairs run concurrently so all host cores are used; benchdetail::timed_op_run
// (H/engine/bench.hpp:144-169) is the model. GeLU / LayerNorm (extensions) are costed as the
// reference blocks they are built from (msb + b2a + exp + reciprocal + muls; square + exp +
// Newton muls). Layer kinds as in the package's model JSON.
struct OpLayer {
  std::string name, kind;
  Shape in;        // input shape
  std::size_t out = 0, kernel = 0, stride = 1, pad = 0, heads = 0;
};

std::vector<OpLayer> opsum_layers(const nlohmann::json& j, Shape& input) {
  input = j.at("input").get<Shape>();
  std::vector<OpLayer> ls;
  std::map<std::string, Shape> outs;
  Shape cur = input;
  for (const auto& l : j.at("layers")) {
    OpLayer o;
    o.name = l.at("name").get<std::string>();
    o.kind = l.at("type").get<std::string>();
    if (l.contains("from")) {
      const std::string f = l.at("from").get<std::string>();
      cur = f == "input" ? input : outs.at(f);
    }
    o.in = cur;
    o.out = l.value("out", std::size_t(0));
    o.kernel = l.value("kernel", std::size_t(0));
    o.stride = l.value("stride", std::size_t(1));
    o.pad = l.value("pad", std::size_t(0));
    o.heads = l.value("heads", std::size_t(0));
    if (o.kind == "conv2d") {
      cur = {cur[0], o.out, (cur[2] + 2 * o.pad - o.kernel) / o.stride + 1, (cur[3] + 2 * o.pad - o.kernel) / o.stride + 1};
    } else if (o.kind == "maxpool2d") {
      cur = {cur[0], cur[1], (cur[2] - o.kernel) / o.stride + 1, (cur[3] - o.kernel) / o.stride + 1};
    } else if (o.kind == "dense") {
      cur.back() = o.out;
    } else if (o.kind == "flatten") {
      cur = {cur[0], shape_numel(cur) / cur[0]};
    } else if (o.kind == "global_avg_pool") {
      cur = {cur[0], cur[1]};
    } else if (o.kind == "mean_pool") {
      cur = {cur[0], cur[2]};
    }
    outs[o.name] = cur;
    ls.push_back(o);
  }
  return ls;
}

int cmd_opsum(const char* model_path, const char* weights, std::size_t div, int pairs, u64 seed) {
  std::ifstream in(model_path);
  if (!in) throw ConfigError(std::string("opsum: cannot open ") + model_path);
  nlohmann::json j;
  in >> j;
  Shape input;
  const auto layers = opsum_layers(j, input);
  const int f = j.value("frac_bits", 20);
  const bool pub = std::string(weights) == "public";
  const std::size_t nl = layers.size();
  // per pair, per layer: sampled seconds (max over the two parties) and the row scale
  std::vector<std::vector<double>> sec(std::size_t(pairs), std::vector<double>(nl, 0.0));
  std::vector<double> scale(nl, 0.0);
  auto rows_of = [&](std::size_t rows) { return std::max<std::size_t>(1, rows / div); };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int pr = 0; pr < pairs; ++pr)
    th.emplace_back([&, pr] {
      auto comms = make_sim_comms(sim2());
      std::vector<std::vector<double>> ps(2, std::vector<double>(nl, 0.0));
      run_parties(2, [&](int p) {
        Communicator& comm = *comms[p];
        SeededDealer dealer(seed, p, 2);
        CounterRng mask(seed ^ 0x9e3779b97f4a7c15ull, static_cast<u64>(p));
        CounterRng vals(seed + 101 * static_cast<u64>(p) + 3 + 7919 * static_cast<u64>(pr), 9);
        ProtoCtx ctx{dealer, comm, mask, f};
        auto rnd = [&](const Shape& s) {  // small fixed-point share words (value range is irrelevant to cost)
          RingTensor t(s, f);
          for (auto& w : t.data()) w = vals() >> 20;
          return AdditiveShare{p, std::move(t)};
        };
        auto linear = [&](std::size_t m, std::size_t K, std::size_t N, const std::string& tag) {
          AdditiveShare x = rnd({m, K}), w = rnd({K, N});
          if (pub) {
            RingTensor z = sar_tensor(matmul(x.tensor, w.tensor), f);
            return z.numel();
          }
          AdditiveShare z = beaver_matmul(x, w, false, dealer, comm, tag);
          z = truncate_shares(z, f, comm, mask);
          return z.tensor.numel();
        };
        for (std::size_t li = 0; li < nl; ++li) {
          const OpLayer& L = layers[li];
          const Shape& s = L.in;
          double sc = 1.0;
          const auto a = std::chrono::steady_clock::now();
          if (L.kind == "conv2d") {
            const std::size_t OH = (s[2] + 2 * L.pad - L.kernel) / L.stride + 1, OW = (s[3] + 2 * L.pad - L.kernel) / L.stride + 1;
            const std::size_t M = s[0] * OH * OW, m = rows_of(M);
            sc = double(M) / double(m);
            linear(m, s[1] * L.kernel * L.kernel, L.out, L.name + ".mm");
          } else if (L.kind == "dense") {
            const std::size_t K = s.back(), M = shape_numel(s) / K, m = rows_of(M);
            sc = double(M) / double(m);
            linear(m, K, L.out, L.name + ".mm");
          } else if (L.kind == "relu") {
            const std::size_t n = shape_numel(s), m = rows_of(n);
            sc = double(n) / double(m);
            relu_shares(rnd({m}), ctx, L.name);
          } else if (L.kind == "maxpool2d") {
            const std::size_t OH = (s[2] - L.kernel) / L.stride + 1, OW = (s[3] - L.kernel) / L.stride + 1;
            const std::size_t w = s[0] * s[1] * OH * OW, m = rows_of(w);
            sc = double(w) / double(m);
            max_last_dim(rnd({m, L.kernel * L.kernel}), L.kernel * L.kernel, ctx, L.name);
          } else if (L.kind == "softmax") {
            const std::size_t Lr = s.back(), r = shape_numel(s) / Lr, m = rows_of(r);
            sc = double(r) / double(m);
            softmax_shares(rnd({m, Lr}), Lr, ctx, L.name);
          } else if (L.kind == "add") {
            const std::size_t n = shape_numel(s), m = rows_of(n);
            sc = double(n) / double(m);
            (void)add(rnd({m}).tensor, rnd({m}).tensor);
          } else if (L.kind == "global_avg_pool" || L.kind == "mean_pool") {
            const std::size_t rows = L.kind == "mean_pool" ? s[0] : s[0] * s[1];
            const std::size_t red = L.kind == "mean_pool" ? s[1] * s[2] : s[2] * s[3];
            const std::size_t m = rows_of(rows);
            sc = double(rows) / double(m);
            RingTensor z = sar_tensor(mul_scalar(sum_last_dim(rnd({m, red}).tensor), encode_fixed(0.5, f)), f);
          } else if (L.kind == "attention") {
            const std::size_t B = s[0], T = s[1], d = s[2], H = L.heads, dh = d / H;
            const std::size_t bh = rows_of(B * H), bt = rows_of(B * T);
            sc = double(B * H) / double(bh);
            const double sc_rows = double(B * T) / double(bt);
            // the projections scale by token rows, the head-batched part by (batch, head)
            const auto a1 = std::chrono::steady_clock::now();
            linear(bt, d, 3 * d, L.name + ".qkv");
            linear(bt, d, d, L.name + ".proj");
            const double proj_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a1).count();
            const auto a2 = std::chrono::steady_clock::now();
            AdditiveShare q = rnd({bh, T, dh}), k = rnd({bh, T, dh}), v = rnd({bh, T, dh});
            AdditiveShare sc1 = beaver_matmul(q, k, true, dealer, comm, L.name + ".qk");
            RingTensor sc2 = sar_tensor(mul_scalar(sar_tensor(sc1.tensor, f), encode_fixed(0.125, f)), f);
            AdditiveShare pr1 = softmax_shares(AdditiveShare{p, reshape(sc2, {bh * T, T})}, T, ctx, L.name + ".softmax");
            AdditiveShare mixed = beaver_matmul(AdditiveShare{p, reshape(pr1.tensor, {bh, T, T})}, v, false, dealer,
                                                comm, L.name + ".av");
            RingTensor merged = sar_tensor(mixed.tensor, f);
            const double head_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a2).count();
            ps[p][li] = proj_s * sc_rows + head_s * sc;
            continue;
          } else if (L.kind == "gelu") {  // x * sigmoid(1.702 x), built from reference blocks
            const std::size_t n = shape_numel(s), m = rows_of(n);
            sc = double(n) / double(m);
            AdditiveShare x = rnd({m});
            BinaryShare b = msb(x, dealer, comm, mask, ctx.adder, L.name + ".msb");
            AdditiveShare bit = b2a_bit(b, dealer, comm, L.name + ".b2a");
            AdditiveShare ax = beaver_mul(x, bit, dealer, comm, L.name + ".abs");
            AdditiveShare e = exp_shares(ax, ctx, L.name + ".exp");
            AdditiveShare r = reciprocal_shares(e, ctx, L.name + ".recip");
            AdditiveShare sg = beaver_mul(r, bit, dealer, comm, L.name + ".sel");
            beaver_mul(x, sg, dealer, comm, L.name + ".out");
          } else if (L.kind == "layernorm") {
            const std::size_t dd = s.back(), rows = shape_numel(s) / dd, m = rows_of(rows);
            sc = double(rows) / double(m);
            AdditiveShare x = rnd({m, dd});
            AdditiveShare sq = beaver_square(x, dealer, comm, L.name + ".sq");
            AdditiveShare v{p, sum_last_dim(sq.tensor)};
            AdditiveShare y = exp_shares(v, ctx, L.name + ".isqrt.exp");
            for (int it = 0; it < 3; ++it) {
              AdditiveShare yy = beaver_square(y, dealer, comm, L.name + ".isqrt.sq" + std::to_string(it));
              y = beaver_mul(yy, v, dealer, comm, L.name + ".isqrt.m" + std::to_string(it));
            }
            AdditiveShare yb{p, broadcast_last(y.tensor, dd)};
            AdditiveShare nrm = beaver_mul(x, yb, dealer, comm, L.name + ".norm");
            if (!pub) beaver_mul(nrm, x, dealer, comm, L.name + ".gamma");
          } else {  // flatten and other reshapes: free
            sc = 0.0;
          }
          ps[p][li] = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count() * sc;
          if (pr == 0 && p == 0) scale[li] = sc;
        }
      });
      for (std::size_t li = 0; li < nl; ++li) sec[std::size_t(pr)][li] = std::max(ps[0][li], ps[1][li]);
    });
  for (auto& t : th) t.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double est = 0;
  std::printf("{\"model\": \"%s\", \"weights\": \"%s\", \"div\": %zu, \"pairs\": %d, \"wall_s\": %.6f, \"layers\": [",
              j.value("name", std::string("model")).c_str(), weights, div, pairs, wall);
  for (std::size_t li = 0; li < nl; ++li) {
    double m = 0;
    for (int pr = 0; pr < pairs; ++pr) m += sec[std::size_t(pr)][li];
    m /= pairs;
    est += m;
    std::printf("%s{\"name\": \"%s\", \"kind\": \"%s\", \"est_s\": %.6f, \"scale\": %.3f}", li ? ", " : "",
                layers[li].name.c_str(), layers[li].kind.c_str(), m, scale[li]);
  }
  std::printf("], \"est_latency_s\": %.6f, \"batch\": %zu}\n", est, input[0]);
  return 0;
}

// Triple-file pin: the triples SeededDealer(5, *, 2) hands out for "t.mul" [3,4] and "t.qk"
// [2,3,4]x[2,5,4]^T (first fetch of each tag, H/sharing/triple.hpp:138-151), written with the
// reference's save_triples (:181-218) — the format the GPU queue loader must read.
int cmd_triples(const char* path) {
  auto stream_of = [](const std::string& tag) {
    u64 h = 0xcbf29ce484222325ull;
    for (char c : tag) h = (h ^ u64(static_cast<unsigned char>(c))) * 0x100000001b3ull;
    return CounterRng::mix(h + 0x51ed270b * 0);
  };
  std::vector<TripleSet> sets;
  {
    CounterRng rng(5, stream_of("t.mul"));
    sets.push_back(dealer_gen_triple(TripleSpec::elementwise(TripleKind::Arith, {3, 4}), 2, rng));
  }
  {
    CounterRng rng(5, stream_of("t.qk"));
    sets.push_back(dealer_gen_triple(TripleSpec::matmul_of({2, 3, 4}, {2, 5, 4}, true), 2, rng));
  }
  save_triples(path, sets);
  return 0;
}

// MPCW interchange check: the reference's own init_weights(model, seed) written by its
// save_weights (H/engine/model.hpp:257-275,277-313), and a file read back by its
// load_weights + check_weights (:315-376) and re-saved, so the package's MPCW reader/writer
// can be compared byte for byte.
int cmd_mpcw(const char* model_path, unsigned long long seed, const char* out_path, const char* in_path) {
  using namespace mpcpipe;
  const ModelGraph g = load_model(model_path);
  if (in_path) {
    WeightMap w = load_weights(in_path);
    check_weights(g, w);
    save_weights(w, out_path);
  } else {
    save_weights(init_weights(g, seed), out_path);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 3 && std::string(argv[1]) == "golden") return cmd_golden(argv[2]);
    if (argc >= 8 && std::string(argv[1]) == "model")
      return cmd_model_golden(argv[2], argv[3], std::atoi(argv[4]), argv[5],
                              std::strtoull(argv[6], nullptr, 10), argv[7]);
    if (argc >= 8 && std::string(argv[1]) == "model_pin")
      return cmd_model_golden(argv[2], argv[3], std::atoi(argv[4]), argv[5],
                              std::strtoull(argv[6], nullptr, 10), argv[7], true);
    if (argc >= 4 && std::string(argv[1]) == "scale") return cmd_scale(argv[2], argv[3]);
    if (argc >= 3 && std::string(argv[1]) == "triples") return cmd_triples(argv[2]);
    if (argc >= 7 && std::string(argv[1]) == "opsum")
      return cmd_opsum(argv[2], argv[3], std::strtoull(argv[4], nullptr, 10), std::atoi(argv[5]),
                       std::strtoull(argv[6], nullptr, 10));
    if (argc >= 7 && std::string(argv[1]) == "bench") return cmd_bench(argc, argv);
    if (argc >= 5 && std::string(argv[1]) == "mpcw")
      return cmd_mpcw(argv[2], std::strtoull(argv[3], nullptr, 10), argv[4], argc >= 6 ? argv[5] : nullptr);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_driver: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr,
               "usage: ref_driver golden <out.bin>\n"
               "       ref_driver model <model.json> <mode> <iters> <private|public> <seed> <out.bin>\n"
               "       ref_driver model_pin <model.json> <mode> <iters> <private|public> <seed> <out.bin>\n"
               "       ref_driver scale <case|all> <out.bin>\n"
               "       ref_driver triples <out.bin>\n"
               "       ref_driver opsum <model.json> <private|public> <div> <pairs> <seed>\n"
               "       ref_driver bench <model.json> <mode> <iters> <private|public> <seed> [chunks thr]\n"
               "       ref_driver mpcw <model.json> <seed> <out.mpcw> [<in.mpcw>]\n");
  return 2;
}
