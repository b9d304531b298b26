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
//   ref_driver bench <model.json> <blocking|pipelined> <iters> <private|public> <seed>
//                    [<chunks> <threshold_bytes>]
//       Times bench_party (H/engine/bench.hpp:36-79) with the two parties as threads
//       over SocketComm on loopback (real wall clock, 1 thread per party) and prints
//       one JSON line: per-iteration wall seconds, bytes, collectives, logits hash.
//
// H/ = /root/reference/proj/include/mpcpipe.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
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

// Model-level golden: per-party logits shares after `iters` runs plus the hash.
int cmd_model_golden(const char* model_path, const char* mode, int iters, const char* weights,
                     u64 seed, const char* out_path) {
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
  put("z0", outs[0]);
  put("z1", outs[1]);
  put("logits", res[0].logits);
  std::vector<u64> meta{fnv1a_words(res[0].logits.data()), res[0].report.bytes_sent,
                        res[0].report.collectives, res[0].report.p2p_sends};
  put("meta", Shape{4}, meta);
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
               "       ref_driver bench <model.json> <mode> <iters> <private|public> <seed> [chunks thr]\n"
               "       ref_driver mpcw <model.json> <seed> <out.mpcw> [<in.mpcw>]\n");
  return 2;
}
