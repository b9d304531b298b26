// extern "C" boundary of libmpcg.so (declared in include/mpcg.h).
#include <cstring>
#include <memory>

#include "../../include/mpcg.h"
#include "core.hpp"
#include "gemm.cuh"
#include "executor.hpp"

using namespace mpcg;

namespace mpcg {
void nccl_unique_id(void* out128);
void nccl_connect(Session& s, const void* id128, int rank);
int& tc_gemm_mode();
}  // namespace mpcg

// Handles share ownership of the session so device memory is always released on a
// live stream, whatever order the host language destroys handles in.
struct mpcg_session {
  std::shared_ptr<Session> s;
};
struct mpcg_tensor {
  std::shared_ptr<Session> s;
  DT t;
};
struct mpcg_model {
  ModelGraph g;
};
struct mpcg_executor {
  std::shared_ptr<Session> s;
  std::unique_ptr<SecureExecutor> e;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MPCG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MPCG_ERR_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return MPCG_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw Error(kUsageError, std::string("null ") + what);
}

mpcg_tensor* wrap(const std::shared_ptr<Session>& s, DT t) { return new mpcg_tensor{s, std::move(t)}; }
const DT& T(const mpcg_tensor* t) {
  need(t, "tensor");
  return t->t;
}
Session& S(mpcg_session* s) {
  need(s, "session");
  return *s->s;
}
const std::shared_ptr<Session>& SP(mpcg_session* s) {
  need(s, "session");
  return s->s;
}
std::string tagstr(const char* t) { return t ? std::string(t) : std::string(); }
}  // namespace

extern "C" {
#pragma GCC visibility push(default)

const char* mpcg_last_error(void) { return g_err.c_str(); }
int mpcg_version(void) { return 1; }

int mpcg_device_count(int* out) {
  return guard([&] {
    need(out, "out");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    cudaGetLastError();
    *out = n;
  });
}

int mpcg_session_create(int device, int n_local, int party, uint64_t seed, uint64_t mask_seed, int frac_bits,
                        mpcg_session** out) {
  return guard([&] {
    need(out, "out");
    auto* h = new mpcg_session;
    try {
      h->s = std::make_shared<Session>(device, n_local, party, seed, mask_seed, frac_bits);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int mpcg_session_destroy(mpcg_session* s) {
  return guard([&] { delete s; });
}

int mpcg_session_set_pipeline(mpcg_session* s, int chunks, uint64_t threshold, int merged) {
  return guard([&] {
    Session& ss = S(s);
    ss.cfg.chunks = chunks;
    ss.cfg.chunk_threshold = threshold;
    ss.cfg.merged_adder = merged != 0;
  });
}

int mpcg_session_set_link(mpcg_session* s, double latency_s, double bw, double msg) {
  return guard([&] {
    Session& ss = S(s);
    // transport/config.hpp:34-38: latency >= 0, bandwidth > 0. (0, 0, 0) removes the emulated
    // link (the real in-device / NVLink transport); a latency-only link is rejected like the
    // reference rejects bandwidth <= 0, instead of silently running as an ideal link.
    if (latency_s < 0) throw Error(kConfigError, "latency must be >= 0");
    if (msg < 0) throw Error(kConfigError, "sec_per_message must be >= 0");
    const bool off = latency_s == 0 && bw == 0 && msg == 0;
    if (!off && !(bw > 0)) throw Error(kConfigError, "bandwidth must be > 0");
    ss.cfg.link_latency_s = latency_s;
    ss.cfg.link_bandwidth = off ? 0 : bw;
    ss.cfg.sec_per_message = msg;
  });
}

int mpcg_session_set_shard(mpcg_session* s, uint64_t local_batch, uint64_t global_batch, uint64_t off) {
  return guard([&] {
    Session& ss = S(s);
    if (local_batch == 0 || global_batch < local_batch || off + local_batch > global_batch)
      throw Error(kConfigError, "bad shard");
    ss.shard_local = local_batch;
    ss.shard_global = global_batch;
    ss.shard_offset = off;
  });
}

int mpcg_nccl_unique_id(uint8_t out[128]) {
  return guard([&] { nccl_unique_id(out); });
}

// ---- triple queues (TripleSource / QueueTripleSource, H/sharing/triple.hpp:126-307)
struct mpcg_triple_queue {
  std::shared_ptr<TripleQueue> q;
};

int mpcg_triple_queue_create(mpcg_triple_queue** out) {
  return guard([&] {
    need(out, "out");
    *out = new mpcg_triple_queue{std::make_shared<TripleQueue>()};
  });
}

int mpcg_triple_queue_destroy(mpcg_triple_queue* q) {
  delete q;
  return 0;
}

int mpcg_triple_queue_size(mpcg_triple_queue* q, uint64_t* records, uint64_t* consumed) {
  return guard([&] {
    need(q, "queue");
    if (records) *records = q->q->items.size();
    if (consumed) *consumed = q->q->next;
  });
}

int mpcg_triple_queue_rewind(mpcg_triple_queue* q) {
  return guard([&] {
    need(q, "queue");
    q->q->next = 0;
  });
}

int mpcg_triple_queue_save(mpcg_triple_queue* q, const char* path) {
  return guard([&] {
    need(q, "queue");
    need(path, "path");
    queue_save(*q->q, path);
  });
}

int mpcg_triple_queue_load(mpcg_triple_queue* q, const char* path) {
  return guard([&] {
    need(q, "queue");
    need(path, "path");
    queue_load(*q->q, path);
  });
}

int mpcg_session_record_triples(mpcg_session* s, mpcg_triple_queue* q) {
  return guard([&] {
    Session& ss = S(s);
    if (q && ss.source_q) throw Error(kUsageError, "record and consume modes are exclusive");
    ss.record_q = q ? q->q : nullptr;
  });
}

int mpcg_session_use_triple_queue(mpcg_session* s, mpcg_triple_queue* q) {
  return guard([&] {
    Session& ss = S(s);
    if (q && ss.record_q) throw Error(kUsageError, "record and consume modes are exclusive");
    ss.source_q = q ? q->q : nullptr;
  });
}

int mpcg_dealer_fetch(mpcg_session* s, int kind, int matmul, int square, int transpose_b, int nda,
                      const uint64_t* dims_a, int ndb, const uint64_t* dims_b, const char* tag, mpcg_tensor** a,
                      mpcg_tensor** b, mpcg_tensor** c) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(c, "c");
    if (nda < 1 || ndb < 1 || nda > 8 || ndb > 8) throw Error(kShapeError, "dealer_fetch: bad rank");
    TripleSpec sp;
    sp.kind = kind ? TripleKind::Bin : TripleKind::Arith;
    sp.matmul = matmul != 0;
    sp.square = square != 0;
    sp.transpose_b = transpose_b != 0;
    sp.shape_a.assign(dims_a, dims_a + nda);
    sp.shape_b.assign(dims_b, dims_b + ndb);
    if (sp.matmul && (sp.square || sp.kind == TripleKind::Bin))
      throw Error(kConfigError, "dealer_fetch: matmul triples are arithmetic and not square");
    if (!sp.matmul && sp.shape_a != sp.shape_b) throw Error(kConfigError, "dealer_gen_triple: elementwise shapes differ");
    DT x, y, z;
    dealer_fetch(S(s), sp, tag ? tag : "", x, y, z);
    *a = wrap(SP(s), x);
    *b = wrap(SP(s), y);
    *c = wrap(SP(s), z);
  });
}

int mpcg_session_connect_p2p(mpcg_session* a, mpcg_session* b) {
  return guard([&] { p2p_connect(S(a), S(b)); });
}

int mpcg_session_connect_socket(mpcg_session* s, const char* host, int port, double timeout_s) {
  return guard([&] {
    need(host, "host");
    if (port <= 0 || port > 65535) throw Error(kConfigError, "bad port");
    socket_connect(S(s), host, port, timeout_s > 0 ? timeout_s : 60.0);
  });
}

int mpcg_session_connect_nccl(mpcg_session* s, const uint8_t id[128], int rank) {
  return guard([&] { nccl_connect(S(s), id, rank); });
}

int mpcg_session_set_persistent(mpcg_session* s, int enable) {
  return guard([&] { S(s).persistent_mode = enable; });
}

int mpcg_session_sync(mpcg_session* s) {
  return guard([&] { S(s).sync(); });
}

int mpcg_session_stats(mpcg_session* s, int slot, uint64_t out[3]) {
  return guard([&] {
    Session& ss = S(s);
    if (slot < 0 || slot >= ss.n_local) throw Error(kUsageError, "bad slot");
    out[0] = ss.stats[slot].bytes_sent;
    out[1] = ss.stats[slot].collectives;
    out[2] = ss.stats[slot].p2p_sends;
  });
}

int mpcg_session_n_local(mpcg_session* s, int* out) {
  return guard([&] { *out = S(s).n_local; });
}

int mpcg_session_trace(mpcg_session* s, int enable) {
  return guard([&] { S(s).set_trace(enable != 0); });
}

int mpcg_session_trace_count(mpcg_session* s, uint64_t* n) {
  return guard([&] {
    need(n, "n");
    *n = S(s).trace_rows().size();
  });
}

int mpcg_session_trace_get(mpcg_session* s, uint64_t i, uint32_t* seq, int* kind, uint64_t* bytes, double t[4],
                           char* tag, int tag_cap) {
  return guard([&] {
    const auto& rows = S(s).trace_rows();
    if (i >= rows.size()) throw Error(kRangeError, "trace row out of range");
    const TraceEvent& r = rows[size_t(i)];
    if (seq) *seq = r.seq;
    if (kind) *kind = int(r.kind);
    if (bytes) *bytes = r.bytes;
    if (t) {
      t[0] = r.t_issue;
      t[1] = r.t_sent;
      t[2] = r.t_wait_begin;
      t[3] = r.t_wait_end;
    }
    if (tag && tag_cap > 0) {
      const size_t n = std::min(r.tag.size(), size_t(tag_cap - 1));
      std::memcpy(tag, r.tag.data(), n);
      tag[n] = 0;
    }
  });
}

int mpcg_session_clear_trace(mpcg_session* s) {
  return guard([&] { S(s).clear_trace(); });
}

int mpcg_session_now(mpcg_session* s, double* out) {
  return guard([&] {
    need(out, "out");
    *out = S(s).now();
  });
}

int mpcg_session_add_delay(mpcg_session* s, double seconds) {
  return guard([&] { S(s).add_delay(seconds); });
}

int mpcg_tensor_create(mpcg_session* s, int ndim, const uint64_t* dims, int scale, const uint64_t* host,
                       mpcg_tensor** out) {
  return guard([&] {
    Session& ss = S(s);
    need(out, "out");
    if (ndim < 0 || ndim > 8) throw Error(kShapeError, "rank must be in [0, 8]");
    Shape sh(dims, dims + ndim);
    DT t = host ? ss.upload(sh, scale, host) : ss.alloc(sh, scale);
    if (!host && t.numel())
      MPCG_CUDA(cudaMemsetAsync(t.mem->ptr, 0, t.numel() * ss.n_local * 8, ss.stream));
    *out = wrap(SP(s), std::move(t));
  });
}

int mpcg_tensor_download(mpcg_tensor* t, uint64_t* host) {
  return guard([&] {
    need(t, "tensor");
    t->s->download(t->t, host);
  });
}

int mpcg_tensor_shape(const mpcg_tensor* t, int* ndim, uint64_t dims[8], int* scale) {
  return guard([&] {
    const DT& d = T(t);
    *ndim = int(d.shape.size());
    for (size_t i = 0; i < d.shape.size() && i < 8; ++i) dims[i] = d.shape[i];
    if (scale) *scale = d.scale;
  });
}

int mpcg_tensor_destroy(mpcg_tensor* t) {
  return guard([&] { delete t; });
}

int mpcg_deal_input(mpcg_session* s, const double* x, int ndim, const uint64_t* gdims, uint64_t off,
                    uint64_t local, uint64_t seed, mpcg_tensor** out) {
  return guard([&] {
    Session& ss = S(s);
    need(x, "input");
    if (ndim < 1) throw Error(kShapeError, "input needs a batch dim");
    Shape g(gdims, gdims + ndim);
    if (off + local > g[0] || local == 0) throw Error(kConfigError, "bad input slice");
    const size_t per = shape_numel(g) / g[0];
    const size_t n = per * local, base = per * off;
    const int f = ss.cfg.frac_bits;
    const u64 key = seed ^ (u64(0x11a9) * kPhi);
    std::vector<u64> host(n * ss.n_local);
    for (size_t i = 0; i < n; ++i) {
      const u64 r = drw(key, 1 + base + i);
      const u64 enc = encode_fixed(x[base + i], f);
      for (int sl = 0; sl < ss.n_local; ++sl) host[sl * n + i] = ss.party_of[sl] == 0 ? enc - r : r;
    }
    Shape ls = g;
    ls[0] = local;
    *out = wrap(SP(s), ss.upload(ls, f, host.data()));
  });
}

#define OP1(expr)                           \
  return guard([&] {                        \
    Session& ss = S(s);                     \
    need(out, "out");                       \
    *out = wrap(SP(s), (expr));                \
  })

int mpcg_open(mpcg_session* s, const mpcg_tensor* x, int reduce, const char* tag, mpcg_tensor** out) {
  OP1(open_value(ss, T(x), reduce == MPCG_REDUCE_XOR ? Reduce::Xor : Reduce::Sum, tagstr(tag)));
}
int mpcg_beaver_mul(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, const char* tag, int chunks,
                    mpcg_tensor** out) {
  OP1(beaver_mul(ss, T(x), T(y), tagstr(tag), chunks));
}
int mpcg_beaver_square(mpcg_session* s, const mpcg_tensor* x, const char* tag, int chunks, mpcg_tensor** out) {
  OP1(beaver_square(ss, T(x), tagstr(tag), chunks));
}
int mpcg_beaver_and(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, const char* tag, int chunks,
                    mpcg_tensor** out) {
  OP1(beaver_and(ss, T(x), T(y), tagstr(tag), chunks));
}
int mpcg_beaver_matmul(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, int tb, const char* tag,
                       int chunks, mpcg_tensor** out) {
  OP1(beaver_matmul(ss, T(x), T(y), tb != 0, tagstr(tag), chunks));
}
int mpcg_binary_add(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, int width, int merged, int chunks,
                    const char* tag, mpcg_tensor** out) {
  AdderOptions o;
  o.width = width;
  o.merged = merged != 0;
  o.chunks = chunks;
  OP1(binary_add(ss, T(x), T(y), o, tagstr(tag)));
}
int mpcg_a2b(mpcg_session* s, const mpcg_tensor* x, int chunks, const char* tag, mpcg_tensor** out) {
  AdderOptions o;
  o.chunks = chunks;
  OP1(a2b(ss, T(x), o, tagstr(tag)));
}
int mpcg_msb(mpcg_session* s, const mpcg_tensor* x, int chunks, const char* tag, mpcg_tensor** out) {
  AdderOptions o;
  o.chunks = chunks;
  OP1(msb(ss, T(x), o, tagstr(tag)));
}
int mpcg_b2a_bit(mpcg_session* s, const mpcg_tensor* b, const char* tag, int chunks, mpcg_tensor** out) {
  OP1(b2a_bit(ss, T(b), tagstr(tag), chunks));
}
int mpcg_less_than(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, int chunks, const char* tag,
                   mpcg_tensor** out) {
  AdderOptions o;
  o.chunks = chunks;
  OP1(less_than(ss, T(x), T(y), o, tagstr(tag)));
}
int mpcg_truncate(mpcg_session* s, const mpcg_tensor* x, int bits, mpcg_tensor** out) {
  OP1(truncate_shares(ss, T(x), bits));
}
int mpcg_relu(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out) {
  OP1(relu_shares(ss, T(x), tagstr(tag)));
}
int mpcg_max_last_dim(mpcg_session* s, const mpcg_tensor* x, uint64_t L, const char* tag, mpcg_tensor** out) {
  OP1(max_last_dim(ss, T(x), L, tagstr(tag)));
}
int mpcg_exp(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out) {
  OP1(exp_shares(ss, T(x), tagstr(tag)));
}
int mpcg_reciprocal(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out) {
  OP1(reciprocal_shares(ss, T(x), tagstr(tag)));
}
int mpcg_softmax(mpcg_session* s, const mpcg_tensor* x, uint64_t L, const char* tag, mpcg_tensor** out) {
  OP1(softmax_shares(ss, T(x), L, tagstr(tag)));
}
int mpcg_maxpool2d(mpcg_session* s, const mpcg_tensor* x, uint64_t N, uint64_t C, uint64_t H, uint64_t W,
                   uint64_t k, uint64_t stride, const char* tag, mpcg_tensor** out) {
  OP1(maxpool2d_shares(ss, T(x), N, C, H, W, k, stride, tagstr(tag)));
}

int mpcg_sigmoid(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out) {
  OP1(sigmoid_shares(ss, T(x), tagstr(tag)));
}
int mpcg_gelu(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out) {
  OP1(gelu_shares(ss, T(x), tagstr(tag)));
}
int mpcg_inv_sqrt(mpcg_session* s, const mpcg_tensor* v, const char* tag, int newton_iters, mpcg_tensor** out) {
  OP1(inv_sqrt_shares(ss, T(v), tagstr(tag), newton_iters));
}
int mpcg_layernorm(mpcg_session* s, const mpcg_tensor* x, uint64_t d, const mpcg_tensor* gamma,
                   const mpcg_tensor* beta, int public_weights, const char* tag, mpcg_tensor** out) {
  OP1(layernorm_shares(ss, T(x), d, T(gamma), T(beta), public_weights != 0, tagstr(tag)));
}
int mpcg_global_avg_pool(mpcg_session* s, const mpcg_tensor* x, uint64_t N, uint64_t C, uint64_t HW,
                         mpcg_tensor** out) {
  OP1(global_avg_pool(ss, T(x), N, C, HW));
}

int mpcg_model_create(const char* name, int frac_bits, int ndim, const uint64_t* dims, mpcg_model** out) {
  return guard([&] {
    need(out, "out");
    if (frac_bits < 1 || frac_bits > 40) throw Error(kConfigError, "frac_bits out of range");
    auto* m = new mpcg_model;
    m->g.name = tagstr(name);
    m->g.frac_bits = frac_bits;
    m->g.input.assign(dims, dims + ndim);
    *out = m;
  });
}

int mpcg_model_add_layer_ex(mpcg_model* m, const char* name, int kind, uint64_t outc, uint64_t kernel,
                            uint64_t stride, uint64_t pad, uint64_t heads, int bias, const char* from,
                            const char* with_) {
  return guard([&] {
    need(m, "model");
    if (kind < 0 || kind > MPCG_LAYER_LAYERNORM) throw Error(kConfigError, "unknown layer kind");
    LayerSpec l;
    l.name = tagstr(name);
    l.kind = static_cast<LayerKind>(kind);
    l.out = outc;
    l.kernel = kernel;
    l.stride = stride;
    l.pad = pad;
    l.heads = heads;
    l.bias = bias != 0;
    l.from = from ? from : "";
    l.with = with_ ? with_ : "";
    m->g.layers.push_back(l);
    try {
      infer_shapes(m->g);  // validate (H/engine/model.hpp:177)
    } catch (...) {
      m->g.layers.pop_back();
      throw;
    }
  });
}

int mpcg_model_add_layer(mpcg_model* m, const char* name, int kind, uint64_t outc, uint64_t kernel, uint64_t stride,
                         uint64_t pad, uint64_t heads, int bias) {
  return mpcg_model_add_layer_ex(m, name, kind, outc, kernel, stride, pad, heads, bias, nullptr, nullptr);
}

int mpcg_model_destroy(mpcg_model* m) {
  return guard([&] { delete m; });
}

int mpcg_executor_create(mpcg_session* s, const mpcg_model* m, int pub, int pipelined, int chunks, uint64_t thr,
                         int merged, mpcg_executor** out) {
  return guard([&] {
    Session& ss = S(s);
    need(m, "model");
    need(out, "out");
    ExecOptions o;
    o.pipelined = pipelined != 0;
    o.chunks = chunks;
    o.chunk_threshold = thr;
    o.merged_adder = merged != 0;
    auto* e = new mpcg_executor;
    e->s = SP(s);
    try {
      e->e = std::make_unique<SecureExecutor>(ss, m->g, pub != 0, o);
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
}

int mpcg_executor_deal_weights(mpcg_executor* e, int count, const char* const* names, const double* const* values,
                               const uint64_t* counts, uint64_t seed) {
  return guard([&] {
    need(e, "executor");
    if (count < 0) throw Error(kConfigError, "negative weight count");
    if (count > 0 && (!names || !values || !counts)) throw Error(kUsageError, "null weight arrays");
    std::vector<std::string> n;
    std::vector<const double*> v;
    std::vector<size_t> k;
    for (int i = 0; i < count; ++i) {
      if (!names[i]) throw Error(kUsageError, "null weight name");
      n.emplace_back(names[i]);
      v.push_back(values[i]);
      k.push_back(size_t(counts[i]));
    }
    e->e->deal_weights(n, v, k, seed);
  });
}

int mpcg_executor_set_linear_chunks(mpcg_executor* e, int on) {
  return guard([&] {
    need(e, "executor");
    if (e->e->captured_) throw Error(kUsageError, "set_linear_chunks after capture");
    e->e->opt_.linear_chunks = on != 0;
  });
}

int mpcg_executor_release_graph(mpcg_executor* e) {
  return guard([&] {
    need(e, "executor");
    e->e->release_graph();
  });
}

int mpcg_executor_run(mpcg_executor* e, const mpcg_tensor* input, mpcg_tensor** out) {
  return guard([&] {
    need(e, "executor");
    need(out, "out");
    *out = wrap(e->s, e->e->run(T(input)));
  });
}

int mpcg_executor_capture(mpcg_executor* e, const mpcg_tensor* input) {
  return guard([&] {
    need(e, "executor");
    e->e->capture(T(input));
  });
}

int mpcg_executor_replay(mpcg_executor* e, mpcg_tensor** out) {
  return guard([&] {
    need(e, "executor");
    DT r = e->e->replay();
    if (out) *out = wrap(e->s, r);
  });
}

int mpcg_executor_time_layers(mpcg_executor* e, int enable) {
  return guard([&] {
    need(e, "executor");
    e->e->time_layers = enable != 0;
  });
}

int mpcg_executor_layer_times(mpcg_executor* e, int max, float* ms, int* count) {
  return guard([&] {
    need(e, "executor");
    if (e->e->captured_ && e->e->time_layers) e->e->collect_timings();  // events of the last replay
    const auto& t = e->e->timings;
    const int n = int(t.size()) < max ? int(t.size()) : max;
    for (int i = 0; i < n; ++i) ms[i] = t[i].ms;
    *count = int(t.size());
  });
}

int mpcg_executor_destroy(mpcg_executor* e) {
  return guard([&] { delete e; });
}

int mpcg_session_connect_loopback(mpcg_session* a, mpcg_session* b) {
  return guard([&] {
    Session& x = S(a);
    Session& y = S(b);
    if (x.n_local != 1 || y.n_local != 1) throw Error(kUsageError, "loopback link needs two single-party sessions");
    if (x.party_of[0] == y.party_of[0]) throw Error(kUsageError, "loopback link needs party 0 and party 1");
    if (x.device != y.device) throw Error(kUsageError, "loopback link: sessions on different devices (use NCCL)");
    auto link = std::make_shared<LoopLink>();
    x.loop = link;
    y.loop = link;
  });
}

int mpcg_debug_tc3_trace(uint64_t* out, int n) {
  return guard([&] { tc3_trace_read(reinterpret_cast<unsigned long long*>(out), n); });
}

namespace {
__global__ void draw_peak_kernel(u64 key, u64* out, int iters) {
  u64 acc = 0;
  const u64 z = key + u64(blockIdx.x * blockDim.x + threadIdx.x) * kPhi * 16;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc ^= mix64(z + u64(i + it * 16) * kPhi);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
}  // namespace

int mpcg_debug_draw_peak(int device, double* draws_per_s) {
  return guard([&] {
    MPCG_CUDA(cudaSetDevice(device));
    const int blocks = num_sms() * 8, threads = 256, iters = 256;
    u64* d = nullptr;
    MPCG_CUDA(cudaMalloc(&d, size_t(blocks) * threads * 8));
    cudaEvent_t a, b;
    MPCG_CUDA(cudaEventCreate(&a));
    MPCG_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      MPCG_CUDA(cudaEventRecord(a));
      draw_peak_kernel<<<blocks, threads>>>(0x1234567ull + rep, d, iters);
      MPCG_CUDA(cudaEventRecord(b));
      MPCG_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      MPCG_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    *draws_per_s = double(blocks) * threads * iters * 16 / (double(best) * 1e-3);
  });
}

int mpcg_debug_tc2_trace(uint64_t* out, int n) {
  return guard([&] { tc2_trace_read(reinterpret_cast<unsigned long long*>(out), n); });
}

int mpcg_set_pair_eval(int on) {
  return guard([&] {
    pair_eval_enabled() = on != 0;
    eps_fuse_enabled() = on != 0;
  });
}

int mpcg_set_gemv(int on) {
  return guard([&] { gemv_mode() = on ? 1 : 0; });
}

int mpcg_set_gemm_mode(int mode) {
  return guard([&] {
    if (mode < 0 || mode > 3) throw Error(kConfigError, "gemm mode must be 0, 1, 2 or 3");
    tc_gemm_mode() = mode == 3 ? 1 : mode;
    tc3_mode() = mode == 3 ? 0 : tc3_default();
  });
}

uint64_t mpcg_launch_count(void) { return g_launches.load(); }

int mpcg_probe_start(int cls) {
  return guard([&] {
    for (auto& [a, b] : g_probe.ev) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    g_probe = Probe{};
    g_probe.cls = cls;
  });
}

int mpcg_probe_stop(double* total_ms, uint64_t* launches, double* units) {
  return guard([&] {
    double ms = 0;
    for (auto& [a, b] : g_probe.ev) {
      MPCG_CUDA(cudaEventSynchronize(b));
      float t = 0;
      MPCG_CUDA(cudaEventElapsedTime(&t, a, b));
      ms += t;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    *total_ms = ms;
    *launches = g_probe.launches;
    *units = g_probe.bytes;
    g_probe = Probe{};
  });
}

int mpcg_pinned_alloc(uint64_t bytes, void** out) {
  return guard([&] { MPCG_CUDA(cudaHostAlloc(out, bytes ? bytes : 8, cudaHostAllocDefault)); });
}

int mpcg_pinned_free(void* p) {
  return guard([&] { MPCG_CUDA(cudaFreeHost(p)); });
}

int mpcg_tensor_copy_from_host(mpcg_tensor* t, const uint64_t* host) {
  return guard([&] {
    need(t, "tensor");
    const size_t n = t->t.numel() * t->s->n_local;
    if (n) MPCG_CUDA(cudaMemcpyAsync(t->t.mem->ptr, host, n * 8, cudaMemcpyHostToDevice, t->s->stream));
  });
}

int mpcg_session_flush_l2(mpcg_session* s) {
  return guard([&] {
    Session& ss = S(s);
    if (!ss.flush_buf) MPCG_CUDA(cudaMalloc(&ss.flush_buf, kFlushBytes));
    MPCG_CUDA(cudaMemsetAsync(ss.flush_buf, ss.flush_val++ & 0xff, kFlushBytes, ss.stream));
  });
}

int mpcg_session_timer(mpcg_session* s, int op, double* total_ms) {
  return guard([&] {
    Session& ss = S(s);
    if (op == 2) {
      for (auto& [a, b] : ss.timer_ev) {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
      ss.timer_ev.clear();
    } else if (op == 0) {
      cudaEvent_t a;
      MPCG_CUDA(cudaEventCreate(&a));
      MPCG_CUDA(cudaEventRecord(a, ss.stream));
      ss.timer_ev.push_back({a, nullptr});
    } else if (op == 1) {
      if (ss.timer_ev.empty() || ss.timer_ev.back().second) throw Error(kUsageError, "timer stop without start");
      cudaEvent_t b;
      MPCG_CUDA(cudaEventCreate(&b));
      MPCG_CUDA(cudaEventRecord(b, ss.stream));
      ss.timer_ev.back().second = b;
    }
    if (total_ms) {
      double ms = 0;
      for (auto& [a, b] : ss.timer_ev) {
        if (!b) continue;
        MPCG_CUDA(cudaEventSynchronize(b));
        float t = 0;
        MPCG_CUDA(cudaEventElapsedTime(&t, a, b));
        ms += t;
      }
      *total_ms = ms;
    }
  });
}

uint64_t mpcg_fnv1a_words(const uint64_t* w, uint64_t n) {
  u64 h = 0xcbf29ce484222325ull;
  for (u64 i = 0; i < n; ++i)
    for (int b = 0; b < 8; ++b) h = (h ^ ((w[i] >> (8 * b)) & 0xff)) * 0x100000001b3ull;
  return h;
}

#pragma GCC visibility pop
}  // extern "C"
