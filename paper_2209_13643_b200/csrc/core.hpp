// Host-side runtime of the B200 2PC engine: sessions, device share tensors, the
// dealer's tag streams and the open/reveal wire.
//
// A Session holds the party slots that live in this process on one GPU:
//   * n_local == 2 — both parties of a 2PC pair on one device (1-GPU mode). Every
//     kernel runs both parties' slots in one launch (blockIdx.y = slot); a slot only
//     touches its own party's state plus the peer payload it opened. An open is then a
//     stream-ordered kernel boundary and the peer reads the poster's outbox in place.
//   * n_local == 1 — one party per process/GPU (2/4/8-GPU runs); the peer's payload
//     crosses NVLink with NCCL send/recv on a dedicated comm stream.
// All protocol code is SPMD over the local slots (H/transport/harness.hpp:23-38 runs
// one thread per party instead; the values and the collective order are identical).
#pragma once

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

typedef struct ncclComm* ncclComm_t;

namespace mpcg {

using Shape = std::vector<size_t>;

inline size_t shape_numel(const Shape& s) {
  size_t n = 1;
  for (auto d : s) n *= d;
  return n;
}
std::string shape_str(const Shape& s);

// round(x * 2^scale), ties toward +inf, in long double (H/ring/fixed.hpp:16-22).
u64 encode_fixed(double x, int scale_bits);

// ------------------------------------------------------------------ device memory
// Eager mode: stream-ordered pool allocation (cudaMallocAsync/cudaFreeAsync), safe after
// every queued reader. Graph capture: a bump arena with fixed addresses and no reuse, so
// one captured inference replays with every buffer at the same place (the arena is laid
// out once; 180 GB of HBM3e leaves room for whole-inference arenas).
struct Block {
  u64* ptr = nullptr;
  size_t words = 0;
  cudaStream_t stream = nullptr;
  bool owned = true;
  bool sync_free = false;  // cudaMalloc'd persistent buffer (outlives graph arenas)
  Block(size_t words, cudaStream_t s);
  Block(u64* arena_ptr, size_t words) : ptr(arena_ptr), words(words), owned(false) {}
  static std::shared_ptr<Block> persistent(size_t words);
  ~Block();
  Block(const Block&) = delete;
  Block& operator=(const Block&) = delete;
};

// One share per local party slot: slot i at base + i*numel (row-major u64).
struct DT {
  std::shared_ptr<Block> mem;
  u64* s[2] = {nullptr, nullptr};
  Shape shape;
  int scale = 0;
  size_t numel() const { return shape_numel(shape); }
  explicit operator bool() const { return mem != nullptr; }
};

enum class Reduce : int { Sum = 0, Xor = 1 };

// One row per collective a party issued (H/transport/transport.hpp:25-37), with device
// timestamps in seconds since the trace was enabled:
//   t_issue      the compute stream reached the post (payload built, send issued)
//   t_sent       sender occupancy charged: the emulated link's busy time (msg + bytes/bw, the
//                sim model of H/transport/sim.hpp:90-92) or the NCCL / loopback transfer done
//   t_wait_begin the compute stream reached wait() (all work before it done)
//   t_wait_end   the stream resumed (the payload had arrived); == t_wait_begin when it was there
// In-device zero-copy opens have no transfer: occupancy and stall are 0. Opens inside a CUDA
// graph capture and in-kernel (persistent chain) opens carry no timestamps (all 0).
struct TraceEvent {
  u32 seq;
  Reduce kind;
  std::string tag;
  u64 bytes;
  double t_issue = 0, t_sent = 0, t_wait_begin = 0, t_wait_end = 0;
  double occupancy() const { return t_sent - t_issue; }
  double stall() const { return t_wait_end - t_wait_begin; }
};
struct CommStats {
  u64 bytes_sent = 0;
  u64 collectives = 0;
  u64 p2p_sends = 0;
};

// ------------------------------------------------------------------ dealer specs
enum class TripleKind : int { Arith = 0, Bin = 1 };
struct TripleSpec {
  TripleKind kind = TripleKind::Arith;
  bool matmul = false;
  bool square = false;
  bool transpose_b = false;
  Shape shape_a, shape_b;
  static TripleSpec elementwise(TripleKind k, Shape s) { return {k, false, false, false, s, s}; }
  static TripleSpec square_of(Shape s) { return {TripleKind::Arith, false, true, false, s, s}; }
  static TripleSpec matmul_of(Shape a, Shape b, bool tb = false) {
    return {TripleKind::Arith, true, false, tb, std::move(a), std::move(b)};
  }
};

// A fetched triple: nothing is materialised; kernels regenerate elements from the key.
struct Triple {
  TripleSpec spec;
  u64 key = 0;
  u64 tag_hash = 0, count = 0;  // FNV-1a of the tag and the fetch count that keyed it
  bool consumed = false;
  EwTriple ew{};  // elementwise view (global numel / shard offsets filled)
  MmTriple mm{};  // matmul view
  void mark_consumed() {
    if (consumed) throw Error(kProtocolError, "beaver triple reused after consumption");
    consumed = true;
  }
};

// ------------------------------------------------------------------ triple queues (pool.cu)
// One materialised triple: the seeded dealer's draw sequence [A | B | r_A | r_B | r_C] (2PC).
struct PoolTriple {
  TripleSpec spec;
  std::shared_ptr<Block> draws;
  u64 words = 0;
};
// QueueTripleSource (H/sharing/triple.hpp:161-179): consumed in order, specs checked.
struct TripleQueue {
  std::vector<PoolTriple> items;
  size_t next = 0;
};
u64 triple_draw_count(const TripleSpec& sp);
bool spec_equal(const TripleSpec& a, const TripleSpec& b);
void queue_save(const TripleQueue& q, const std::string& path);
void queue_load(TripleQueue& q, const std::string& path);

// ------------------------------------------------------------------ the wire
// One collective: each local slot's build kernel writes its payload into own(slot);
// after wait() the peer's payload for the same slot is readable at peer(slot).
struct ConvGeom {
  u32 N, C, H, W, k, stride, pad, OH, OW;
};
// An eps open whose opened value E = x0 + x1 - A (two local slots, pair evaluation) is not
// materialised: the combine GEMM (gemm_tc3.cu) generates it in its producer warps from the
// activation shares and the dealer's A. mode 1 = dense rows x[a_off + m*K + k], 2 = im2col rows
// of a convolution (global row a_off/K + m). The open is still posted and accounted.
struct EpsDefer {
  int mode = 0;  // 1 dense eps, 2 im2col eps (gemm_tc3.cu), 3 weight-side delta F = x0 + x1 - B (ring_gemv_pair)
  const u64* x0 = nullptr;
  const u64* x1 = nullptr;
  ConvGeom g{};
  u64 a_off = 0;
};

struct Open {
  std::shared_ptr<Block> out;    // n_local * n words: own payloads
  std::shared_ptr<Block> in;     // n words: received peer payload (n_local == 1 only)
  size_t n = 0;
  Reduce kind = Reduce::Sum;
  u32 seq = 0;
  bool waited = false;
  bool posted = false;
  long trace_idx = -1;           // row in Session::trace when its timestamps are recorded
  u64 trace_gen = 0;             // Session::trace_gen_ when the row was made (clear_trace bumps it)
  cudaEvent_t ready = nullptr;   // arrival (throttled link or NCCL), or null
  // n_local == 2 only, set by the caller before the build: the build writes the opened value
  // (own0 + own1 — what both parties read after the zero-copy open) once into own(0) instead
  // of the two payloads; consumers read it as one operand (beaver_combine).
  bool summed = false;
  EpsDefer defer{};              // summed eps built inside the combine GEMM (defer.mode != 0)
  u64* own(int slot) const { return out->ptr + size_t(slot) * n; }
  u64 tag_hash = 0;              // FNV-1a of the post tag (collective header)
  const u64* peer(int slot) const;
  int n_local = 2;
};

struct SessionConfig {
  int frac_bits = 16;
  int chunks = 1;                 // ProtoCtx::chunks (H/protocols/context.hpp:17-35)
  u64 chunk_threshold = 0;        // bytes
  bool merged_adder = true;
  double link_latency_s = 0;      // optional throttled link (H/transport/config.hpp:41-43)
  double link_bandwidth = 0;      // bytes/s; 0 = no throttle (NVLink / in-device)
  double sec_per_message = 0;
};

constexpr size_t kFlushBytes = size_t(256) << 20;  // > 126 MB L2

// In-process link between two single-party sessions on one GPU (party 0 and party 1 driven
// by two host threads): the same one-party-per-session code path a 2-GPU pair runs, with the
// NCCL send/recv replaced by device copies, so it can be exercised on one device. The second
// party to post a collective enqueues both directions on its comm stream; both wait on it.
struct LoopLink {
  struct Slot {
    u64 tag_hash[2] = {0, 0};
    cudaEvent_t trailer_done[2] = {nullptr, nullptr};
    const u64* own[2] = {nullptr, nullptr};
    u64* in[2] = {nullptr, nullptr};
    cudaEvent_t built[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;
    size_t n = 0;
    int arrived = 0;
    bool completed = false;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::map<u64, Slot> slots;
};

struct SocketLink;  // link.cu: TCP link between one-party sessions in different processes
struct P2PLink;     // link.cu: device-flag peer-store link between one-party sessions of a process

class Session {
 public:
  Session(int device, int n_local, int party, u64 seed, u64 mask_seed, int frac_bits);
  ~Session();

  int device = 0;
  int n_local = 2;
  int party_of[2] = {0, 1};   // party id of each local slot
  u64 seed = 1;
  SessionConfig cfg;
  cudaStream_t stream = nullptr;       // compute stream (all local slots)
  cudaStream_t comm_stream = nullptr;  // link emulation / NCCL
  ncclComm_t nccl = nullptr;
  std::shared_ptr<LoopLink> loop;      // in-process peer (tests of the one-party path on one GPU)
  std::shared_ptr<SocketLink> sock;    // peer process over TCP (link.cu, the SocketComm counterpart)
  std::shared_ptr<P2PLink> p2p_link;        // peer session of this process: device-initiated stores + flags
  struct SockPending {                 // received frames staged host->device, buffer not yet reusable
    cudaEvent_t ev;
    u64* p;
    size_t words;
  };
  std::vector<SockPending> sock_pending;

  // data-parallel shard (batch-leading tensors): local rows are a slice of the global batch
  u64 shard_local = 1, shard_global = 1, shard_offset = 0;
  u64 dp_global(u64 numel_local) const { return numel_local / shard_local * shard_global; }
  u64 dp_offset(u64 numel_local) const { return numel_local / shard_local * shard_offset; }

  // ---- tensors
  DT alloc(const Shape& shape, int scale = 0);
  DT upload(const Shape& shape, int scale, const u64* host);  // host holds n_local*numel words
  void download(const DT& t, u64* host);
  std::shared_ptr<Block> raw(size_t words);

  // ---- dealer (H/sharing/triple.hpp:138-151): stream per tag and fetch count
  Triple fetch(const TripleSpec& spec, const std::string& tag, bool batch_b = false);
  u64 tag_stream(const std::string& tag);
  std::unordered_map<u64, u64> tag_counts;
  u64 untagged_index = 0;
  // TripleSource plugin (H/sharing/triple.hpp:126-179): record every fetched triple into a
  // queue (offline dealer) and/or consume triples from a queue instead of the seeded dealer.
  std::shared_ptr<TripleQueue> record_q, source_q;

  // ---- party mask rng (CounterRng(mask_seed, party)): sequential counters per slot
  u64 mask_key[2] = {0, 0};
  u64 mask_ctr = 0;  // same count for every party: each a2b draws numel per party
  struct MaskRef {
    u64 base;
    const u64* bp;  // device slot (graph replay) or null
  };
  MaskRef take_mask(u64 numel_local);  // first counter of this call's draws, advances

  // ---- CUDA-graph capture of a whole inference (executor)
  static constexpr size_t kMaxKeys = 1 << 15, kMaxMasks = 1 << 13;
  struct Capture {
    bool active = false;
    u64* tab = nullptr;              // device: keys [0,kMaxKeys), mask bases [kMaxKeys, +kMaxMasks)
    u64* meta = nullptr;             // device: h[], c0[], mbase0[] for the rekey kernel
    u64* iter = nullptr;             // device replay counter
    u64* seqd = nullptr;             // device: collectives per replay (p2p flag values)
    std::vector<u64> hs, c0s, mb0;
    std::vector<char> carried;  // key slot adopted from a fetch made before the capture
    bool comm_used = false;     // the comm stream was forked into the capture
    u64 mask_per_run = 0;
    CommStats stats_delta[2];
    u64 seq_delta = 0;
    std::vector<std::pair<u64*, size_t>> chunks;  // arena (cudaMalloc'd, persistent)
    size_t chunk = 0, off = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    u64 kernels = 0;                 // kernel nodes in the graph
    u64 replays = 0;
  } cap;
  u64* arena_alloc(size_t words);
  // A triple fetched before the capture but consumed inside it (the pipelined wrap-around
  // prefetch): give it a key slot that tracks the previous replay's prefetch.
  void capture_adopt(Triple& t);
  void begin_capture();
  void end_capture();
  void replay();
  void release_graph();
  void require_eager_streams(const char* what) const;

  // ---- wire
  // Collective header (H/transport/sim.hpp:101-110 checks seq / shape per reveal): with one
  // party per session every payload crosses the link with a 3-word trailer {seq, n, tag hash}
  // written on the comm stream; after the transfer a check kernel compares the peer's trailer
  // with this party's own and records a mismatch in host-mapped memory. The next wait() /
  // sync() throws ProtocolError (a desync can only be seen once the payload landed).
  static constexpr size_t kTrailer = 3;
  struct Desync {
    unsigned int bad;
    unsigned int pad;
    unsigned long long want[3], got[3];
  };
  Desync* desync_ = nullptr;      // host-mapped
  Desync* desync_dev_ = nullptr;  // its device alias
  void check_desync();
  Open begin_open(size_t nwords, Reduce kind, std::shared_ptr<Block> out = nullptr,
                  std::shared_ptr<Block> in = nullptr);
  void post(Open& o, const std::string& tag, bool p2p = false);
  void wait(Open& o);
  // Collective bookkeeping only (stats, trace, order) for opens that a persistent kernel
  // performs in-device; returns the sequence number.
  u32 account(size_t nwords, Reduce kind, const std::string& tag, bool p2p = false);
  // 1-GPU mode without an emulated link: chains of rounds may run as one persistent kernel.
  // Auto (2): small chains are launch-latency bound and run persistent; large ones run one
  // kernel per round at full occupancy. 0 = never, 1 = always (MPCG_PERSISTENT / set_persistent).
  bool persistent_ok(size_t n) const;
  int persistent_mode = 2;
  // In-device opens without an emulated link and without tracing (two local slots): a chunked
  // op runs the lanes of each round as ONE launch over the whole tensor, and accounts the
  // collectives per lane in the reference's order (round-major, lanes in order), so tags,
  // counts and bytes are those of the lane-by-lane schedule. There is no transfer for the
  // lanes to overlap; splitting the launches only adds ramp and tail per round.
  // MPCG_FUSE_LANES=0 keeps one launch per lane.
  bool fuse_lanes() const;
  // Post `o` (the whole tensor's payload, already built) as `ch` lane collectives: lane k
  // carries words_per_elem x |chunk_range(n, ch, k)| words under tag_of(k).
  template <class TagOf>
  void post_lanes(Open& o, size_t n, int ch, size_t words_per_elem, TagOf tag_of) {
    if (o.posted) throw Error(kUsageError, "open posted twice");
    o.posted = true;
    for (int k = 0; k < ch; ++k) {
      const size_t lo = n * size_t(k) / size_t(ch), hi = n * size_t(k + 1) / size_t(ch);
      const u32 seq = account(words_per_elem * (hi - lo), o.kind, tag_of(k));
      if (k == 0) o.seq = seq;
    }
    check();
  }
  // measured with whole-inference graph replay: 16384 beats 32768 / 65536 on LeNet-5 (0.604 vs
  // 0.626 ms) and is level on BERT-base (46.5 vs 46.6 ms)
  static constexpr size_t kPersistentMaxElems = 16384;
  u32 next_seq = 0;
  CommStats stats[2];
  std::vector<TraceEvent> trace;
  bool trace_on = false;
  void set_trace(bool on);
  void clear_trace();
  // Synchronises, resolves the device timestamps of every traced row and returns them.
  const std::vector<TraceEvent>& trace_rows();
  // Host wall seconds since the session was created (Communicator::now, socket backend).
  double now() const;
  // Fault injection (Communicator::add_delay): the compute stream idles `seconds` here.
  void add_delay(double seconds);

  void sync();
  void check();  // debug: sync + error check when MPCG_DEBUG_SYNC=1
  bool debug_sync = false;

  // measurement helpers (bench.py)
  void* flush_buf = nullptr;
  int flush_val = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timer_ev;

 private:
  void throttle(Open& o);
  cudaEvent_t pool_event();
  cudaEvent_t trace_event(cudaStream_t st);  // timing event recorded on `st`, owned by the trace
  struct TraceMarks {
    cudaEvent_t issue = nullptr, sent = nullptr, wait_begin = nullptr, wait_end = nullptr;
    double busy_s = -1;  // emulated link: modelled sender occupancy
  };
  std::vector<TraceMarks> trace_marks_;
  std::vector<cudaEvent_t> trace_events_;
  cudaEvent_t trace_epoch_ = nullptr;
  size_t trace_resolved_ = 0;
 public:
  u64 trace_gen_ = 0;
 private:
  double created_ = 0;
  std::vector<cudaEvent_t> events_;
  size_t event_next_ = 0;
  u64* link_state_ = nullptr;  // device: [next free ns]
};

void pool_on_fetch(Session& s, Triple& t);
void dealer_fetch(Session& s, const TripleSpec& spec, const std::string& tag, DT& a, DT& b, DT& c);
void socket_connect(Session& s, const char* host, int port, double timeout_s);
void socket_post(Session& s, Open& o, size_t words);
void socket_receive(Session& s, Open& o);
void socket_reap(Session& s, bool all);
void p2p_connect(Session& a, Session& b);
void p2p_post(Session& s, Open& o);
void p2p_wait(Session& s, const Open& o);
void p2p_replay_barrier(Session& s);

// ------------------------------------------------------------------ protocol ops
// Mirrors of the reference free functions; arguments keep their meaning, each DT
// carries every local party's share (H/protocols/*.hpp, H/nonlinear/*.hpp).
void require_same_shape(const DT& a, const DT& b, const char* op);
int clamp_chunks(int chunks, size_t numel);
inline std::pair<size_t, size_t> chunk_range(size_t total, int chunks, int k) {
  return {total * size_t(k) / size_t(chunks), total * (size_t(k) + 1) / size_t(chunks)};
}

struct AdderOptions {
  int width = 64;
  bool merged = true;
  int chunks = 1;
};

int chunks_for(const Session& s, size_t numel);

DT beaver_mul(Session& s, const DT& x, const DT& y, const std::string& tag = "mul", int chunks = 1);
DT beaver_square(Session& s, const DT& x, const std::string& tag = "square", int chunks = 1);
DT beaver_and(Session& s, const DT& x, const DT& y, const std::string& tag = "and", int chunks = 1);
DT beaver_matmul(Session& s, const DT& x, const DT& y, bool transpose_b, const std::string& tag = "matmul",
                 int chunks = 1);
DT binary_add(Session& s, const DT& x, const DT& y, const AdderOptions& opt = {},
              const std::string& tag = "badd");
DT a2b(Session& s, const DT& x, const AdderOptions& opt = {}, const std::string& tag = "a2b");
DT msb(Session& s, const DT& x, const AdderOptions& opt = {}, const std::string& tag = "msb");
DT b2a_bit(Session& s, const DT& b, const std::string& tag = "b2a", int chunks = 1);
DT less_than(Session& s, const DT& x, const DT& y, const AdderOptions& opt = {},
             const std::string& tag = "lt");
DT truncate_shares(Session& s, const DT& x, int bits);
DT relu_shares(Session& s, const DT& x, const std::string& tag = "relu");
DT max_last_dim(Session& s, const DT& x, size_t L, const std::string& tag = "max");
DT exp_shares(Session& s, const DT& x, const std::string& tag = "exp", int square_iters = 7);
DT reciprocal_shares(Session& s, const DT& x, const std::string& tag = "recip", int newton_iters = 10);
DT softmax_shares(Session& s, const DT& x, size_t L, const std::string& tag = "softmax");
DT maxpool2d_shares(Session& s, const DT& x, size_t N, size_t C, size_t H, size_t W, size_t k,
                    size_t stride, const std::string& tag = "maxpool");
DT open_value(Session& s, const DT& x, Reduce kind, const std::string& tag);  // reveal, every slot gets it

// Extensions the ResNet-18 / BERT-base configs need and the reference lacks (ext.cu;
// restated in oracle/mpc_oracle.py, parity unpinned by the reference).
constexpr double kLnEps = 1e-5;
constexpr int kIsqrtIters = 3;
int recip_unit_iters(int frac_bits);  // Newton steps for 1/d on [1, 2] from a linear seed (sigmoid)
DT sigmoid_shares(Session& s, const DT& x, const std::string& tag = "sigmoid");
DT gelu_shares(Session& s, const DT& x, const std::string& tag = "gelu");
DT inv_sqrt_shares(Session& s, const DT& v, const std::string& tag = "isqrt", int newton_iters = kIsqrtIters);
DT layernorm_shares(Session& s, const DT& x, size_t d, const DT& gamma, const DT& beta, bool public_weights,
                    const std::string& tag = "ln");
DT global_avg_pool(Session& s, const DT& x, size_t N, size_t C, size_t HW);

// local tensor helpers (fused into producers where it matters)
DT add_public(Session& s, const DT& x, u64 v);     // party 0 absorbs
DT scale_public(Session& s, const DT& x, u64 k);
DT sub_t(Session& s, const DT& a, const DT& b);
DT add_t(Session& s, const DT& a, const DT& b);
DT reshape(const DT& a, Shape shape);

}  // namespace mpcg
