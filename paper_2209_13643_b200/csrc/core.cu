// Session runtime: device memory, dealer tag streams, the open/reveal wire.
#include <cstdio>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "core.hpp"

namespace mpcg {

std::string shape_str(const Shape& s) {
  std::string out = "[";
  for (size_t i = 0; i < s.size(); ++i) {
    if (i) out += "x";
    out += std::to_string(s[i]);
  }
  return out + "]";
}

u64 encode_fixed(double x, int scale_bits) {
  const long double t = std::floor(static_cast<long double>(x) * std::exp2l(scale_bits) + 0.5L);
  if (t < -9223372036854775808.0L || t >= 9223372036854775808.0L)
    throw Error(kRangeError, "encode_fixed: " + std::to_string(x) + " exceeds representable range at scale " +
                                 std::to_string(scale_bits));
  return static_cast<u64>(static_cast<i64>(t));
}

// ------------------------------------------------------------------ memory
Block::Block(size_t w, cudaStream_t s) : words(w), stream(s) {
  if (w) MPCG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), w * sizeof(u64), s));
}
Block::~Block() {
  if (ptr && owned) {
    if (sync_free)
      cudaFree(ptr);
    else
      cudaFreeAsync(ptr, stream);  // stream-ordered: safe after every queued reader
  }
}

std::shared_ptr<Block> Block::persistent(size_t words) {
  u64* p = nullptr;
  MPCG_CUDA(cudaMalloc(&p, (words ? words : 1) * sizeof(u64)));
  auto b = std::make_shared<Block>(p, words);
  b->owned = true;
  b->sync_free = true;
  return b;
}

std::shared_ptr<Block> Session::raw(size_t words) {
  if (cap.active) return std::make_shared<Block>(arena_alloc(words), words);
  return std::make_shared<Block>(words, stream);
}

u64* Session::arena_alloc(size_t words) {
  const size_t w = (words + 31) / 32 * 32;  // 256-byte aligned
  while (true) {
    if (cap.chunk < cap.chunks.size()) {
      auto& [p, n] = cap.chunks[cap.chunk];
      if (cap.off + w <= n) {
        u64* r = p + cap.off;
        cap.off += w;
        return r;
      }
      ++cap.chunk;
      cap.off = 0;
      continue;
    }
    const size_t n = std::max<size_t>(w, size_t(32) << 20);  // >= 256 MiB chunks
    u64* p = nullptr;
    MPCG_CUDA(cudaMalloc(&p, n * sizeof(u64)));
    cap.chunks.push_back({p, n});
  }
}

DT Session::alloc(const Shape& shape, int scale) {
  DT t;
  t.shape = shape;
  t.scale = scale;
  const size_t n = shape_numel(shape);
  t.mem = raw(n * size_t(n_local) + 1);
  for (int i = 0; i < n_local; ++i) t.s[i] = t.mem->ptr + size_t(i) * n;
  return t;
}

DT Session::upload(const Shape& shape, int scale, const u64* host) {
  DT t = alloc(shape, scale);
  const size_t n = shape_numel(shape);
  if (n)
    MPCG_CUDA(cudaMemcpyAsync(t.mem->ptr, host, n * n_local * sizeof(u64), cudaMemcpyHostToDevice, stream));
  return t;
}

void Session::download(const DT& t, u64* host) {
  const size_t n = t.numel();
  if (n)
    MPCG_CUDA(cudaMemcpyAsync(host, t.mem->ptr, n * n_local * sizeof(u64), cudaMemcpyDeviceToHost, stream));
  MPCG_CUDA(cudaStreamSynchronize(stream));
}

// ------------------------------------------------------------------ NCCL (dlopen'd)
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) throw Error(kNcclError, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(a.h, n);
      if (!p) throw Error(kNcclError, std::string("missing NCCL symbol ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(kNcclError, std::string(what) + ": " + nccl_api().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

void nccl_connect(Session& s, const void* id128, int rank) {
  if (s.n_local != 1) throw Error(kUsageError, "NCCL link needs a single-party session");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  MPCG_CUDA(cudaSetDevice(s.device));
  nccl_check(nccl_api().CommInitRank(&s.nccl, 2, id, rank), "ncclCommInitRank");
}

// ------------------------------------------------------------------ session
Session::Session(int dev, int nl, int party, u64 sd, u64 mask_seed, int frac_bits)
    : device(dev), n_local(nl), seed(sd) {
  if (nl != 1 && nl != 2) throw Error(kConfigError, "n_local must be 1 or 2");
  if (nl == 1 && (party < 0 || party > 1)) throw Error(kConfigError, "bad party index");
  if (frac_bits < 1 || frac_bits > 40) throw Error(kConfigError, "frac_bits out of range");
  cfg.frac_bits = frac_bits;
  if (nl == 2) {
    party_of[0] = 0;
    party_of[1] = 1;
  } else {
    party_of[0] = party;
  }
  for (int i = 0; i < nl; ++i) mask_key[i] = mask_seed ^ (u64(party_of[i]) * kPhi);
  MPCG_CUDA(cudaSetDevice(device));
  MPCG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  MPCG_CUDA(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  MPCG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  u64 thr = ~u64(0);
  MPCG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  MPCG_CUDA(cudaMalloc(&link_state_, 64));
  MPCG_CUDA(cudaMemset(link_state_, 0, 64));
  if (nl == 1) {
    MPCG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&desync_), sizeof(Desync), cudaHostAllocMapped));
    std::memset(desync_, 0, sizeof(Desync));
    MPCG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&desync_dev_), desync_, 0));
  }
  const char* dbg = std::getenv("MPCG_DEBUG_SYNC");
  debug_sync = dbg && dbg[0] == '1';
  const char* per = std::getenv("MPCG_PERSISTENT");
  if (per && (per[0] == '0' || per[0] == '1')) persistent_mode = per[0] - '0';
  created_ = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

double Session::now() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - created_;
}

Session::~Session() {
  cudaStreamSynchronize(stream);
  cudaStreamSynchronize(comm_stream);
  try {
    socket_reap(*this, true);
  } catch (...) {
  }
  sock.reset();
  for (auto e : events_) cudaEventDestroy(e);
  for (auto e : trace_events_) cudaEventDestroy(e);
  if (trace_epoch_) cudaEventDestroy(trace_epoch_);
  for (auto& [a, b] : timer_ev) {
    cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  if (flush_buf) cudaFree(flush_buf);
  if (cap.exec) cudaGraphExecDestroy(cap.exec);
  if (cap.graph) cudaGraphDestroy(cap.graph);
  for (auto& [p, n] : cap.chunks) cudaFree(p);
  if (cap.tab) cudaFree(cap.tab);
  if (cap.meta) cudaFree(cap.meta);
  if (cap.iter) cudaFree(cap.iter);
  if (cap.seqd) cudaFree(cap.seqd);
  if (nccl) nccl_api().CommDestroy(nccl);
  if (desync_) cudaFreeHost(desync_);
  cudaFree(link_state_);
  cudaStreamDestroy(comm_stream);
  cudaStreamDestroy(stream);
}

void Session::sync() {
  MPCG_CUDA(cudaStreamSynchronize(comm_stream));
  MPCG_CUDA(cudaStreamSynchronize(stream));
  socket_reap(*this, true);
  check_desync();
}

void Session::check_desync() {
  if (!desync_ || !reinterpret_cast<volatile Desync*>(desync_)->bad) return;
  const Desync d = *desync_;
  desync_->bad = 0;
  throw Error(kProtocolError, "collective desync with the peer: expected seq " + std::to_string(d.want[0]) + " (" +
                                  std::to_string(d.want[1]) + " words, tag hash " + std::to_string(d.want[2]) +
                                  "), peer sent seq " + std::to_string(d.got[0]) + " (" + std::to_string(d.got[1]) +
                                  " words, tag hash " + std::to_string(d.got[2]) + ")");
}

void Session::check() {
  if (!debug_sync) return;
  MPCG_CUDA(cudaGetLastError());
  sync();
}

// ------------------------------------------------------------------ dealer
u64 Session::tag_stream(const std::string& tag) {
  if (tag.empty()) return 0x7452u ^ untagged_index++;
  u64 h = 0xcbf29ce484222325ull;
  for (char c : tag) h = (h ^ u64(static_cast<unsigned char>(c))) * 0x100000001b3ull;
  return mix64(h + 0x51ed270bull * tag_counts[h]++);
}

void Session::require_eager_streams(const char* what) const {
  // A captured graph replays fixed fetch/mask positions from host counters it advances per
  // replay; an eager fetch in between would desynchronise the two and make the next replay
  // reuse triples. Release the graph first.
  if (cap.exec && !cap.active)
    throw Error(kUsageError, std::string(what) + ": the session holds a captured graph that owns its dealer "
                                                 "streams; release it (mpcg_executor_release_graph) first");
}

void Session::release_graph() {
  if (cap.active) throw Error(kUsageError, "release_graph during a capture");
  if (cap.exec) {
    MPCG_CUDA(cudaStreamSynchronize(stream));
    cudaGraphExecDestroy(cap.exec);
    cudaGraphDestroy(cap.graph);
    cap.exec = nullptr;
    cap.graph = nullptr;
  }
}

Triple Session::fetch(const TripleSpec& spec, const std::string& tag, bool batch_b) {
  require_eager_streams("fetch");
  Triple t;
  t.spec = spec;
  const u64* kp = nullptr;
  if (cap.active && !tag.empty()) {  // replayed fetch: key slot refreshed per replay
    u64 h = 0xcbf29ce484222325ull;
    for (char c : tag) h = (h ^ u64(static_cast<unsigned char>(c))) * 0x100000001b3ull;
    if (cap.hs.size() >= kMaxKeys) throw Error(kConfigError, "graph capture: too many triple fetches");
    kp = cap.tab + cap.hs.size();
    cap.hs.push_back(h);
    cap.c0s.push_back(tag_counts[h]);
    cap.carried.push_back(0);
  } else if (cap.active) {
    throw Error(kUsageError, "graph capture needs tagged fetches");
  }
  if (!tag.empty()) {
    u64 h = 0xcbf29ce484222325ull;
    for (char c : tag) h = (h ^ u64(static_cast<unsigned char>(c))) * 0x100000001b3ull;
    t.tag_hash = h;
    t.count = tag_counts[h];
  }
  const u64 stream_id = tag_stream(tag);
  t.key = seed ^ (stream_id * kPhi);
  t.ew.kp = kp;
  t.mm.kp = kp;
  const u64 na = shape_numel(spec.shape_a);
  if (!spec.matmul) {
    if (spec.shape_a != spec.shape_b) throw Error(kConfigError, "dealer_gen_triple: elementwise shapes differ");
    // stacked [2, ...] specs (adder levels) map each half separately
    const bool stacked = batch_b;
    const u64 half = stacked ? na / 2 : na;
    t.ew.key = t.key;
    t.ew.ghalf = dp_global(half);
    t.ew.off = dp_offset(half);
    t.ew.mg = stacked ? 2 * t.ew.ghalf : t.ew.ghalf;
    t.ew.square = spec.square;
    t.ew.bin = spec.kind == TripleKind::Bin;
    t.ew.set_phis();
  } else {
    const Shape& a = spec.shape_a;
    const Shape& b = spec.shape_b;
    if (a.size() < 2 || b.size() < 2) throw Error(kConfigError, "dealer_gen_triple: matmul shapes must have rank >= 2");
    const size_t k = a.back();
    const size_t bk = spec.transpose_b ? b.back() : b[b.size() - 2];
    if (k != bk) throw Error(kConfigError, "dealer_gen_triple: matmul inner dims incompatible");
    const size_t N = spec.transpose_b ? b[b.size() - 2] : b.back();
    const u64 nb = shape_numel(b);
    const u64 nc = na / k * N;
    const bool bb = b.size() > 2;  // batched rhs is batch-leading (attention)
    t.mm.key = t.key;
    t.mm.na = dp_global(na);
    t.mm.offA = dp_offset(na);
    t.mm.nb = bb ? dp_global(nb) : nb;
    t.mm.offB = bb ? dp_offset(nb) : 0;
    t.mm.nc = dp_global(nc);
    t.mm.offC = dp_offset(nc);
    t.mm.set_phis();
  }
  pool_on_fetch(*this, t);
  return t;
}

Session::MaskRef Session::take_mask(u64 numel_local) {
  require_eager_streams("a2b mask");
  const u64 base = mask_ctr + dp_offset(numel_local);
  mask_ctr += dp_global(numel_local);
  MaskRef r{base, nullptr};
  if (cap.active) {
    if (cap.mb0.size() >= kMaxMasks) throw Error(kConfigError, "graph capture: too many a2b calls");
    r.bp = cap.tab + kMaxKeys + cap.mb0.size();
    cap.mb0.push_back(base);
    cap.mask_per_run += dp_global(numel_local);
  }
  return r;
}

// ------------------------------------------------------------------ graph capture
namespace {
// Refresh the replay's key table: tag h fetched with count c0 + iter (the reference's
// per-tag counter, H/sharing/triple.hpp:146), mask bases advanced by whole runs.
__global__ void rekey_kernel(u64* tab, const u64* meta, u32 nkeys, u32 nmasks, u64* iter, u64 seed,
                             u64 mask_per_run, u32 kmax) {
  const u64 it = *iter;
  for (u32 i = threadIdx.x; i < nkeys; i += blockDim.x)
    tab[i] = seed ^ (mix64(meta[i] + 0x51ed270bull * (meta[nkeys + i] + it * meta[2 * nkeys + i])) * kPhi);
  for (u32 j = threadIdx.x; j < nmasks; j += blockDim.x) tab[kmax + j] = meta[3 * nkeys + j] + it * mask_per_run;
  __syncthreads();
  if (threadIdx.x == 0) *iter = it + 1;
}
}  // namespace

void Session::capture_adopt(Triple& t) {
  if (!cap.active) throw Error(kUsageError, "capture_adopt outside a capture");
  if (t.ew.kp || t.mm.kp) return;
  if (cap.hs.size() >= kMaxKeys) throw Error(kConfigError, "graph capture: too many triple fetches");
  const u64* kp = cap.tab + cap.hs.size();
  cap.hs.push_back(t.tag_hash);
  cap.c0s.push_back(t.count);
  cap.carried.push_back(1);
  t.ew.kp = kp;
  t.mm.kp = kp;
}

void Session::begin_capture() {
  if (cap.active) throw Error(kUsageError, "capture already active");
  sync();
  if (cap.exec) {
    cudaGraphExecDestroy(cap.exec);
    cudaGraphDestroy(cap.graph);
    cap.exec = nullptr;
    cap.graph = nullptr;
  }
  if (!cap.tab) {
    MPCG_CUDA(cudaMalloc(&cap.tab, (kMaxKeys + kMaxMasks) * sizeof(u64)));
    MPCG_CUDA(cudaMalloc(&cap.iter, 64));
    MPCG_CUDA(cudaMalloc(&cap.seqd, 64));
  }
  MPCG_CUDA(cudaMemset(cap.iter, 0, 64));
  cap.hs.clear();
  cap.c0s.clear();
  cap.mb0.clear();
  cap.carried.clear();
  cap.mask_per_run = 0;
  cap.chunk = 0;
  cap.off = 0;
  cap.replays = 0;
  cap.comm_used = false;
  for (int i = 0; i < 2; ++i) cap.stats_delta[i] = stats[i];
  cap.seq_delta = next_seq;
  cap.kernels = g_launches.load();
  cap.active = true;
  MPCG_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed));
}

void Session::end_capture() {
  if (p2p_link) p2p_replay_barrier(*this);  // replay r+1 must not overwrite inboxes the peer still reads
  if (cap.comm_used) {  // rejoin the comm stream (opens still in flight at the end of the run)
    cudaEvent_t j = pool_event();
    MPCG_CUDA(cudaEventRecord(j, comm_stream));
    MPCG_CUDA(cudaStreamWaitEvent(stream, j, 0));
  }
  cap.active = false;
  cudaError_t e = cudaStreamEndCapture(stream, &cap.graph);
  MPCG_CUDA(e);
  MPCG_CUDA(cudaGraphInstantiate(&cap.exec, cap.graph, 0));
  cap.kernels = g_launches.load() - cap.kernels;
  for (int i = 0; i < 2; ++i) {
    cap.stats_delta[i].bytes_sent = stats[i].bytes_sent - cap.stats_delta[i].bytes_sent;
    cap.stats_delta[i].collectives = stats[i].collectives - cap.stats_delta[i].collectives;
    cap.stats_delta[i].p2p_sends = stats[i].p2p_sends - cap.stats_delta[i].p2p_sends;
  }
  cap.seq_delta = next_seq - cap.seq_delta;
  MPCG_CUDA(cudaMemcpy(cap.seqd, &cap.seq_delta, sizeof(u64), cudaMemcpyHostToDevice));
  const size_t nk = cap.hs.size(), nm = cap.mb0.size();
  std::vector<u64> meta(3 * nk + nm + 1);
  std::unordered_map<u64, u64> per_run;  // fetches of each tag per replay (its count stride)
  for (size_t i = 0; i < nk; ++i)
    if (!cap.carried[i]) per_run[cap.hs[i]]++;
  std::copy(cap.hs.begin(), cap.hs.end(), meta.begin());
  std::copy(cap.c0s.begin(), cap.c0s.end(), meta.begin() + nk);
  for (size_t i = 0; i < nk; ++i) meta[2 * nk + i] = per_run[cap.hs[i]];
  std::copy(cap.mb0.begin(), cap.mb0.end(), meta.begin() + 3 * nk);
  if (cap.meta) cudaFree(cap.meta);
  MPCG_CUDA(cudaMalloc(&cap.meta, meta.size() * sizeof(u64)));
  MPCG_CUDA(cudaMemcpy(cap.meta, meta.data(), meta.size() * sizeof(u64), cudaMemcpyHostToDevice));
}

void Session::replay() {
  if (!cap.exec) throw Error(kUsageError, "replay without a captured graph");
  if (cap.replays > 0) {  // keep host dealer state in step with the device's draws
    for (size_t i = 0; i < cap.hs.size(); ++i)
      if (!cap.carried[i]) tag_counts[cap.hs[i]]++;
    mask_ctr += cap.mask_per_run;
    for (int i = 0; i < n_local; ++i) {
      stats[i].bytes_sent += cap.stats_delta[i].bytes_sent;
      stats[i].collectives += cap.stats_delta[i].collectives;
      stats[i].p2p_sends += cap.stats_delta[i].p2p_sends;
    }
    next_seq += u32(cap.seq_delta);
  }
  cap.replays++;
  rekey_kernel<<<1, 1024, 0, stream>>>(cap.tab, cap.meta, u32(cap.hs.size()), u32(cap.mb0.size()), cap.iter,
                                       seed, cap.mask_per_run, u32(kMaxKeys));
  MPCG_CUDA(cudaGetLastError());
  MPCG_CUDA(cudaGraphLaunch(cap.exec, stream));
  g_launches.fetch_add(cap.kernels + 1);
  check();
}

// ------------------------------------------------------------------ wire
const u64* Open::peer(int slot) const {
  return n_local == 2 ? out->ptr + size_t(1 - slot) * n : in->ptr;
}

cudaEvent_t Session::pool_event() {
  // Ring of events; an event is re-recorded only 4096 opens later, long after its wait.
  constexpr size_t kRing = 4096;
  if (events_.size() < kRing) {
    cudaEvent_t e;
    MPCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events_.push_back(e);
    return e;
  }
  cudaEvent_t e = events_[event_next_];
  event_next_ = (event_next_ + 1) % kRing;
  return e;
}

Open Session::begin_open(size_t nwords, Reduce kind, std::shared_ptr<Block> out, std::shared_ptr<Block> in) {
  Open o;
  o.n = nwords;
  o.kind = kind;
  o.n_local = n_local;
  // one-party sessions: room for the collective trailer behind the payload
  o.out = out ? out : raw(nwords * size_t(n_local) + (n_local == 1 ? kTrailer : 1));
  if (n_local == 1) o.in = in ? in : raw(nwords + kTrailer);
  return o;
}

namespace {
__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Emulated link (H/transport/sim.hpp:83-166 model): the sender's link is busy for
// msg + bytes/bw (serialised in issue order), the payload lands `latency` later.
__global__ void link_delay_kernel(u64* state, u64 busy_ns, u64 latency_ns) {
  const u64 now = globaltimer_ns();
  const u64 start = now > state[0] ? now : state[0];
  const u64 end = start + busy_ns;
  state[0] = end;
  const u64 arrive = end + latency_ns;
  while (globaltimer_ns() < arrive) __nanosleep(500);
}
}  // namespace

__global__ void trailer_kernel(u64* tail, u64 seq, u64 n, u64 h) {
  tail[0] = seq;
  tail[1] = n;
  tail[2] = h;
}
__global__ void trailer_check_kernel(const u64* got, u64 seq, u64 n, u64 h, Session::Desync* d) {
  if (got[0] != seq || got[1] != n || got[2] != h) {
    if (atomicExch(&d->bad, 1u) == 0u) {
      d->want[0] = seq, d->want[1] = n, d->want[2] = h;
      d->got[0] = got[0], d->got[1] = got[1], d->got[2] = got[2];
    }
  }
}

void Session::throttle(Open& o) {
  const double busy = cfg.sec_per_message + double(o.n * 8) / cfg.link_bandwidth;
  link_delay_kernel<<<1, 1, 0, comm_stream>>>(link_state_, u64(busy * 1e9), u64(cfg.link_latency_s * 1e9));
  MPCG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ trace
void Session::set_trace(bool on) {
  if (on && !trace_epoch_) {
    MPCG_CUDA(cudaEventCreate(&trace_epoch_));
    MPCG_CUDA(cudaEventRecord(trace_epoch_, stream));
  }
  trace_on = on;
}

void Session::clear_trace() {
  sync();
  trace.clear();
  trace_marks_.clear();
  for (auto e : trace_events_) cudaEventDestroy(e);
  trace_events_.clear();
  trace_resolved_ = 0;
  ++trace_gen_;
  if (trace_epoch_) MPCG_CUDA(cudaEventRecord(trace_epoch_, stream));
}

cudaEvent_t Session::trace_event(cudaStream_t st) {
  cudaEvent_t e;
  MPCG_CUDA(cudaEventCreate(&e));
  trace_events_.push_back(e);
  MPCG_CUDA(cudaEventRecord(e, st));
  return e;
}

const std::vector<TraceEvent>& Session::trace_rows() {
  sync();
  auto at = [&](cudaEvent_t e) {
    float ms = 0;
    MPCG_CUDA(cudaEventElapsedTime(&ms, trace_epoch_, e));
    return double(ms) * 1e-3;
  };
  for (; trace_resolved_ < trace.size(); ++trace_resolved_) {
    TraceEvent& r = trace[trace_resolved_];
    const TraceMarks& m = trace_marks_[trace_resolved_];
    if (!m.issue) continue;  // captured / in-kernel open: no timestamps
    r.t_issue = at(m.issue);
    r.t_sent = m.busy_s >= 0 ? r.t_issue + m.busy_s : (m.sent ? std::max(r.t_issue, at(m.sent)) : r.t_issue);
    r.t_wait_begin = m.wait_begin ? at(m.wait_begin) : r.t_sent;
    r.t_wait_end = m.wait_end ? std::max(r.t_wait_begin, at(m.wait_end)) : r.t_wait_begin;
  }
  return trace;
}

namespace {
__global__ void delay_kernel(u64 ns) {
  u64 t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
    __nanosleep(1000);
  }
}
}  // namespace

void Session::add_delay(double seconds) {
  if (!(seconds >= 0)) throw Error(kConfigError, "add_delay: seconds must be >= 0");
  if (seconds == 0) return;
  delay_kernel<<<1, 1, 0, stream>>>(u64(seconds * 1e9));
  MPCG_CUDA(cudaGetLastError());
}

u32 Session::account(size_t nwords, Reduce kind, const std::string& tag, bool p2p) {
  const u32 seq = next_seq++;  // collective order = post order (what both parties must agree on)
  for (int i = 0; i < n_local; ++i) {
    stats[i].bytes_sent += nwords * 8;
    if (p2p)
      stats[i].p2p_sends++;
    else
      stats[i].collectives++;
  }
  if (trace_on) {
    trace.push_back(TraceEvent{seq, kind, tag, nwords * 8});
    trace_marks_.push_back(TraceMarks{});
  }
  return seq;
}

bool Session::persistent_ok(size_t n) const {
  // (queue-sourced triples run the per-round kernels: the persistent chains draw in place)
  if (n_local != 2 || cfg.link_bandwidth > 0 || persistent_mode == 0 || source_q) return false;
  static const size_t max_elems = [] {  // MPCG_PERSIST_MAX overrides the measured default
    const char* e = std::getenv("MPCG_PERSIST_MAX");
    return e ? size_t(std::strtoull(e, nullptr, 10)) : kPersistentMaxElems;
  }();
  return persistent_mode == 1 || n <= max_elems;
}

bool Session::fuse_lanes() const {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_FUSE_LANES");
    return !(e && e[0] == '0');
  }();
  return on && n_local == 2 && !(cfg.link_bandwidth > 0) && !trace_on;
}

void Session::post(Open& o, const std::string& tag, bool p2p) {
  if (o.posted) throw Error(kUsageError, "open posted twice");
  o.posted = true;
  o.seq = account(o.n, o.kind, tag, p2p);
  {
    u64 h = 0xcbf29ce484222325ull;
    for (char ch : tag) h = (h ^ u64(static_cast<unsigned char>(ch))) * 0x100000001b3ull;
    o.tag_hash = h ^ (p2p ? 1 : 0) ^ (u64(o.kind) << 1);
  }
  const bool throttled = cfg.link_bandwidth > 0;
  TraceMarks* tm = nullptr;
  if (trace_on && !cap.active) {
    o.trace_idx = long(trace.size()) - 1;
    o.trace_gen = trace_gen_;
    tm = &trace_marks_.back();
    tm->issue = trace_event(stream);
    if (throttled) tm->busy_s = cfg.sec_per_message + double(o.n * 8) / cfg.link_bandwidth;
  }
  if (n_local == 2 && !throttled) {
    check();
    return;  // zero-copy: the peer reads our outbox after the stream-ordered kernel boundary
  }
  cudaEvent_t built = pool_event();
  MPCG_CUDA(cudaEventRecord(built, stream));
  MPCG_CUDA(cudaStreamWaitEvent(comm_stream, built, 0));
  if (cap.active) cap.comm_used = true;
  if (n_local == 1 && sock) {  // TCP to a peer process: framed message with its own header
    if (cap.active) throw Error(kUsageError, "socket link: graph capture is not supported (host I/O)");
    socket_reap(*this, false);
    socket_post(*this, o, o.n);
    if (tm) tm->sent = trace_event(comm_stream);  // staged for the wire
    check();
    return;
  }
  if (n_local == 1 && p2p_link) {  // device-initiated peer stores + flag (link.cu)
    p2p_post(*this, o);
    if (tm) tm->sent = trace_event(comm_stream);
    o.ready = pool_event();  // the push has read our payload (its lifetime is the compute stream's)
    MPCG_CUDA(cudaEventRecord(o.ready, comm_stream));
    check();
    return;
  }
  const size_t wire = n_local == 1 ? o.n + kTrailer : o.n;  // words on the link
  if (n_local == 1) {
    trailer_kernel<<<1, 1, 0, comm_stream>>>(o.own(0) + o.n, o.seq, o.n, o.tag_hash);
    MPCG_CUDA(cudaGetLastError());
    g_launches.fetch_add(1);
  }
  if (n_local == 1 && loop) {
    if (cap.active) throw Error(kUsageError, "loopback link: graph capture is not supported (use the p2p link)");
    const int me = party_of[0];
    static const bool dbg = std::getenv("MPCG_LINK_DEBUG") != nullptr;  // diagnosis of a rare stall
    if (dbg) std::fprintf(stderr, "loopback party %d post seq %u n %zu\n", me, unsigned(o.seq), o.n);
    std::unique_lock<std::mutex> lk(loop->mu);
    LoopLink::Slot& sl = loop->slots[u64(o.seq)];
    sl.own[me] = o.own(0);
    sl.in[me] = o.in->ptr;
    sl.built[me] = built;
    sl.tag_hash[me] = o.tag_hash;
    if (sl.arrived == 1 && sl.n != o.n) {
      // wake the peer so it fails too instead of waiting for a transfer that never comes
      sl.completed = true;
      sl.n = ~size_t(0);
      loop->cv.notify_all();
      throw Error(kProtocolError, "loopback link: collective size mismatch at seq " + std::to_string(o.seq));
    }
    sl.n = o.n;
    if (++sl.arrived == 2) {
      // the peer wrote its trailer on its own comm stream: order the copies behind it too
      MPCG_CUDA(cudaStreamWaitEvent(comm_stream, sl.built[1 - me], 0));
      if (sl.trailer_done[1 - me]) MPCG_CUDA(cudaStreamWaitEvent(comm_stream, sl.trailer_done[1 - me], 0));
      MPCG_CUDA(cudaMemcpyAsync(sl.in[me], sl.own[1 - me], wire * sizeof(u64), cudaMemcpyDeviceToDevice, comm_stream));
      MPCG_CUDA(cudaMemcpyAsync(sl.in[1 - me], sl.own[me], wire * sizeof(u64), cudaMemcpyDeviceToDevice, comm_stream));
      sl.done = pool_event();
      MPCG_CUDA(cudaEventRecord(sl.done, comm_stream));
      sl.completed = true;
      loop->cv.notify_all();
    } else {
      sl.trailer_done[me] = pool_event();
      MPCG_CUDA(cudaEventRecord(sl.trailer_done[me], comm_stream));
      loop->cv.notify_all();
      loop->cv.wait(lk, [&] { return sl.completed; });
      if (sl.n == ~size_t(0)) {
        loop->slots.erase(u64(o.seq));
        throw Error(kProtocolError, "loopback link: collective size mismatch at seq " + std::to_string(o.seq));
      }
      MPCG_CUDA(cudaStreamWaitEvent(comm_stream, sl.done, 0));
      loop->slots.erase(u64(o.seq));
    }
  } else if (n_local == 1) {
    if (!nccl) throw Error(kTransportError, "single-party session has no peer link (connect NCCL first)");
    const int peer = 1 - party_of[0];
    auto& api = nccl_api();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    nccl_check(api.Send(o.own(0), wire, ncclUint64, peer, nccl, comm_stream), "ncclSend");
    nccl_check(api.Recv(o.in->ptr, wire, ncclUint64, peer, nccl, comm_stream), "ncclRecv");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
  if (n_local == 1) {
    trailer_check_kernel<<<1, 1, 0, comm_stream>>>(o.in->ptr + o.n, o.seq, o.n, o.tag_hash, desync_dev_);
    MPCG_CUDA(cudaGetLastError());
    g_launches.fetch_add(1);
  }
  if (tm && n_local == 1) tm->sent = trace_event(comm_stream);  // transfer done
  if (throttled) throttle(o);
  o.ready = pool_event();
  MPCG_CUDA(cudaEventRecord(o.ready, comm_stream));
  check();
}

void Session::wait(Open& o) {
  if (o.waited) throw Error(kUsageError, "wait() called twice on one handle");
  if (!o.posted) throw Error(kUsageError, "wait() on an open that was never posted");
  o.waited = true;
  check_desync();  // a mismatch the comm stream has already seen
  const bool timed = o.trace_idx >= 0 && o.trace_gen == trace_gen_ && size_t(o.trace_idx) < trace_marks_.size() &&
                     !cap.active;
  if (timed) trace_marks_[size_t(o.trace_idx)].wait_begin = trace_event(stream);
  if (sock && n_local == 1 && !o.ready) socket_receive(*this, o);  // blocks until the peer's frame is here
  if (p2p_link && n_local == 1) p2p_wait(*this, o);                      // device spin on the peer's flag
  if (o.ready) MPCG_CUDA(cudaStreamWaitEvent(stream, o.ready, 0));
  if (timed) trace_marks_[size_t(o.trace_idx)].wait_end = o.ready ? trace_event(stream) : nullptr;
}

}  // namespace mpcg
