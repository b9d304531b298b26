// Socket link between two one-party sessions in different processes (or hosts): the GPU
// engine's counterpart of the reference's SocketComm (H/transport/socket.hpp:60-413).
//
// Each post() stages the party's payload device->host on the comm stream into a pinned buffer
// and hands it to a sender thread, which waits for the copy and writes one framed message to
// the peer: {seq, words, tag hash} header (the reference's per-collective sequence check,
// socket.hpp:326-330) + the little-endian payload. A receiver thread reads frames into pinned
// buffers keyed by seq. wait() blocks the host until the peer's frame for that seq arrived,
// checks the header (ProtocolError on a desync, as the reference does), copies it host->device
// into the open's inbox on the comm stream and orders the compute stream behind it. Host I/O
// runs off the issuing thread, so a party keeps enqueueing kernels while its payloads travel.
// Party 0 listens, party 1 connects (socket.hpp:345-402). Not capturable into a CUDA graph.
#include <arpa/inet.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstring>
#include <deque>
#include <thread>

#include "core.hpp"

namespace mpcg {

namespace {
struct Frame {
  u64 seq = 0, words = 0, tag_hash = 0;
};

void write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = ::send(fd, c, n, MSG_NOSIGNAL);
    if (w < 0) {
      if (errno == EINTR) continue;
      throw Error(kTransportError, std::string("socket link: send failed: ") + std::strerror(errno));
    }
    c += w;
    n -= size_t(w);
  }
}

bool read_all(int fd, void* p, size_t n) {  // false on orderly close before any byte
  char* c = static_cast<char*>(p);
  size_t got = 0;
  while (got < n) {
    const ssize_t r = ::recv(fd, c + got, n - got, 0);
    if (r == 0) {
      if (got == 0) return false;
      throw Error(kTransportError, "socket link: peer closed mid-frame");
    }
    if (r < 0) {
      if (errno == EINTR) continue;
      throw Error(kTransportError, std::string("socket link: recv failed: ") + std::strerror(errno));
    }
    got += size_t(r);
  }
  return true;
}

struct Pinned {
  u64* p = nullptr;
  size_t words = 0;
};
}  // namespace

struct SocketLink {
  int fd = -1;
  std::mutex mu;
  std::condition_variable cv;
  // sender side
  struct Job {
    Frame f;
    Pinned buf;
    cudaEvent_t staged;
  };
  std::deque<Job> sendq;
  // receiver side
  std::map<u64, std::pair<Frame, Pinned>> inbox;
  std::vector<Pinned> free_bufs;
  std::string error;  // first I/O error of either thread
  bool closing = false;
  std::thread tx, rx;
  int device = 0;

  Pinned take(size_t words) {  // caller holds mu
    for (size_t i = 0; i < free_bufs.size(); ++i)
      if (free_bufs[i].words >= words) {
        Pinned b = free_bufs[i];
        free_bufs.erase(free_bufs.begin() + long(i));
        return b;
      }
    Pinned b;
    b.words = words < 4096 ? 4096 : words;
    MPCG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b.p), b.words * 8, cudaHostAllocDefault));
    return b;
  }
  void give(Pinned b) {  // caller holds mu
    free_bufs.push_back(b);
  }

  void fail(const std::string& e) {
    std::lock_guard<std::mutex> lk(mu);
    if (error.empty()) error = e;
    cv.notify_all();
  }

  void tx_loop() {
    cudaSetDevice(device);
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return closing || !sendq.empty(); });
        if (sendq.empty()) return;
        j = sendq.front();
        sendq.pop_front();
      }
      try {
        MPCG_CUDA(cudaEventSynchronize(j.staged));
        write_all(fd, &j.f, sizeof j.f);
        write_all(fd, j.buf.p, j.f.words * 8);
      } catch (const std::exception& e) {
        fail(e.what());
      }
      std::lock_guard<std::mutex> lk(mu);
      cudaEventDestroy(j.staged);
      give(j.buf);
    }
  }

  void rx_loop() {
    cudaSetDevice(device);
    try {
      for (;;) {
        Frame f;
        if (!read_all(fd, &f, sizeof f)) return;
        Pinned b;
        {
          std::lock_guard<std::mutex> lk(mu);
          b = take(f.words);
        }
        read_all(fd, b.p, f.words * 8);
        std::lock_guard<std::mutex> lk(mu);
        inbox[f.seq] = {f, b};
        cv.notify_all();
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(mu);
      if (!closing) error = e.what();
      cv.notify_all();
    }
  }

  ~SocketLink() {
    {
      std::lock_guard<std::mutex> lk(mu);
      closing = true;
      cv.notify_all();
    }
    if (tx.joinable()) tx.join();
    if (fd >= 0) ::shutdown(fd, SHUT_RDWR);
    if (rx.joinable()) rx.join();
    if (fd >= 0) ::close(fd);
    for (auto& b : free_bufs) cudaFreeHost(b.p);
    for (auto& [k, v] : inbox) cudaFreeHost(v.second.p);
  }
};

void socket_connect(Session& s, const char* host, int port, double timeout_s) {
  if (s.n_local != 1) throw Error(kUsageError, "socket link needs a single-party session");
  if (s.sock || s.nccl || s.loop || s.p2p_link) throw Error(kUsageError, "session already has a peer link");
  auto L = std::make_shared<SocketLink>();
  L->device = s.device;
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  sockaddr_in addr{};
  addr.sin_family = AF_INET;
  addr.sin_port = htons(static_cast<uint16_t>(port));
  if (::inet_pton(AF_INET, host, &addr.sin_addr) != 1) {
    hostent* he = ::gethostbyname(host);
    if (!he) throw Error(kConfigError, std::string("socket link: cannot resolve ") + host);
    std::memcpy(&addr.sin_addr, he->h_addr_list[0], sizeof addr.sin_addr);
  }
  if (s.party_of[0] == 0) {  // party 0 listens (H/transport/socket.hpp:345-402)
    const int ls = ::socket(AF_INET, SOCK_STREAM, 0);
    int one = 1;
    ::setsockopt(ls, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
    if (::bind(ls, reinterpret_cast<sockaddr*>(&addr), sizeof addr) != 0 || ::listen(ls, 1) != 0) {
      ::close(ls);
      throw Error(kTransportError, std::string("socket link: cannot listen: ") + std::strerror(errno));
    }
    timeval tv{};
    const double left = std::chrono::duration<double>(deadline - std::chrono::steady_clock::now()).count();
    tv.tv_sec = long(left > 0 ? left : 0);
    ::setsockopt(ls, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
    L->fd = ::accept(ls, nullptr, nullptr);
    ::close(ls);
    if (L->fd < 0) throw Error(kTransportError, "socket link: no peer connected before the timeout");
  } else {
    for (;;) {
      const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
      if (::connect(fd, reinterpret_cast<sockaddr*>(&addr), sizeof addr) == 0) {
        L->fd = fd;
        break;
      }
      ::close(fd);
      if (std::chrono::steady_clock::now() > deadline)
        throw Error(kTransportError, "socket link: cannot connect to the peer before the timeout");
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
  }
  int one = 1;
  ::setsockopt(L->fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
  // hello: both sides agree on the party pairing and the dealer seed before any payload
  const u64 hello[2] = {u64(s.party_of[0]), s.seed};
  write_all(L->fd, hello, sizeof hello);
  u64 peer[2];
  if (!read_all(L->fd, peer, sizeof peer)) throw Error(kTransportError, "socket link: peer closed during hello");
  if (peer[0] != u64(1 - s.party_of[0])) throw Error(kProtocolError, "socket link: both ends claim the same party");
  if (peer[1] != s.seed) throw Error(kProtocolError, "socket link: the parties' session seeds differ");
  L->tx = std::thread([p = L.get()] { p->tx_loop(); });
  L->rx = std::thread([p = L.get()] { p->rx_loop(); });
  s.sock = L;
}

void socket_post(Session& s, Open& o, size_t words) {
  SocketLink& L = *s.sock;
  SocketLink::Job j;
  j.f = Frame{o.seq, o.n, o.tag_hash};
  {
    std::lock_guard<std::mutex> lk(L.mu);
    if (!L.error.empty()) throw Error(kTransportError, "socket link: " + L.error);
    j.buf = L.take(words);
  }
  MPCG_CUDA(cudaMemcpyAsync(j.buf.p, o.own(0), o.n * 8, cudaMemcpyDeviceToHost, s.comm_stream));
  MPCG_CUDA(cudaEventCreateWithFlags(&j.staged, cudaEventDisableTiming | cudaEventBlockingSync));
  MPCG_CUDA(cudaEventRecord(j.staged, s.comm_stream));
  std::lock_guard<std::mutex> lk(L.mu);
  L.sendq.push_back(j);
  L.cv.notify_all();
}

// Blocks until the peer's frame for o.seq arrived; stages it into o.in on the comm stream.
void socket_receive(Session& s, Open& o) {
  SocketLink& L = *s.sock;
  Frame f;
  Pinned b;
  {
    std::unique_lock<std::mutex> lk(L.mu);
    L.cv.wait(lk, [&] { return !L.error.empty() || L.inbox.count(o.seq); });
    if (!L.inbox.count(o.seq)) throw Error(kTransportError, "socket link: " + L.error);
    f = L.inbox[o.seq].first;
    b = L.inbox[o.seq].second;
    L.inbox.erase(o.seq);
  }
  if (f.words != o.n || f.tag_hash != o.tag_hash) {
    std::lock_guard<std::mutex> lk(L.mu);
    L.give(b);
    throw Error(kProtocolError, "collective desync with the peer at seq " + std::to_string(o.seq) + ": expected " +
                                    std::to_string(o.n) + " words (tag hash " + std::to_string(o.tag_hash) +
                                    "), peer sent " + std::to_string(f.words) + " (tag hash " +
                                    std::to_string(f.tag_hash) + ")");
  }
  MPCG_CUDA(cudaMemcpyAsync(o.in->ptr, b.p, o.n * 8, cudaMemcpyHostToDevice, s.comm_stream));
  // the pinned buffer returns to the pool once the copy has read it
  cudaEvent_t done;
  MPCG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  MPCG_CUDA(cudaEventRecord(done, s.comm_stream));
  o.ready = done;
  s.sock_pending.push_back({done, b.p, b.words});
}

void socket_reap(Session& s, bool all) {
  if (!s.sock) return;
  auto& q = s.sock_pending;
  size_t k = 0;
  for (; k < q.size(); ++k) {
    if (!all && cudaEventQuery(q[k].ev) == cudaErrorNotReady) break;
    if (all) cudaEventSynchronize(q[k].ev);
    cudaEventDestroy(q[k].ev);
    std::lock_guard<std::mutex> lk(s.sock->mu);
    s.sock->give(Pinned{q[k].p, q[k].words});
  }
  q.erase(q.begin(), q.begin() + long(k));
}


// ------------------------------------------------------------------ device-flag P2P link
// Two one-party sessions driven by two host threads of one process, on one GPU or on two GPUs
// with peer access over NVLink. An open is device-initiated on both ends: the sender's comm
// stream copies its payload straight into the receiver's inbox (peer stores) and then publishes
// a per-collective flag in the receiver's memory with a system-scope release; the receiver's
// compute stream waits on that flag with an acquire spin (no host event crosses the parties,
// no staging copy). Hosts only exchange the inbox address of each collective once (and check
// the {size, tag} header, H/transport/sim.hpp:101-110). Flags are monotonic sequence values, so
// nothing is ever reset. Under CUDA-graph capture the flag value is derived on device from the
// replay counter (seq + replay * collectives-per-run), and every replay ends with a two-party
// device barrier so a replay never overwrites an inbox the peer is still reading.
namespace {
constexpr u32 kFlagRing = 1u << 16;
// per party: [0, kFlagRing) collective flags, [kFlagRing] replay-barrier word, then from
// kReadyOff a second ring: "my inbox for collective s is free to overwrite" (see p2p_post)
constexpr u32 kReadyOff = kFlagRing + 8;
constexpr u32 kFlagWords = kReadyOff + kFlagRing;

// The sequence number of a collective in this run: the baked capture-time number plus one run's
// worth of collectives per replay after the first. Both the flag SLOT and its value derive from
// it, so a collective posted in replay r and waited in replay r+1 (the pipelined executor's
// wrap-around weight-side opening) meets in the same slot.
__device__ __forceinline__ u64 run_seq(u64 base, const u64* iter, const u64* delta) {
  return base + (iter ? (*iter - 1) * *delta : 0);
}
__global__ void p2p_push_kernel(const u64* __restrict__ src, u64* __restrict__ dst, u64 n) {
  const u64 stride = u64(gridDim.x) * blockDim.x;
  u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (u64 j = i; j < n / 2; j += stride) d4[j] = s4[j];
    if (i == 0 && (n & 1)) dst[n - 1] = src[n - 1];
  } else {
    for (u64 j = i; j < n; j += stride) dst[j] = src[j];
  }
}
__device__ __forceinline__ void flag_release(u64* flag, u64 v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}
__device__ __forceinline__ void flag_acquire(const u64* flag, u64 v) {
  for (;;) {
    u64 f;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(flag) : "memory");
    if (f >= v) break;
    __nanosleep(256);
  }
}
// collective flags: ring[run_seq % kFlagRing] = run_seq + 1 (monotonic, never reset)
__global__ void p2p_signal_kernel(u64* ring, u64 base, const u64* iter, const u64* delta) {
  const u64 s = run_seq(base, iter, delta);
  flag_release(ring + s % kFlagRing, s + 1);
}
__global__ void p2p_wait_kernel(const u64* ring, u64 base, const u64* iter, const u64* delta) {
  const u64 s = run_seq(base, iter, delta);
  flag_acquire(ring + s % kFlagRing, s + 1);
}
// end-of-replay barrier word (after the ring): value = replay index (*iter)
__global__ void p2p_barrier_kernel(u64* peer_word, const u64* own_word, const u64* iter) {
  flag_release(peer_word, *iter);
  flag_acquire(own_word, *iter);
}
}  // namespace

struct P2PLink {
  std::mutex mu;
  std::condition_variable cv;
  struct Slot {
    u64* inbox[2] = {nullptr, nullptr};
    size_t n[2] = {0, 0};
    u64 h[2] = {0, 0};
    int arrived = 0, taken = 0;
    bool bad = false;
  };
  std::map<u64, Slot> slots;
  u64* flags[2] = {nullptr, nullptr};  // kFlagRing collective flags + 1 replay-barrier word, per party
  int device[2] = {0, 0};
  ~P2PLink() {
    for (int p = 0; p < 2; ++p)
      if (flags[p]) {
        cudaSetDevice(device[p]);
        cudaFree(flags[p]);
      }
  }
};

void p2p_connect(Session& a, Session& b) {
  if (a.n_local != 1 || b.n_local != 1 || a.party_of[0] == b.party_of[0])
    throw Error(kUsageError, "p2p link joins party 0's and party 1's single-party sessions");
  for (Session* s : {&a, &b})
    if (s->sock || s->nccl || s->loop || s->p2p_link) throw Error(kUsageError, "session already has a peer link");
  if (a.seed != b.seed) throw Error(kProtocolError, "p2p link: the parties' session seeds differ");
  auto L = std::make_shared<P2PLink>();
  for (Session* s : {&a, &b}) {
    const int p = s->party_of[0];
    L->device[p] = s->device;
    MPCG_CUDA(cudaSetDevice(s->device));
    MPCG_CUDA(cudaMalloc(&L->flags[p], kFlagWords * sizeof(u64)));
    MPCG_CUDA(cudaMemset(L->flags[p], 0, kFlagWords * sizeof(u64)));
  }
  if (a.device != b.device) {  // peer stores over NVLink both ways
    for (auto [x, y] : {std::pair<int, int>{a.device, b.device}, {b.device, a.device}}) {
      int ok = 0;
      MPCG_CUDA(cudaDeviceCanAccessPeer(&ok, x, y));
      if (!ok) throw Error(kConfigError, "p2p link: no peer access between the two GPUs");
      MPCG_CUDA(cudaSetDevice(x));
      const cudaError_t e = cudaDeviceEnablePeerAccess(y, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) MPCG_CUDA(e);
      cudaGetLastError();
    }
  }
  MPCG_CUDA(cudaDeviceSynchronize());
  MPCG_CUDA(cudaSetDevice(a.device));
  a.p2p_link = L;
  b.p2p_link = L;
}

void p2p_post(Session& s, Open& o) {
  P2PLink& L = *s.p2p_link;
  const int me = s.party_of[0];
  u64* peer_inbox = nullptr;
  {
    std::unique_lock<std::mutex> lk(L.mu);
    P2PLink::Slot& sl = L.slots[u64(o.seq)];
    sl.inbox[me] = o.in->ptr;
    sl.n[me] = o.n;
    sl.h[me] = o.tag_hash;
    if (++sl.arrived == 2) {
      sl.bad = sl.n[0] != sl.n[1] || sl.h[0] != sl.h[1];
      L.cv.notify_all();
    } else {
      L.cv.wait(lk, [&] { return sl.arrived == 2; });
    }
    const bool bad = sl.bad;
    const size_t pn = sl.n[1 - me];
    const u64 ph = sl.h[1 - me];
    peer_inbox = sl.inbox[1 - me];
    if (++sl.taken == 2) L.slots.erase(u64(o.seq));
    if (bad)
      throw Error(kProtocolError, "collective desync with the peer at seq " + std::to_string(o.seq) + ": " +
                                      std::to_string(o.n) + " words (tag hash " + std::to_string(o.tag_hash) +
                                      ") vs the peer's " + std::to_string(pn) + " (tag hash " + std::to_string(ph) +
                                      ")");
  }
  const u64* it = s.cap.active ? s.cap.iter : nullptr;
  const u64* dl = s.cap.active ? s.cap.seqd : nullptr;
  if (o.n) {
    // Inbox reuse: this party's inbox for seq may be pool memory whose previous reader (the
    // consumer of an earlier collective) is queued on this party's compute stream but has not
    // run yet; the peer pushes from ITS comm stream, which nothing orders behind that reader.
    // So publish "inbox free" from the compute stream (after everything queued so far) and
    // let the push wait for the peer's.
    p2p_signal_kernel<<<1, 1, 0, s.stream>>>(L.flags[1 - me] + kReadyOff, o.seq, it, dl);
    MPCG_CUDA(cudaGetLastError());
    p2p_wait_kernel<<<1, 1, 0, s.comm_stream>>>(L.flags[me] + kReadyOff, o.seq, it, dl);
    MPCG_CUDA(cudaGetLastError());
    g_launches.fetch_add(2);
    u64 blocks = (o.n / 2 + 255) / 256;
    const u64 cap = u64(num_sms()) * 2;
    blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
    p2p_push_kernel<<<unsigned(blocks), 256, 0, s.comm_stream>>>(o.own(0), peer_inbox, o.n);
    MPCG_CUDA(cudaGetLastError());
  }
  p2p_signal_kernel<<<1, 1, 0, s.comm_stream>>>(L.flags[1 - me], o.seq, it, dl);
  MPCG_CUDA(cudaGetLastError());
  g_launches.fetch_add(o.n ? 2 : 1);
}

void p2p_wait(Session& s, const Open& o) {
  P2PLink& L = *s.p2p_link;
  const int me = s.party_of[0];
  const u64* it = s.cap.active ? s.cap.iter : nullptr;
  const u64* dl = s.cap.active ? s.cap.seqd : nullptr;
  p2p_wait_kernel<<<1, 1, 0, s.stream>>>(L.flags[me], o.seq, it, dl);
  MPCG_CUDA(cudaGetLastError());
  g_launches.fetch_add(1);
}

// End of a captured inference: each party tells the other it is done with this replay and waits
// for the peer's word, so replay r+1 never pushes into an inbox the peer still reads in replay r.
void p2p_replay_barrier(Session& s) {
  P2PLink& L = *s.p2p_link;
  const int me = s.party_of[0];
  // both parties' comm streams are joined into the capture at end_capture: order the signal
  // behind everything this party enqueued in the replay (the compute stream)
  p2p_barrier_kernel<<<1, 1, 0, s.stream>>>(L.flags[1 - me] + kFlagRing, L.flags[me] + kFlagRing, s.cap.iter);
  MPCG_CUDA(cudaGetLastError());
  g_launches.fetch_add(1);
}

}  // namespace mpcg
