// Shared device/host primitives for the B200 2PC engine (sm_100a).
//
// Ring Z_2^64 arithmetic and the counter-mode splitmix64 PRG of the reference
// (H/ring/ring_ops.hpp:13-25, H/sharing/rng.hpp:10-32), plus the closed-form dealer
// element functions that regenerate any party's triple share in registers
// (H/sharing/triple.hpp:85-151, H/sharing/share.hpp:22-50).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace mpcg {

using u64 = std::uint64_t;
using u32 = std::uint32_t;
using i64 = std::int64_t;

constexpr u64 kPhi = 0x9E3779B97F4A7C15ull;

// ------------------------------------------------------------------ errors
// Codes mirror the reference exception hierarchy (H/errors.hpp:8-45).
enum ErrCode : int {
  kOk = 0,
  kRangeError = 1,
  kShapeError = 2,
  kConfigError = 3,
  kProtocolError = 4,
  kTransportError = 5,
  kBudgetError = 6,
  kUsageError = 7,
  kCudaError = 8,
  kNcclError = 9,
  kInternalError = 10,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(kCudaError, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                                std::to_string(line));
}
#define MPCG_CUDA(x) ::mpcg::cuda_check((x), #x, __FILE__, __LINE__)

// ------------------------------------------------------------------ ring ops
__host__ __device__ __forceinline__ u64 sar64(u64 v, int k) {
  return static_cast<u64>(static_cast<i64>(v) >> k);
}

__host__ __device__ __forceinline__ u64 mix64(u64 z) {
#if defined(MPCG_NO_DEALER) && defined(__CUDA_ARCH__)
  // Measurement build (make dealerless): device-side dealer/mask draws cost nothing, so timing
  // it beside the real build separates the online protocol from the dealer's work (SURVEY
  // 8f row 4). Its shares are NOT the reference's; it is never used for parity.
  return z;
#endif
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// draw #c (c >= 1) of the stream keyed `key` (already key ^ stream*phi).
__host__ __device__ __forceinline__ u64 drw(u64 key, u64 c) { return mix64(key + c * kPhi); }

// Dealer draw at counter position z = key + c*phi of a triple stream. With a materialised triple
// (queue / pool source, TripleSource plugin: H/sharing/triple.hpp:126-179) the stream's draws
// live in device memory, draw c at pool[c - 1] (c = (z - key) * phi^-1 mod 2^64), laid out as
// the seeded dealer's counters: [A | B | r_A | r_B | r_C] for 2 parties.
constexpr u64 kPhiInv = 0xF1DE83E19937733Dull;  // phi * kPhiInv == 1 (mod 2^64)
__device__ __forceinline__ u64 pool_at(const u64* pool, u64 z, u64 key) {
  return __ldg(pool + ((z - key) * kPhiInv - 1));
}
__device__ __forceinline__ u64 dmix(u64 z, u64 key, const u64* pool) {
#ifndef MPCG_SEEDED_ONLY  // (A/B measurement build: seeded dealer only, no queue source)
  if (__builtin_expect(pool != nullptr, 0)) return pool_at(pool, z, key);
#endif
  return mix64(z);
}

// The triple source is decided once per call site, not per draw: f(std::true_type) reads the
// materialised draws, f(std::false_type) runs the seeded dealer's splitmix64 straight-line (a
// branch per draw would split the independent draws of an element into separate blocks).
template <class F>
__device__ __forceinline__ auto by_source(const u64* pool, F f) {
  if (__builtin_expect(pool != nullptr, 0)) return f(std::true_type{});  // cold: queue source
  return f(std::false_type{});
}
template <bool P>
__device__ __forceinline__ u64 drawp(u64 z, u64 key, const u64* pool) {
  return P ? pool_at(pool, z, key) : mix64(z);
}

// ------------------------------------------------------------------ dealer
// Triple stream keys are either immediates (eager launches) or read from a device key
// table that a rekey kernel refreshes at the head of every CUDA-graph replay, so a
// replayed inference draws the next iteration's triples exactly as the reference's
// per-tag fetch counter does (H/sharing/triple.hpp:146).
//
// One elementwise triple as seen by one party, with the local->global index map that
// lets a data-parallel shard regenerate exactly its slice of the full-batch triple.
// A tensor of `half` local elements per stacked half lives at global index
// s*ghalf + off + i (s = stacked half, 0 for unstacked specs).
struct EwTriple {
  u64 key;        // seed ^ (stream * phi)
  const u64* kp;  // device key slot (graph replay), or null
  const u64* pool = nullptr;  // materialised draws (queue source), or null = seeded dealer
  u64 mg;         // global numel of A (== of B, C)
  u64 ghalf;      // global elements per stacked half (== mg when unstacked)
  u64 off;        // global offset of this shard inside each half
  int square;     // B == A as a secret; only A drawn
  int bin;        // XOR sharing + AND product
  // draw c of element g is mix(key + (base + g)*phi) = mix((key + base*phi) + g*phi): the
  // base*phi terms of the five streams are host constants (set_phis), so a thread pays one
  // 64-bit multiply (g*phi) per element instead of one per draw.
  u64 pA, pB, pra, prb, prc;
  __host__ void set_phis() {
    const u64 nbd = square ? 0 : mg;
    const u64 baseA = 1 + mg + nbd, baseB = baseA + mg;
    pA = kPhi;
    pB = square ? kPhi : (1 + mg) * kPhi;
    pra = baseA * kPhi;
    prb = baseB * kPhi;
    prc = (baseB + mg) * kPhi;
  }
};

__device__ __forceinline__ u64 tkey(u64 key, const u64* kp) { return kp ? __ldg(kp) : key; }

// Raw dealer draws of elementwise triple element g (H/sharing/triple.hpp:62-94): the masks
// rA, rB (, rC) that party 1 receives and, when `p0` is asked for, the secrets A, B that
// party 0's shares absorb. Splitting draws from shares lets a thread that evaluates BOTH
// co-located party slots (1-GPU mode) run the dealer once per element, as the dealer does.
struct Dw {
  u64 A, B, ra, rb, rc;
};
// Pool = true: the triple is materialised (queue source) and its draws are read from HBM;
// false: the seeded dealer's straight-line splitmix64 code. Hot kernels (the SPK adder rounds)
// are instantiated per mode; others take the runtime-checked ew_draw / ew_secrets.
template <bool WithC, bool Pool>
__device__ __forceinline__ Dw ew_draw_t(const EwTriple& t, u64 g, bool p0) {
  const u64 key = tkey(t.key, t.kp);
  const u64 gp = g * kPhi;
  Dw d;
  auto dr = [&](u64 z) { return Pool ? pool_at(t.pool, z, key) : mix64(z); };
  d.ra = dr(key + t.pra + gp);
  d.rb = dr(key + t.prb + gp);
  d.rc = WithC ? dr(key + t.prc + gp) : 0;
  d.A = d.B = 0;
  if (p0) {
    d.A = dr(key + t.pA + gp);
    d.B = t.square ? d.A : dr(key + t.pB + gp);
  }
  return d;
}
template <bool WithC>
__device__ __forceinline__ Dw ew_draw(const EwTriple& t, u64 g, bool p0) {
  if (__builtin_expect(t.pool != nullptr, 0)) return ew_draw_t<WithC, true>(t, g, p0);  // cold: queue source
  return ew_draw_t<WithC, false>(t, g, p0);
}
// The same draws with the stream key and (global index)*phi supplied by the caller: hot loops
// resolve the key once per thread and share one 64-bit multiply between an element's triples.
template <bool WithC, bool Pool>
__device__ __forceinline__ Dw ew_draw_kg(const EwTriple& t, u64 key, u64 gp, bool p0) {
  Dw d;
  auto dr = [&](u64 z) { return Pool ? pool_at(t.pool, z, key) : mix64(z); };
  d.ra = dr(key + t.pra + gp);
  d.rb = dr(key + t.prb + gp);
  d.rc = WithC ? dr(key + t.prc + gp) : 0;
  d.A = d.B = 0;
  if (p0) {
    d.A = dr(key + t.pA + gp);
    d.B = t.square ? d.A : dr(key + t.pB + gp);
  }
  return d;
}
template <bool Pool>
__device__ __forceinline__ Dw ew_secrets_kg(const EwTriple& t, u64 key, u64 gp) {
  auto dr = [&](u64 z) { return Pool ? pool_at(t.pool, z, key) : mix64(z); };
  Dw d;
  d.ra = d.rb = d.rc = 0;
  d.A = dr(key + t.pA + gp);
  d.B = t.square ? d.A : dr(key + t.pB + gp);
  return d;
}

// Only the dealer's secrets A, B of element g: what the two parties' shares reconstruct to
// (a0 ^ a1 or a0 + a1), all an opened-wire issue needs — the masks cancel in the open.
template <bool Pool>
__device__ __forceinline__ Dw ew_secrets_t(const EwTriple& t, u64 g) {
  const u64 key = tkey(t.key, t.kp);
  const u64 gp = g * kPhi;
  auto dr = [&](u64 z) { return Pool ? pool_at(t.pool, z, key) : mix64(z); };
  Dw d;
  d.ra = d.rb = d.rc = 0;
  d.A = dr(key + t.pA + gp);
  d.B = t.square ? d.A : dr(key + t.pB + gp);
  return d;
}
__device__ __forceinline__ Dw ew_secrets(const EwTriple& t, u64 g) {
  if (__builtin_expect(t.pool != nullptr, 0)) return ew_secrets_t<true>(t, g);  // cold: queue source
  return ew_secrets_t<false>(t, g);
}
// `party`'s shares of a drawn element (0 absorbs the secret).
template <bool WithC>
__device__ __forceinline__ void ew_share(const EwTriple& t, int party, const Dw& d, u64& a, u64& b, u64& c) {
  if (party != 0) {
    a = d.ra;
    b = d.rb;
    if (WithC) c = d.rc;
    return;
  }
  if (t.bin) {
    a = d.A ^ d.ra;
    b = d.B ^ d.rb;
    if (WithC) c = (d.A & d.B) ^ d.rc;
  } else {
    a = d.A - d.ra;
    b = d.B - d.rb;
    if (WithC) c = d.A * d.B - d.rc;
  }
}

// a, b shares of element g (global index) for `party` (0 absorbs the secret).
__device__ __forceinline__ void ew_ab(const EwTriple& t, int party, u64 g, u64& a, u64& b) {
  u64 c;
  ew_share<false>(t, party, ew_draw<false>(t, g, party == 0), a, b, c);
}

__device__ __forceinline__ void ew_abc(const EwTriple& t, int party, u64 g, u64& a, u64& b, u64& c) {
  ew_share<true>(t, party, ew_draw<true>(t, g, party == 0), a, b, c);
}

// Square triples only need a and c (b is never used by the combine).
__device__ __forceinline__ void sq_ac(const EwTriple& t, int party, u64 g, u64& a, u64& c) {
  const u64 key = tkey(t.key, t.kp);
  const u64 gp = g * kPhi;
  by_source(t.pool, [&](auto src) {
    constexpr bool P = decltype(src)::value;
    const u64 ra = drawp<P>(key + t.pra + gp, key, t.pool), rc = drawp<P>(key + t.prc + gp, key, t.pool);
    if (party != 0) {
      a = ra;
      c = rc;
      return 0;
    }
    const u64 A = drawp<P>(key + t.pA + gp, key, t.pool);
    a = A - ra;
    c = A * A - rc;
    return 0;
  });
}

__device__ __forceinline__ u64 sq_a(const EwTriple& t, int party, u64 g) {
  const u64 key = tkey(t.key, t.kp);
  const u64 gp = g * kPhi;
  return by_source(t.pool, [&](auto src) {
    constexpr bool P = decltype(src)::value;
    const u64 ra = drawp<P>(key + t.pra + gp, key, t.pool);
    return party != 0 ? ra : drawp<P>(key + t.pA + gp, key, t.pool) - ra;
  });
}

// Matmul triple (H/sharing/triple.hpp:96-114): draws A (na), B (nb), then r_A, r_B, r_C.
struct MmTriple {
  u64 key;
  const u64* kp;
  const u64* pool = nullptr;  // materialised draws (queue source), or null = seeded dealer
  u64 na, nb, nc;     // global numels
  u64 offA, offB, offC;
  u64 pA, pB, prA, prB, prC;  // (stream base + shard offset) * phi, see EwTriple::set_phis
  __host__ void set_phis() {
    pA = (1 + offA) * kPhi;
    pB = (1 + na + offB) * kPhi;
    prA = (1 + na + nb + offA) * kPhi;
    prB = (1 + 2 * na + nb + offB) * kPhi;
    prC = (1 + 2 * na + 2 * nb + offC) * kPhi;
  }
};
__device__ __forceinline__ u64 mm_draw(const MmTriple& t, u64 base_phi, u64 i) {
  const u64 key = tkey(t.key, t.kp);
  return dmix(key + base_phi + i * kPhi, key, t.pool);
}
__device__ __forceinline__ u64 mm_A(const MmTriple& t, u64 i) { return mm_draw(t, t.pA, i); }
__device__ __forceinline__ u64 mm_B(const MmTriple& t, u64 j) { return mm_draw(t, t.pB, j); }
__device__ __forceinline__ u64 mm_rA(const MmTriple& t, u64 i) { return mm_draw(t, t.prA, i); }
__device__ __forceinline__ u64 mm_rB(const MmTriple& t, u64 j) { return mm_draw(t, t.prB, j); }
__device__ __forceinline__ u64 mm_rC(const MmTriple& t, u64 k) { return mm_draw(t, t.prC, k); }

// ------------------------------------------------------------------ launch helpers
// SM count of the current device, queried once per device (148 on a full B200; fewer under
// MIG / MPS partitions). Sizes persistent/cooperative grids and the split-K heuristics.
inline int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

// Instrumentation: count of kernels this library launched, and an optional probe that
// brackets every launch of one kernel class with CUDA events (bench.py's live roofline).
enum KernelClass : int { kClsOther = 0, kClsAdderRound = 1, kClsGemm = 2, kClsBeaver = 3, kClsChain = 4, kClsChainReg = 5 };
struct Probe {
  int cls = -1;             // class being timed, -1 = off
  double bytes = 0;         // algorithmic bytes of the probed launches
  u64 launches = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
};
inline std::atomic<u64> g_launches{0};
inline Probe g_probe;
inline thread_local int t_cls = kClsOther;
inline thread_local double t_bytes = 0;
struct ClassScope {  // tags launches issued in this scope: ClassScope cs(kClsAdderRound, bytes)
  int prev;
  double pb;
  ClassScope(int c, double bytes) : prev(t_cls), pb(t_bytes) {
    t_cls = c;
    t_bytes = bytes;
  }
  ~ClassScope() {
    t_cls = prev;
    t_bytes = pb;
  }
};
inline void probe_begin(cudaStream_t st, cudaEvent_t* a) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  *a = nullptr;
  if (g_probe.cls >= 0 && g_probe.cls == t_cls) {
    cudaEventCreate(a);
    cudaEventRecord(*a, st);
  }
}
inline void probe_end(cudaStream_t st, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, st);
  g_probe.ev.push_back({a, b});
  g_probe.bytes += t_bytes;
  g_probe.launches++;
}

// Programmatic dependent launch: every kernel lets the next one in the stream be scheduled
// as soon as its own CTAs are all resident, and waits (griddepcontrol.wait) for the
// previous grid's completion + memory flush before touching data. In a CUDA graph this
// overlaps the ~µs launch latency of each dependent round kernel with its predecessor.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool& pdl_enabled() {
  static bool on = [] {
    const char* e = std::getenv("MPCG_PDL");
    return e && e[0] == '1';  // measured neutral-to-negative inside graphs: opt-in (MPCG_PDL=1)
  }();
  return on;
}

// cudaLaunchKernelEx with the PDL attribute (when enabled).
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = &attr;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  MPCG_CUDA(cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...));
}

template <class F>
__global__ void __launch_bounds__(256) ew_kernel(u64 n, F f) {
  pdl_enter();
  const int slot = blockIdx.y;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    f(slot, i);
}

inline unsigned ew_blocks(u64 n) {
  u64 b = (n + 255) / 256;
  const u64 cap = u64(num_sms()) * 8;  // 8 resident 256-thread CTAs per SM
  return static_cast<unsigned>(b < 1 ? 1 : (b > cap ? cap : b));
}

// Pair evaluation (1-GPU mode, both party slots local): a functor that defines both(i)
// evaluates element i for slot 0 and slot 1 in one thread, running the dealer's draws for
// that element once. Each slot still writes its own outbox and reads the peer's payload
// from memory, exactly as in per-slot evaluation. MPCG_PAIR_EVAL=0 turns it off.
template <class F, class = void>
struct has_both : std::false_type {};
template <class F>
struct has_both<F, std::void_t<decltype(std::declval<const F&>().both(u64(0)))>> : std::true_type {};

inline bool& pair_eval_enabled() {
  static bool on = [] {
    const char* e = std::getenv("MPCG_PAIR_EVAL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// Summed in-device opens of the matmul combine's eps / delta (MPCG_EPS_FUSE=0: both payloads).
inline bool& eps_fuse_enabled() {
  static bool on = [] {
    const char* e = std::getenv("MPCG_EPS_FUSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// f for slot `slot`, or for both slots when `pair`.
template <class F>
__device__ __forceinline__ void eval_slots(const F& f, bool pair, int slot, u64 i) {
  if (!pair) {
    f(slot, i);
  } else if constexpr (has_both<F>::value) {
    f.both(i);
  } else {
    f(0, i);
    f(1, i);
  }
}

// Functors may define prep() -> P (per-thread values computed once before the grid-stride
// loop, e.g. the dealer keys of graph replay) and both_p(i, P); the functor itself stays in
// the kernel's parameter space (a local copy of a large functor lands in local memory).
template <class F, class = void>
struct has_prep : std::false_type {};
template <class F>
struct has_prep<F, std::void_t<decltype(std::declval<const F&>().prep())>> : std::true_type {};

template <class F>
__global__ void __launch_bounds__(256, 4) ew_pair_kernel(u64 n, F f) {
  pdl_enter();
  if constexpr (has_prep<F>::value) {
    const auto p = f.prep();
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) f.both_p(i, p);
  } else {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) f.both(i);
  }
}

// Launch f(slot, i) for i in [0, n) and every local party slot, on `stream`.
template <class F>
void launch_ew(cudaStream_t stream, int nslots, u64 n, F f) {
  if (n == 0) return;
  cudaEvent_t pe;
  probe_begin(stream, &pe);
  if constexpr (has_both<F>::value) {
    if (nslots == 2 && pair_eval_enabled()) {
      launch_pdl(ew_pair_kernel<F>, dim3(ew_blocks(n)), dim3(256), 0, stream, n, f);
      probe_end(stream, pe);
      return;
    }
  }
  launch_pdl(ew_kernel<F>, dim3(ew_blocks(n), nslots), dim3(256), 0, stream, n, f);
  probe_end(stream, pe);
}

}  // namespace mpcg
