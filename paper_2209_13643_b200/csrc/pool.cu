// Offline/online split: materialised triple queues (the reference's TripleSource plugin,
// H/sharing/triple.hpp:126-179) and its triple-file format (save_triples / load_triples,
// H/sharing/triple.hpp:181-307).
//
// A queue entry is one triple stored the way the seeded dealer lays out its stream (SURVEY
// Appendix A): the draw sequence [A | B | r_A | r_B | r_C] (2PC; B is not drawn for a square
// triple), so every protocol kernel reads it through the same counter arithmetic it uses to
// regenerate draws (dmix, common.cuh) and the per-party shares it derives are exactly the
// triple's: party 1 holds (r_A, r_B, r_C), party 0 (A - r_A, B - r_B, A*B - r_C).
//   * offline phase: a session in record mode materialises every triple it fetches (one
//     dealer kernel per fetch: draw c -> pool[c-1]) into a queue, or a queue is loaded from a
//     reference triple file;
//   * online phase: a session in queue mode pops triples in fetch order — QueueTripleSource
//     semantics: specs are checked ("triple queue spec mismatch at record i"), tags are
//     irrelevant, running out is "triple queue exhausted" (ProtocolError) — and its kernels
//     read the draws from HBM instead of running splitmix64.
#include <cstdio>
#include <cstring>

#include "core.hpp"
#include "ew.cuh"
#include "gemm.cuh"

namespace mpcg {

namespace {
__global__ void pool_fill_kernel(u64* out, u64 key, u64 n) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    out[i] = mix64(key + (i + 1) * kPhi);  // draw c = i + 1 of the stream
}

struct Sizes {
  u64 na, nb, nc, nb_draw;
};
Sizes spec_sizes(const TripleSpec& sp) {
  Sizes z{};
  z.na = shape_numel(sp.shape_a);
  z.nb = shape_numel(sp.shape_b);
  if (!sp.matmul) {
    z.nc = z.na;
  } else {
    const size_t k = sp.shape_a.back();
    const size_t N = sp.transpose_b ? sp.shape_b[sp.shape_b.size() - 2] : sp.shape_b.back();
    z.nc = z.na / k * N;
  }
  z.nb_draw = sp.square ? 0 : z.nb;
  return z;
}
}  // namespace

u64 triple_draw_count(const TripleSpec& sp) {
  const Sizes z = spec_sizes(sp);
  return z.na + z.nb_draw + z.na + z.nb + z.nc;  // 2 parties: one masked copy of A, B, C
}

bool spec_equal(const TripleSpec& a, const TripleSpec& b) {
  return a.kind == b.kind && a.matmul == b.matmul && a.square == b.square && a.transpose_b == b.transpose_b &&
         a.shape_a == b.shape_a && a.shape_b == b.shape_b;
}

// Session::fetch hook: record (offline dealer) and/or consume (queue source).
void pool_on_fetch(Session& s, Triple& t) {
  if (!s.record_q && !s.source_q) return;
  if (s.cap.active) throw Error(kUsageError, "triple queues and CUDA-graph capture do not mix");
  if (s.shard_local != s.shard_global) throw Error(kUsageError, "triple queues need an unsharded session");
  if (s.source_q) {
    TripleQueue& q = *s.source_q;
    if (q.next >= q.items.size()) throw Error(kProtocolError, "triple queue exhausted");
    const PoolTriple& it = q.items[q.next];
    if (!spec_equal(it.spec, t.spec))
      throw Error(kProtocolError, "triple queue spec mismatch at record " + std::to_string(q.next));
    ++q.next;
    t.ew.pool = it.draws->ptr;
    t.mm.pool = it.draws->ptr;
    t.ew.kp = t.mm.kp = nullptr;
    return;
  }
  PoolTriple it;
  it.spec = t.spec;
  it.words = triple_draw_count(t.spec);
  it.draws = Block::persistent(it.words);
  const u64 blocks = std::max<u64>(1, std::min<u64>((it.words + 255) / 256, u64(num_sms()) * 8));
  pool_fill_kernel<<<unsigned(blocks), 256, 0, s.stream>>>(it.draws->ptr, t.key, it.words);
  MPCG_CUDA(cudaGetLastError());
  g_launches.fetch_add(1);
  s.record_q->items.push_back(std::move(it));
}

// ---------------------------------------------------------------- triple files (2PC)
namespace {
void put_u64(std::string& b, u64 v) {
  for (int i = 0; i < 8; ++i) b.push_back(char((v >> (8 * i)) & 0xFF));
}
u64 get_u64(const unsigned char* p) {
  u64 v = 0;
  for (int i = 0; i < 8; ++i) v |= u64(p[i]) << (8 * i);
  return v;
}

// C = A (x) B on the host: wrapping multiply, AND for binary, batched / transposed matmul
// (H/sharing/triple.hpp:74-79, H/ring/tensor.hpp:242-281).
std::vector<u64> host_product(const TripleSpec& sp, const u64* A, const u64* B) {
  const Sizes z = spec_sizes(sp);
  std::vector<u64> C(z.nc, 0);
  if (!sp.matmul) {
    for (u64 i = 0; i < z.na; ++i) C[i] = sp.kind == TripleKind::Bin ? (A[i] & B[i]) : A[i] * B[i];
    return C;
  }
  const u64 K = sp.shape_a.back(), M = sp.shape_a[sp.shape_a.size() - 2];
  const u64 N = sp.transpose_b ? sp.shape_b[sp.shape_b.size() - 2] : sp.shape_b.back();
  const u64 batch = z.na / (M * K);
  const bool bb = sp.shape_b.size() > 2;
  for (u64 b = 0; b < batch; ++b)
    for (u64 m = 0; m < M; ++m)
      for (u64 n = 0; n < N; ++n) {
        u64 acc = 0;
        const u64* a = A + (b * M + m) * K;
        const u64* bm = B + (bb ? b * K * N : 0);
        for (u64 k = 0; k < K; ++k) acc += a[k] * (sp.transpose_b ? bm[n * K + k] : bm[k * N + n]);
        C[(b * M + m) * N + n] = acc;
      }
  return C;
}
}  // namespace

void queue_save(const TripleQueue& q, const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw Error(kTransportError, "save_triples: cannot open " + path);
  for (const PoolTriple& it : q.items) {
    const TripleSpec& sp = it.spec;
    const Sizes z = spec_sizes(sp);
    std::vector<u64> d(it.words);
    MPCG_CUDA(cudaMemcpy(d.data(), it.draws->ptr, it.words * 8, cudaMemcpyDeviceToHost));
    const u64* A = d.data();
    const u64* B = sp.square ? A : A + z.na;
    const u64* rA = A + z.na + z.nb_draw;
    const u64* rB = rA + z.na;
    const u64* rC = rB + z.nb;
    const std::vector<u64> C = host_product(sp, A, B);
    const bool bin = sp.kind == TripleKind::Bin;
    std::string body;
    body.push_back(char(sp.kind));
    body.push_back(char(sp.matmul ? 1 : 0));
    body.push_back(char(sp.square ? 1 : 0));
    body.push_back(char(sp.transpose_b ? 1 : 0));
    body.push_back(char(2));
    body.push_back(char(sp.shape_a.size()));
    for (auto v : sp.shape_a) put_u64(body, v);
    body.push_back(char(sp.shape_b.size()));
    for (auto v : sp.shape_b) put_u64(body, v);
    for (u64 i = 0; i < z.na; ++i) put_u64(body, bin ? A[i] ^ rA[i] : A[i] - rA[i]);  // party 0
    for (u64 i = 0; i < z.nb; ++i) put_u64(body, bin ? B[i] ^ rB[i] : B[i] - rB[i]);
    for (u64 i = 0; i < z.nc; ++i) put_u64(body, bin ? C[i] ^ rC[i] : C[i] - rC[i]);
    for (u64 i = 0; i < z.na; ++i) put_u64(body, rA[i]);  // party 1
    for (u64 i = 0; i < z.nb; ++i) put_u64(body, rB[i]);
    for (u64 i = 0; i < z.nc; ++i) put_u64(body, rC[i]);
    std::string head;
    put_u64(head, body.size());
    std::fwrite(head.data(), 1, head.size(), f);
    std::fwrite(body.data(), 1, body.size(), f);
  }
  std::fclose(f);
}

void queue_load(TripleQueue& q, const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw Error(kTransportError, "load_triples: cannot open " + path);
  std::vector<PoolTriple> out;
  for (size_t rec = 0;; ++rec) {
    unsigned char head[8];
    const size_t got = std::fread(head, 1, 8, f);
    if (got == 0) break;
    if (got != 8) {
      std::fclose(f);
      throw Error(kTransportError, "load_triples: truncated record header");
    }
    const u64 len = get_u64(head);
    std::vector<unsigned char> body(len);
    if (std::fread(body.data(), 1, len, f) != len) {
      std::fclose(f);
      throw Error(kTransportError, "load_triples: truncated record body");
    }
    size_t off = 0;
    auto need = [&](size_t n) {
      if (off + n > body.size()) {
        std::fclose(f);
        throw Error(kTransportError, "load_triples: malformed record");
      }
    };
    need(6);
    TripleSpec sp;
    sp.kind = body[off++] ? TripleKind::Bin : TripleKind::Arith;
    sp.matmul = body[off++] != 0;
    sp.square = body[off++] != 0;
    sp.transpose_b = body[off++] != 0;
    const int n = body[off++];
    if (n != 2) {
      std::fclose(f);
      throw Error(kConfigError, "load_triples: only 2-party triple files are supported (3PC is out of scope)");
    }
    const int nda = body[off++];
    for (int i = 0; i < nda; ++i) {
      need(8);
      sp.shape_a.push_back(get_u64(body.data() + off));
      off += 8;
    }
    need(1);
    const int ndb = body[off++];
    for (int i = 0; i < ndb; ++i) {
      need(8);
      sp.shape_b.push_back(get_u64(body.data() + off));
      off += 8;
    }
    const Sizes z = spec_sizes(sp);
    need(16 * (z.na + z.nb + z.nc));
    auto word = [&](u64 i) { return get_u64(body.data() + off + 8 * i); };
    const u64 p1 = z.na + z.nb + z.nc;  // party 1's block
    const bool bin = sp.kind == TripleKind::Bin;
    PoolTriple it;
    it.spec = sp;
    it.words = triple_draw_count(sp);
    std::vector<u64> d(it.words);
    u64* A = d.data();
    u64* B = sp.square ? nullptr : A + z.na;
    u64* rA = A + z.na + z.nb_draw;
    u64* rB = rA + z.na;
    u64* rC = rB + z.nb;
    std::vector<u64> Bs(z.nb), c0(z.nc);
    for (u64 i = 0; i < z.na; ++i) {
      rA[i] = word(p1 + i);
      A[i] = bin ? word(i) ^ rA[i] : word(i) + rA[i];
    }
    for (u64 i = 0; i < z.nb; ++i) {
      rB[i] = word(p1 + z.na + i);
      Bs[i] = bin ? word(z.na + i) ^ rB[i] : word(z.na + i) + rB[i];
      if (B) B[i] = Bs[i];
    }
    for (u64 i = 0; i < z.nc; ++i) {
      rC[i] = word(p1 + z.na + z.nb + i);
      c0[i] = word(z.na + z.nb + i);
    }
    // The kernels derive party 0's c share as A*B - r_C: the record must be a valid triple.
    if (sp.square)
      for (u64 i = 0; i < z.na; ++i)
        if (Bs[i] != A[i]) throw Error(kProtocolError, "load_triples: square record " + std::to_string(rec) + " has B != A");
    const std::vector<u64> C = host_product(sp, A, sp.square ? A : Bs.data());
    for (u64 i = 0; i < z.nc; ++i)
      if ((bin ? (c0[i] ^ rC[i]) : (c0[i] + rC[i])) != C[i])
        throw Error(kProtocolError, "load_triples: record " + std::to_string(rec) + " is not a valid Beaver triple");
    it.draws = Block::persistent(it.words);
    MPCG_CUDA(cudaMemcpy(it.draws->ptr, d.data(), it.words * 8, cudaMemcpyHostToDevice));
    out.push_back(std::move(it));
    off += 16 * (z.na + z.nb + z.nc);
  }
  std::fclose(f);
  for (auto& it : out) q.items.push_back(std::move(it));
}

// TripleSource::fetch (H/sharing/triple.hpp:126-130) at the boundary: this session's local
// party shares (a, b, c) of the next triple for `spec` / `tag`, from the seeded dealer or the
// queue in use. A matmul triple's party-0 C share is a ring GEMM (A*B - r_C).
void dealer_fetch(Session& s, const TripleSpec& spec, const std::string& tag, DT& a, DT& b, DT& c) {
  const bool stacked = false;
  Triple t = s.fetch(spec, tag, spec.matmul ? spec.shape_b.size() > 2 : stacked);
  t.mark_consumed();
  const Sizes z = spec_sizes(spec);
  Shape cs = spec.shape_a;
  if (spec.matmul) cs.back() = spec.transpose_b ? spec.shape_b[spec.shape_b.size() - 2] : spec.shape_b.back();
  a = s.alloc(spec.shape_a);
  b = s.alloc(spec.shape_b);
  c = s.alloc(cs);
  const Pid2 pid = pids(s);
  const Ptr2 ap = ptrs(a), bp = ptrs(b), cp = ptrs(c);
  if (!spec.matmul) {
    const EwTriple T = t.ew;
    launch_ew(s.stream, s.n_local, z.na, [=] __device__(int slot, u64 i) {
      u64 x, y, w;
      ew_abc(T, pid.v[slot], T.off + i, x, y, w);
      sel(ap, slot)[i] = x;
      sel(bp, slot)[i] = y;
      sel(cp, slot)[i] = w;
    });
    return;
  }
  const MmTriple mm = t.mm;
  launch_ew(s.stream, s.n_local, z.na, [=] __device__(int slot, u64 i) {
    const u64 ra = mm_rA(mm, i);
    sel(ap, slot)[i] = pid.v[slot] ? ra : mm_A(mm, i) - ra;
  });
  launch_ew(s.stream, s.n_local, z.nb, [=] __device__(int slot, u64 j) {
    const u64 rb = mm_rB(mm, j);
    sel(bp, slot)[j] = pid.v[slot] ? rb : mm_B(mm, j) - rb;
  });
  // c: party 1 = r_C; party 0 = A*B - r_C (one-segment ring GEMM with dealer-drawn operands)
  const u64 K = spec.shape_a.back(), M = spec.shape_a[spec.shape_a.size() - 2];
  const u64 N = cs.back(), batch = z.na / (M * K);
  GemmArgs g{};
  g.nslots = s.n_local;
  g.M = u32(M);
  g.N = u32(N);
  g.K = u32(K);
  g.nbatch = u32(batch);
  g.tb = spec.transpose_b ? 1 : 0;
  for (int i = 0; i < s.n_local; ++i) {
    GemmSlotArgs& S = g.sl[i];
    S.out = c.s[i];
    S.ckey = t.mm.key;
    S.ckp = t.mm.kp;
    S.cbase = 1 + 2 * t.mm.na + 2 * t.mm.nb + t.mm.offC;
    S.mm = t.mm;
    if (s.party_of[i] == 0) {
      S.nseg = 1;
      S.cterm = -1;
      S.lk[0] = kOpA;
      S.rk[0] = kOpB;
      S.sL[0] = M * K;
      S.sR[0] = spec.shape_b.size() > 2 ? K * N : 0;
    } else {
      S.nseg = 0;  // r_C only
      S.cterm = +1;
    }
  }
  const bool all_p1 = s.n_local == 1 && s.party_of[0] == 1;
  if (all_p1) {
    const u64 nc = z.nc;
    launch_ew(s.stream, 1, nc, [=] __device__(int slot, u64 k) { sel(cp, slot)[k] = mm_rC(mm, k); });
    return;
  }
  if (s.n_local == 2) {  // party 1's slot: r_C directly; the GEMM runs party 0's slot only
    const u64 nc = z.nc;
    const int p1slot = s.party_of[0] == 1 ? 0 : 1;
    u64* c1 = c.s[p1slot];
    launch_ew(s.stream, 1, nc, [=] __device__(int, u64 k) { c1[k] = mm_rC(mm, k); });
    g.nslots = 1;
    if (p1slot == 0) g.sl[0] = g.sl[1];
  }
  ring_gemm_launch(s, g);
}

}  // namespace mpcg
