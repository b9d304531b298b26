// Ring GEMM interfaces (gemm.cu SIMT / GEMV / row paths, gemm_tc2.cu tcgen05 int8-limb path).
#pragma once

#include "core.hpp"

namespace mpcg {

// Operand kinds of a GEMM segment. Plain loads, or generated on the fly in the SIMT tile
// loader from the dealer's stream / the two halves of an opened payload, so the Beaver
// combine needs no operand-materialisation pass (matmul triple draws: H/sharing/triple.hpp:96-114).
enum OpKind : int {
  kOpMem = 0,   // p[idx]
  kOpSum = 1,   // p[idx] + q[idx]               (opened E or F = own + peer payload)
  kOpA = 2,     // dealer A                       (party 0)
  kOpA0 = 3,    // a0 = A - r_A                   (party 0 share of A)
  kOpRA = 4,    // r_A                            (party 1 share of A)
  kOpB = 5,     // dealer B                       (party 0)
  kOpB0F = 6,   // (B - r_B) + p[idx] + q[idx]    (party 0: b0 + F)
  kOpRB = 7,    // r_B                            (party 1 share of B)
  kOpBF = 8,    // B + p[idx] + q[idx]            (party 0, tensor-core split: A*(B + F))
  kOpNegSum = 9,  // -(p[idx] + q[idx])           (party 0, tensor-core split: -r_A*F)
};

// One party slot of a multi-segment ring GEMM: out = epi( sum_g L_g * R_g ).
struct GemmSlotArgs {
  int nseg = 0;
  const u64* L[3] = {};   // [batch][M][K], batch stride sL (0 = shared)
  const u64* R[3] = {};   // [batch][K][N] or, transposed, [batch][N][K]; stride sR
  u64 sL[3] = {}, sR[3] = {};
  int lk[3] = {0, 0, 0}, rk[3] = {0, 0, 0};   // OpKind per segment (kOpMem = plain)
  const u64* L2[3] = {};  // second addend of kOpSum
  const u64* R2[3] = {};  // second addend of kOpSum / kOpB0F
  MmTriple mm{};          // dealer view for generated operands
  u64 aoff = 0, boff = 0; // element offset of this call inside A / B (PRG index base)
  u64* out = nullptr;
  const u64* bias = nullptr;  // [N], added after truncation
  const u64* addend = nullptr;  // fused residual add: same layout as out, added last (or null)
  int cterm = 0;              // +1 / -1: add / subtract the triple's r_C
  u64 ckey = 0, cbase = 0;    // r_C(idx) = drw(ckey, cbase + idx)
  const u64* ckp = nullptr;   // device key slot (graph replay)
};

struct GemmArgs {
  GemmSlotArgs sl[2];
  int nslots = 1;
  u32 M = 0, N = 0, K = 0, nbatch = 1;
  int tb = 0;          // R transposed
  int trunc_bits = 0;  // 2PC local truncation (H/protocols/trunc.hpp:41)
  int col2im = 0;      // store NCHW with row = (n, oh, ow)  (H/engine/executor.hpp:110-123)
  u32 OHW = 1;
  u32 row0 = 0;        // col2im: global row of this call's row 0 (row-block chunks of one conv)
  // split-K over the concatenated K' = nseg*K axis: partial sums are added mod 2^64 into
  // acc[slot] ([nbatch][M][N], zeroed) and a second kernel applies the epilogue.
  u32 ksplit = 1, kchunk = 0;
  u64* acc[2] = {nullptr, nullptr};
  int vec16 = 0;  // every L (and transposed R) row start is 16-byte aligned (K even, bases aligned)
  EpsDefer ed{};  // E generated in the GEMM (gemm_tc3.cu only; ed.mode != 0)
  int fdefer = 0;  // F = R + R2 - B: the weight-side delta open not built (ring_gemv_pair only)
};

struct Epi {
  int trunc_bits = 0;
  const u64* bias[2] = {nullptr, nullptr};
  const u64* addend[2] = {nullptr, nullptr};  // fused residual add (the layer's full output layout)
  int col2im = 0;
  u32 OHW = 1;
};


struct FastDiv {  // q = n / d for any 32-bit n (Granlund-Montgomery, round-up multiplier)
  u32 d, m, l;
  FastDiv() = default;
  explicit FastDiv(u32 dv) : d(dv) {
    l = 0;
    while ((u64(1) << l) < dv) ++l;
    m = u32(((u64(1) << 32) * ((u64(1) << l) - dv)) / dv + 1);
  }
  __device__ __forceinline__ u32 div(u32 n) const { return u32((u64(__umulhi(m, n)) + n) >> l); }
};

// Element idx (call-local linear index in the segment's stored layout) of a segment.
__device__ __forceinline__ u64 load_l(const GemmSlotArgs& S, int sg, u64 idx) {
  switch (S.lk[sg]) {
    case kOpMem: return S.L[sg][idx];
    case kOpSum: return S.L[sg][idx] + S.L2[sg][idx];
    case kOpA: return mm_A(S.mm, S.aoff + idx);
    case kOpA0: return mm_A(S.mm, S.aoff + idx) - mm_rA(S.mm, S.aoff + idx);
    default: return mm_rA(S.mm, S.aoff + idx);
  }
}
// The opened F = own + peer delta, or (R2 null: the open summed at build time) R alone.
__device__ __forceinline__ u64 load_f(const GemmSlotArgs& S, int sg, u64 idx) {
  return S.R2[sg] ? S.R[sg][idx] + S.R2[sg][idx] : S.R[sg][idx];
}
__device__ __forceinline__ u64 load_r(const GemmSlotArgs& S, int sg, u64 idx) {
  switch (S.rk[sg]) {
    case kOpMem: return S.R[sg][idx];
    case kOpSum: return load_f(S, sg, idx);
    case kOpB: return mm_B(S.mm, S.boff + idx);
    case kOpB0F: return (mm_B(S.mm, S.boff + idx) - mm_rB(S.mm, S.boff + idx)) + load_f(S, sg, idx);
    case kOpBF: return mm_B(S.mm, S.boff + idx) + load_f(S, sg, idx);
    case kOpNegSum: return u64(0) - load_f(S, sg, idx);
    default: return mm_rB(S.mm, S.boff + idx);
  }
}

__device__ __forceinline__ void gemm_epilogue(const GemmArgs& a, const GemmSlotArgs& S, u32 b, u32 m, u32 n,
                                              u64 v) {
  const u64 lin = (u64(b) * a.M + m) * a.N + n;
  if (S.cterm) {
    const u64 rc = S.mm.pool ? __ldg(S.mm.pool + S.cbase + lin - 1) : drw(tkey(S.ckey, S.ckp), S.cbase + lin);
    v = S.cterm > 0 ? v + rc : v - rc;
  }
  if (a.trunc_bits) v = sar64(v, a.trunc_bits);
  if (S.bias) v += S.bias[n];
  if (a.col2im) {
    const u32 mg = m + a.row0, img = mg / a.OHW, rem = mg - img * a.OHW;
    const u64 o = (u64(img) * a.N + n) * a.OHW + rem;
    S.out[o] = S.addend ? v + __ldg(S.addend + o) : v;
  } else {
    S.out[lin] = S.addend ? v + __ldg(S.addend + lin) : v;
  }
}

void ring_gemm_launch(Session& s, const GemmArgs& a);
// Split-K epilogue: sums a.ksplit partial tiles from a.acc[slot] mod 2^64, then the Beaver epilogue.
__global__ void gemm_splitk_epilogue(GemmArgs a);
using splitk_epilogue_t = void (*)(GemmArgs);
splitk_epilogue_t gemm_splitk_epilogue_fn();
bool gemv_eligible_shape(u32 M, u32 nbatch, bool tb, int col2im);  // the small-M path takes it
// Deferred weight-side delta: the summed delta open of a combine the pair-evaluated GEMV will
// run is not built (o.defer.mode = 3); the GEMV forms F = W0 + W1 - B from the weight shares.
bool delta_defer(Session& s, Open& o, const u64* const w[2], u32 M, u32 N, u32 K);
// Small-M fused-segment path (ring_gemv): 1 = on (default), 0 = off (MPCG_GEMV=0).
inline int& gemv_mode() {
  static int m = [] {
    const char* e = std::getenv("MPCG_GEMV");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return m;
}
int& tc_gemm_mode();  // 0 = never tensor cores, 1 = whenever exact, 2 = auto by size
// Warp-specialised tcgen05 path (gemm_tc2.cu): operands generated by producer warps or packed
// once and bulk-copied; takes every operand kind.
bool ring_gemm_tc2_wants(const GemmArgs& a);
bool ring_gemm_tc2_try(Session& s, const GemmArgs& a);
// Both party slots of a pair-evaluated Beaver combine in one CTA (gemm_tc3.cu); false = not taken.
bool ring_gemm_tc3_try(Session& s, const GemmArgs& a);
int& tc3_mode();
bool tc3_shape_ok(const Session& s, u32 M, u32 N, u32 K, bool col2im);
bool ring_gemm_tc3_accepts(const Session& s, const GemmArgs& a);
// Defer a summed eps open into the combine GEMM when the both-slots kernel will run it (sets
// o.defer; the caller then skips the build and still posts o). false = build it as usual.
bool eps_defer(Session& s, Open& o, const u64* const x[2], const ConvGeom* g, size_t a_off, u32 M, u32 N, u32 K);    // 1 = both-slots kernel where it applies (default), 0 = tc2 only
int tc3_default();  // MPCG_TC3 (0 = off)
void tc2_trace_read(unsigned long long* out, int n);
void tc3_trace_read(unsigned long long* out, int n);  // debug: MPCG_TC3_TRACE=1 stage stamps  // debug: stage timestamps (MPCG_TC2_TRACE=1)
void beaver_combine(Session& s, const Triple& t, const Open& e, size_t a_off, size_t na, const Open& d, size_t nb,
                    DT* rcache, u64* const out[2], size_t out_off, u32 nbatch, u32 M, u32 N, u32 K, bool tb,
                    bool batched_r, size_t r_batch0, const Epi& ep, const DT* aops = nullptr);
bool beaver_combine_fuses_eps(const Session& s, u32 nbatch, u32 M, u32 N, u32 K);
bool beaver_combine_wants_aops(const Session& s, u32 nbatch, u32 M, u32 N, u32 K);

void delta_build_mem(Session& s, const Triple& t, const u64* const y[2], size_t nb, Open& o);
// eps = x - a payload; with `aops` ([2, na] per slot) also the A-side combine operands.
void eps_build_mem(Session& s, const Triple& t, const u64* const x[2], size_t a_off, size_t na, Open& o,
                   const DT* aops = nullptr);
void eps_build_im2col(Session& s, const Triple& t, const u64* const x[2], const ConvGeom& g, size_t a_off,
                      size_t na, Open& o, const DT* aops = nullptr);
void public_gemm(Session& s, const u64* const x[2], const u64* W, u64* const out[2], u32 M, u32 N, u32 K,
                 const Epi& ep);

}  // namespace mpcg
