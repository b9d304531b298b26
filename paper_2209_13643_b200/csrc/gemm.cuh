// Ring GEMM interfaces (gemm.cu SIMT path, gemm_tc.cu tcgen05 int8-limb path).
#pragma once

#include "core.hpp"

namespace mpcg {

// One party slot of a multi-segment ring GEMM: out = epi( sum_g L_g * R_g ).
struct GemmSlotArgs {
  int nseg = 0;
  const u64* L[3] = {};   // [batch][M][K], batch stride sL (0 = shared)
  const u64* R[3] = {};   // [batch][K][N] or, transposed, [batch][N][K]; stride sR
  u64 sL[3] = {}, sR[3] = {};
  u64* out = nullptr;
  const u64* bias = nullptr;  // [N], added after truncation
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
  // split-K over the concatenated K' = nseg*K axis: partial sums are added mod 2^64 into
  // acc[slot] ([nbatch][M][N], zeroed) and a second kernel applies the epilogue.
  u32 ksplit = 1, kchunk = 0;
  u64* acc[2] = {nullptr, nullptr};
  int vec16 = 0;  // every L (and transposed R) row start is 16-byte aligned (K even, bases aligned)
};

struct Epi {
  int trunc_bits = 0;
  const u64* bias[2] = {nullptr, nullptr};
  int col2im = 0;
  u32 OHW = 1;
};

struct ConvGeom {
  u32 N, C, H, W, k, stride, pad, OH, OW;
};

__device__ __forceinline__ void gemm_epilogue(const GemmArgs& a, const GemmSlotArgs& S, u32 b, u32 m, u32 n,
                                              u64 v) {
  const u64 lin = (u64(b) * a.M + m) * a.N + n;
  if (S.cterm) {
    const u64 rc = drw(tkey(S.ckey, S.ckp), S.cbase + lin);
    v = S.cterm > 0 ? v + rc : v - rc;
  }
  if (a.trunc_bits) v = sar64(v, a.trunc_bits);
  if (S.bias) v += S.bias[n];
  if (a.col2im) {
    const u32 img = m / a.OHW, rem = m - img * a.OHW;
    S.out[(u64(img) * a.N + n) * a.OHW + rem] = v;
  } else {
    S.out[lin] = v;
  }
}

void ring_gemm_launch(Session& s, const GemmArgs& a);
bool ring_gemm_tc_try(Session& s, const GemmArgs& a);

void delta_build_mem(Session& s, const Triple& t, const u64* const y[2], size_t nb, Open& o);
void eps_build_mem(Session& s, const Triple& t, const u64* const x[2], size_t a_off, size_t na, Open& o);
void eps_build_im2col(Session& s, const Triple& t, const u64* const x[2], const ConvGeom& g, size_t a_off,
                      size_t na, Open& o);
DT prepare_R(Session& s, const Triple& t, const Open& d, size_t nb);
DT prepare_L(Session& s, const Triple& t, const Open& e, size_t a_off, size_t na);
void mm_combine(Session& s, const Triple& t, const DT& L, size_t na, const DT& R, size_t nb, u64* const out[2],
                size_t out_off, u32 nbatch, u32 M, u32 N, u32 K, bool tb, bool batched_r, size_t r_batch0,
                const Epi& ep);
void public_gemm(Session& s, const u64* const x[2], const u64* W, u64* const out[2], u32 M, u32 N, u32 K,
                 const Epi& ep);

}  // namespace mpcg
