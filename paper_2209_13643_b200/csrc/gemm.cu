// Ring GEMM over Z_2^64 and the Beaver matmul combine.
//
// The combine of a matmul triple (H/protocols/beaver.hpp:175-180) is evaluated as ONE
// multi-segment GEMM per party, exact in Z_2^64 by distributivity:
//   party 1: z = +r_C + E*r_B + r_A*F
//   party 0: z = -r_C + A*B + E*(b0 + F) + a0*F        (A*B is the dealer's C = A*B)
// with E, F the opened eps/delta. The epilogue fuses the 2PC truncation, the bias and
// the conv col2im scatter (H/engine/executor.hpp:110-136,319-324).
#include "ew.cuh"
#include "gemm.cuh"

namespace mpcg {

namespace {

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(256) ring_gemm_simt(GemmArgs a) {
  constexpr int BK = 16, TX = BN / TN, TY = BM / TM;
  static_assert(TX * TY == 256, "256 threads");
  __shared__ u64 As[BK][BM + 1];
  __shared__ u64 Bs[BK][BN + 1];
  pdl_enter();
  // blockIdx.z = (split * nbatch + b) * nslots + slot
  const int slot = blockIdx.z % a.nslots;
  const u32 zb = blockIdx.z / a.nslots;
  const u32 b = zb % a.nbatch, split = zb / a.nbatch;
  const GemmSlotArgs& S = a.sl[slot];
  const u32 M = a.M, N = a.N, K = a.K;
  const u32 m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  u64 acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0;
  // this block's slice [kb, ke) of the concatenated K' = nseg*K axis
  const u32 kb = a.ksplit > 1 ? split * a.kchunk : 0;
  const u32 ke = a.ksplit > 1 ? min(kb + a.kchunk, u32(S.nseg) * K) : u32(S.nseg) * K;

  for (int sg = 0; sg < S.nseg; ++sg) {
    const u32 sb = u32(sg) * K;
    if (sb + K <= kb || sb >= ke) continue;
    const u32 lo = kb > sb ? kb - sb : 0, hi = min(K, ke - sb);
    const u64 lb = u64(b) * S.sL[sg], rbb = u64(b) * S.sR[sg];
    for (u32 k0 = lo; k0 < hi; k0 += BK) {
      for (int e = threadIdx.x; e < BM * BK; e += 256) {
        const int kk = e % BK, mm = e / BK;
        u64 v = 0;
        if (m0 + mm < M && k0 + kk < hi) v = load_l(S, sg, lb + u64(m0 + mm) * K + k0 + kk);
        As[kk][mm] = v;
      }
      if (!a.tb) {
        for (int e = threadIdx.x; e < BN * BK; e += 256) {
          const int nn = e % BN, kk = e / BN;
          u64 v = 0;
          if (k0 + kk < hi && n0 + nn < N) v = load_r(S, sg, rbb + u64(k0 + kk) * N + n0 + nn);
          Bs[kk][nn] = v;
        }
      } else {
        for (int e = threadIdx.x; e < BN * BK; e += 256) {
          const int kk = e % BK, nn = e / BK;
          u64 v = 0;
          if (k0 + kk < hi && n0 + nn < N) v = load_r(S, sg, rbb + u64(n0 + nn) * K + k0 + kk);
          Bs[kk][nn] = v;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        u64 ar[TM], br[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) ar[i] = As[kk][ty + i * TY];
#pragma unroll
        for (int j = 0; j < TN; ++j) br[j] = Bs[kk][tx + j * TX];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] += ar[i] * br[j];
      }
      __syncthreads();
    }
  }
  u64* accp = a.ksplit > 1 ? a.acc[slot] : nullptr;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const u32 m = m0 + ty + i * TY;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const u32 n = n0 + tx + j * TX;
      if (n >= N) continue;
      if (accp)  // this split's partial sum (summed mod 2^64 by the epilogue kernel)
        accp[u64(split) * a.nbatch * M * N + (u64(b) * M + m) * N + n] = acc[i][j];
      else
        gemm_epilogue(a, S, b, m, n, acc[i][j]);
    }
  }
}

}  // namespace
__global__ void __launch_bounds__(256) gemm_splitk_epilogue(GemmArgs a) {
  pdl_enter();
  const u64 per = u64(a.nbatch) * a.M * a.N;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < per * a.nslots; i += u64(gridDim.x) * blockDim.x) {
    const int slot = int(i / per);
    const u64 r = i - slot * per;
    const u32 n = u32(r % a.N), m = u32((r / a.N) % a.M), b = u32(r / (u64(a.N) * a.M));
    u64 v = 0;
    for (u32 sp = 0; sp < a.ksplit; ++sp) v += a.acc[slot][u64(sp) * per + r];
    gemm_epilogue(a, a.sl[slot], b, m, n, v);
  }
}
splitk_epilogue_t gemm_splitk_epilogue_fn() { return gemm_splitk_epilogue; }
namespace {

template <int BM, int BN, int TM, int TN>
void launch_simt(Session& s, GemmArgs a) {
  cudaStream_t st = s.stream;
  const u64 tiles = u64((a.N + BN - 1) / BN) * ((a.M + BM - 1) / BM) * a.nslots * a.nbatch;
  int maxseg = 0;
  for (int i = 0; i < a.nslots; ++i) maxseg = a.sl[i].nseg > maxseg ? a.sl[i].nseg : maxseg;
  const u32 kp = u32(maxseg) * a.K;
  // split K' until ~2 waves of CTAs exist, keeping >= 2 k-steps of 16 per split
  u32 split = 1;
  if (tiles < 2 * u64(num_sms())) {
    split = u32((2 * u64(num_sms()) + tiles - 1) / tiles);
    split = split > 16 ? 16 : split;  // the epilogue kernel sums the partials serially
    const u32 maxsplit = (kp + 31) / 32;
    split = split > maxsplit ? maxsplit : split;
    split = split < 1 ? 1 : split;
  }
  std::shared_ptr<Block> ws;
  if (split > 1) {
    a.ksplit = split;
    a.kchunk = ((kp + split - 1) / split + 15) / 16 * 16;
    a.ksplit = (kp + a.kchunk - 1) / a.kchunk;
    const u64 per = u64(a.nbatch) * a.M * a.N;  // one partial tile set per split, no zeroing pass
    ws = s.raw(per * a.ksplit * a.nslots);
    for (int i = 0; i < a.nslots; ++i) a.acc[i] = ws->ptr + i * per * a.ksplit;
  }
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, a.nslots * a.nbatch * a.ksplit);
  cudaEvent_t pe;
  probe_begin(st, &pe);
  launch_pdl(ring_gemm_simt<BM, BN, TM, TN>, grid, dim3(256), 0, st, a);
  if (a.ksplit > 1) {
    const u64 n = u64(a.nbatch) * a.M * a.N * a.nslots;
    launch_pdl(gemm_splitk_epilogue, dim3(ew_blocks(n)), dim3(256), 0, st, a);
  }
  probe_end(st, pe);
}

// ---------------------------------------------------------------- small-M (GEMV-shaped) path
// Dense heads at batch 1..16 (MLP, VGG fc6/fc7/fc8, LeNet fc): the combine streams the
// weight-side operands R_g[k][n] (dealer B / r_B draws and the opened F = own + peer delta)
// exactly once per (k, n) for ALL segments of a slot — party 0's three segments share one
// B / r_B draw and one F load — while the few L rows of a K-chunk are staged in shared
// memory. Bound by reading F (2 x 8 B per (k, n) per party) and the dealer draws.
constexpr int kGvMax = 16;  // the small-M path takes M <= kGvMax (M=64 x N=120 measured 6x slower than SIMT)
constexpr int kGvKC = 64;   // K chunk staged in smem (512 for M = 1 measured: -4% on VGG fc6, +20% on MLP)

template <int MR>
__global__ void __launch_bounds__(256) ring_gemv(GemmArgs a) {
  // block = 32 columns x 8 warps: lane = column (coalesced R reads), warp = K slice of every
  // staged chunk; the 8 warp partials are summed in shared memory at the end.
  __shared__ u64 Ls[3][MR][kGvKC];
  constexpr int kRG = MR < 4 ? MR : 4;  // rows reduced per pass
  __shared__ u64 red[8][kRG][32];
  pdl_enter();
  const int slot = int(blockIdx.z % a.nslots);
  const u32 m0 = (blockIdx.z / a.nslots) * MR;  // row group (M > MR: the R stream is re-read per group)
  const GemmSlotArgs& S = a.sl[slot];
  const u32 M = a.M, N = a.N, K = a.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 n = blockIdx.x * 32 + lane;
  const u32 kb = blockIdx.y * a.kchunk, ke = min(K, kb + a.kchunk);
  bool needB = false, needRB = false, needF = false;
  for (int g = 0; g < S.nseg; ++g) {
    const int rk = S.rk[g];
    needB |= rk == kOpB || rk == kOpB0F || rk == kOpBF;
    needRB |= rk == kOpRB || rk == kOpB0F;
    needF |= rk == kOpSum || rk == kOpB0F || rk == kOpBF || rk == kOpNegSum;
  }
  const u64* Fo = nullptr;
  const u64* Fp = nullptr;
  for (int g = 0; g < S.nseg; ++g)
    if (S.rk[g] == kOpSum || S.rk[g] == kOpB0F || S.rk[g] == kOpBF || S.rk[g] == kOpNegSum)
      Fo = S.R[g], Fp = S.R2[g];
  u64 acc[MR];
#pragma unroll
  for (int m = 0; m < MR; ++m) acc[m] = 0;
  for (u32 k0 = kb; k0 < ke; k0 += kGvKC) {
    const u32 kc = min(u32(kGvKC), ke - k0);
    __syncthreads();
    for (u32 e = threadIdx.x; e < u32(S.nseg) * MR * kGvKC; e += 256) {
      const u32 kk = e % kGvKC, m = (e / kGvKC) % MR, g = e / (kGvKC * MR);
      Ls[g][m][kk] = (m0 + m < M && kk < kc) ? load_l(S, int(g), u64(m0 + m) * K + k0 + kk) : 0;
    }
    __syncthreads();
    if (n >= N) continue;
    for (u32 kk = u32(warp); kk < kc; kk += 8) {
      const u64 idx = u64(k0 + kk) * N + n;
      const u64 B = needB ? mm_B(S.mm, S.boff + idx) : 0;
      const u64 rB = needRB ? mm_rB(S.mm, S.boff + idx) : 0;
      const u64 F = needF ? (Fp ? __ldg(Fo + idx) + __ldg(Fp + idx) : __ldg(Fo + idx)) : 0;
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        if (g >= S.nseg) break;
        u64 r;
        switch (S.rk[g]) {
          case kOpMem: r = __ldg(S.R[g] + idx); break;
          case kOpSum: r = F; break;
          case kOpB: r = B; break;
          case kOpB0F: r = (B - rB) + F; break;
          case kOpBF: r = B + F; break;
          case kOpNegSum: r = u64(0) - F; break;
          default: r = rB; break;
        }
#pragma unroll
        for (int m = 0; m < MR; ++m) acc[m] += Ls[g][m][kk] * r;
      }
    }
  }
  const u64 per = u64(M) * N;
#pragma unroll
  for (int mb = 0; mb < MR; mb += kRG) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRG; ++j) red[warp][j][lane] = acc[mb + j];
    __syncthreads();
    if (warp == 0 && n < N) {
#pragma unroll
      for (int j = 0; j < kRG; ++j) {
        u64 v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += red[w][j][lane];
        if (m0 + u32(mb + j) < M) a.acc[slot][u64(blockIdx.y) * per + u64(m0 + mb + j) * N + n] = v;
      }
    }
  }
}

// Pair-evaluated form (both party slots on this device, one dealer stream): one thread per
// column n evaluates BOTH slots' combines, so B and r_B are drawn and F is loaded once per
// (k, n) instead of per slot (2 draws + 8 B instead of 3 + 16 B; the per-slot blocks also ran
// a whole slot apart, so the second F read missed L2). Segment forms (beaver_combine):
//   party 0: A*B + E*((B - r_B) + F) + (A - r_A)*F,   party 1: E*r_B + r_A*F
// with the left values A, E, A - r_A, r_A of the staged K chunk in shared memory.
template <int MR>
__global__ void __launch_bounds__(256) ring_gemv_pair(GemmArgs a, int p0) {
  __shared__ u64 Ls[4][MR][kGvKC];  // A, E, A - r_A, r_A
  constexpr int kRG = MR < 4 ? MR : 4;
  __shared__ u64 red[8][kRG][32];
  pdl_enter();
  const GemmSlotArgs& S0 = a.sl[p0];
  const GemmSlotArgs& S1 = a.sl[1 - p0];
  const u32 m0 = blockIdx.z * MR;
  const u32 M = a.M, N = a.N, K = a.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 n = blockIdx.x * 32 + lane;
  const u32 kb = blockIdx.y * a.kchunk, ke = min(K, kb + a.kchunk);
  const u64* const Fo = S0.R[1];
  const u64* const Fp = S0.R2[1];
  u64 acc0[MR], acc1[MR];
#pragma unroll
  for (int m = 0; m < MR; ++m) acc0[m] = acc1[m] = 0;
  for (u32 k0 = kb; k0 < ke; k0 += kGvKC) {
    const u32 kc = min(u32(kGvKC), ke - k0);
    __syncthreads();
    for (u32 e = threadIdx.x; e < 4u * MR * kGvKC; e += 256) {
      const u32 kk = e % kGvKC, m = (e / kGvKC) % MR, g = e / (kGvKC * MR);
      u64 v = 0;
      if (m0 + m < M && kk < kc) {
        const u64 idx = u64(m0 + m) * K + k0 + kk;
        v = g == 3 ? load_l(S1, 1, idx) : load_l(S0, int(g), idx);
      }
      Ls[g][m][kk] = v;
    }
    __syncthreads();
    if (n >= N) continue;
    for (u32 kk = u32(warp); kk < kc; kk += 8) {
      const u64 idx = u64(k0 + kk) * N + n;
      const u64 B = mm_B(S0.mm, S0.boff + idx), rB = mm_rB(S0.mm, S0.boff + idx);
      const u64 F = Fp ? __ldg(Fo + idx) + __ldg(Fp + idx) - (a.fdefer ? B : 0) : __ldg(Fo + idx);
      const u64 b0F = (B - rB) + F;
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        const u64 e = Ls[1][m][kk];
        acc0[m] += Ls[0][m][kk] * B + e * b0F + Ls[2][m][kk] * F;
        acc1[m] += e * rB + Ls[3][m][kk] * F;
      }
    }
  }
  const u64 per = u64(M) * N;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const u64* acc = q == 0 ? acc0 : acc1;
    u64* const dst = a.acc[q == 0 ? p0 : 1 - p0];
#pragma unroll
    for (int mb = 0; mb < MR; mb += kRG) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kRG; ++j) red[warp][j][lane] = acc[mb + j];
      __syncthreads();
      if (warp == 0 && n < N) {
#pragma unroll
        for (int j = 0; j < kRG; ++j) {
          u64 v = 0;
#pragma unroll
          for (int w = 0; w < 8; ++w) v += red[w][j][lane];
          if (m0 + u32(mb + j) < M) dst[u64(blockIdx.y) * per + u64(m0 + mb + j) * N + n] = v;
        }
      }
    }
  }
}

// The pair-evaluated combine pattern of beaver_combine's non-tensor-core form on one dealer
// stream: party 0's slot [A*B, E*(b0+F), a0*F], party 1's [E*r_B, r_A*F]; returns party 0's
// slot or -1 (then the per-slot kernel runs).
bool gemv_pair_on() {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_GEMV_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

int gemv_pair_pattern(const GemmArgs& a) {
  if (!gemv_pair_on() || !pair_eval_enabled() || a.nslots != 2 || a.nbatch != 1) return -1;
  int p0 = -1;
  for (int i = 0; i < 2; ++i)
    if (a.sl[i].nseg == 3) p0 = i;
  if (p0 < 0 || a.sl[1 - p0].nseg != 2) return -1;
  const GemmSlotArgs& S0 = a.sl[p0];
  const GemmSlotArgs& S1 = a.sl[1 - p0];
  const int ek = S0.lk[1];
  if ((ek != kOpMem && ek != kOpSum) || S1.lk[0] != ek) return -1;
  if (S0.lk[0] != kOpA || S0.lk[2] != kOpA0 || S1.lk[1] != kOpRA) return -1;
  if (S0.rk[0] != kOpB || S0.rk[1] != kOpB0F || S0.rk[2] != kOpSum || S1.rk[0] != kOpRB || S1.rk[1] != kOpSum)
    return -1;
  // one opened E and one opened F for both slots (as (own, peer) of either slot)
  auto same = [](const u64* x0, const u64* x1, const u64* y0, const u64* y1) {
    return (x0 == y0 && x1 == y1) || (x1 && x0 == y1 && x1 == y0);
  };
  if (!same(S0.L[1], S0.L2[1], S1.L[0], S1.L2[0])) return -1;
  if (S0.R[1] != S0.R[2] || S0.R2[1] != S0.R2[2] || !same(S0.R[1], S0.R2[1], S1.R[1], S1.R2[1])) return -1;
  if (S0.aoff != S1.aoff || S0.boff != S1.boff || S0.sL[0] != S1.sL[0]) return -1;
  if (S0.mm.key != S1.mm.key || S0.mm.kp != S1.mm.kp || S0.mm.pool != S1.mm.pool || S0.mm.pA != S1.mm.pA ||
      S0.mm.prA != S1.mm.prA || S0.mm.pB != S1.mm.pB || S0.mm.prB != S1.mm.prB)
    return -1;
  return p0;
}

template <int MR>
void launch_gemv(Session& s, GemmArgs a) {
  cudaStream_t st = s.stream;
  const u32 ncol = (a.N + 31) / 32;
  const u32 mgrp = (a.M + MR - 1) / MR;
  // split K until ~16 blocks per SM (two full waves of 8 resident 256-thread blocks: the
  // per-(k, n) dealer draws are latency-bound chains, so the kernel needs every warp slot;
  // VGG fc6 1 x 25088 x 4096: 1.61 ms at ~3 blocks per SM), >= one staged chunk per split
  const int p0 = gemv_pair_pattern(a);
  const u64 base = u64(ncol) * (p0 >= 0 ? 1 : a.nslots) * mgrp;
  u32 split = u32((16 * u64(num_sms()) + base - 1) / base);
  const u32 maxsplit = (a.K + kGvKC - 1) / kGvKC;
  split = split > maxsplit ? maxsplit : (split < 1 ? 1 : split);
  a.kchunk = ((a.K + split - 1) / split + kGvKC - 1) / kGvKC * kGvKC;
  a.ksplit = (a.K + a.kchunk - 1) / a.kchunk;
  const u64 per = u64(a.M) * a.N;
  std::shared_ptr<Block> ws = s.raw(per * a.ksplit * a.nslots);
  for (int i = 0; i < a.nslots; ++i) a.acc[i] = ws->ptr + i * per * a.ksplit;
  cudaEvent_t pe;
  probe_begin(st, &pe);
  if (p0 >= 0)
    launch_pdl(ring_gemv_pair<MR>, dim3(ncol, a.ksplit, mgrp), dim3(256), 0, st, a, p0);
  else
    launch_pdl(ring_gemv<MR>, dim3(ncol, a.ksplit, a.nslots * mgrp), dim3(256), 0, st, a);
  launch_pdl(gemm_splitk_epilogue, dim3(ew_blocks(per * a.nslots)), dim3(256), 0, st, a);
  probe_end(st, pe);
}

// ---------------------------------------------------------------- skinny-N (row) path
// Convolutions with few output channels (LeNet conv0: M=50176, K=25, N=6): one thread owns
// one output row of one slot and streams its left-operand rows (every segment), while the
// right operand of a K chunk (nseg x KC x N words) is staged in shared memory. The tiled SIMT
// kernel wastes its BN-wide tile and syncs every 16 K; this one is bound by reading L.
constexpr int kRowN = 8;    // max N
constexpr int kRowKC = 64;  // K chunk of R staged in smem

template <int NR>
__global__ void __launch_bounds__(256) ring_gemm_rows(GemmArgs a) {
  __shared__ u64 Rs[3][kRowKC][NR];
  pdl_enter();
  const int slot = int(blockIdx.x % a.nslots);  // both slots of a row block co-scheduled (shared E in L2)
  const GemmSlotArgs& S = a.sl[slot];
  const u32 M = a.M, N = a.N, K = a.K;
  const u32 m = (blockIdx.x / a.nslots) * 256 + threadIdx.x;
  u64 acc[NR];
#pragma unroll
  for (int n = 0; n < NR; ++n) acc[n] = 0;
  for (u32 k0 = 0; k0 < K; k0 += kRowKC) {
    const u32 kc = min(u32(kRowKC), K - k0);
    __syncthreads();
    for (u32 e = threadIdx.x; e < u32(S.nseg) * kRowKC * NR; e += 256) {
      const u32 n = e % NR, kk = (e / NR) % kRowKC, g = e / (NR * kRowKC);
      Rs[g][kk][n] = (n < N && kk < kc) ? load_r(S, int(g), u64(k0 + kk) * N + n) : 0;
    }
    __syncthreads();
    if (m >= M) continue;
    for (int g = 0; g < S.nseg; ++g) {
      const u64 rowbase = u64(m) * K + k0;
      const int kind = S.lk[g];
      u32 kk = 0;
      if (kind == kOpMem || kind == kOpSum) {  // 8 independent loads in flight per thread
        const u64* p = S.L[g] + rowbase;
        const u64* p2 = S.L2[g] + rowbase;
        for (; kk + 8 <= kc; kk += 8) {
          u64 v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = __ldg(p + kk + i);
          if (kind == kOpSum) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += __ldg(p2 + kk + i);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int n = 0; n < NR; ++n) acc[n] += v[i] * Rs[g][kk + i][n];
        }
      }
      if (kind == kOpA || kind == kOpRA || kind == kOpA0) {  // dealer draws: counters advance by phi
        const u64 key = tkey(S.mm.key, S.mm.kp);
        const u64 e0 = S.aoff + rowbase + kk;
        u64 z = key + (kind == kOpRA ? S.mm.prA : S.mm.pA) + e0 * kPhi, z2 = key + S.mm.prA + e0 * kPhi;
        const u64* pool = S.mm.pool;
        for (; kk < kc; ++kk, z += kPhi, z2 += kPhi) {
          u64 v = pool ? pool_at(pool, z, key) : mix64(z);
          if (kind == kOpA0) v -= pool ? pool_at(pool, z2, key) : mix64(z2);
#pragma unroll
          for (int n = 0; n < NR; ++n) acc[n] += v * Rs[g][kk][n];
        }
      }
      for (; kk < kc; ++kk) {
        const u64 v = load_l(S, g, rowbase + kk);
#pragma unroll
        for (int n = 0; n < NR; ++n) acc[n] += v * Rs[g][kk][n];
      }
    }
  }
  if (m >= M) return;
#pragma unroll
  for (int n = 0; n < NR; ++n)
    if (u32(n) < N) gemm_epilogue(a, S, 0, m, u32(n), acc[n]);
}

}  // namespace

static bool rows_eligible(const GemmArgs& a) { return a.N <= u32(kRowN) && a.M >= 1024 && a.nbatch == 1 && !a.tb; }

bool gemv_eligible_shape(u32 M, u32 nbatch, bool tb, int col2im) {
  return M <= u32(kGvMax) && nbatch == 1 && !tb && !col2im;
}
static bool gemv_eligible(const GemmArgs& a) { return gemv_eligible_shape(a.M, a.nbatch, a.tb, a.col2im); }

void ring_gemm_launch(Session& s, const GemmArgs& a) {
  if (a.M == 0 || a.N == 0 || a.nbatch == 0) return;
  if (a.M > 65535u * 64u) throw Error(kShapeError, "ring_gemm: M too large");
  // algorithmic work: ring MACs of every segment of every slot
  double macs = 0;
  for (int i = 0; i < a.nslots; ++i) macs += double(a.sl[i].nseg) * a.M * a.N * a.K * a.nbatch;
  ClassScope cs(kClsGemm, macs);
  if (a.fdefer && !(gemv_eligible(a) && gemv_mode() != 0 && gemv_pair_pattern(a) >= 0))
    throw Error(kInternalError, "deferred delta: the pair-evaluated GEMV did not take the combine");
  if (gemv_eligible(a) && gemv_mode() != 0) {
    if (a.M <= 1) launch_gemv<1>(s, a);
    else if (a.M <= 4) launch_gemv<4>(s, a);
    else launch_gemv<16>(s, a);
    s.check();
    return;
  }
  if (rows_eligible(a) && gemv_mode() != 0) {  // skinny N: one thread per output row
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    const dim3 grid((a.M + 255) / 256 * a.nslots);  // accumulators sized to N (no padded columns)
    if (a.N <= 2)
      launch_pdl(ring_gemm_rows<2>, grid, dim3(256), 0, s.stream, a);
    else if (a.N <= 4)
      launch_pdl(ring_gemm_rows<4>, grid, dim3(256), 0, s.stream, a);
    else if (a.N <= 6)
      launch_pdl(ring_gemm_rows<6>, grid, dim3(256), 0, s.stream, a);
    else
      launch_pdl(ring_gemm_rows<kRowN>, grid, dim3(256), 0, s.stream, a);
    probe_end(s.stream, pe);
    s.check();
    return;
  }
  if (ring_gemm_tc2_wants(a) && ring_gemm_tc3_try(s, a)) return;  // both slots per CTA (tcgen05)
  if (a.ed.mode) throw Error(kInternalError, "deferred eps: the both-slots GEMM did not take the combine");
  if (ring_gemm_tc2_try(s, a)) return;  // warp-specialised tcgen05 int8-limb path
  if (a.M <= 16) {
    if (a.N <= 16)
      launch_simt<16, 16, 1, 1>(s, a);
    else
      launch_simt<16, 64, 1, 4>(s, a);
  } else if (a.N <= 8) {
    launch_simt<256, 8, 1, 8>(s, a);
  } else if (a.N <= 16) {
    launch_simt<256, 16, 2, 8>(s, a);
  } else if (a.N <= 32) {
    launch_simt<64, 32, 4, 2>(s, a);
  } else {
    launch_simt<64, 64, 4, 4>(s, a);
  }
  s.check();
}

// ---------------------------------------------------------------- matmul triple operands
namespace {
__device__ __forceinline__ u64 mm_b_share(const MmTriple& t, int party, u64 j) {
  const u64 rb = mm_rB(t, j);
  return party ? rb : mm_B(t, j) - rb;
}
}  // namespace

// own payload = y - b  (delta; H/engine/executor.hpp:283, H/protocols/beaver.hpp:194)
template <class YF>
static void delta_build(Session& s, const Triple& t, size_t nb, Open& o, YF yf) {
  const Pid2 pid = pids(s);
  const Ptr2 own = own_ptrs(o);
  const MmTriple mm = t.mm;
  if (o.summed) {  // fused in-device open: delta0 + delta1 = y0 + y1 - B (the r_B masks cancel)
    if (s.n_local != 2) throw Error(kUsageError, "summed delta open needs both slots");
    launch_ew(s.stream, 1, nb, [=] __device__(int, u64 j) { own.p[0][j] = yf(0, j) + yf(1, j) - mm_B(mm, j); });
    return;
  }
  launch_ew(s.stream, s.n_local, nb, [=] __device__(int slot, u64 j) {
    sel(own, slot)[j] = yf(slot, j) - mm_b_share(mm, pid.v[slot], j);
  });
}

void delta_build_mem(Session& s, const Triple& t, const u64* const y[2], size_t nb, Open& o) {
  delta_build(s, t, nb, o, SrcMem{CPtr2{{y[0], y[1]}}});
}

// own payload = x - a over A elements [a_off, a_off + na)  (eps; beaver.hpp:205,216)
// a-share of A element i; also emits the party's A-side GEMM operands into aop (if given):
// party 0 {A, a0 = A - r_A} at [j] and [na + j], party 1 {r_A} at [j]. The draws are the ones
// the eps payload needs anyway, so the combine GEMM reads them instead of redrawing.
__device__ __forceinline__ u64 a_share_out(const MmTriple& t, int party, u64 i, u64* aop, u64 j, u64 na) {
  const u64 key = tkey(t.key, t.kp), ip = i * kPhi;
  const u64 ra = dmix(key + t.prA + ip, key, t.pool);
  if (party) {
    if (aop) aop[j] = ra;
    return ra;
  }
  const u64 A = dmix(key + t.pA + ip, key, t.pool), a0 = A - ra;
  if (aop) {
    aop[j] = A;
    aop[na + j] = a0;
  }
  return a0;
}

void eps_build_mem(Session& s, const Triple& t, const u64* const x[2], size_t a_off, size_t na, Open& o,
                   const DT* aops) {
  const Pid2 pid = pids(s);
  const Ptr2 own = own_ptrs(o);
  const MmTriple mm = t.mm;
  const CPtr2 xp{{x[0], x[1]}};
  const Ptr2 ap{{aops ? aops->s[0] : nullptr, aops ? aops->s[1] : nullptr}};
  if (o.summed) {  // fused in-device open: both payloads, summed in registers
    if (s.n_local != 2 || aops) throw Error(kUsageError, "summed eps open needs both slots and no A operands");
    launch_ew(s.stream, 1, na, [=] __device__(int, u64 j) {  // eps0 + eps1 = x0 + x1 - A
      const u64 key = tkey(mm.key, mm.kp);
      own.p[0][j] = xp.p[0][a_off + j] + xp.p[1][a_off + j] - dmix(key + mm.pA + (a_off + j) * kPhi, key, mm.pool);
    });
    return;
  }
  launch_ew(s.stream, s.n_local, na, [=] __device__(int slot, u64 j) {
    sel(own, slot)[j] = sel(xp, slot)[a_off + j] - a_share_out(mm, pid.v[slot], a_off + j, sel(ap, slot), j, na);
  });
}

// im2col-fused eps build for conv layers (H/engine/executor.hpp:82-108): row=(n,oh,ow),
// col=(ci,ki,kj), padding taps read zero.
// One thread per im2col element (consecutive threads write consecutive words: fully
// coalesced payload stores), index decomposition by invariant-divisor multiplication instead of
// hardware-less 32-bit division, and, when both party slots are local, one r_A draw per element
// for both slots (party 0 also draws A), as the dealer does.
namespace {
struct EpsIm2colPair {
  MmTriple mm;
  Pid2 pid;
  Ptr2 own, ap;
  CPtr2 xp;
  ConvGeom g;
  FastDiv fKK, fk, fOW, fOH;
  u64 a_off, na;
  int nslots;
  int summed;  // fused in-device open: write own0 + own1 into own.p[0] only
  __device__ void operator()(u64 j) const {
    const u32 jj = u32(j);
    const u32 r = fKK.div(jj), c = jj - r * fKK.d;
    const u32 rq = fOW.div(r), ow = r - rq * g.OW;
    const u32 n = fOH.div(rq), oh = rq - n * g.OH;
    const u32 c1 = fk.div(c), kj = c - c1 * g.k;
    const u32 ci = fk.div(c1), ki = c1 - ci * g.k;
    const int ih = int(oh * g.stride + ki) - int(g.pad), iw = int(ow * g.stride + kj) - int(g.pad);
    const bool in = ih >= 0 && iw >= 0 && ih < int(g.H) && iw < int(g.W);
    const u64 src = ((u64(n) * g.C + ci) * g.H + u32(ih)) * g.W + u32(iw);
    const u64 key = tkey(mm.key, mm.kp);
    const u64 ip = (a_off + j) * kPhi;
    if (summed) {  // eps0 + eps1 = (x0 + x1) - (a0 + a1), a0 + a1 = A: the r_A masks cancel
      const u64 v = in ? xp.p[0][src] + xp.p[1][src] : 0;
      own.p[0][j] = v - dmix(key + mm.pA + ip, key, mm.pool);
      return;
    }
    const u64 ra = dmix(key + mm.prA + ip, key, mm.pool);
    u64 A = 0;
    bool haveA = false;
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      if (sl >= nslots) break;
      const u64 v = in ? xp.p[sl][src] : 0;
      u64 a;
      if (pid.v[sl] == 0) {
        if (!haveA) {
          A = dmix(key + mm.pA + ip, key, mm.pool);
          haveA = true;
        }
        a = A - ra;
        if (ap.p[sl]) {
          ap.p[sl][j] = A;
          ap.p[sl][na + j] = a;
        }
      } else {
        a = ra;
        if (ap.p[sl]) ap.p[sl][j] = ra;
      }
      own.p[sl][j] = v - a;
    }
  }
};
// Fused in-device open of the im2col eps (Open::summed): E[r][c] = x0[src] + x1[src] - A[r][c].
// A warp owns an im2col row r = (n, oh, ow) and walks its K = C*k*k columns 32 at a time; the
// column decomposition c -> (x offset, ki, kj) comes from a per-block shared table built once,
// so an element costs one table read, two gathers, one dealer draw (the counter advances by
// 32*phi per step) and a coalesced store — instead of five divisions per element.
__global__ void __launch_bounds__(256) eps_im2col_summed_kernel(MmTriple mm, ConvGeom g, const u64* __restrict__ x0,
                                                               const u64* __restrict__ x1, u64* __restrict__ out,
                                                               u32 rows, u64 a_off) {
  extern __shared__ int2 tab[];  // per column: {ci*H*W + ki*W + kj, ki | kj << 16}
  pdl_enter();
  const u32 K = g.C * g.k * g.k, kk = g.k * g.k;
  for (u32 c = threadIdx.x; c < K; c += blockDim.x) {
    const u32 ci = c / kk, rem = c - ci * kk, ki = rem / g.k, kj = rem - ki * g.k;
    tab[c] = make_int2(int(ci * g.H * g.W + ki * g.W + kj), int(ki | (kj << 16)));
  }
  __syncthreads();
  const u64 key = tkey(mm.key, mm.kp) + mm.pA;
  const u32 lane = threadIdx.x & 31;
  const u32 wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const u64 chw = u64(g.C) * g.H * g.W;
  for (u32 r = wg; r < rows; r += nw) {
    const u32 ow = r % g.OW, t = r / g.OW, oh = t % g.OH, n = t / g.OH;
    const int ih0 = int(oh * g.stride) - int(g.pad), iw0 = int(ow * g.stride) - int(g.pad);
    const long long xb = (long long)(u64(n) * chw) + (long long)ih0 * g.W + iw0;
    const u64 j0 = u64(r) * K;
    u64 z = key + (a_off + j0 + lane) * kPhi;
    for (u32 c = lane; c < K; c += 32, z += 32 * kPhi) {
      const int2 e = tab[c];
      const int ih = ih0 + (e.y & 0xFFFF), iw = iw0 + (e.y >> 16);
      u64 v = 0;
      if (unsigned(ih) < g.H && unsigned(iw) < g.W) {
        const long long src = xb + e.x;
        v = x0[src] + x1[src];
      }
      out[j0 + c] = v - dmix(z, key - mm.pA, mm.pool);  // eps0 + eps1 = x0 + x1 - (a0 + a1), a0 + a1 = A
    }
  }
}

// The same, tiled for input reuse: a block owns 8 consecutive output columns (ow) of one
// output row (n, oh) — warp w the im2col row of ow0 + w — and stages, per chunk of cc input
// channels, the summed input window x0 + x1 (cc x k x (7*stride + k) words, zero padded) in
// shared memory once; every tap is then a shared-memory read instead of two gathers, so the
// kernel is bound by its coalesced E stores.
__global__ void __launch_bounds__(256) eps_im2col_tile_kernel(MmTriple mm, ConvGeom g, const u64* __restrict__ x0,
                                                             const u64* __restrict__ x1, u64* __restrict__ out,
                                                             u32 cc_max, FastDiv fkk, FastDiv fk, u32 rowid0) {
  extern __shared__ u64 sx[];
  pdl_enter();
  const u32 owt = (g.OW + 7) / 8;
  // rowid = n*OH + oh; this call covers rowids [rowid0, rowid0 + gridDim.x / owt) and writes
  // them from out[0] (a row-block chunk of the eps payload), drawing A at the global index
  const u32 bt = blockIdx.x % owt, rowid = rowid0 + blockIdx.x / owt;
  const u32 oh = rowid % g.OH, n = rowid / g.OH;
  const u32 ow0 = bt * 8, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u32 ow = ow0 + warp;
  const u32 K = g.C * g.k * g.k, kk = g.k * g.k;
  const u32 ww = 7 * g.stride + g.k;  // window width
  const int ih0 = int(oh * g.stride) - int(g.pad), iw0 = int(ow0 * g.stride) - int(g.pad);
  const u64 r = u64(rowid) * g.OW + ow;
  const u64 key = tkey(mm.key, mm.kp) + mm.pA;
  for (u32 c0 = 0; c0 < g.C; c0 += cc_max) {
    const u32 cc = min(cc_max, g.C - c0);
    __syncthreads();
    const u32 wn = cc * g.k * ww;
    for (u32 e = threadIdx.x; e < wn; e += blockDim.x) {
      const u32 cl = e / (g.k * ww), rem = e - cl * (g.k * ww), ki = rem / ww, wx = rem - ki * ww;
      const int ih = ih0 + int(ki), iw = iw0 + int(wx);
      u64 v = 0;
      if (unsigned(ih) < g.H && unsigned(iw) < g.W) {
        const u64 src = ((u64(n) * g.C + c0 + cl) * g.H + u32(ih)) * g.W + u32(iw);
        v = x0[src] + x1[src];
      }
      sx[e] = v;
    }
    __syncthreads();
    if (ow >= g.OW) continue;
    const u32 ncol = cc * kk;
    const u64 jb = r * K + u64(c0) * kk;
    const u64 ob = jb - u64(rowid0) * g.OW * K;
    u64 z = key + (jb + lane) * kPhi;
    for (u32 cl = lane; cl < ncol; cl += 32, z += 32 * kPhi) {
      const u32 ci = fkk.div(cl), t2 = cl - ci * kk, ki = fk.div(t2), kj = t2 - ki * g.k;
      const u64 v = sx[(ci * g.k + ki) * ww + warp * g.stride + kj];
      out[ob + cl] = v - dmix(z, key - mm.pA, mm.pool);  // eps0 + eps1 = x0 + x1 - (a0 + a1), a0 + a1 = A
    }
  }
}

template <class F>
__global__ void __launch_bounds__(256) strip_kernel(u64 n, F f) {
  pdl_enter();
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) f(i);
}
}  // namespace

static bool tile_eps_enabled() {  // MPCG_EPS_TILE=0: the warp-per-row gather kernel instead
  static const bool on = [] {
    const char* e = std::getenv("MPCG_EPS_TILE");
    return !(e && e[0] == '0');
  }();
  return on;
}

void eps_build_im2col(Session& s, const Triple& t, const u64* const x[2], const ConvGeom& gm, size_t a_off,
                      size_t na, Open& o, const DT* aops) {
  const u32 Kc = gm.C * gm.k * gm.k;
  const u32 ww = 7 * gm.stride + gm.k;
  const u32 cc_max = u32((48 * 1024) / (8 * gm.k * ww));
  const u64 row_words = u64(gm.OW) * Kc;  // one (n, oh) output row of the im2col matrix
  if (o.summed && s.n_local == 2 && !aops && a_off % row_words == 0 && na % row_words == 0 && cc_max >= 1 &&
      tile_eps_enabled()) {
    const u32 cc = cc_max < gm.C ? cc_max : gm.C;
    const size_t smem = size_t(cc) * gm.k * ww * 8;
    const u64 blocks = u64(na / row_words) * ((gm.OW + 7) / 8);
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    launch_pdl(eps_im2col_tile_kernel, dim3(unsigned(blocks)), dim3(256), smem, s.stream, t.mm, gm, x[0], x[1],
               o.own(0), cc, FastDiv(gm.k * gm.k), FastDiv(gm.k), u32(a_off / row_words));
    probe_end(s.stream, pe);
    return;
  }
  if (o.summed && s.n_local == 2 && !aops && a_off % Kc == 0 && na % Kc == 0 && Kc * sizeof(int2) <= 96 * 1024) {
    const u32 rows = u32(na / Kc);
    const size_t smem = Kc * sizeof(int2);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      MPCG_CUDA(cudaFuncSetAttribute(eps_im2col_summed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr = smem;
    }
    u64 blocks = (u64(rows) + 7) / 8;
    const u64 cap = u64(num_sms()) * 8;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    launch_pdl(eps_im2col_summed_kernel, dim3(unsigned(blocks)), dim3(256), smem, s.stream, t.mm, gm, x[0], x[1],
               o.own(0), rows, u64(a_off));
    probe_end(s.stream, pe);
    return;
  }
  if (a_off == 0 && na < (u64(1) << 32)) {  // call-local indices fit the 32-bit fast division
    EpsIm2colPair f{t.mm, pids(s), own_ptrs(o),
                    Ptr2{{aops ? aops->s[0] : nullptr, aops && s.n_local == 2 ? aops->s[1] : nullptr}},
                    CPtr2{{x[0], s.n_local == 2 ? x[1] : nullptr}}, gm, FastDiv(gm.C * gm.k * gm.k), FastDiv(gm.k),
                    FastDiv(gm.OW), FastDiv(gm.OH), a_off, na, s.n_local, o.summed ? 1 : 0};
    if (o.summed && (s.n_local != 2 || aops))
      throw Error(kUsageError, "summed eps open needs both slots and no A operands");
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    launch_pdl(strip_kernel<EpsIm2colPair>, dim3(ew_blocks(na)), dim3(256), 0, s.stream, u64(na), f);
    probe_end(s.stream, pe);
    return;
  }
  const Pid2 pid = pids(s);
  const Ptr2 own = own_ptrs(o);
  const MmTriple mm = t.mm;
  const CPtr2 xp{{x[0], x[1]}};
  const ConvGeom g = gm;
  const Ptr2 ap{{aops ? aops->s[0] : nullptr, aops ? aops->s[1] : nullptr}};
  if (o.summed) throw Error(kUsageError, "summed eps open: call-local im2col indices must fit 32 bits");
  launch_ew(s.stream, s.n_local, na, [=] __device__(int slot, u64 j) {
    const u64 idx = a_off + j;
    const u32 KK = g.C * g.k * g.k;
    const u32 r = u32(idx) / KK, c = u32(idx) - r * KK;
    const u32 ow = r % g.OW, oh = (r / g.OW) % g.OH, n = r / (g.OW * g.OH);
    const u32 kj = c % g.k, ki = (c / g.k) % g.k, ci = c / (g.k * g.k);
    const int ih = int(oh * g.stride + ki) - int(g.pad), iw = int(ow * g.stride + kj) - int(g.pad);
    u64 v = 0;
    if (ih >= 0 && iw >= 0 && ih < int(g.H) && iw < int(g.W))
      v = sel(xp, slot)[((u64(n) * g.C + ci) * g.H + u32(ih)) * g.W + u32(iw)];
    sel(own, slot)[j] = v - a_share_out(mm, pid.v[slot], idx, sel(ap, slot), j, na);
  });
}

// The eps build also emits the A-side operands (A, a0 / r_A) only for combines that read them
// from memory (tiled SIMT and first-generation tcgen05); the small-M path, the skinny-N row
// path and the warp-specialised tcgen05 path draw them in place.
bool beaver_combine_wants_aops(const Session& s, u32 nbatch, u32 M, u32 N, u32 K) {
  GemmArgs a{};
  a.nslots = s.n_local;
  a.M = M;
  a.N = N;
  a.K = K;
  a.nbatch = nbatch;
  for (int i = 0; i < s.n_local; ++i) a.sl[i].nseg = s.party_of[i] == 0 ? 3 : 2;
  if (gemv_eligible_shape(M, nbatch, false, 0) && gemv_mode() != 0) return false;
  if (rows_eligible(a) && gemv_mode() != 0) return false;  // the row kernel draws A / r_A itself
  return !ring_gemm_tc2_wants(a);
}

// The eps open can be fused into its build (Open::summed) when both slots are local and the
// combine reads E as a GEMM operand (not through the A-operand path).
bool delta_defer(Session& s, Open& o, const u64* const w[2], u32 M, u32 N, u32 K) {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_DELTA_DEFER");
    return !(e && e[0] == '0');
  }();
  if (!on || !o.summed || s.n_local != 2 || s.cfg.link_bandwidth > 0 || !gemv_pair_on() || !pair_eval_enabled())
    return false;
  if (!(gemv_eligible_shape(M, 1, false, 0) && gemv_mode() != 0) || beaver_combine_wants_aops(s, 1, M, N, K))
    return false;
  o.defer.mode = 3;
  o.defer.x0 = w[0];
  o.defer.x1 = w[1];
  return true;
}

bool beaver_combine_fuses_eps(const Session& s, u32 nbatch, u32 M, u32 N, u32 K) {
  return eps_fuse_enabled() && s.n_local == 2 && !beaver_combine_wants_aops(s, nbatch, M, N, K);
}

void beaver_combine(Session& s, const Triple& t, const Open& e, size_t a_off, size_t na, const Open& d, size_t nb,
                    DT* rcache, u64* const out[2], size_t out_off, u32 nbatch, u32 M, u32 N, u32 K, bool tb,
                    bool batched_r, size_t r_batch0, const Epi& ep, const DT* aops) {
  GemmArgs a{};
  a.nslots = s.n_local;
  a.M = M;
  a.N = N;
  a.K = K;
  a.tb = tb;
  a.nbatch = nbatch;
  a.trunc_bits = ep.trunc_bits;
  a.col2im = ep.col2im;
  a.OHW = ep.OHW;
  a.row0 = ep.col2im ? u32(out_off / N) : 0;
  for (int i = 0; i < s.n_local; ++i) a.sl[i].nseg = s.party_of[i] == 0 ? 3 : 2;
  const u64 sL = u64(M) * K, sR = batched_r ? u64(K) * N : 0;
  const u64 rboff = batched_r ? r_batch0 * u64(K) * N : 0;
  const bool tc2 = !(gemv_eligible_shape(M, nbatch, tb, ep.col2im) && gemv_mode() != 0) && ring_gemm_tc2_wants(a);
  for (int i = 0; i < s.n_local; ++i) {
    GemmSlotArgs& S = a.sl[i];
    const u64* E0 = e.summed ? e.own(0) : e.own(i);
    const u64* E1 = e.summed ? nullptr : e.peer(i);
    const int ek = e.summed ? kOpMem : kOpSum;  // E = own + peer, or already summed
    const u64* F0 = (d.defer.mode == 3 ? d.defer.x0 : d.summed ? d.own(0) : d.own(i)) + rboff;
    const u64* F1 = d.defer.mode == 3 ? d.defer.x1 + rboff  // deferred: F = W0 + W1 - B in the GEMV
                    : d.summed ? nullptr : d.peer(i) + rboff;  // null: F summed at build time
    S.out = ep.col2im ? out[i] : out[i] + out_off;  // col2im scatters by global row (a.row0)
    S.addend = ep.addend[i] ? (ep.col2im ? ep.addend[i] : ep.addend[i] + out_off) : nullptr;
    S.bias = ep.bias[i];
    S.ckey = t.mm.key;
    S.ckp = t.mm.kp;
    S.cbase = 1 + 2 * t.mm.na + 2 * t.mm.nb + t.mm.offC + out_off;
    S.mm = t.mm;
    S.aoff = a_off;
    S.boff = rboff;
    const u64* ao = aops ? aops->s[i] : nullptr;  // A-side operands emitted by the eps build
    if (s.party_of[i] == 0 && !ao && tc2) {  // -r_C + A*(B + F) + E*(b0 + F) - r_A*F  (= a0*F split)
      S.cterm = -1;
      S.lk[0] = kOpA;
      S.rk[0] = kOpBF, S.R[0] = F0, S.R2[0] = F1;
      S.lk[1] = ek, S.L[1] = E0, S.L2[1] = E1;
      S.rk[1] = kOpB0F, S.R[1] = F0, S.R2[1] = F1;
      S.lk[2] = kOpRA;
      S.rk[2] = kOpNegSum, S.R[2] = F0, S.R2[2] = F1;
    } else if (s.party_of[i] == 0) {  // -r_C + A*B + E*(b0 + F) + a0*F
      S.cterm = -1;
      if (ao) S.lk[0] = kOpMem, S.L[0] = ao;
      else S.lk[0] = kOpA;
      S.rk[0] = kOpB;
      S.lk[1] = ek, S.L[1] = E0, S.L2[1] = E1;
      S.rk[1] = kOpB0F, S.R[1] = F0, S.R2[1] = F1;
      if (ao) S.lk[2] = kOpMem, S.L[2] = ao + na;
      else S.lk[2] = kOpA0;
      S.rk[2] = kOpSum, S.R[2] = F0, S.R2[2] = F1;
    } else {  // +r_C + E*r_B + r_A*F
      S.cterm = +1;
      S.lk[0] = ek, S.L[0] = E0, S.L2[0] = E1;
      S.rk[0] = kOpRB;
      if (ao) S.lk[1] = kOpMem, S.L[1] = ao;
      else S.lk[1] = kOpRA;
      S.rk[1] = kOpSum, S.R[1] = F0, S.R2[1] = F1;
    }
    for (int g = 0; g < 3; ++g) {
      S.sL[g] = sL;
      S.sR[g] = sR;
    }
  }
  if (d.defer.mode == 3) {  // F formed by the pair-evaluated GEMV (delta_defer)
    a.fdefer = 1;
    if (!(gemv_eligible(a) && gemv_mode() != 0 && gemv_pair_pattern(a) >= 0)) {  // not expected: build it
      Open o = d;
      o.defer = EpsDefer{};
      const u64* const w[2] = {d.defer.x0, d.defer.x1};
      delta_build_mem(s, t, w, nb, o);
      a.fdefer = 0;
      for (int i = 0; i < s.n_local; ++i)
        for (int g = 0; g < a.sl[i].nseg; ++g)
          if (a.sl[i].R2[g] == d.defer.x1 + rboff || a.sl[i].R2[g] == d.defer.x0 + rboff) {
            a.sl[i].R[g] = d.own(0) + rboff;
            a.sl[i].R2[g] = nullptr;
          }
    }
  }
  if (e.defer.mode) {  // E is generated by the both-slots GEMM's producers (eps_defer)
    a.ed = e.defer;
    if (!ring_gemm_tc3_accepts(s, a)) {  // not expected: build the opened value after all
      Open o = e;
      o.defer = EpsDefer{};
      const u64* const x[2] = {e.defer.x0, e.defer.x1};
      if (e.defer.mode == 2) eps_build_im2col(s, t, x, e.defer.g, a_off, na, o);
      else eps_build_mem(s, t, x, a_off, na, o);
      a.ed = EpsDefer{};
    }
  }
  ring_gemm_launch(s, a);
}

// Public-weight product x2d * W (H/engine/executor.hpp:294-298): one segment, no triple.
void public_gemm(Session& s, const u64* const x[2], const u64* W, u64* const out[2], u32 M, u32 N, u32 K,
                 const Epi& ep) {
  GemmArgs a{};
  a.nslots = s.n_local;
  a.M = M;
  a.N = N;
  a.K = K;
  a.nbatch = 1;
  a.trunc_bits = ep.trunc_bits;
  a.col2im = ep.col2im;
  a.OHW = ep.OHW;
  for (int i = 0; i < s.n_local; ++i) {
    GemmSlotArgs& S = a.sl[i];
    S.nseg = 1;
    S.L[0] = x[i];
    S.R[0] = W;
    S.out = out[i];
    S.addend = ep.addend[i];
    S.bias = ep.bias[i];
  }
  ring_gemm_launch(s, a);
}

// ---------------------------------------------------------------- beaver_matmul
DT beaver_matmul(Session& s, const DT& x, const DT& y, bool transpose_b, const std::string& tag, int chunks) {
  if (x.shape.size() < 2 || y.shape.size() < 2) throw Error(kShapeError, "matmul: operands must have rank >= 2");
  const bool batched_b = y.shape.size() > 2;
  Triple t = s.fetch(TripleSpec::matmul_of(x.shape, y.shape, transpose_b), tag, batched_b);
  t.mark_consumed();
  const size_t M = x.shape[x.shape.size() - 2], K = x.shape.back();
  const size_t N = transpose_b ? y.shape[y.shape.size() - 2] : y.shape.back();
  const size_t nb = y.numel(), na = x.numel();
  const size_t batch = na / (M * K);
  if (batched_b && nb / (K * N) != batch) throw Error(kShapeError, "matmul: batch mismatch");

  Open hd = s.begin_open(nb, Reduce::Sum);
  delta_build_mem(s, t, y.s, nb, hd);
  s.post(hd, tag + ".delta");

  const size_t rows = batched_b ? batch : na / K;
  const size_t row_w = batched_b ? M * K : K;
  chunks = clamp_chunks(chunks, rows);
  std::vector<Open> he(static_cast<size_t>(chunks));
  std::vector<DT> aops(static_cast<size_t>(chunks));
  for (int k = 0; k < chunks; ++k) {
    const auto r = chunk_range(rows, chunks, k);
    const size_t cnt = r.second - r.first;
    he[k] = s.begin_open(cnt * row_w, Reduce::Sum);
    const bool want = batched_b ? beaver_combine_wants_aops(s, u32(cnt), u32(M), u32(N), u32(K))
                                : beaver_combine_wants_aops(s, 1, u32(cnt), u32(N), u32(K));
    if (want) aops[k] = s.alloc(Shape{2, cnt * row_w});  // A-side combine operands from the eps draws
    else
      he[k].summed = batched_b ? beaver_combine_fuses_eps(s, u32(cnt), u32(M), u32(N), u32(K))
                               : beaver_combine_fuses_eps(s, 1, u32(cnt), u32(N), u32(K));
    if (want || batched_b || !eps_defer(s, he[k], x.s, nullptr, r.first * row_w, u32(cnt), u32(N), u32(K)))
      eps_build_mem(s, t, x.s, r.first * row_w, cnt * row_w, he[k], want ? &aops[k] : nullptr);
    s.post(he[k], chunks == 1 ? tag + ".eps" : tag + ".eps.chunk" + std::to_string(k));
  }
  s.wait(hd);
  DT rcache;
  Shape out_shape(x.shape.begin(), x.shape.end() - 1);
  out_shape.push_back(N);
  DT z = s.alloc(out_shape, x.scale);
  const size_t out_row_w = batched_b ? M * N : N;
  for (int k = 0; k < chunks; ++k) {
    const auto r = chunk_range(rows, chunks, k);
    const size_t cnt = r.second - r.first;
    s.wait(he[k]);
    Epi ep{};
    if (batched_b)
      beaver_combine(s, t, he[k], r.first * row_w, cnt * row_w, hd, nb, &rcache, z.s, r.first * out_row_w,
                     u32(cnt), u32(M), u32(N), u32(K), transpose_b, true, r.first, ep, aops[k] ? &aops[k] : nullptr);
    else
      beaver_combine(s, t, he[k], r.first * row_w, cnt * row_w, hd, nb, &rcache, z.s, r.first * out_row_w, 1,
                     u32(cnt), u32(N), u32(K), transpose_b, false, 0, ep, aops[k] ? &aops[k] : nullptr);
  }
  s.check();
  return z;
}

}  // namespace mpcg
