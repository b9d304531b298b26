// tcgen05 int8-limb ring GEMM over Z_2^64, warp-specialised (sm_100a).
//
// u64 operands split into 8 u8 limbs; the 36 limb pairs with
// l+m <= 7 run as tcgen05.mma.kind::i8 into 8 s32 TMEM accumulators, one per diagonal
// d = l+m; the epilogue recombines z = sum_d D_d << 8d mod 2^64 — the int8 form of
// LimbPlan/limb_matmul, H/ring/limb.hpp:15-99), restructured as a Blackwell pipeline:
//
//   warps 0-15 L producers: generate the left operand of every segment straight from its
//              source — the opened E = own + peer eps (two vector loads) or the dealer's
//              A / r_A draws (counter PRG, H/sharing/triple.hpp:96-114) — byte-transpose it
//              into K-major limb planes and publish the stage with an mbarrier arrive;
//   warp 16    bulk loader: the right operands (weight side, packed once per layer into the
//              exact shared-memory image of a stage) arrive by cp.async.bulk (TMA engine)
//              on the same mbarrier with expect_tx;
//   warp 17    MMA issuer (one thread): per stage, A plane l against the B planes 0..7-l
//              stacked along N (the packed B image interleaves the planes per K chunk) — 8
//              MMAs of N = (8-l)*BN (split at 256), 12 for BN = 64 instead of 36 per-pair
//              MMAs, since the issue cost is per instruction; tcgen05.commit frees the stage;
//   warps 0-15 epilogue: tcgen05.ld of the 8 diagonals, recombination, Beaver epilogue.
//
// A 4-stage ring of 32-byte K slabs keeps HBM loads, PRG work and MMAs in flight together.
// When N spans several BN tiles the left operand is also packed once (pack kernel) and both
// sides arrive by cp.async.bulk, so the generation is not repeated per N tile.
// Exactness: per-diagonal sums over K' = nseg*K <= 16384 (see below).
#include "tc_common.cuh"

namespace mpcg {

namespace {

constexpr int kM = 128;        // tile rows (UMMA M)
#ifndef MPCG_TC2_STAGES
#define MPCG_TC2_STAGES 4
#endif
constexpr int kStages = MPCG_TC2_STAGES;
constexpr int kProdWarps = 16;                 // L producers (and epilogue): warps 0-15
constexpr int kLoadWarp = kProdWarps;          // bulk loader
constexpr int kMmaWarp = kProdWarps + 1;       // MMA issuer, TMEM owner
constexpr int kThreads = (kProdWarps + 2) * 32;
constexpr u32 kMaxKPrime = 16384;

}  // namespace

// Debug trace (MPCG_TC2_TRACE=1): stage timestamps of CTA (0,0,0) — MMA thread wait-for-full
// start/end + issue end, producer warps 0 (generated) and 8 (memory) empty-wait start/end and
// arrive — read back with mpcg_debug_tc2_trace. Off by default; no effect on values.
constexpr int kTraceStages = 256;
__device__ unsigned long long g_tc2_trace[kTraceStages][10];

struct Tc2Args {
  GemmArgs g;
  const char* Rpk[2] = {nullptr, nullptr};  // packed right operand per slot
  u64 Rpk_b[2] = {0, 0};                    // bytes per batch (0 = shared across the batch)
  const char* Lpk[2] = {nullptr, nullptr};  // packed left operand (multi-N-tile shapes) or null
  u64 Lpk_b[2] = {0, 0};
  u32 lmask[2] = {0, 0};  // segments whose left operand is in Lpk (all: fully packed; else hybrid)
  // packed-left image layout per slot: segments per K block in the image and this slot's first
  // segment in it (party 1 may read E and r_A from party 0's image: lnpk 3, lseg0 1)
  u32 lnpk[2] = {0, 0}, lseg0[2] = {0, 0};
  u32 nkb = 0;                              // K blocks of 32
  int vec = 0;                              // L row loads: 2 = 32-byte, 1 = 16-byte, 0 = scalar
  u32 ksplit = 1, kbper = 0;                // split-K over K blocks (partials summed by the epilogue kernel)
  u32 l2ahead = 3;                          // K blocks of L2 prefetch ahead of the register loads (0 = off)
  int trace = 0;
};

namespace {

// AT: the left operand's limb planes live in TMEM (4 stages x 8 planes x 8 columns after the
// 8*BN accumulator columns), written by the producers with tcgen05.st; each MMA then reads
// only its B plane from shared memory. Without it every MMA re-reads a 4 KB A plane and the
// 36-MMA stage is shared-memory-bandwidth bound (~51-70 cycles per M128xN64 MMA, measured)
// rather than tensor bound (32). Needs 8*BN + 256 <= 512 columns, i.e. BN = 32.
template <int BN, bool SPLIT, bool AT>
__global__ void __launch_bounds__(kThreads, 1) ring_gemm_tc2(const __grid_constant__ Tc2Args P) {
  constexpr u32 kA = AT ? 0 : kM * kKB;  // bytes per A limb plane per shared-memory stage
  constexpr u32 kB = BN * kKB;           // bytes per B limb plane per stage
  constexpr u32 kStage = 8 * (kA + kB);
  constexpr u32 kAcols = 8 * BN;
  constexpr u32 kCols = AT ? 512 : kAcols;
  static_assert(!AT || kAcols + kStages * 64 <= 512, "TMEM budget (A stages)");
  static_assert(kCols <= 512, "TMEM budget");
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) u64 full[kStages], empty[kStages], done;
  __shared__ u32 tmem_slot;

  pdl_enter();
  const GemmArgs& a = P.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // grid.x = (N tile, slot) with the slot fastest: the CTAs that read the same opened-E rows
  // (both party slots of an M tile, every N tile) are co-scheduled, so the rows come from L2.
  const int slot = int(blockIdx.x % a.nslots);
  const u32 ntile = blockIdx.x / a.nslots;
  const u32 b = blockIdx.z % a.nbatch;
  const u32 split = blockIdx.z / a.nbatch;
  const GemmSlotArgs& S = a.sl[slot];
  const u32 M = a.M, N = a.N, K = a.K;
  const u32 m0 = blockIdx.y * kM, n0 = ntile * BN;
  const int nseg = S.nseg;
  const u32 kb0 = split * P.kbper, kb1 = min(P.nkb, kb0 + P.kbper);  // this CTA's K blocks
  const u32 nst = (kb1 - kb0) * u32(nseg);
  // left operand: fully packed (every segment bulk-copied), hybrid (the dealer-drawn segments
  // packed once per layer, the memory segments loaded by the producers), or generated
  const u32 lm = P.Lpk[slot] ? P.lmask[slot] : 0u;
  const bool packedL = lm != 0 && lm == (1u << nseg) - 1;
  const u32 npk = __popc(lm);

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], packedL ? 1 : (SPLIT ? kProdWarps / 2 : kProdWarps) + 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = tmem_slot;

  if (SPLIT && warp < kProdWarps && !packedL) {
    // ---- split producers: warps 0-7 own the generated segments (dealer draws), warps 8-15
    // the memory segments (opened E); each unit is 16 K-consecutive values of one row, so a
    // stage is written by one group of 8 warps and the E loads of block kb+1 stay in flight
    // while the other group generates — the E group has nothing else to wait on.
    const int gt = tid & 255;             // thread within the group
    const bool egroup = warp >= kProdWarps / 2;
    const int r = gt & (kM - 1), hf = gt >> 7;
    const u32 m = m0 + u32(r);
    const bool rowok = m < M;
    const u64 rowoff = u64(b) * S.sL[0] + u64(m) * K;
    const u64 key = tkey(S.mm.key, S.mm.kp);
    const u64 iA = 1 + S.mm.offA + S.aoff;
    const u64 iRA = 1 + S.mm.na + S.mm.nb + S.mm.offA + S.aoff;
    const u32 off = (u32(hf) * (kM / 8) + u32(r) / 8) * 128 + (u32(r) % 8) * 16;
    u64 pr[16], pr2[16];
    // issue the loads of memory segment g for K block kb into pr/pr2 (E = own + peer)
    auto fetch = [&](int g, u32 kb) {
      const u32 k0 = kb * kKB + u32(hf) * 16;
      const bool sum = S.lk[g] == kOpSum;
      if (!rowok || k0 >= K) {
#pragma unroll
        for (int i = 0; i < 16; ++i) pr[i] = pr2[i] = 0;
      } else if (k0 + 16 <= K && P.vec) {
        // 256-bit loads where aligned: one L1 wavefront per 32-byte sector, not two
        if (P.vec == 2) load16w(S.L[g] + rowoff + k0, pr);
        else load16(S.L[g] + rowoff + k0, pr);
        if (!sum) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pr2[i] = 0;
        } else if (P.vec == 2) {
          load16w(S.L2[g] + rowoff + k0, pr2);
        } else {
          load16(S.L2[g] + rowoff + k0, pr2);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const bool in = k0 + i < K;
          pr[i] = in ? __ldg(S.L[g] + rowoff + k0 + i) : 0;
          pr2[i] = (in && sum) ? __ldg(S.L2[g] + rowoff + k0 + i) : 0;
        }
      }
    };
    // the memory segments this group serves, in stage order
    auto is_mem = [&](int g) { return S.lk[g] == kOpMem || S.lk[g] == kOpSum; };
    int firstmem = -1;
    for (int g = 0; g < nseg && firstmem < 0; ++g)
      if (is_mem(g)) firstmem = g;
    const bool tr = P.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 &&
                    (warp == 0 || warp == kProdWarps / 2);
    const int tcol = warp == 0 ? 3 : 6;
    auto publish = [&](const u64 (&v)[16], u32 it) {
      const int stg = int(it % kStages);
      if (tr && it < kTraceStages) g_tc2_trace[it][tcol] = clock64();
      if (it >= kStages) mbar_wait(&empty[stg], ((it / kStages) & 1) ^ 1);
      if (tr && it < kTraceStages) g_tc2_trace[it][tcol + 1] = clock64();
      if constexpr (AT) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        transpose16_tmem(v, tmem + ((u32(r) & ~31u) << 16) + kAcols + u32(stg) * 64 + u32(hf) * 4);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else {
        transpose16_store(v, smem + stg * kStage, kA, off);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[stg]);
      if (tr && it < kTraceStages) g_tc2_trace[it][tcol + 2] = clock64();
    };
    if (egroup) {  // memory segments: loads of the next one in flight while this one is published
      if (firstmem >= 0) fetch(firstmem, kb0);
      u32 it = 0;
      for (u32 kb = kb0; kb < kb1; ++kb)
        for (int g = 0; g < nseg; ++g, ++it) {
          if (!is_mem(g)) continue;
#pragma unroll
          for (int i = 0; i < 16; ++i) pr[i] += pr2[i];  // in place: E = own + peer
          publish(pr, it);
          int ng = -1;
          for (int h = g + 1; h < nseg && ng < 0; ++h)
            if (is_mem(h)) ng = h;
          if (ng >= 0) fetch(ng, kb);
          else if (kb + 1 < kb1) fetch(firstmem, kb + 1);
        }
    } else {  // generated segments: the dealer's A / r_A draws
      u32 it = 0;
      for (u32 kb = kb0; kb < kb1; ++kb) {
        const u32 k0 = kb * kKB + u32(hf) * 16;
        for (int g = 0; g < nseg; ++g, ++it) {
          if (is_mem(g)) continue;
          if ((lm >> g) & 1u) {  // hybrid: this stage's left operand is bulk-copied by the loader
            const int stg = int(it % kStages);
            if (it >= kStages) mbar_wait(&empty[stg], ((it / kStages) & 1) ^ 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[stg]);
            continue;
          }
          const int kind = S.lk[g];
          const u64 e0 = rowoff + k0;
          u64 v[16];
          if (!rowok || k0 >= K) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0;
          } else {
            draws16(key, (kind == kOpRA ? iRA : iA) + e0, v, S.mm.pool);
            if (kind == kOpA0) {
              u64 w[16];
              draws16(key, iRA + e0, w, S.mm.pool);
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] -= w[i];
            }
            if (k0 + 16 > K) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (k0 + i >= K) v[i] = 0;
            }
          }
          publish(v, it);
        }
      }
    }
  } else if (warp < kProdWarps) {
    if (!packedL) {
      // ---- L producers: unit = (row r, quarter q) = 8 K-consecutive values of one row per
      // stage; each becomes one 8-byte row segment in every limb plane.
      const int r = tid & (kM - 1), q = tid >> 7;
      const u32 m = m0 + u32(r);
      const bool rowok = m < M;
      const u64 rowoff = u64(b) * S.sL[0] + u64(m) * K;  // same stride for every segment
      const u64 key = tkey(S.mm.key, S.mm.kp);
      const u64 iA = 1 + S.mm.offA + S.aoff;                       // draw index of A[0]
      const u64 iRA = 1 + S.mm.na + S.mm.nb + S.mm.offA + S.aoff;  // of r_A[0]
      const u32 off = (u32(q >> 1) * (kM / 8) + u32(r) / 8) * 128 + (u32(r) % 8) * 16 + u32(q & 1) * 8;
      // The first memory segment (the opened E = own + peer, or a plain operand) is software-
      // pipelined one K block ahead: its loads for block kb+1 are issued as soon as block kb's
      // values are consumed, so they fly behind the next block's dealer draws and transposes.
      int pf = -1;
      for (int g = 0; g < nseg && pf < 0; ++g)
        if (S.lk[g] == kOpMem || S.lk[g] == kOpSum) pf = g;
      u64 pr[kVW], pr2[kVW];
      auto fetch = [&](u32 kb) {
        const u32 k0 = kb * kKB + u32(q) * kVW;
        const bool sum = S.lk[pf] == kOpSum;
        if (!rowok || kb >= kb1 || k0 >= K) {
#pragma unroll
          for (int i = 0; i < kVW; ++i) pr[i] = pr2[i] = 0;
        } else if (k0 + kVW <= K && P.vec) {
          if (P.vec == 2) {
            load_vecw(S.L[pf] + rowoff + k0, pr);
            if (sum) load_vecw(S.L2[pf] + rowoff + k0, pr2);
          } else {
            load_vec(S.L[pf] + rowoff + k0, pr);
            if (sum) load_vec(S.L2[pf] + rowoff + k0, pr2);
          }
        } else {
#pragma unroll
          for (int i = 0; i < kVW; ++i) {
            const bool in = k0 + i < K;
            pr[i] = in ? __ldg(S.L[pf] + rowoff + k0 + i) : 0;
            pr2[i] = (in && sum) ? __ldg(S.L2[pf] + rowoff + k0 + i) : 0;
          }
        }
        if (!sum) {
#pragma unroll
          for (int i = 0; i < kVW; ++i) pr2[i] = 0;
        }
        // deeper, register-free prefetch: pull block kb+kL2Ahead into L2 so that the register
        // load issued one block ahead finds it there (HBM latency > one block of producer work)
        const u32 kp = (kb + P.l2ahead) * kKB + u32(q) * kVW;
        if (P.l2ahead && rowok && kb + P.l2ahead < kb1 && kp < K) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(S.L[pf] + rowoff + kp));
          if (sum) asm volatile("prefetch.global.L2 [%0];" ::"l"(S.L2[pf] + rowoff + kp));
        }
      };
      if (pf >= 0) fetch(kb0);
      u32 it = 0;
      for (u32 kb = kb0; kb < kb1; ++kb) {
        const u32 k0 = kb * kKB + u32(q) * kVW;
        const bool fullv = rowok && k0 + kVW <= K;
        for (int g = 0; g < nseg; ++g, ++it) {
          const int stg = int(it % kStages);
          if ((lm >> g) & 1u) {  // hybrid: bulk-copied by the loader
            if (it >= kStages) mbar_wait(&empty[stg], ((it / kStages) & 1) ^ 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[stg]);
            continue;
          }
          u64 v[kVW];
          const int kind = S.lk[g];
          if (g == pf) {
#pragma unroll
            for (int i = 0; i < kVW; ++i) v[i] = pr[i] + pr2[i];
            fetch(kb + 1);
          } else if (!rowok || k0 >= K) {
#pragma unroll
            for (int i = 0; i < kVW; ++i) v[i] = 0;
          } else if (kind == kOpMem || kind == kOpSum) {
#pragma unroll
            for (int i = 0; i < kVW; ++i) {
              u64 x = 0;
              if (k0 + i < K) {
                x = __ldg(S.L[g] + rowoff + k0 + i);
                if (kind == kOpSum) x += __ldg(S.L2[g] + rowoff + k0 + i);
              }
              v[i] = x;
            }
          } else {  // dealer draws: A, r_A (party 0 splits a0*F as A*F - r_A*F), or a0 = A - r_A
            const u64 e0 = rowoff + k0;
            draws_vec(key, (kind == kOpRA ? iRA : iA) + e0, v, S.mm.pool);
            if (kind == kOpA0) {
              u64 w[kVW];
              draws_vec(key, iRA + e0, w, S.mm.pool);
#pragma unroll
              for (int i = 0; i < kVW; ++i) v[i] -= w[i];
            }
            if (!fullv) {
#pragma unroll
              for (int i = 0; i < kVW; ++i)
                if (k0 + i >= K) v[i] = 0;
            }
          }
          if (it >= kStages) mbar_wait(&empty[stg], ((it / kStages) & 1) ^ 1);
          if constexpr (AT) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            transpose8_tmem(v, tmem + ((u32(r) & ~31u) << 16) + kAcols + u32(stg) * 64 + u32(q) * 2);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          } else {
            transpose8_store(v, smem + stg * kStage, kA, off);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[stg]);
        }
      }
    }
  } else if (warp == kLoadWarp) {
    if (lane == 0) {  // ---- bulk loader
      const char* Rb = P.Rpk[slot] + u64(b) * P.Rpk_b[slot] +
                       (u64(ntile) * P.nkb + kb0) * u64(nseg) * 8 * kB;
      const char* Lb =
          lm ? P.Lpk[slot] + u64(b) * P.Lpk_b[slot] + (u64(blockIdx.y) * P.nkb + kb0) * u64(P.lnpk[slot]) * 8 * kA
             : nullptr;
      for (u32 it = 0; it < nst; ++it) {
        const int stg = int(it % kStages);
        if (it >= kStages) mbar_wait(&empty[stg], ((it / kStages) & 1) ^ 1);
        char* sA = smem + stg * kStage;
        const u32 g = it % u32(nseg), kr = it / u32(nseg);
        const bool pl = (lm >> g) & 1u;
        mbar_arrive_tx(&full[stg], 8 * kB + (pl ? 8 * kA : 0));
        bulk_g2s(sA + 8 * kA, Rb + u64(it) * 8 * kB, 8 * kB, &full[stg]);
        if (pl)
          bulk_g2s(sA, Lb + (u64(kr) * P.lnpk[slot] + P.lseg0[slot] + __popc(lm & ((1u << g) - 1))) * 8 * kA, 8 * kA,
                   &full[stg]);
      }
    }
  } else {
    if (lane == 0) {  // ---- MMA issuer
      for (u32 it = 0; it < nst; ++it) {
        const int stg = int(it % kStages);
        const bool tr = P.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && it < kTraceStages;
        if (tr) g_tc2_trace[it][0] = clock64();
        mbar_wait(&full[stg], (it / kStages) & 1);
        if (tr) g_tc2_trace[it][1] = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const u32 aBase = smem_u32(smem + stg * kStage), bBase = aBase + 8 * kA;
        // A plane l times B planes 0..7-l (stacked along N) -> diagonals l..7 (adjacent TMEM
        // column blocks): one MMA of N = (8-l)*BN, split at the 256-column MMA limit. Issue
        // cost is per instruction (~50 cycles measured for any N <= 64), so 12 wide MMAs
        // instead of 36 narrow ones leave the stage tensor-bound.
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const u32 acc = (it > 0 || l > 0) ? 1u : 0u;
#pragma unroll
          for (u32 c0 = 0; c0 < u32(8 - l) * BN; c0 += 256) {
            const u32 nn = min(256u, u32(8 - l) * BN - c0);
            const u64 bd = smem_desc(bBase + (c0 / 8) * 128, BN * 128, 128);
            const u32 dcol = tmem + u32(l) * BN + c0;
            if constexpr (AT)
              mma_i8_ts(dcol, tmem + kAcols + u32(stg) * 64 + u32(l) * 8, bd, idesc_i8(kM, nn), acc);
            else
              mma_i8(dcol, smem_desc(aBase + l * kA, (kM / 8) * 128, 128), bd, idesc_i8(kM, nn), acc);
          }
        }
        mma_commit(&empty[stg]);
        if (P.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && it < kTraceStages)
          g_tc2_trace[it][2] = clock64();
      }
      mma_commit(&done);
    }
  }

  // ---- epilogue (producer warps): warp w reads TMEM lanes 32*(w%4).. and column group w/4
  if (warp < kProdWarps) {
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    constexpr int kGrp = kProdWarps / 4;
    constexpr int kCW = BN / kGrp;  // columns per warp: 16 / 8 / 4 for BN = 64 / 32 / 16
    const int qd = warp & 3, cg = warp >> 2;
    const u32 row = u32(qd) * 32 + u32(lane);
    const u32 m = m0 + row;
    const u32 lane_addr = tmem + ((u32(qd) * 32) << 16) + u32(cg * kCW);
    u64 acc[kCW];
#pragma unroll
    for (int c = 0; c < kCW; ++c) acc[c] = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      u32 rr[kCW];
      tmem_ld<kCW>(lane_addr + u32(d) * BN, rr);
#pragma unroll
      for (int c = 0; c < kCW; ++c) acc[c] += u64(rr[c]) << (8 * d);
    }
    if (m < M) {
      u64* part = P.ksplit > 1 ? a.acc[slot] + u64(split) * a.nbatch * M * N : nullptr;
#pragma unroll
      for (int c = 0; c < kCW; ++c) {
        const u32 n = n0 + u32(cg * kCW + c);
        if (n < N) {
          if (part)
            part[(u64(b) * M + m) * N + n] = acc[c];
          else
            gemm_epilogue(a, S, b, m, n, acc[c]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}

// Packs one operand into the shared-memory image of every stage it feeds:
// [batch][row tile][K block][segment][limb plane][BR rows x 32 B], core matrices K-major
// (row group r/8, K chunk kc) at (kc*(BR/8) + r/8)*128, row r%8 at +16*(r%8).
// left: value = load_l(S, g, b*sL + row*K + k); right: load_r at (b*sR + k*N + row) or,
// transposed, (b*sR + row*K + k).
template <int BR>
__global__ void __launch_bounds__(256) pack_limbs(GemmArgs a, int left, u32 rows, u32 nbatch, u32 nkb, char* out0,
                                                  char* out1, u32 mask0, u32 mask1, int both) {
  pdl_enter();
  // every local slot in one launch: one slot per grid row, or (both: the pair combine's right
  // operand, one dealer stream and one F) both slots per thread, B / r_B drawn and F read once
  const int slot = both ? 0 : int(blockIdx.y);
  const GemmSlotArgs& S = a.sl[slot];
  const u32 K = a.K, N = a.N;
  const u32 tiles = (rows + BR - 1) / BR;
  // unit = 4 K-consecutive values of one row for EVERY packed segment of the slot: one 4-byte
  // word in each limb plane of each segment. The dealer draws (A, r_A / B, r_B) and the
  // opened F of a value are produced once and shared by the segments that use them
  // (the launcher guarantees one stride and one F for all segments).
  const u32 units = nbatch * tiles * nkb * BR * 8;
  constexpr u32 plane = BR * kKB;
  bool dA = false, dRA = false, dB = false, dRB = false, dF = false;
  int fseg = 0, fslot = slot;
  for (int sl = slot; sl < slot + (both ? 2 : 1); ++sl)
  for (u32 g = 0; g < u32(a.sl[sl].nseg); ++g) {
    if (!(((sl ? mask1 : mask0) >> g) & 1u)) continue;
    const int k = left ? a.sl[sl].lk[g] : a.sl[sl].rk[g];
    if (left) {
      dA |= k == kOpA || k == kOpA0;
      dRA |= k == kOpRA || k == kOpA0;
    } else {
      dB |= k == kOpB || k == kOpB0F || k == kOpBF;
      dRB |= k == kOpRB || k == kOpB0F;
      if (k == kOpSum || k == kOpB0F || k == kOpBF || k == kOpNegSum) dF = true, fseg = int(g), fslot = sl;
    }
  }
  // Unit order: when the source rows are K-contiguous (left operand, transposed right operand)
  // the 8 K-quarters of a row are the fastest index, so a warp reads 4 rows x 256 contiguous
  // bytes and writes whole 16-byte core-matrix rows; otherwise (right operand [K][N]) the row
  // index is fastest, so a warp reads 32 consecutive N columns of each K.
  const bool kfast = left || a.tb;
  // unit index math in 32 bits (the launcher guarantees units < 2^32)
  for (u32 uid = blockIdx.x * blockDim.x + threadIdx.x; uid < units; uid += gridDim.x * blockDim.x) {
    u32 t = uid;
    u32 r, kq;
    if (kfast) {
      kq = t % 8;
      t /= 8;
      r = t % BR;
      t /= BR;
    } else {
      r = t % BR;
      t /= BR;
      kq = t % 8;  // 4-value quarter of the 32-value K block
      t /= 8;
    }
    const u32 kb = t % nkb;
    t /= nkb;
    const u32 tile = t % tiles;
    const u32 bb = t / tiles;
    const u32 row = tile * BR + r;
    const u32 k0 = kb * kKB + kq * 4;
    u64 A[4], RA[4], F[4];  // per value: the shared draws (left: A, r_A; right: B, r_B) and F
    u64 idx[4];
    bool in[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const u32 k = k0 + u32(i);
      in[i] = row < rows && k < K;
      idx[i] = left ? u64(bb) * S.sL[0] + u64(row) * K + k
                    : u64(bb) * S.sR[0] + (a.tb ? u64(row) * K + k : u64(k) * N + row);
      A[i] = RA[i] = F[i] = 0;
      if (in[i]) {
        if (left) {
          if (dA) A[i] = mm_A(S.mm, S.aoff + idx[i]);
          if (dRA) RA[i] = mm_rA(S.mm, S.aoff + idx[i]);
        } else {
          if (dB) A[i] = mm_B(S.mm, S.boff + idx[i]);
          if (dRB) RA[i] = mm_rB(S.mm, S.boff + idx[i]);
          if (dF) F[i] = load_f(a.sl[fslot], fseg, idx[i]);
        }
      }
    }
    const u32 kc = kq / 4;  // which 16-byte K chunk of the core matrix
    // left: plane-major (one MMA A operand per plane); right: the 8 planes stacked along N
    // inside each K chunk, so planes 0..7-l form one B operand of N = (8-l)*BR rows
    const u32 off = left ? (kc * (BR / 8) + r / 8) * 128 + (r % 8) * 16 + (kq % 4) * 4
                         : kc * (BR * 128) + (r / 8) * 128 + (r % 8) * 16 + (kq % 4) * 4;
    const u32 pstride = left ? plane : BR * 16;
    for (int sl = slot; sl < slot + (both ? 2 : 1); ++sl) {
    const GemmSlotArgs& S = a.sl[sl];
    char* out = sl ? out1 : out0;
    // packed segments: all (right operand, full left pack) or the masked ones (hybrid left)
    const u32 smask = (sl ? mask1 : mask0) & ((1u << S.nseg) - 1);
    const u32 nseg = u32(__popc(smask));
    const u64 img = (((u64(bb) * tiles + tile) * nkb + kb) * nseg) * 8 * plane;
    u32 gp = 0;
    for (int g = 0; g < S.nseg; ++g) {
      if (!((smask >> g) & 1u)) continue;
      const int kind = left ? S.lk[g] : S.rk[g];
      u32 lo[4], hi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        u64 x = 0;
        if (in[i]) {
          if (left) {
            switch (kind) {
              case kOpMem: x = S.L[g][idx[i]]; break;
              case kOpSum: x = S.L[g][idx[i]] + S.L2[g][idx[i]]; break;
              case kOpA: x = A[i]; break;
              case kOpA0: x = A[i] - RA[i]; break;
              default: x = RA[i]; break;
            }
          } else {
            switch (kind) {
              case kOpMem: x = S.R[g][idx[i]]; break;
              case kOpSum: x = F[i]; break;
              case kOpB: x = A[i]; break;
              case kOpB0F: x = (A[i] - RA[i]) + F[i]; break;
              case kOpBF: x = A[i] + F[i]; break;
              case kOpNegSum: x = u64(0) - F[i]; break;
              default: x = RA[i]; break;
            }
          }
        }
        lo[i] = u32(x);
        hi[i] = u32(x >> 32);
      }
      char* base = out + img + u64(gp) * 8 * plane;
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const u32* w = l < 4 ? lo : hi;
        *reinterpret_cast<u32*>(base + l * pstride + off) = gather4(w[0], w[1], w[2], w[3], u32(l & 3));
      }
      ++gp;
    }
    }
  }
}

// The pair-evaluated Beaver combine's tensor-core operand pattern (beaver_combine): party 0's
// slot [A, E, r_A] and party 1's [E, r_A] on one dealer stream; returns party 0's slot or -1.
int pair_combine_p0(const GemmArgs& a) {
  if (a.nslots != 2) return -1;
  int p0 = -1;
  for (int i = 0; i < 2; ++i)
    if (a.sl[i].nseg == 3) p0 = i;
  if (p0 < 0 || a.sl[1 - p0].nseg != 2) return -1;
  const GemmSlotArgs& S0 = a.sl[p0];
  const GemmSlotArgs& S1 = a.sl[1 - p0];
  const bool e0 = S0.lk[1] == kOpMem || S0.lk[1] == kOpSum, e1 = S1.lk[0] == kOpMem || S1.lk[0] == kOpSum;
  if (S0.lk[0] != kOpA || !e0 || S0.lk[2] != kOpRA || !e1 || S1.lk[1] != kOpRA) return -1;
  if (S0.aoff != S1.aoff || S0.sL[0] != S1.sL[0] || S0.mm.key != S1.mm.key || S0.mm.kp != S1.mm.kp ||
      S0.mm.pool != S1.mm.pool || S0.mm.prA != S1.mm.prA)
    return -1;
  return p0;
}

bool pack_pair_on() {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_PACK_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}
// both slots' right operands come from one dealer stream (B, r_B at the same offset and
// stride) and one opened F (as (own, peer) of either slot)
bool pair_same_right(const GemmArgs& a) {
  const GemmSlotArgs& S0 = a.sl[0];
  const GemmSlotArgs& S1 = a.sl[1];
  if (S0.boff != S1.boff || S0.sR[0] != S1.sR[0] || S0.mm.key != S1.mm.key || S0.mm.kp != S1.mm.kp ||
      S0.mm.pool != S1.mm.pool || S0.mm.pB != S1.mm.pB || S0.mm.prB != S1.mm.prB)
    return false;
  const u64* f0 = nullptr;
  const u64* f1 = nullptr;
  bool any = false;
  for (int i = 0; i < 2; ++i)
    for (int g = 0; g < a.sl[i].nseg; ++g) {
      const int k = a.sl[i].rk[g];
      if (k == kOpMem) return false;
      if (k == kOpSum || k == kOpB0F || k == kOpBF || k == kOpNegSum) {
        const u64* x0 = a.sl[i].R[g];
        const u64* x1 = a.sl[i].R2[g];
        if (!any) {
          f0 = x0, f1 = x1, any = true;
        } else if (!((x0 == f0 && x1 == f1) || (x1 && x0 == f1 && x1 == f0))) {
          return false;
        }
      }
    }
  return true;
}

template <int BR>
void launch_pack(Session& s, const GemmArgs& a, bool left, u32 rows, u32 nbatch, u32 nkb, char* out0, char* out1,
                 u32 mask0 = ~0u, u32 mask1 = ~0u) {
  const u32 tiles = (rows + BR - 1) / BR;
  int maxseg = 0;
  for (int i = 0; i < a.nslots; ++i) {
    const int np = __builtin_popcount((i ? mask1 : mask0) & ((1u << a.sl[i].nseg) - 1));
    maxseg = np > maxseg ? np : maxseg;
  }
  const u64 units = u64(nbatch) * tiles * nkb * BR * 8;  // a unit packs every segment of its slot
  if (units * (maxseg > 0 ? 1 : 0) >= (u64(1) << 32)) throw Error(kShapeError, "tcgen05 pack: operand too large");
  cudaEvent_t pe;
  probe_begin(s.stream, &pe);
  // the pair combine's right operand: both slots per thread (one B / r_B draw and F load)
  const int both = !left && pack_pair_on() && pair_combine_p0(a) >= 0 && pair_same_right(a) ? 1 : 0;
  launch_pdl(pack_limbs<BR>, dim3(ew_blocks(units), both ? 1 : a.nslots), dim3(256), 0, s.stream, a, left ? 1 : 0,
             rows, nbatch, nkb, out0, out1, mask0, mask1, both);
  probe_end(s.stream, pe);
}

// packL: 0 = left operand generated by the producers, 1 = fully packed, 2 = hybrid (the
// dealer-drawn segments packed once, the memory segments loaded by the producers)
template <int BN, bool AT = false>
void launch_tc2(Session& s, const GemmArgs& a, int packL) {
  constexpr u32 kStage = 8 * ((AT ? 0 : kM * kKB) + BN * kKB);
  const size_t smem = kStages * kStage;
  static bool attr = false;
  if (!attr) {
    MPCG_CUDA(
        cudaFuncSetAttribute(ring_gemm_tc2<BN, false, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    MPCG_CUDA(
        cudaFuncSetAttribute(ring_gemm_tc2<BN, true, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  Tc2Args P{};
  P.g = a;
  P.nkb = (a.K + kKB - 1) / kKB;
  static const u32 l2ahead = [] {
    const char* e = std::getenv("MPCG_TC2_L2AHEAD");
    return e ? u32(std::atoi(e)) : 3u;
  }();
  P.l2ahead = l2ahead;
  static const int trace = [] {
    const char* e = std::getenv("MPCG_TC2_TRACE");
    return e && e[0] == '1' ? 1 : 0;
  }();
  P.trace = trace;
  const u32 ntiles = (a.N + BN - 1) / BN, mtiles = (a.M + kM - 1) / kM;
  // right operand: batched only when some segment's R has a batch stride
  bool rbatched = false;
  for (int i = 0; i < a.nslots; ++i)
    for (int g = 0; g < a.sl[i].nseg; ++g) rbatched |= a.sl[i].sR[g] != 0;
  const u32 rb = rbatched ? a.nbatch : 1;
  std::vector<std::shared_ptr<Block>> keep;
  // Fully packed pair combine: party 1's left segments (E, r_A) are party 0's segments 1 and 2
  // (the opened E and the dealer's r_A are the same values for both slots), so party 1 reads
  // party 0's image and only one image is packed (MPCG_TC2_SHAREL=0: one per slot).
  int share_slot = -1;
  {
    static const bool share_on = [] {
      const char* e = std::getenv("MPCG_TC2_SHAREL");
      return !(e && e[0] == '0');
    }();
    const int p0 = packL == 1 && share_on ? pair_combine_p0(a) : -1;
    if (p0 >= 0) share_slot = 1 - p0;
  }
  // the shared slot must come after party 0's image is allocated
  {
    ClassScope pack_scope(kClsOther, 0);  // the roofline probe times the GEMM kernel itself
    char* rp[2] = {nullptr, nullptr};
    char* lp[2] = {nullptr, nullptr};
    for (int ii = 0; ii < a.nslots; ++ii) {
      const int i = share_slot == 0 ? 1 - ii : ii;  // the image owner (party 0) first
      const u64 rbytes = u64(ntiles) * P.nkb * a.sl[i].nseg * 8 * BN * kKB;
      auto blk = s.raw((rbytes * rb + 7) / 8);
      keep.push_back(blk);
      rp[i] = reinterpret_cast<char*>(blk->ptr);
      P.Rpk[i] = rp[i];
      P.Rpk_b[i] = rbatched ? rbytes : 0;
      u32 lmask = 0;
      for (int g = 0; g < a.sl[i].nseg; ++g) {
        const int k = a.sl[i].lk[g];
        if (packL == 1 || (packL == 2 && k != kOpMem && k != kOpSum)) lmask |= 1u << g;
      }
      P.lmask[i] = lmask;
      P.lnpk[i] = u32(__builtin_popcount(lmask));
      P.lseg0[i] = 0;
      if (lmask && i == share_slot) {  // reads party 0's image (E, r_A are the same values)
        P.lnpk[i] = P.lnpk[1 - i];
        P.lseg0[i] = 1;
        P.Lpk[i] = P.Lpk[1 - i];
        P.Lpk_b[i] = P.Lpk_b[1 - i];
        lp[i] = nullptr;
        continue;
      }
      if (lmask) {
        const u64 lbytes = u64(mtiles) * P.nkb * __builtin_popcount(lmask) * 8 * kM * kKB;
        auto lb = s.raw((lbytes * a.nbatch + 7) / 8);
        keep.push_back(lb);
        lp[i] = reinterpret_cast<char*>(lb->ptr);
        P.Lpk[i] = lp[i];
        P.Lpk_b[i] = lbytes;
      }
    }
    launch_pack<BN>(s, a, false, a.N, rb, P.nkb, rp[0], rp[1]);
    if (P.lmask[0] | P.lmask[1])
      launch_pack<kM>(s, a, true, a.M, a.nbatch, P.nkb, lp[0], lp[1], share_slot == 0 ? 0u : P.lmask[0],
                      share_slot == 1 ? 0u : P.lmask[1]);
  }
  // vector width of the L row loads: 2 = 32-byte (LDG.256), 1 = 16-byte, 0 = scalar
  auto aligned = [&](u32 vals) {
    bool ok = (a.K % vals) == 0;
    for (int i = 0; i < a.nslots && ok; ++i)
      for (int g = 0; g < a.sl[i].nseg; ++g) {
        const GemmSlotArgs& S = a.sl[i];
        if (S.lk[g] == kOpMem || S.lk[g] == kOpSum)
          ok = ok && reinterpret_cast<uintptr_t>(S.L[g]) % (8 * vals) == 0 && S.sL[g] % vals == 0;
        if (S.lk[g] == kOpSum) ok = ok && reinterpret_cast<uintptr_t>(S.L2[g]) % (8 * vals) == 0;
      }
    return ok;
  };
  P.vec = aligned(4) ? 2 : aligned(2) ? 1 : 0;
  static const bool wave_split = [] {
    const char* e = std::getenv("MPCG_TC2_WAVESPLIT");
    return !(e && e[0] == '0');
  }();
  // split K when the tile grid cannot fill the SMs (small-M layers): >= 2 K blocks per split
  const u64 ctas = u64(ntiles) * mtiles * a.nslots * a.nbatch;
  u32 split = 1;
  if (ctas < u64(num_sms())) {
    split = u32((num_sms() + ctas - 1) / ctas);
    split = split > 16 ? 16 : split;
    const u32 maxs = P.nkb / 2 > 0 ? P.nkb / 2 : 1;
    split = split > maxs ? maxs : split;
  } else if (wave_split) {
    // wave quantisation (one resident CTA per SM): a grid of 1.3 waves idles a third of the
    // last wave (BERT-base ffn2, 192 CTAs). Split K when it fills the waves >= 15% better and
    // each split keeps >= 48 pipeline stages (shorter splits pay the CTA fill and the partials
    // pass: BERT-base attention out, 24-36 stages per split, measured slower).
    // MPCG_TC2_WAVESPLIT=0 disables.
    const u64 sms = num_sms();
    u32 maxseg = 1;
    for (int i = 0; i < a.nslots; ++i) maxseg = u32(a.sl[i].nseg) > maxseg ? u32(a.sl[i].nseg) : maxseg;
    auto eff = [&](u64 sp) { const u64 c = ctas * sp; return double(c) / double((c + sms - 1) / sms * sms); };
    double best = eff(1);
    for (u32 sp = 2; sp <= 4; ++sp)
      if (P.nkb * maxseg / sp >= 48 && eff(sp) >= 1.15 * eff(1) && eff(sp) > best + 1e-9) {
        best = eff(sp);
        split = sp;
      }
  }
  P.kbper = (P.nkb + split - 1) / split;
  P.ksplit = (P.nkb + P.kbper - 1) / P.kbper;
  std::shared_ptr<Block> ws;
  if (P.ksplit > 1) {
    const u64 per = u64(a.nbatch) * a.M * a.N;
    ws = s.raw(per * P.ksplit * a.nslots);
    for (int i = 0; i < a.nslots; ++i) P.g.acc[i] = ws->ptr + i * per * P.ksplit;
    P.g.ksplit = P.ksplit;
  }
  dim3 grid(ntiles * a.nslots, mtiles, a.nbatch * P.ksplit);
  cudaEvent_t pe;
  probe_begin(s.stream, &pe);
  static const bool split_groups = [] {  // measured ~3-5% faster on ResNet-18 / VGG-16 convs
    const char* e = std::getenv("MPCG_TC2_SPLIT");
    return !(e && e[0] == '0');
  }();
  if (split_groups)
    launch_pdl(ring_gemm_tc2<BN, true, AT>, grid, dim3(kThreads), smem, s.stream, P);
  else
    launch_pdl(ring_gemm_tc2<BN, false, AT>, grid, dim3(kThreads), smem, s.stream, P);
  probe_end(s.stream, pe);
  if (P.ksplit > 1) {
    ClassScope ep_scope(kClsOther, 0);
    const u64 n = u64(a.nbatch) * a.M * a.N * a.nslots;
    launch_pdl(gemm_splitk_epilogue_fn(), dim3(ew_blocks(n)), dim3(256), 0, s.stream, P.g);
  }
  // the packed buffers are stream-ordered pool blocks (or graph-arena blocks): released
  // after the GEMM's queued reads by the Block destructor
}

}  // namespace

// 0 = never, 1 = every shape within the exactness budget, 2 = auto (large shapes).
int& tc_gemm_mode() {
  static int mode = [] {
    const char* e = std::getenv("MPCG_TC_GEMM");
    return (e && (e[0] == '0' || e[0] == '1')) ? e[0] - '0' : 2;
  }();
  return mode;
}

bool ring_gemm_tc2_wants(const GemmArgs& a) {
  if (tc_gemm_mode() == 0) return false;
  int maxseg = 0;
  for (int i = 0; i < a.nslots; ++i) maxseg = a.sl[i].nseg > maxseg ? a.sl[i].nseg : maxseg;
  if (u64(maxseg) * a.K > kMaxKPrime) return false;
  if (a.ksplit > 1) return false;
  const double work = double(a.M) * a.N * a.K * maxseg * a.nbatch * a.nslots;
  // partial-row tiles pay off on short, wide linear layers too (LeNet fc0 64x256x120: SIMT
  // split-K 50.5 us -> 36.2 us measured); below ~5e6 ring MACs the SIMT kernel's latency wins
  return tc_gemm_mode() == 1 || (a.M >= 128 && a.N >= 16 && work >= 3e7) || (a.M < 128 && a.N >= 16 && work >= 5e6);
}

bool ring_gemm_tc2_try(Session& s, const GemmArgs& a) {
  if (!ring_gemm_tc2_wants(a)) return false;
  for (int i = 0; i < a.nslots; ++i)
    for (int g = 0; g < a.sl[i].nseg; ++g) {
      const GemmSlotArgs& S = a.sl[i];
      if (S.sL[g] != S.sL[0]) return false;  // the producer uses one row stride for every segment
      if (S.sR[g] != S.sR[0]) return false;  // the pack shares draws across segments
      const bool fk = S.rk[g] == kOpSum || S.rk[g] == kOpB0F || S.rk[g] == kOpBF || S.rk[g] == kOpNegSum;
      for (int h = 0; h < g && fk; ++h) {
        const bool fh = S.rk[h] == kOpSum || S.rk[h] == kOpB0F || S.rk[h] == kOpBF || S.rk[h] == kOpNegSum;
        if (fh && (S.R[h] != S.R[g] || S.R2[h] != S.R2[g])) return false;  // ... and one opened F
      }
    }
  // several N tiles: pack the left operand once (bulk-copied per tile) or regenerate it per
  // tile in the producers (CTAs of one M tile run side by side, so E re-reads hit L2).
  // Measured: regenerating wins up to 8 tiles (ResNet-18 / VGG-16 convs), packing beyond
  // (BERT's 768..3072-wide projections, where the dealer draws would repeat 12..48 times).
  static const int packl = [] {
    const char* e = std::getenv("MPCG_TC2_PACKL");  // 0 = never, 1 = whenever N > 64, else auto
    return e ? e[0] - '0' : 2;
  }();
  const bool multiN = a.N > 64 && (packl == 1 || (packl == 2 && a.N > 512));
  // left operand in TMEM (BN = 32 tiles) for the regenerated-L shapes: opt-in only — with the
  // wide MMAs the stage is no longer shared-memory bound, and halving BN doubles the L
  // regeneration (measured ResNet-18 51.4 vs 43.3 ms)
  static const int at = [] {
    const char* e = std::getenv("MPCG_TC2_AT");  // 1 = on, 0 = off
    return e ? e[0] - '0' : 0;
  }();
  // five or more N tiles but not fully packed: pack only the dealer-drawn segments (their draws
  // would repeat per N tile) and let the producers load E (MPCG_TC2_HYBRID=0: regenerate
  // everything). Measured per layer: a win at 8 tiles (ResNet-18 layer4 / VGG-16 conv4-5, up to
  // -15%), a loss at 2-4 (the packed planes' HBM round trip outweighs 2-4 regenerations).
  static const bool hybrid = [] {
    const char* e = std::getenv("MPCG_TC2_HYBRID");
    return !(e && e[0] == '0');
  }();
  const int lmode = multiN ? 1 : (hybrid && a.N > 4 * 64 ? 2 : 0);
  if (at == 1 && !multiN && a.N > 16)
    launch_tc2<32, true>(s, a, 0);
  else if (a.N > 32)
    launch_tc2<64>(s, a, lmode);
  else if (a.N > 16)
    launch_tc2<32>(s, a, 0);
  else
    launch_tc2<16>(s, a, 0);
  s.check();
  return true;
}

void tc2_trace_read(unsigned long long* out, int n) {
  const int m = n < kTraceStages * 10 ? n : kTraceStages * 10;
  MPCG_CUDA(cudaMemcpyFromSymbol(out, g_tc2_trace, sizeof(unsigned long long) * size_t(m)));
}

}  // namespace mpcg
