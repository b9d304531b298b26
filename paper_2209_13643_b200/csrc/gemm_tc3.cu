// tcgen05 int8-limb ring GEMM for the pair-evaluated Beaver combine: BOTH party slots of a
// private linear layer in one CTA (sm_100a).
//
// The combine of H/protocols/beaver.hpp:175-180 (matmul_combine) is, per party slot,
//   party 0:  z0 = -r_C + A*(B + F) + E*(b0 + F) - r_A*F      (b0 = B - r_B; dealer C = A*B online)
//   party 1:  z1 = +r_C + E*r_B     + r_A*F
// The left operands are only three matrices, {A, E, r_A}, and E and r_A are shared by the two
// slots. gemm_tc2.cu runs one CTA per slot, so E is transposed into limb planes twice and r_A
// drawn and transposed twice; its producers (dealer splitmix64 draws + byte transposes, ALU
// pipe) bound it, not the tensor pipe (ncu: ALU 57% / tensor 46% active, profiles/r02_tc3_*).
// Here the GEMM is computed transposed, Z^T = R^T * L^T, with the two slots' right operands
// stacked as the UMMA M dimension:
//
//   UMMA A (M = 128 rows, packed once per call, bulk-copied): rows 0-63 = party 0's right
//          operand for this left operand, rows 64-127 = party 1's (zero for the A stage);
//   UMMA B (N = 64 rows of L per CTA, generated in place by the producers): one stage per
//          left operand per 32-wide K slab, in the order A, E, r_A.
//
// so each left value is generated and transposed ONCE for both slots (2 draws + 3 transposes
// per (m, k) instead of 3 + 5). The cost is the A stage's idle upper half (1/6 of the MMAs).
// Limb form as in gemm_tc2.cu (H/ring/limb.hpp:15-99): 8 u8 limb planes per operand; the UMMA
// A plane l (weights) against the generated planes 0..7-l stacked along N gives diagonals l..7
// in adjacent TMEM column blocks (12 MMAs per stage), D_d summed mod 2^32 per diagonal, and the
// epilogue recombines z = sum_d D_d << 8d mod 2^64 (exact for K' = 3K <= 16384).
//
// Warp roles (18 warps): warps 0-15 = four producer groups of 4 warps (one warp per SM
// sub-partition each); group j owns ring stage j (4 stages) and so every 4th pipeline stage;
// warp 16 = bulk loader of the packed weight images; warp 17 = MMA issuer (one thread) and
// TMEM owner; warps 0-15 = epilogue (TMEM lane quadrant = (party, 32 output columns)).
#include "tc_common.cuh"

namespace mpcg {

namespace {

constexpr int kT3Rows = 64;                    // L rows per CTA (UMMA N per plane)
constexpr int kT3Stages = 4;                   // = producer groups
constexpr int kT3Groups = 4;
constexpr int kT3Warps = 4 * kT3Groups + 2;
constexpr int kT3Threads = kT3Warps * 32;
constexpr u32 kT3A = 128 * kKB;                // bytes per weight limb plane per stage (4 KB)
constexpr u32 kT3B = kT3Rows * kKB;            // bytes per generated limb plane per stage (2 KB)
constexpr u32 kT3Stage = 8 * (kT3A + kT3B);    // 48 KB
constexpr u32 kT3MaxKPrime = 16384;

// Debug trace (MPCG_TC3_TRACE=1): per-stage clock64 stamps of CTA (0,0,0) — MMA thread: wait
// start, stage full, MMAs issued; the producing group's first warp: generation start, empty
// wait start, empty acquired, arrived — plus the epilogue start/end (row kT3TraceRows - 1).
// Read back with mpcg_debug_tc3_trace; off by default, no effect on values.
constexpr int kT3TraceRows = 256;
__device__ unsigned long long g_tc3_trace[kT3TraceRows][8];

struct Tc3Args {
  GemmArgs g;
  int p0slot = 0;             // slot index of party 0 (image rows 0-63)
  const u64* E = nullptr;     // opened E = own + peer (summed at build time), [M][K]
  const char* Wpk = nullptr;  // packed weights: [ntile][kb][3][8 planes][128 rows x 32 B]
  u32 nkb = 0;
  int vec = 0;                // 2 = E rows 32-byte aligned (LDG.256), 1 = 16-byte, 0 = scalar
  FastDiv fkk, fk;            // deferred conv eps: k*k and k
  FastDiv fohw;               // col2im epilogue: OH*OW
  int trace = 0;
  int mfast = 0;              // grid x = M tiles (see the kernel)
};

// gemm_epilogue's value (+-r_C, truncation, bias) without the store.
__device__ __forceinline__ u64 epi_value(const GemmArgs& a, const GemmSlotArgs& S, u32 m, u32 n, u64 v) {
  const u64 lin = u64(m) * a.N + n;
  if (S.cterm) {
    const u64 rc = S.mm.pool ? __ldg(S.mm.pool + S.cbase + lin - 1) : drw(tkey(S.ckey, S.ckp), S.cbase + lin);
    v = S.cterm > 0 ? v + rc : v - rc;
  }
  if (a.trunc_bits) v = sar64(v, a.trunc_bits);
  if (S.bias) v += S.bias[n];
  return v;
}

// 16 K-consecutive values of E row `row` starting at k0 (zero past M / K).
__device__ __forceinline__ void e_fetch(const Tc3Args& P, u32 row, u32 k0, u64 (&v)[16]) {
  const u32 M = P.g.M, K = P.g.K;
  if (row >= M || k0 >= K) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0;
    return;
  }
  const u64* p = P.E + u64(row) * K + k0;
  if (k0 + 16 <= K && P.vec == 2) {
    load16w(p, v);
  } else if (k0 + 16 <= K && P.vec == 1) {
    load16(p, v);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (k0 + u32(i) < K) ? __ldg(p + i) : 0;
  }
}

// 18 warps: SM sub-partitions hold 5 warps x 96 registers at most (16K registers each)
// Deferred eps (EpsDefer): the 16 opened values E = x0 + x1 - A of row m from the activation
// shares and the dealer's A, in the producer (what the summed eps build kernels write,
// eps_build_mem / eps_build_im2col in gemm.cu, H/protocols/beaver.hpp:186-196 + im2col of
// H/engine/executor.hpp:82-108). v holds the A draws on entry. Conv rows: the thread's output
// pixel is decoded once (GatherRow); per stage the (ci, ki, kj) of k0 by two multiply-shift
// divisions, then the input index advances incrementally; rows whose 3x3 (k x k) window lies
// inside the image skip the bounds tests.
struct GatherRow {
  u32 img;       // n * C
  int ih0, iw0;  // top-left input coordinate of the window
  bool inside;
};
__device__ __forceinline__ GatherRow gather_row(const EpsDefer& ed, u32 K, u32 m) {
  const ConvGeom& g = ed.g;
  GatherRow gr{};
  const u32 row = u32(ed.a_off / K) + m;  // global im2col row (n, oh, ow)
  const u32 ow = row % g.OW, rq = row / g.OW, oh = rq % g.OH, n = rq / g.OH;
  gr.img = n * g.C;
  gr.ih0 = int(oh * g.stride) - int(g.pad);
  gr.iw0 = int(ow * g.stride) - int(g.pad);
  gr.inside = gr.ih0 >= 0 && gr.iw0 >= 0 && gr.ih0 + int(g.k) <= int(g.H) && gr.iw0 + int(g.k) <= int(g.W);
  return gr;
}
__device__ __forceinline__ void e_gen(const Tc3Args& P, const GatherRow& gr, u32 m, u32 k0, u64 (&v)[16]) {
  const EpsDefer& ed = P.g.ed;
  const u32 K = P.g.K;
  if (ed.mode == 1) {
    const u64 base = ed.a_off + u64(m) * K + k0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      v[i] = (k0 + u32(i) < K) ? __ldg(ed.x0 + base + i) + __ldg(ed.x1 + base + i) - v[i] : 0;
    return;
  }
  const u32 ks = ed.g.k, H = ed.g.H, W = ed.g.W;
  const u32 ci = P.fkk.div(k0), rem = k0 - ci * P.fkk.d, ki0 = P.fk.div(rem), kj0 = rem - ki0 * ks;
  int ki = int(ki0), kj = int(kj0);
  int idx = int(((gr.img + ci) * H) * W) + (gr.ih0 + ki) * int(W) + gr.iw0 + kj;
  const int wstep = int(W) - int(ks), cstep = int(H - ks) * int(W);
  if (gr.inside && k0 + 16 <= K) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = __ldg(ed.x0 + idx) + __ldg(ed.x1 + idx) - v[i];
      ++idx;
      if (++kj == int(ks)) {
        kj = 0;
        idx += wstep;
        if (++ki == int(ks)) ki = 0, idx += cstep;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int ih = gr.ih0 + ki, iw = gr.iw0 + kj;
    u64 x = 0;
    if (k0 + u32(i) < K && ih >= 0 && iw >= 0 && ih < int(H) && iw < int(W)) x = __ldg(ed.x0 + idx) + __ldg(ed.x1 + idx);
    v[i] = (k0 + u32(i) < K) ? x - v[i] : 0;
    ++idx;
    if (++kj == int(ks)) {
      kj = 0;
      idx += wstep;
      if (++ki == int(ks)) ki = 0, idx += cstep;
    }
  }
}

__global__ void __launch_bounds__(kT3Threads, 1) ring_gemm_tc3(const __grid_constant__ Tc3Args P) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) u64 full[kT3Stages], empty[kT3Stages], done;
  __shared__ u32 tmem_slot;

  pdl_enter();
  const GemmArgs& a = P.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const u32 M = a.M, N = a.N, K = a.K;
  // grid: (N tile, M tile) — the CTAs of one M tile run together (their gathered / loaded L
  // rows shared in L2) — or, with P.mfast, (M tile, N tile): the CTAs in flight share one N
  // tile's weight images (large-N layers, where all images would not stay in L2 together)
  const u32 ntile = P.mfast ? blockIdx.y : blockIdx.x;
  const u32 m0 = (P.mfast ? blockIdx.x : blockIdx.y) * kT3Rows, n0 = ntile * 64;
  const u32 nst = P.nkb * 3;

  if (tid == 0) {
    for (int i = 0; i < kT3Stages; ++i) {
      mbar_init(&full[i], 4 + 1);  // the 4 warps of the owning producer group + the loader
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kT3Warps - 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = tmem_slot;

  if (warp < 4 * kT3Groups) {
    // ---- producer group j = warp / 4 owns ring stage j: pipeline stages it = j, j+4, ...
    // (stage type it % 3: 0 = A, 1 = E, 2 = r_A; 3 and 4 coprime, so every group serves all
    // three). Thread t: row r = t % 64, K half hf = t / 64 -> 16 K-consecutive values.
    const int j = warp >> 2, t = tid & 127;
    const u32 r = u32(t) & 63u, hf = u32(t) >> 6;
    const u32 m = m0 + r;
    const GemmSlotArgs& S0 = a.sl[P.p0slot];
    const u64 key = tkey(S0.mm.key, S0.mm.kp);
    const u64 iA = 1 + S0.mm.offA + S0.aoff;
    const u64 iRA = 1 + S0.mm.na + S0.mm.nb + S0.mm.offA + S0.aoff;
    // plane p, K chunk hf, row r: hf*8 KB + (p*8 + r/8)*128 + (r%8)*16
    const u32 off = hf * (8 * kT3Rows * 16) + (r / 8) * 128 + (r % 8) * 16;
    char* const sB = smem + u32(j) * kT3Stage + 8 * kT3A;
    // The E rows of this group's next E stage are pulled into L2 one group-stage (or two)
    // ahead; the register loads are issued at the stage itself, under the other three groups'
    // dealer draws (a register prefetch would cost 32 registers, and 5 warps x 96 fill an SM
    // sub-partition's register file).
    auto next_e = [&](u32 it) {  // first E stage of group j at or after stage it (or nst)
      u32 x = it;
      while (x < nst && x % 3 != 1) x += kT3Stages;
      return x;
    };
    auto l2_prefetch = [&](u32 ite) {
      const u32 kp = (ite / 3) * kKB + hf * 16;
      if (ite < nst && m < M && kp < K) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.E + u64(m) * K + kp));
    };
    if (a.ed.mode == 0) l2_prefetch(next_e(u32(j)));
    const GatherRow gr = a.ed.mode == 2 ? gather_row(a.ed, K, m) : GatherRow{};
    const bool tr = P.trace && blockIdx.x == 0 && blockIdx.y == 0 && (tid & 127) == 0;
    for (u32 it = u32(j), use = 0; it < nst; it += kT3Stages, ++use) {
      const u32 kb = it / 3, type = it % 3;
      const u32 k0 = kb * kKB + hf * 16;
      if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][3] = clock64();
      u64 v[16];
      if (type == 1 && a.ed.mode != 0) {  // deferred eps: E = x0 + x1 - A generated here
        if (m >= M || k0 >= K) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0;
        } else {
          draws16(key, iA + u64(m) * K + k0, v, S0.mm.pool);
          e_gen(P, gr, m, k0, v);
        }
      } else if (type == 1) {
        e_fetch(P, m, k0, v);
        l2_prefetch(next_e(it + kT3Stages));
      } else if (m >= M || k0 >= K) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0;
      } else {
        draws16(key, (type == 2 ? iRA : iA) + u64(m) * K + k0, v, S0.mm.pool);
        if (k0 + 16 > K) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (k0 + u32(i) >= K) v[i] = 0;
        }
      }
      if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][4] = clock64();
      if (use > 0) mbar_wait(&empty[j], (use - 1) & 1);
      if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][5] = clock64();
      limb_store16(v, sB + off, 8 * 128);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[j]);
      if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][6] = clock64();
    }
  } else if (warp == 4 * kT3Groups) {
    if (lane == 0) {  // ---- bulk loader: the packed weight image of each stage
      const char* Wb = P.Wpk + u64(ntile) * P.nkb * 3 * 8 * kT3A;
      for (u32 it = 0; it < nst; ++it) {
        const int stg = int(it % kT3Stages);
        if (it >= u32(kT3Stages)) mbar_wait(&empty[stg], ((it / kT3Stages) - 1) & 1);
        mbar_arrive_tx(&full[stg], 8 * kT3A);
        bulk_g2s(smem + stg * kT3Stage, Wb + u64(it) * 8 * kT3A, 8 * kT3A, &full[stg]);
      }
    }
  } else {
    if (lane == 0) {  // ---- MMA issuer
      const bool tr = P.trace && blockIdx.x == 0 && blockIdx.y == 0;
      for (u32 it = 0; it < nst; ++it) {
        const int stg = int(it % kT3Stages);
        if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][0] = clock64();
        mbar_wait(&full[stg], (it / kT3Stages) & 1);
        if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][1] = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const u32 aBase = smem_u32(smem + stg * kT3Stage), bBase = aBase + 8 * kT3A;
        // weight plane l x generated planes 0..7-l stacked along N -> diagonals l..7
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const u32 acc = (it > 0 || l > 0) ? 1u : 0u;
#pragma unroll
          for (u32 c0 = 0; c0 < u32(8 - l) * kT3Rows; c0 += 256) {
            const u32 nn = min(256u, u32(8 - l) * kT3Rows - c0);
            const u64 bd = smem_desc(bBase + (c0 / 8) * 128, 8 * kT3Rows * 16, 128);
            const u64 ad = smem_desc(aBase + u32(l) * kT3A, (128 / 8) * 128, 128);
            mma_i8(tmem + u32(l) * kT3Rows + c0, ad, bd, idesc_i8(128, nn), acc);
          }
        }
        mma_commit(&empty[stg]);
        if (tr && it < kT3TraceRows - 1) g_tc3_trace[it][2] = clock64();
      }
      mma_commit(&done);
    }
  }

  // ---- epilogue: warp w reads TMEM lane quadrant q = w % 4 (rows 32q..32q+31 = party q/2,
  // output columns n0 + (q%2)*32 + lane) and L-row group cg = w / 4 (16 rows)
  if (warp < 4 * kT3Groups) {
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool tre = P.trace && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0;
    if (tre) g_tc3_trace[kT3TraceRows - 1][0] = clock64();
    const int q = warp & 3, cg = warp >> 2;
    const int slot = (q >> 1) == 0 ? P.p0slot : 1 - P.p0slot;
    const u32 n = n0 + u32(q & 1) * 32 + u32(lane);
    const GemmSlotArgs& S = a.sl[slot];
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {  // 8 L rows at a time
      const u32 lane_addr = tmem + ((u32(q) * 32) << 16) + u32(cg) * 16 + u32(h) * 8;
      u64 acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0;
#pragma unroll
      for (int d0 = 0; d0 < 8; d0 += 4) {  // 4 diagonals in flight per wait
        u32 rr[32];
        tmem_ld4x8(lane_addr + u32(d0) * kT3Rows, lane_addr + u32(d0 + 1) * kT3Rows,
                   lane_addr + u32(d0 + 2) * kT3Rows, lane_addr + u32(d0 + 3) * kT3Rows, rr);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] += u64(rr[8 * i + c]) << (8 * (d0 + i));
      }
      if (a.col2im) {  // staged in shared memory, stored below with lanes along the rows
        u64* tile = reinterpret_cast<u64*>(smem) + (u32(q >> 1) * 64 + u32(q & 1) * 32 + u32(lane)) * kT3Rows;
        // Beaver epilogue per value (gemm_epilogue's +-r_C, truncation, bias), with the r_C
        // stream position advanced by N*phi per row instead of recomputed, and the key, bias
        // and slot fields read once
        const u32 mb = m0 + u32(cg) * 16 + u32(h) * 8;
        const u64 ck = S.cterm ? (S.mm.pool ? 0 : tkey(S.ckey, S.ckp)) : 0;
        u64 z = ck + (S.cbase + u64(mb) * N + n) * kPhi;
        const u64 dz = u64(N) * kPhi;
        const u64 bias = (S.bias && n < N) ? S.bias[n] : 0;
        const int cterm = S.cterm, tb = a.trunc_bits;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const u32 mloc = u32(cg) * 16 + u32(h) * 8 + u32(c);
          u64 v = acc[c];
          if (cterm) {
            const u64 rc = S.mm.pool ? __ldg(S.mm.pool + S.cbase + (u64(mb + c) * N + n) - 1) : mix64(z);
            v = cterm > 0 ? v + rc : v - rc;
          }
          if (tb) v = sar64(v, tb);
          tile[mloc] = (n < N && m0 + mloc < M) ? v + bias : 0;
          z += dz;
        }
      } else if (n < N) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const u32 mm = m0 + u32(cg) * 16 + u32(h) * 8 + u32(c);
          if (mm < M) gemm_epilogue(a, S, 0, mm, n, acc[c]);
        }
      }
    }
    if (a.col2im) {
      // col2im (H/engine/executor.hpp:110-123): out[(img*N + n)*OHW + rem] for global row
      // m0 + row0 + mloc = img*OHW + rem. Lanes run along the rows, so a warp writes up to 32
      // consecutive words of one output plane instead of 32 planes one word each.
      asm volatile("bar.sync 1, %0;" ::"r"(4 * kT3Groups * 32) : "memory");
      const u64* tile = reinterpret_cast<const u64*>(smem);
      // element e = tid + 512 i: row mloc = tid % 64 is fixed per thread (512 % 64 == 0), so the
      // image / position decode is done once; the (party, column) index advances by 8 per step
      constexpr u32 kEpiThreads = 4 * kT3Groups * 32;
      static_assert(kEpiThreads % kT3Rows == 0, "epilogue row mapping");
      const u32 mloc = u32(tid) % kT3Rows, mm = m0 + mloc;
      if (mm < M) {
        const u32 mg = mm + a.row0, img = P.fohw.div(mg), rem = mg - img * a.OHW;
        u64* const out0 = a.sl[P.p0slot].out;
        u64* const out1 = a.sl[1 - P.p0slot].out;
        const u64* const add0 = a.sl[P.p0slot].addend;  // fused residual add (or null)
        const u64* const add1 = a.sl[1 - P.p0slot].addend;
        const u64 ibase = u64(img) * N;
        constexpr u32 kStep = kEpiThreads / kT3Rows, kIt = 128 / kStep;
        if (add0 || add1) {  // fused residual add: every addend load in flight before the stores
          u64 adv[kIt];
#pragma unroll
          for (u32 it = 0; it < kIt; ++it) {
            const u32 nq = u32(tid) / kT3Rows + it * kStep, n = n0 + (nq & 63u);
            const u64* const ad = nq < 64 ? add0 : add1;
            adv[it] = (ad && n < N) ? __ldg(ad + (ibase + n) * a.OHW + rem) : 0;
          }
#pragma unroll
          for (u32 it = 0; it < kIt; ++it) {
            const u32 nq = u32(tid) / kT3Rows + it * kStep, n = n0 + (nq & 63u);
            if (n < N) (nq < 64 ? out0 : out1)[(ibase + n) * a.OHW + rem] = tile[nq * kT3Rows + mloc] + adv[it];
          }
        } else {
#pragma unroll 4
          for (u32 nq = u32(tid) / kT3Rows; nq < 128; nq += kStep) {
            const u32 n = n0 + (nq & 63u);
            if (n < N) (nq < 64 ? out0 : out1)[(ibase + n) * a.OHW + rem] = tile[nq * kT3Rows + mloc];
          }
        }
      }
    }
    if (tre) g_tc3_trace[kT3TraceRows - 1][1] = clock64();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kT3Warps - 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

// Weight image of every stage: [ntile][kb][type][plane][128 rows x 32 B], K-major core
// matrices (row group r/8, K chunk kc) at (kc*16 + r/8)*128 + (r%8)*16. Row r < 64: party 0's
// right operand for column n0 + r, r >= 64: party 1's for n0 + r - 64. Per (k, n) the dealer's
// B, r_B and the opened F are read once for the three stage types:
//   type 0 (left A):   party 0: B + F,           party 1: 0
//   type 1 (left E):   party 0: (B - r_B) + F,   party 1: r_B
//   type 2 (left r_A): party 0: -F,              party 1: F
// Unit = 4 K-consecutive values of one image row for all three types.
__global__ void __launch_bounds__(256) pack_tc3(const __grid_constant__ Tc3Args P, char* out) {
  pdl_enter();
  const GemmArgs& a = P.g;
  const GemmSlotArgs& S = a.sl[P.p0slot];
  const u32 K = a.K, N = a.N, nkb = P.nkb;
  const u32 ntiles = (N + 63) / 64;
  const u32 units = ntiles * nkb * 128 * 8;
  for (u32 uid = blockIdx.x * blockDim.x + threadIdx.x; uid < units; uid += gridDim.x * blockDim.x) {
    u32 t = uid, rr, kq;
    if (a.tb) {  // R stored [N][K]: K-quarters fastest (contiguous reads)
      kq = t % 8;
      t /= 8;
      rr = t % 128;
      t /= 128;
    } else {  // R stored [K][N]: columns fastest
      rr = t % 128;
      t /= 128;
      kq = t % 8;
      t /= 8;
    }
    const u32 kb = t % nkb, nt = t / nkb;
    const bool p1 = rr >= 64;
    const u32 n = nt * 64 + (rr & 63u), k0 = kb * kKB + kq * 4;
    u64 x[3][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const u32 k = k0 + u32(i);
      x[0][i] = x[1][i] = x[2][i] = 0;
      if (n < N && k < K) {
        const u64 idx = a.tb ? u64(n) * K + k : u64(k) * N + n;
        const u64 F = load_f(S, 0, idx);  // segment 0 (B + F) carries the opened F
        const u64 rB = mm_rB(S.mm, S.boff + idx);
        if (p1) {
          x[1][i] = rB;
          x[2][i] = F;
        } else {
          const u64 B = mm_B(S.mm, S.boff + idx);
          x[0][i] = B + F;
          x[1][i] = (B - rB) + F;
          x[2][i] = u64(0) - F;
        }
      }
    }
    const u32 kc = kq / 4;
    const u32 off = (kc * 16 + rr / 8) * 128 + (rr % 8) * 16 + (kq % 4) * 4;
    char* base = out + (u64(nt) * nkb + kb) * 3 * 8 * kT3A;
#pragma unroll
    for (int ty = 0; ty < 3; ++ty) {
      u32 lo[4], hi[4];
      bt4(u32(x[ty][0]), u32(x[ty][1]), u32(x[ty][2]), u32(x[ty][3]), lo);
      bt4(u32(x[ty][0] >> 32), u32(x[ty][1] >> 32), u32(x[ty][2] >> 32), u32(x[ty][3] >> 32), hi);
      char* tb = base + u32(ty) * 8 * kT3A + off;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        *reinterpret_cast<u32*>(tb + u32(p) * kT3A) = lo[p];
        *reinterpret_cast<u32*>(tb + u32(p + 4) * kT3A) = hi[p];
      }
    }
  }
}

// The exact operand pattern beaver_combine builds for the tensor-core path with a summed E:
// returns the party-0 slot index, or -1.
int tc3_pattern(const GemmArgs& a) {
  if (a.nslots != 2 || a.nbatch != 1 || a.ksplit > 1) return -1;
  int p0 = -1;
  for (int i = 0; i < 2; ++i)
    if (a.sl[i].nseg == 3) p0 = i;
  if (p0 < 0) return -1;
  const GemmSlotArgs& S0 = a.sl[p0];
  const GemmSlotArgs& S1 = a.sl[1 - p0];
  if (S1.nseg != 2) return -1;
  if (S0.lk[0] != kOpA || S0.lk[1] != kOpMem || S0.lk[2] != kOpRA) return -1;
  if (S0.rk[0] != kOpBF || S0.rk[1] != kOpB0F || S0.rk[2] != kOpNegSum) return -1;
  if (S1.lk[0] != kOpMem || S1.lk[1] != kOpRA || S1.rk[0] != kOpRB || S1.rk[1] != kOpSum) return -1;
  if (S0.L[1] != S1.L[0] || S0.aoff != S1.aoff || S0.boff != S1.boff) return -1;
  if (S0.mm.key != S1.mm.key || S0.mm.kp != S1.mm.kp || S0.mm.pool != S1.mm.pool || S0.mm.pA != S1.mm.pA ||
      S0.mm.prA != S1.mm.prA || S0.mm.pB != S1.mm.pB || S0.mm.prB != S1.mm.prB)
    return -1;
  for (int g = 0; g < 3; ++g)  // one opened F for every right operand of both slots
    if (S0.R[g] != S0.R[0] || S0.R2[g] != S0.R2[0]) return -1;
  // party 1's F: the same opened value, as (own, peer) of either slot
  const bool sameF = S1.R[1] == S0.R[0] && S1.R2[1] == S0.R2[0];
  const bool swapF = S0.R2[0] && S1.R[1] == S0.R2[0] && S1.R2[1] == S0.R[0];
  if (!sameF && !swapF) return -1;
  return p0;
}

}  // namespace

// 0 = off, 1 = on (default): the both-slots tcgen05 kernel where its pattern applies.
bool tc3_shape_ok(const Session& s, u32 M, u32 N, u32 K, bool col2im);
int tc3_default() {
  const char* e = std::getenv("MPCG_TC3");
  return (e && e[0] == '0') ? 0 : 1;
}
int& tc3_mode() {
  static int mode = tc3_default();
  return mode;
}

static u32 tc3_maxn() {
  static const u32 maxn = [] {  // N tiles regenerating the left operand (MPCG_TC3_MAXN)
    const char* e = std::getenv("MPCG_TC3_MAXN");
    return e ? u32(std::atoi(e)) : 8u;  // 8 measured faster than the tc2 hybrid at N = 512
  }();
  return maxn;
}

// Shape policy of the both-slots kernel for a pair-evaluated unbatched combine of an M x K by
// K x N product: the dispatch order of ring_gemm_launch (small-M GEMV, skinny-N rows, then the
// tcgen05 size policy) and this kernel's own limits.
bool tc3_shape_ok(const Session& s, u32 M, u32 N, u32 K, bool col2im) {
  if (tc3_mode() == 0 || tc_gemm_mode() == 0 || s.n_local != 2) return false;
  if (gemv_mode() != 0 && (gemv_eligible_shape(M, 1, false, col2im ? 1 : 0) || (N <= 8 && M >= 1024)))
    return false;
  GemmArgs a{};
  a.nslots = 2;
  a.M = M;
  a.N = N;
  a.K = K;
  a.sl[0].nseg = 3;
  a.sl[1].nseg = 2;
  if (!ring_gemm_tc2_wants(a)) return false;
  if (u64(3) * K > kT3MaxKPrime) return false;
  const u32 ntiles = (N + 63) / 64, mtiles = (M + kT3Rows - 1) / kT3Rows;
  if (ntiles > tc3_maxn()) return false;
  if (tc_gemm_mode() != 1 && u64(ntiles) * mtiles < u64(num_sms())) return false;  // forced: any grid
  return true;
}

bool ring_gemm_tc3_accepts(const Session& s, const GemmArgs& a) {
  return tc3_pattern(a) >= 0 && tc3_shape_ok(s, a.M, a.N, a.K, a.col2im != 0);
}

// Deferred eps (EpsDefer): the summed eps open of a combine that the both-slots kernel will
// run is not built; its producers generate E. MPCG_EPS_DEFER=0 keeps the build kernels.
bool eps_defer(Session& s, Open& o, const u64* const x[2], const ConvGeom* g, size_t a_off, u32 M, u32 N, u32 K) {
  static const bool on = [] {
    const char* e = std::getenv("MPCG_EPS_DEFER");
    return !(e && e[0] == '0');
  }();
  if (!on || !o.summed || s.n_local != 2 || s.cfg.link_bandwidth > 0) return false;
  if (!tc3_shape_ok(s, M, N, K, g != nullptr)) return false;
  if (g && u64(g->N) * g->C * g->H * g->W >= (u64(1) << 32)) return false;  // 32-bit gather index
  o.defer.mode = g ? 2 : 1;
  o.defer.x0 = x[0];
  o.defer.x1 = x[1];
  if (g) o.defer.g = *g;
  o.defer.a_off = a_off;
  return true;
}

bool ring_gemm_tc3_try(Session& s, const GemmArgs& a) {
  const int p0 = tc3_pattern(a);
  if (p0 < 0 || !tc3_shape_ok(s, a.M, a.N, a.K, a.col2im != 0)) return false;
  const u32 ntiles = (a.N + 63) / 64, mtiles = (a.M + kT3Rows - 1) / kT3Rows;
  static bool attr = false;
  if (!attr) {
    MPCG_CUDA(cudaFuncSetAttribute(ring_gemm_tc3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(kT3Stages * kT3Stage)));
    attr = true;
  }
  Tc3Args P{};
  P.g = a;
  P.p0slot = p0;
  P.E = a.sl[p0].L[1];
  P.nkb = (a.K + kKB - 1) / kKB;
  if (a.ed.mode == 2) {
    P.fkk = FastDiv(a.ed.g.k * a.ed.g.k);
    P.fk = FastDiv(a.ed.g.k);
  }
  if (a.col2im) P.fohw = FastDiv(a.OHW);
  static const int trace = [] {
    const char* e = std::getenv("MPCG_TC3_TRACE");
    return e && e[0] == '1' ? 1 : 0;
  }();
  P.trace = trace;
  const uintptr_t ea = reinterpret_cast<uintptr_t>(P.E);
  P.vec = (a.K % 4 == 0 && ea % 32 == 0) ? 2 : (a.K % 2 == 0 && ea % 16 == 0) ? 1 : 0;
  const u64 wbytes = u64(ntiles) * P.nkb * 3 * 8 * kT3A;
  auto wblk = s.raw((wbytes + 7) / 8);
  P.Wpk = reinterpret_cast<const char*>(wblk->ptr);
  {
    ClassScope pack_scope(kClsOther, 0);  // the roofline probe times the GEMM kernel itself
    cudaEvent_t pe;
    probe_begin(s.stream, &pe);
    const u64 units = u64(ntiles) * P.nkb * 128 * 8;
    launch_pdl(pack_tc3, dim3(ew_blocks(units)), dim3(256), 0, s.stream, P, reinterpret_cast<char*>(wblk->ptr));
    probe_end(s.stream, pe);
  }
  cudaEvent_t pe;
  probe_begin(s.stream, &pe);
  static const u32 mfast_min = [] {  // N tiles from which the grid runs M tiles fastest
    const char* e = std::getenv("MPCG_TC3_MFAST");
    return e ? u32(std::atoi(e)) : 1000u;
  }();
  P.mfast = ntiles >= mfast_min ? 1 : 0;
  const dim3 grid = P.mfast ? dim3(mtiles, ntiles, 1) : dim3(ntiles, mtiles, 1);
  launch_pdl(ring_gemm_tc3, grid, dim3(kT3Threads), size_t(kT3Stages) * kT3Stage, s.stream, P);
  probe_end(s.stream, pe);
  s.check();
  return true;
}

void tc3_trace_read(unsigned long long* out, int n) {
  const int m = n < kT3TraceRows * 8 ? n : kT3TraceRows * 8;
  MPCG_CUDA(cudaMemcpyFromSymbol(out, g_tc3_trace, sizeof(unsigned long long) * size_t(m)));
}

}  // namespace mpcg
