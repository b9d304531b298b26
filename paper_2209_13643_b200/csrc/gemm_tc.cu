// tcgen05 int8-limb ring GEMM over Z_2^64 (sm_100a).
//
// x*y mod 2^64 = sum_{l+m<=7} x_l*y_m * 2^(8(l+m)) for the u8 limbs x_l, y_m of the u64
// operands (the int8 plan generalising LimbPlan, H/ring/limb.hpp:15-99). For one output tile
// the 36 limb-pair products run as tcgen05.mma.kind::i8 (u8 x u8 -> s32) into 8 TMEM
// accumulators, one per diagonal d = l+m:
//   D_d = sum_{l+m=d} L_l * R_m        (K' = nseg*K products per pair)
// and the epilogue recombines  z = sum_d 2^(8d) * D_d  mod 2^64.
// Exactness: diagonals d >= 4 are only needed mod 2^(64-8d) <= 2^32, so the s32 wrap is
// harmless; d <= 3 need the exact sum, i.e. 4*K'*255^2 < 2^32  =>  K' <= 16384 per pass.
//
// Operands are u64 matrices in HBM (segments of the Beaver combine, see gemm.cu). Producer
// threads load u64 values, byte-transpose 16 K-consecutive values into 8 limb planes in
// registers (PRMT) and store 16-byte rows of K-major core matrices (8 rows x 16 B,
// SWIZZLE_NONE) into shared memory; one elected thread issues the MMAs; tcgen05.commit on
// an mbarrier releases each smem stage back to the producers (2-stage pipeline).
#include "gemm.cuh"

namespace mpcg {

namespace {

constexpr int kTM = 128;        // tile rows (UMMA M)
constexpr int kKB = 64;         // K elements (= bytes per limb row) per pipeline stage
constexpr int kThreads = 512;   // 16 warps: producers (1 A unit each), MMA issuer (thread 0), epilogue
constexpr u32 kMaxKPrime = 16384;

__device__ __forceinline__ u32 smem_u32(const void* p) {
  return static_cast<u32>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// K-major, no-swizzle UMMA shared-memory descriptor (version 1 for Blackwell).
// LBO: byte distance between the two 16-byte K chunks of an MMA; SBO: between 8-row groups.
__device__ __forceinline__ u64 smem_desc(u32 addr, u32 lbo, u32 sbo) {
  u64 d = 0;
  d |= u64((addr >> 4) & 0x3FFF);
  d |= u64((lbo >> 4) & 0x3FFF) << 16;
  d |= u64((sbo >> 4) & 0x3FFF) << 32;
  d |= u64(1) << 46;  // version
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor: kind::i8, D = s32, A/B unsigned 8-bit, both K-major.
__host__ __device__ constexpr u32 idesc_i8(u32 M, u32 N) {
  return (2u << 4)            // c_format = S32
         | (0u << 7)          // a_format = unsigned 8-bit
         | (0u << 10)         // b_format = unsigned 8-bit
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

__device__ __forceinline__ void mma_i8(u32 d_tmem, u64 adesc, u64 bdesc, u32 idesc, u32 accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Byte l (0..3) of four 32-bit words a,b,c,d packed into one word [a_l, b_l, c_l, d_l].
__device__ __forceinline__ u32 gather4(u32 a, u32 b, u32 c, u32 d, u32 l) {
  const u32 sel = l | ((l + 4) << 4);
  const u32 t0 = __byte_perm(a, b, sel);
  const u32 t1 = __byte_perm(c, d, sel);
  return __byte_perm(t0, t1, 0x5410);
}

// 16 u64 values (K-consecutive) -> 8 limb rows of 16 bytes, stored to the planes.
// plane p row is at base + p*plane_bytes + off.
__device__ __forceinline__ void transpose_store(const u64 (&v)[16], char* base, u32 plane_bytes, u32 off) {
  u32 lo[16], hi[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    lo[i] = u32(v[i]);
    hi[i] = u32(v[i] >> 32);
  }
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    const u32* s = l < 4 ? lo : hi;
    const u32 b = u32(l & 3);
    uint4 w;
    w.x = gather4(s[0], s[1], s[2], s[3], b);
    w.y = gather4(s[4], s[5], s[6], s[7], b);
    w.z = gather4(s[8], s[9], s[10], s[11], b);
    w.w = gather4(s[12], s[13], s[14], s[15], b);
    *reinterpret_cast<uint4*>(base + l * plane_bytes + off) = w;
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) ring_gemm_tc_kernel(const __grid_constant__ GemmArgs a) {
  constexpr u32 kAPlane = kTM * kKB;       // bytes per A limb plane per stage (8 KB)
  constexpr u32 kBPlane = BN * kKB;        // bytes per B limb plane per stage
  constexpr u32 kStage = 8 * (kAPlane + kBPlane);
  constexpr u32 kCols = 8 * BN;            // TMEM columns: one s32 accumulator per diagonal
  constexpr int kBUnits = BN * (kKB / 16);
  static_assert(kCols <= 512, "TMEM budget");
  static_assert(kTM * (kKB / 16) == kThreads, "one A unit per thread per stage");
  extern __shared__ __align__(1024) char smem[];
  __shared__ u64 bar_empty[2];
  __shared__ u64 bar_done;
  __shared__ u32 tmem_base_slot;

  pdl_enter();
  const int tid = threadIdx.x, warp = tid >> 5;
  const int slot = blockIdx.z % a.nslots;
  const u32 b = blockIdx.z / a.nslots;
  const GemmSlotArgs& S = a.sl[slot];
  const u32 M = a.M, N = a.N, K = a.K;
  const u32 m0 = blockIdx.y * kTM, n0 = blockIdx.x * BN;

  if (tid == 0) {
    mbar_init(&bar_empty[0], 1);
    mbar_init(&bar_empty[1], 1);
    mbar_init(&bar_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = tmem_base_slot;

  const u32 steps = (u32(S.nseg) * K + kKB - 1) / kKB;
  constexpr u32 idesc = idesc_i8(kTM, BN);
  u32 phase[2] = {0, 0};

  // this thread's units: A (row ra, k-chunk ka) always; B (row rb, k-chunk kb) if tid < kBUnits
  const int ra = tid % kTM, ka = tid / kTM;
  const bool hasB = tid < kBUnits;
  const int rb = tid % BN, kbc = tid / BN;
  u64 va[16], vb[16];
  // Register prefetch of step `st`'s operands (issued while earlier MMAs run). The segments
  // are packed back to back along K' = nseg*K, so small K (e.g. 25) is not padded per segment.
  const u32 KP = u32(S.nseg) * K;
  // base2: second addend of kOpSum segments (the opened E = own + peer eps), L side only.
  auto load16 = [&](const u64* const* base, const u64* const* base2, const int* kind, const u64* stride, bool trans,
                    u32 row, u32 rows, u32 kp, u64 (&v)[16]) {
    // 16 K'-consecutive values of `row` starting at packed index kp
    const u32 sg0 = kp / K;
    if (row < rows && kp + 16 <= KP && sg0 == (kp + 15) / K && a.vec16 && (trans || base == S.L)) {
      const u32 k = kp - sg0 * K;
      const u64 off = u64(b) * stride[sg0] + u64(row) * K + k;
      const uint4* p4 = reinterpret_cast<const uint4*>(base[sg0] + off);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 w = __ldg(p4 + i);
        v[2 * i] = (u64(w.y) << 32) | w.x;
        v[2 * i + 1] = (u64(w.w) << 32) | w.z;
      }
      if (kind && kind[sg0] == kOpSum) {
        const uint4* q4 = reinterpret_cast<const uint4*>(base2[sg0] + off);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 w = __ldg(q4 + i);
          v[2 * i] += (u64(w.y) << 32) | w.x;
          v[2 * i + 1] += (u64(w.w) << 32) | w.z;
        }
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      u64 x = 0;
      const u32 q = kp + i;
      if (row < rows && q < KP) {
        const u32 sg = q / K, k = q - sg * K;
        const u64 off = u64(b) * stride[sg] + (trans ? u64(row) * K + k : u64(k) * N + row);
        x = __ldg(base[sg] + off);
        if (kind && kind[sg] == kOpSum) x += __ldg(base2[sg] + off);
      }
      v[i] = x;
    }
  };
  auto load_step = [&](u32 st) {
    const u32 k0 = st * kKB;
    load16(S.L, S.L2, S.lk, S.sL, true, m0 + ra, M, k0 + ka * 16, va);  // A rows are K-contiguous
    if (hasB) load16(S.R, nullptr, nullptr, S.sR, a.tb != 0, n0 + rb, N, k0 + kbc * 16, vb);
  };

  if (steps > 0) load_step(0);
  for (u32 st = 0; st < steps; ++st) {
    const u32 stage = st & 1;
    char* sA = smem + stage * kStage;
    char* sB = sA + 8 * kAPlane;
    if (st >= 2) {  // the MMAs that read this stage two steps ago must be done
      mbar_wait(&bar_empty[stage], phase[stage]);
      phase[stage] ^= 1;
    }
    // core matrix (row group r/8, k chunk kc) at (kc*(rows/8) + r/8)*128, row r%8 at +16*(r%8)
    transpose_store(va, sA, kAPlane, (ka * (kTM / 8) + ra / 8) * 128 + (ra % 8) * 16);
    if (hasB) transpose_store(vb, sB, kBPlane, (kbc * (BN / 8) + rb / 8) * 128 + (rb % 8) * 16);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const u32 aBase = smem_u32(sA), bBase = smem_u32(sB);
#pragma unroll
      for (int j = 0; j < kKB / 32; ++j) {  // MMA K-slabs of 32 bytes per stage
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const u64 ad = smem_desc(aBase + l * kAPlane + 2 * j * (kTM / 8) * 128, (kTM / 8) * 128, 128);
#pragma unroll
          for (int mm = 0; mm + l < 8; ++mm) {
            const u64 bd = smem_desc(bBase + mm * kBPlane + 2 * j * (BN / 8) * 128, (BN / 8) * 128, 128);
            const u32 acc = (st > 0 || j > 0 || l > 0) ? 1u : 0u;  // first MMA of a diagonal initialises
            mma_i8(tmem + u32(l + mm) * BN, ad, bd, idesc, acc);
          }
        }
      }
      mma_commit(&bar_empty[stage]);
    }
    if (st + 1 < steps) load_step(st + 1);
  }
  if (tid == 0) mma_commit(&bar_done);
  mbar_wait(&bar_done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- epilogue: warp w reads TMEM lanes 32*(w%4).. (its rows) and column group w/4;
  // recombine the diagonals z = sum_d D_d << 8d (mod 2^64) and apply the Beaver epilogue.
  constexpr int kCW = BN / 4;  // columns per warp
  const int q = warp & 3, cg = warp >> 2;
  const u32 row = u32(q) * 32 + (tid & 31);
  const u32 m = m0 + row;
  const u32 lane_addr = tmem + ((u32(q) * 32) << 16) + u32(cg * kCW);
  u64 acc[kCW];
#pragma unroll
  for (int c = 0; c < kCW; ++c) acc[c] = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    u32 r[kCW];
    if constexpr (kCW == 16) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(lane_addr + u32(d) * BN));
    } else if constexpr (kCW == 8) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(lane_addr + u32(d) * BN));
    } else {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                   : "r"(lane_addr + u32(d) * BN));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int c = 0; c < kCW; ++c) acc[c] += u64(r[c]) << (8 * d);
  }
  if (m < M) {
#pragma unroll
    for (int c = 0; c < kCW; ++c) {
      const u32 n = n0 + u32(cg * kCW + c);
      if (n < N) gemm_epilogue(a, S, b, m, n, acc[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}

template <int BN>
void launch_tc(Session& s, const GemmArgs& a) {
  constexpr u32 kStage = 8 * (kTM * kKB + BN * kKB);
  const size_t smem = 2 * kStage;
  static bool attr_set = false;
  if (!attr_set) {
    MPCG_CUDA(cudaFuncSetAttribute(ring_gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
    attr_set = true;
  }
  dim3 grid((a.N + BN - 1) / BN, (a.M + kTM - 1) / kTM, a.nslots * a.nbatch);
  cudaEvent_t pe;
  probe_begin(s.stream, &pe);
  launch_pdl(ring_gemm_tc_kernel<BN>, grid, dim3(kThreads), smem, s.stream, a);
  probe_end(s.stream, pe);
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

// Shapes worth the tensor cores: full 128-row tiles, N >= 32, exact-accumulation budget.
bool ring_gemm_tc_wants(const GemmArgs& a) {
  const int mode = tc_gemm_mode();
  if (mode == 0) return false;
  int maxseg = 0;
  for (int i = 0; i < a.nslots; ++i) maxseg = a.sl[i].nseg > maxseg ? a.sl[i].nseg : maxseg;
  if (u64(maxseg) * a.K > kMaxKPrime) return false;  // needs the multi-pass drain (not yet)
  if (a.ksplit > 1) return false;
  const double work = double(a.M) * a.N * a.K * maxseg * a.nbatch * a.nslots;
  // Full 128-row tiles and enough work to amortise the operand materialisation; the SIMT
  // path is issue-bound at ~9 instructions per ring MAC, so even N=6 convs win on the
  // tensor cores (N padded to 16).
  return mode == 1 || (a.M >= 128 && a.N >= 16 && work >= 3e7);
}

bool ring_gemm_tc_try(Session& s, const GemmArgs& a) {
  if (!ring_gemm_tc_wants(a)) return false;
  for (int i = 0; i < a.nslots; ++i)  // the producer reads memory operands (L: plain or own + peer)
    for (int g = 0; g < a.sl[i].nseg; ++g)
      if ((a.sl[i].lk[g] != kOpMem && a.sl[i].lk[g] != kOpSum) || a.sl[i].rk[g] != kOpMem) return false;
  GemmArgs v = a;
  bool al = (a.K % 2) == 0;
  for (int i = 0; i < a.nslots && al; ++i)
    for (int g = 0; g < a.sl[i].nseg; ++g) {
      al = al && (reinterpret_cast<uintptr_t>(a.sl[i].L[g]) % 16 == 0) && (a.sl[i].sL[g] % 2 == 0);
      if (a.sl[i].lk[g] == kOpSum) al = al && (reinterpret_cast<uintptr_t>(a.sl[i].L2[g]) % 16 == 0);
      if (a.tb) al = al && (reinterpret_cast<uintptr_t>(a.sl[i].R[g]) % 16 == 0) && (a.sl[i].sR[g] % 2 == 0);
    }
  v.vec16 = al ? 1 : 0;
  if (a.N > 32)
    launch_tc<64>(s, v);
  else if (a.N > 16)
    launch_tc<32>(s, v);
  else
    launch_tc<16>(s, v);
  s.check();
  return true;
}

}  // namespace mpcg
