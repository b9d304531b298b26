// tcgen05 / mbarrier / bulk-copy helpers shared by the int8-limb ring GEMMs (gemm_tc2.cu,
// gemm_tc3.cu): PTX wrappers, UMMA descriptors, limb-plane byte transposes, TMEM loads and the
// dealer draw / operand load vectors of the producer warps.
#pragma once
#include "gemm.cuh"

namespace mpcg {
namespace {

constexpr int kKB = 32;  // K values (= limb bytes) per stage: one UMMA K slab
constexpr int kVW = 8;   // K values per producer unit of the unsplit tc2 producers

__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// The waiting thread is suspended in try_wait (time hint 10 ms, i.e. until the phase completes)
// instead of re-issuing the test: spinning waiters (producers ahead of the MMA, the loader)
// otherwise take issue slots from the producer warps that share their SM sub-partition.
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// K-major SWIZZLE_NONE descriptor (version 1): LBO between the two 16-B K chunks, SBO between
// 8-row groups.
__device__ __forceinline__ u64 smem_desc(u32 addr, u32 lbo, u32 sbo) {
  return u64((addr >> 4) & 0x3FFF) | (u64((lbo >> 4) & 0x3FFF) << 16) | (u64((sbo >> 4) & 0x3FFF) << 32) |
         (u64(1) << 46);
}
// kind::i8, D = s32, A/B unsigned 8-bit, both K-major.
__host__ __device__ constexpr u32 idesc_i8(u32 M, u32 N) { return (2u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24); }

__device__ __forceinline__ void mma_i8(u32 d_tmem, u64 adesc, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// A operand from TMEM (lanes = rows, 4 K bytes per 32-bit column), B from shared memory.
__device__ __forceinline__ void mma_i8_ts(u32 d_tmem, u32 a_tmem, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ u32 gather4(u32 a, u32 b, u32 c, u32 d, u32 l) {
  const u32 sel = l | ((l + 4) << 4);
  return __byte_perm(__byte_perm(a, b, sel), __byte_perm(c, d, sel), 0x5410);
}


__device__ __forceinline__ void draws16(u64 key, u64 c0, u64 (&v)[16], const u64* pool) {
  if (pool) {  // materialised triple (queue source): draw c at pool[c - 1]
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __ldg(pool + c0 - 1 + i);
    return;
  }
  u64 z = key + c0 * kPhi;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = mix64(z);
    z += kPhi;
  }
}
__device__ __forceinline__ void load16(const u64* p, u64 (&v)[16]) {
  const uint4* p4 = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 w = __ldg(p4 + i);
    v[2 * i] = (u64(w.y) << 32) | w.x;
    v[2 * i + 1] = (u64(w.w) << 32) | w.z;
  }
}
__device__ __forceinline__ void load16w(const u64* p, u64 (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(v[4 * i]), "=l"(v[4 * i + 1]), "=l"(v[4 * i + 2]), "=l"(v[4 * i + 3])
        : "l"(p + 4 * i));
}
// The same 16-value unit stored into a TMEM A stage instead: this thread's lane, columns
// plane*8 + base (+0..3) — 8 tcgen05.st of 4 columns.
__device__ __forceinline__ void transpose16_tmem(const u64 (&v)[16], u32 taddr) {
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    const int sh = (l & 3), hi = l >> 2;
    u32 w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = hi ? u32(v[i] >> 32) : u32(v[i]);
    const u32 x = gather4(w[0], w[1], w[2], w[3], sh), y = gather4(w[4], w[5], w[6], w[7], sh),
              z = gather4(w[8], w[9], w[10], w[11], sh), t = gather4(w[12], w[13], w[14], w[15], sh);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr + u32(l) * 8), "r"(x),
                 "r"(y), "r"(z), "r"(t)
                 : "memory");
  }
}

// kVW dealer draws c0, c0+1, ... of one stream (key + c*phi advances by phi).
__device__ __forceinline__ void draws_vec(u64 key, u64 c0, u64 (&v)[kVW], const u64* pool) {
  if (pool) {
#pragma unroll
    for (int i = 0; i < kVW; ++i) v[i] = __ldg(pool + c0 - 1 + i);
    return;
  }
  u64 z = key + c0 * kPhi;
#pragma unroll
  for (int i = 0; i < kVW; ++i) {
    v[i] = mix64(z);
    z += kPhi;
  }
}
__device__ __forceinline__ void load_vec(const u64* p, u64 (&v)[kVW]) {
  const uint4* p4 = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < kVW / 2; ++i) {
    const uint4 w = __ldg(p4 + i);
    v[2 * i] = (u64(w.y) << 32) | w.x;
    v[2 * i + 1] = (u64(w.w) << 32) | w.z;
  }
}
__device__ __forceinline__ void load_vecw(const u64* p, u64 (&v)[kVW]) {
#pragma unroll
  for (int i = 0; i < kVW / 4; ++i)
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(v[4 * i]), "=l"(v[4 * i + 1]), "=l"(v[4 * i + 2]), "=l"(v[4 * i + 3])
        : "l"(p + 4 * i));
}
__device__ __forceinline__ void transpose8_tmem(const u64 (&v)[kVW], u32 taddr) {
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    const int sh = (l & 3), hi = l >> 2;
    u32 w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = hi ? u32(v[i] >> 32) : u32(v[i]);
    const u32 x = gather4(w[0], w[1], w[2], w[3], sh), y = gather4(w[4], w[5], w[6], w[7], sh);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr + u32(l) * 8), "r"(x), "r"(y)
                 : "memory");
  }
}
// tcgen05.ld of W consecutive 32-bit TMEM columns of this warp's 32 lanes.
template <int W>
__device__ __forceinline__ void tmem_ld(u32 addr, u32 (&r)[W]) {
  if constexpr (W == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
  } else if constexpr (W == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
  } else {
    static_assert(W == 4, "tmem_ld width");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}



// 4x4 byte transpose: o[b] byte j = byte b of w[j] (8 PRMT for 4 output words, against 12 with
// gather4) — byte b of 4 K-consecutive values is one 4-byte word of limb plane b.
__device__ __forceinline__ void bt4(u32 w0, u32 w1, u32 w2, u32 w3, u32 (&o)[4]) {
  const u32 t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
  const u32 t2 = __byte_perm(w2, w3, 0x5140), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t2, 0x5410);
  o[1] = __byte_perm(t0, t2, 0x7632);
  o[2] = __byte_perm(t1, t3, 0x5410);
  o[3] = __byte_perm(t1, t3, 0x7632);
}
// 16 K-consecutive u64 -> the 16-byte row of each of the 8 limb planes: row[p] (uint4).
__device__ __forceinline__ void limb_rows16(const u64 (&v)[16], uint4 (&row)[8]) {
  u32 lo[4][4], hi[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bt4(u32(v[4 * j]), u32(v[4 * j + 1]), u32(v[4 * j + 2]), u32(v[4 * j + 3]), lo[j]);
    bt4(u32(v[4 * j] >> 32), u32(v[4 * j + 1] >> 32), u32(v[4 * j + 2] >> 32), u32(v[4 * j + 3] >> 32), hi[j]);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    row[p] = make_uint4(lo[0][p], lo[1][p], lo[2][p], lo[3][p]);
    row[p + 4] = make_uint4(hi[0][p], hi[1][p], hi[2][p], hi[3][p]);
  }
}

// limb_rows16 + stores, low planes first so the low words die before the high ones are
// transposed (register pressure): row p at base + p*pstride.
__device__ __forceinline__ void limb_store16(const u64 (&v)[16], char* base, u32 pstride) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    u32 o[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      bt4(u32(v[4 * j] >> (32 * h)), u32(v[4 * j + 1] >> (32 * h)), u32(v[4 * j + 2] >> (32 * h)),
          u32(v[4 * j + 3] >> (32 * h)), o[j]);
#pragma unroll
    for (int p = 0; p < 4; ++p)
      *reinterpret_cast<uint4*>(base + u32(4 * h + p) * pstride) = make_uint4(o[0][p], o[1][p], o[2][p], o[3][p]);
  }
}
// 16 K-consecutive u64 -> one 16-byte row in each of the 8 limb planes.
__device__ __forceinline__ void transpose16_store(const u64 (&v)[16], char* base, u32 plane, u32 off) {
  limb_store16(v, base + off, plane);
}
// 8 K-consecutive u64 -> one 8-byte row segment in each of the 8 limb planes.
__device__ __forceinline__ void transpose8_store(const u64 (&v)[kVW], char* base, u32 plane, u32 off) {
  u32 lo[2][4], hi[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    bt4(u32(v[4 * j]), u32(v[4 * j + 1]), u32(v[4 * j + 2]), u32(v[4 * j + 3]), lo[j]);
    bt4(u32(v[4 * j] >> 32), u32(v[4 * j + 1] >> 32), u32(v[4 * j + 2] >> 32), u32(v[4 * j + 3] >> 32), hi[j]);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    *reinterpret_cast<uint2*>(base + p * plane + off) = make_uint2(lo[0][p], lo[1][p]);
    *reinterpret_cast<uint2*>(base + (p + 4) * plane + off) = make_uint2(hi[0][p], hi[1][p]);
  }
}
// Four 8-column TMEM loads in flight, one wait: the wait names the 32 destination registers so
// the compiler cannot consume them before the loads have landed.
__device__ __forceinline__ void tmem_ld4x8(u32 a0, u32 a1, u32 a2, u32 a3, u32 (&r)[32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const u32 ad = i == 0 ? a0 : i == 1 ? a1 : i == 2 ? a2 : a3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[8 * i]), "=r"(r[8 * i + 1]), "=r"(r[8 * i + 2]), "=r"(r[8 * i + 3]), "=r"(r[8 * i + 4]),
                   "=r"(r[8 * i + 5]), "=r"(r[8 * i + 6]), "=r"(r[8 * i + 7])
                 : "r"(ad));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
                 "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

}  // namespace
}  // namespace mpcg
