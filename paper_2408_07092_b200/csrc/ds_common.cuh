// ds_common.cuh -- element types and sm_100a PTX helpers shared by the
// Double Sparsity kernels (product code; shares nothing with oracle/).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace ds {

// ---------------------------------------------------------------- types
template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kBytes = 2;
  __device__ static __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ static __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
  // unpack two packed elements of a 32-bit word (lo = element 0)
  __device__ static __forceinline__ float2 unpack2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  }
};
template <> struct Elem<__half> {
  static constexpr int kBytes = 2;
  __device__ static __forceinline__ float to_f(__half x) { return __half2float(x); }
  __device__ static __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
  __device__ static __forceinline__ float2 unpack2(uint32_t w) {
    __half2 h = *reinterpret_cast<__half2 *>(&w);
    return __half22float2(h);
  }
};
template <> struct Elem<float> {
  static constexpr int kBytes = 4;
  __device__ static __forceinline__ float to_f(float x) { return x; }
  __device__ static __forceinline__ float from_f(float x) { return x; }
};

// ------------------------------------------------------- cp.async (LDGSTS)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy global->shared; src_bytes = 0 zero-fills the 16 bytes.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ------------------------------------------------------ tensor-core MMA
__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                            uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
template <typename T> struct Mma;
template <> struct Mma<__nv_bfloat16> {
  __device__ static __forceinline__ void run(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                             uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};
template <> struct Mma<__half> {
  __device__ static __forceinline__ void run(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                             uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};

// m16n8k8: A 16x8 (a0 rows 0-7, a1 rows 8-15), B 8x8 (one register)
template <typename T> struct Mma8;
template <> struct Mma8<__nv_bfloat16> {
  __device__ static __forceinline__ void run(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(b0));
  }
};
template <> struct Mma8<__half> {
  __device__ static __forceinline__ void run(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(b0));
  }
};

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                                  uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// pack two fp32 into a 16-bit pair (lo = first), round-to-nearest-even
template <typename T> __device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
template <> __device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ----------------------------------------- programmatic dependent launch
// Kernels launched with cudaLaunchAttributeProgrammaticStreamSerialization
// may start while their predecessor drains.  Each kernel only touches data
// written by its immediate predecessor after pdl_wait(), and triggers its own
// dependents after that wait, so any pre-wait read is of data written two or
// more launches earlier (complete by then).  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// L2 prefetch of [p, p + bytes) (bulk, asynchronous, no data returned to the
// SM): safe before pdl_wait() even for data the predecessor may still write,
// since the L2 stays coherent and nothing is read into registers.  p and
// bytes are 16-B multiples.
__device__ __forceinline__ void prefetch_l2(const void *p, size_t bytes) {
  const char *a = static_cast<const char *>(p);
  for (size_t off = 0; off < bytes; off += 65536) {
    const uint32_t n = (uint32_t)(bytes - off < 65536 ? bytes - off : 65536) & ~15u;
    if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a + off), "r"(n) : "memory");
  }
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ------------------------------------------------------------- misc
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Monotone u32 key of an fp32 score: larger score <=> larger key; -0 and
// +0 map to the same key (DESIGN reading R6).
__device__ __forceinline__ uint32_t order_key(float s) {
  uint32_t u = __float_as_uint(s);
  if ((u & 0x7fffffffu) == 0u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ---------------------------------------------- 4-bit label (reading R16)
// code j of a packed row: nibble j (byte j/2, low nibble first), 4-bit
// two's complement
__device__ __forceinline__ int q4_code(const uint8_t *row, int j) {
  const int by = row[j >> 1];
  return (j & 1) ? ((int)(int8_t)by >> 4) : ((int)(int8_t)(by << 4) >> 4);
}
// fma chain over the 8 codes of a packed word (j ascending), each code
// exact and without an int->float conversion (I2F is a low-throughput pipe).
// a = w ^ 0x88888888 holds u_j = c_j + 8 in [1, 15] in nibble j.  Nibble j at
// bits [4j, 4j + 4) (j <= 4), masked out and OR-ed with the exponent of
// 2^(23 - 4j), is the float 2^(23 - 4j) + u_j exactly (its lowest set
// mantissa bit weighs 1), so c_j = that - (2^(23 - 4j) + 8); nibbles 5..7 do
// the same on a >> 20.  One LOP3 + one FADD per code, one SHF per word.
template <uint32_t MASK>
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t orv) {
  uint32_t d;  // (a & MASK) | orv in one LOP3
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(MASK), "r"(orv));
  return d;
}
__device__ __forceinline__ float q4_word_dot(uint32_t w, const float *ql, float acc) {
  const uint32_t a = w ^ 0x88888888u, b = a >> 20;
  const float c0 = __uint_as_float(lop3_and_or<0x0000Fu>(a, 0x4B000000u)) - 8388616.0f;  // 2^23 + 8
  const float c1 = __uint_as_float(lop3_and_or<0x000F0u>(a, 0x49000000u)) - 524296.0f;   // 2^19 + 8
  const float c2 = __uint_as_float(lop3_and_or<0x00F00u>(a, 0x47000000u)) - 32776.0f;    // 2^15 + 8
  const float c3 = __uint_as_float(lop3_and_or<0x0F000u>(a, 0x45000000u)) - 2056.0f;     // 2^11 + 8
  const float c4 = __uint_as_float(lop3_and_or<0xF0000u>(a, 0x43000000u)) - 136.0f;      // 2^7 + 8
  const float c5 = __uint_as_float(lop3_and_or<0x0000Fu>(b, 0x4B000000u)) - 8388616.0f;
  const float c6 = __uint_as_float(lop3_and_or<0x000F0u>(b, 0x49000000u)) - 524296.0f;
  const float c7 = __uint_as_float(lop3_and_or<0x00F00u>(b, 0x47000000u)) - 32776.0f;
  acc = fmaf(ql[0], c0, acc);
  acc = fmaf(ql[1], c1, acc);
  acc = fmaf(ql[2], c2, acc);
  acc = fmaf(ql[3], c3, acc);
  acc = fmaf(ql[4], c4, acc);
  acc = fmaf(ql[5], c5, acc);
  acc = fmaf(ql[6], c6, acc);
  acc = fmaf(ql[7], c7, acc);
  return acc;
}
// Two 4-bit label rows at once with packed fp32 pairs (sm_100 FADD2 /
// FFMA2): each lane of add.rn.f32x2 / fma.rn.f32x2 is the scalar RN
// operation, so both chains are bit-identical to q4_word_dot's (same codes,
// same j order).  A pair instruction issues in 2 cycles against 1 for the
// scalar one -- the same fp32 rate -- but half the issue slots, and the
// 4-bit stream is issue-bound (~40 instructions per token with scalars).
typedef unsigned long long u64;
__device__ __forceinline__ u64 pack_u2(uint32_t lo, uint32_t hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack_f2(u64 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ u64 fadd2(u64 x, u64 y) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  return r;
}
__device__ __forceinline__ u64 fmul2(u64 x, u64 y) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  return r;
}
__device__ __forceinline__ void ffma2(u64 &acc, u64 x, u64 y) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(y));
}
template <uint32_t MASK, uint32_t E, uint32_t NEGK>
__device__ __forceinline__ u64 q4_code2(uint32_t a, uint32_t b) {  // {c_j of a, c_j of b} as exact fp32
  return fadd2(pack_u2(lop3_and_or<MASK>(a, E), lop3_and_or<MASK>(b, E)), ((u64)NEGK << 32) | NEGK);
}
// qp[j] = {q_label[j], q_label[j]}; returns the two chains (no scale)
__device__ __forceinline__ float2 q4_pair_dot(uint32_t wa, uint32_t wb, const u64 *qp) {
  const uint32_t a = wa ^ 0x88888888u, as = a >> 20, b = wb ^ 0x88888888u, bs = b >> 20;
  u64 acc = 0ull;  // {+0, +0}, as q4_word_dot's acc = 0
  ffma2(acc, qp[0], q4_code2<0x0000Fu, 0x4B000000u, 0xcb000008u>(a, b));  // - (2^23 + 8)
  ffma2(acc, qp[1], q4_code2<0x000F0u, 0x49000000u, 0xc9000080u>(a, b));  // - (2^19 + 8)
  ffma2(acc, qp[2], q4_code2<0x00F00u, 0x47000000u, 0xc7000800u>(a, b));  // - (2^15 + 8)
  ffma2(acc, qp[3], q4_code2<0x0F000u, 0x45000000u, 0xc5008000u>(a, b));  // - (2^11 + 8)
  ffma2(acc, qp[4], q4_code2<0xF0000u, 0x43000000u, 0xc3080000u>(a, b));  // - (2^7 + 8)
  ffma2(acc, qp[5], q4_code2<0x0000Fu, 0x4B000000u, 0xcb000008u>(as, bs));
  ffma2(acc, qp[6], q4_code2<0x000F0u, 0x49000000u, 0xc9000080u>(as, bs));
  ffma2(acc, qp[7], q4_code2<0x00F00u, 0x47000000u, 0xc7000800u>(as, bs));
  return unpack_f2(acc);
}
// 16-B / 8-B read-only loads issued where they are written (asm volatile:
// the compiler cannot sink a prefetch below the work it overlaps)
__device__ __forceinline__ uint4 ldg_nc_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void *p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];\n" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
// line 2 over a 4-bit label row: (fp32 fma chain of q_label[j] * c_j) * s
template <typename T>
__device__ __forceinline__ float q4_score(const uint8_t *row, T scale, const float *ql, int r) {
  float acc = 0.0f;
  for (int j = 0; j < r; ++j) acc = fmaf(ql[j], (float)q4_code(row, j), acc);
  return acc * Elem<T>::to_f(scale);
}

// Inverse of order_key (the canonical +0 for the zero key).
__device__ __forceinline__ float key_to_float(uint32_t key) {
  const uint32_t u = (key & 0x80000000u) ? (key & 0x7fffffffu) : ~key;
  return __uint_as_float(u);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --------------------------------------------------- histogram boundary
// One warp: boundary of a histogram held NPL bins per lane, bins in
// descending order hi_bin - NPL*lane - j.  With `base` keys above the
// first bin and `need` wanted from the top, returns the bin d with
// above(d) < need <= above(d) + cnt(d).
template <int NPL>
struct Boundary {
  int bin;
  uint32_t above, cnt;
};
template <int NPL>
__device__ __forceinline__ Boundary<NPL> warp_boundary(const uint32_t (&v)[NPL], int hi_bin, uint32_t base,
                                                       uint32_t need) {
  const int lane = threadIdx.x & 31;
  uint32_t tot = 0;
#pragma unroll
  for (int j = 0; j < NPL; ++j) tot += v[j];
  uint32_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  uint32_t run = base + incl - tot;
  int hit = -1;
  uint32_t ha = 0, hc = 0;
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    if (hit < 0 && run < need && run + v[j] >= need) {
      hit = j;
      ha = run;
      hc = v[j];
    }
    run += v[j];
  }
  const uint32_t m = __ballot_sync(0xffffffffu, hit >= 0);
  const int src = m ? __ffs(m) - 1 : 31;
  Boundary<NPL> r;
  r.bin = hi_bin - NPL * src - __shfl_sync(0xffffffffu, hit < 0 ? 0 : hit, src);
  r.above = __shfl_sync(0xffffffffu, ha, src);
  r.cnt = __shfl_sync(0xffffffffu, hc, src);
  return r;
}

// named barriers (id 0 is __syncthreads)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace ds

// ------------------------------------------------------------ tracing
// Debug builds only (-DDS_TRACE, libds_trace.so): thread 0 of each CTA
// stamps %globaltimer at phase boundaries; read back with
// ds_debug_read_trace().  The product library compiles these to nothing.
#ifdef DS_TRACE
namespace ds {
constexpr int kTraceCtas = 4096, kTraceSlots = 16;
__device__ unsigned long long g_trace[3][kTraceCtas][kTraceSlots];  // unity trace build: one TU
}
#define DS_TRACE_AT(kind, slot) DS_TRACE_BY(kind, slot, 0)
#define DS_TRACE_BY(kind, slot, thread)                                                      \
  do {                                                                                       \
    const unsigned cta_ = blockIdx.x + blockIdx.y * gridDim.x;                              \
    if (threadIdx.x == (thread) && cta_ < (unsigned)ds::kTraceCtas) {                        \
      unsigned long long t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
      ds::g_trace[kind][cta_][slot] = t_;                                                    \
    }                                                                                        \
  } while (0)
#else
#define DS_TRACE_AT(kind, slot) \
  do {                          \
  } while (0)
#define DS_TRACE_BY(kind, slot, thread) \
  do {                                  \
  } while (0)
#endif
