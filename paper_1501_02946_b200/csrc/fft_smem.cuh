// Shared-memory power-of-two FFTs used by the lateral, NER and inverse
// kernels.  In-place radix-2^R decimation in time: the caller stores the
// input in bit-reversed order, every thread then owns 2^R points of one
// transform per pass and does R radix-2 stages in registers.
//
// Layout is abstracted by an address functor so the same passes run on
//  * a single long transform with bank-conflict padding (NER rows), and
//  * P interleaved transforms of a [len][P] tile whose fast axis is the
//    batch (lateral FFTs over a chunk of consecutive time samples), which
//    is conflict-free because neighbouring threads own neighbouring batches.
//
// Twiddles come from one table tw[k] = exp(-2 pi i k / 2^LMAX); a length-2^L
// transform reads it with stride 2^(LMAX-L).
#pragma once
#include <type_traits>

#include <cuda_runtime.h>

namespace patfft {
namespace fft {

constexpr int kLogTwiddles = 14;  // table length 16384
// Per-pass twiddle tables behind the main table (host: make_twiddles): for a
// pass at half-length H = 2^LOGH (1 <= LOGH <= kPassTwMaxLog), item offset k
// reads its R <= 4 stage twiddles W_{H 2^(i+1)}^k, i = 0..3, as 4 consecutive
// float2 at kPassTwOffset(LOGH) + 4k.  Neighbouring items (lanes) then read
// neighbouring 32-byte blocks instead of gathering single float2 at a stride
// of 2^(14-LOGH-i-1) -- in the single-transform NER passes those strided
// gathers were 60% of the L1 data-pipe wavefronts.
constexpr int kPassTwMaxLog = 12;
__host__ __device__ constexpr int kPassTwOffset(int logh) { return (1 << kLogTwiddles) + 4 * ((1 << logh) - 2); }
constexpr int kTwiddleTableLen = kPassTwOffset(kPassTwMaxLog + 1);

// Packed FP32 (sm_100a FADD2 / FMUL2 / FFMA2): one issue slot per complex
// add, two per complex multiply.  The compiler folds broadcast scalars,
// operand swaps and negations into the packed instructions' operand modifiers.
#define PATFFT_F2_BINOP(op)                                                                                  \
  __device__ __forceinline__ float2 f2##op(float2 a, float2 b) {                                           \
    float2 d;                                                                                               \
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t" #op                 \
        ".rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n}"                                                \
        : "=f"(d.x), "=f"(d.y)                                                                              \
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                                          \
    return d;                                                                                               \
  }
PATFFT_F2_BINOP(add)
PATFFT_F2_BINOP(sub)
PATFFT_F2_BINOP(mul)
#undef PATFFT_F2_BINOP

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// a * b = a.x * (b.x, b.y) + a.y * (-b.y, b.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return f2fma(make_float2(a.y, a.y), make_float2(-b.y, b.x), f2mul(make_float2(a.x, a.x), b));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return f2add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return f2sub(a, b); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return f2mul(a, make_float2(s, s)); }

// exp(-+2 pi i j / 32)
template <bool INV>
__device__ __forceinline__ float2 w32(int j) {
  const float c[32] = {1.0f, 0.98078528040323043f, 0.92387953251128674f, 0.83146961230254524f,
                       0.70710678118654752f, 0.55557023301960218f, 0.38268343236508977f, 0.19509032201612827f,
                       0.0f, -0.19509032201612827f, -0.38268343236508977f, -0.55557023301960218f,
                       -0.70710678118654752f, -0.83146961230254524f, -0.92387953251128674f, -0.98078528040323043f,
                       -1.0f, -0.98078528040323043f, -0.92387953251128674f, -0.83146961230254524f,
                       -0.70710678118654752f, -0.55557023301960218f, -0.38268343236508977f, -0.19509032201612827f,
                       0.0f, 0.19509032201612827f, 0.38268343236508977f, 0.55557023301960218f,
                       0.70710678118654752f, 0.83146961230254524f, 0.92387953251128674f, 0.98078528040323043f};
  const float s = c[(j + 24) & 31];  // sin(2 pi j/32) = cos(2 pi (j-8)/32)
  return make_float2(c[j & 31], INV ? s : -s);
}

struct PadAddr {  // single transform, 1 pad element per 16 (bank-conflict free radix-16 passes)
  __device__ __forceinline__ int operator()(int i, int) const { return i + (i >> 4); }
};
// Single transform of length 2^L, XOR-swizzled: the low 4 bits (the 8-byte
// slot within a 128-byte row) are XOR-ed with bits 4..7 and with the top 4
// bits.  Bijective, no padding, and conflict-free for the radix-16 passes,
// the bit-reversed input scatter (stride 2^(L-5) between lanes) and the
// stride-~4 interpolation gathers of the NER.
struct SwzAddr {
  int sh;  // L - 4 (31 when L < 8)
  __device__ __forceinline__ int operator()(int i, int) const { return i ^ (((i >> 4) ^ (i >> sh)) & 15); }
  static __device__ __forceinline__ SwzAddr for_log(int L) { return SwzAddr{L >= 8 ? L - 4 : 31}; }
};
struct TileAddr {  // [len][P] tile, batch fastest
  int plog;
  __device__ __forceinline__ int operator()(int i, int p) const { return (i << plog) + p; }
};

// One pass: stages logh+1 .. logh+R of P transforms of length 2^L.
template <int R, bool INV, class Addr>
__device__ __forceinline__ void dit_pass(float2* __restrict__ buf, int L, int plog, int logh,
                                         const float2* __restrict__ tw, int tid, int nth, Addr addr) {
  constexpr int PR = 1 << R;
  const int h = 1 << logh;
  const int items = 1 << (L - R + plog);
  const int pmask = (1 << plog) - 1;
  for (int it = tid; it < items; it += nth) {
    const int p = it & pmask;
    const int q = it >> plog;
    const int k = q & (h - 1);
    const int base = ((q >> logh) << (logh + R)) + k;
    float2 e[PR];
#pragma unroll
    for (int m = 0; m < PR; ++m) e[m] = buf[addr(base + m * h, p)];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      float2 wi = __ldg(&tw[k << (kLogTwiddles - logh - i - 1)]);  // W_{h 2^{i+1}}^k
      if (INV) wi.y = -wi.y;
#pragma unroll
      for (int r = 0; r < (1 << i); ++r) {
        const float2 t = (r == 0) ? wi : cmul(wi, w32<INV>(r << (4 - i)));
#pragma unroll
        for (int m0 = 0; m0 < PR; m0 += (2 << i)) {
          const int m = m0 + r;
          const float2 x = cmul(e[m + (1 << i)], t);
          e[m + (1 << i)] = csub(e[m], x);
          e[m] = cadd(e[m], x);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < PR; ++m) buf[addr(base + m * h, p)] = e[m];
  }
}

// Radix of the pass starting at stage logh of a length-2^L transform: as few
// passes as possible (at most MAXR stages, i.e. 2^MAXR points per thread),
// split evenly so no pass degenerates to radix 2.
// EVEN: split the stages evenly over the passes (e.g. 10 = 4+3+3) instead of
// greedily (10 = 4+4+2); which one is faster depends on the kernel's
// threads per transform and register budget (measured).
template <int MAXR, bool EVEN>
__device__ __forceinline__ int pass_radix(int L, int logh) {
  const int left = L - logh;
  if (!EVEN) return left < MAXR ? left : MAXR;
  const int passes = (left + MAXR - 1) / MAXR;
  return (left + passes - 1) / passes;
}

// Full transform (input already bit-reversed); ends with __syncthreads.
template <bool INV, int MAXR, bool EVEN, class Addr>
__device__ __forceinline__ void fft_inplace(float2* __restrict__ buf, int L, int plog, const float2* __restrict__ tw,
                                            int tid, int nth, Addr addr) {
  int logh = 0;
  while (logh < L) {
    const int R = pass_radix<MAXR, EVEN>(L, logh);
    switch (R) {
      case 5: if constexpr (MAXR >= 5) dit_pass<5, INV>(buf, L, plog, logh, tw, tid, nth, addr); break;
      case 4: dit_pass<4, INV>(buf, L, plog, logh, tw, tid, nth, addr); break;
      case 3: dit_pass<3, INV>(buf, L, plog, logh, tw, tid, nth, addr); break;
      case 2: dit_pass<2, INV>(buf, L, plog, logh, tw, tid, nth, addr); break;
      default: dit_pass<1, INV>(buf, L, plog, logh, tw, tid, nth, addr); break;
    }
    logh += R;
    __syncthreads();
  }
}

__device__ __forceinline__ int brev(int i, int L) { return L ? (int)(__brev((unsigned)i) >> (32 - L)) : 0; }

// ---------------------------------------------------------------------------
// Compile-time variants: transform length 2^L, batch 2^PLOG and the CTA size
// NTH are template parameters, so the pass schedule, strides, masks and
// item loops fold to constants (used for the common power-of-two sizes; the
// runtime versions above remain the fallback).
// ---------------------------------------------------------------------------
template <int L>
struct SwzC {  // SwzAddr with a compile-time shift
  static constexpr bool kXorLinear = true;  // addr(a ^ b) == addr(a) ^ addr(b)
  static constexpr int sh = L >= 8 ? L - 4 : 31;
  __device__ __forceinline__ int operator()(int i, int) const { return i ^ (((i >> 4) ^ (i >> sh)) & 15); }
};
template <int PLOG>
struct TileC {
  __device__ __forceinline__ int operator()(int i, int p) const { return (i << PLOG) + p; }
};

// Element address of base + m*H.  The pass's base never shares a bit with
// m*H (base = k + multiples of H << R, k < H), so for an XOR-linear layout
// the address is addr(base) ^ addr(m*H) with the second term a compile-time
// constant: one LOP3 per access instead of the full swizzle.
template <class Addr, class = void>
struct XorLinear : std::false_type {};
template <class Addr>
struct XorLinear<Addr, std::void_t<decltype(Addr::kXorLinear)>> : std::bool_constant<Addr::kXorLinear> {};

// Radix-2^R DIT butterflies of one pass item (stages LOGH+1 .. LOGH+R),
// item offset k within the current half-length 2^LOGH.
template <int R, bool INV, int LOGH>
__device__ __forceinline__ void pass_butterflies(float2 (&e)[1 << R], int k, const float2* __restrict__ tw) {
  constexpr int PR = 1 << R;
  float2 wst[4];
  if constexpr (LOGH > 0 && LOGH <= kPassTwMaxLog) {
    const float4* pt = reinterpret_cast<const float4*>(tw + kPassTwOffset(LOGH) + 4 * k);
    const float4 a = __ldg(pt);
    wst[0] = make_float2(a.x, a.y);
    wst[1] = make_float2(a.z, a.w);
    if constexpr (R > 2) {
      const float4 b = __ldg(pt + 1);
      wst[2] = make_float2(b.x, b.y);
      wst[3] = make_float2(b.z, b.w);
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    float2 wi = make_float2(1.f, 0.f);
    if constexpr (LOGH > 0) {
      if constexpr (LOGH <= kPassTwMaxLog) wi = wst[i];
      else wi = __ldg(&tw[k << (kLogTwiddles - LOGH - i - 1)]);  // W_{H 2^{i+1}}^k
      if (INV) wi.y = -wi.y;
    }
#pragma unroll
    for (int r = 0; r < (1 << i); ++r) {
      const float2 t = (r == 0) ? wi : (LOGH > 0 ? cmul(wi, w32<INV>(r << (4 - i))) : w32<INV>(r << (4 - i)));
#pragma unroll
      for (int m0 = 0; m0 < PR; m0 += (2 << i)) {
        const int m = m0 + r;
        const float2 x = (LOGH == 0 && r == 0) ? e[m + (1 << i)] : cmul(e[m + (1 << i)], t);
        e[m + (1 << i)] = csub(e[m], x);
        e[m] = cadd(e[m], x);
      }
    }
  }
}

template <int R, bool INV, int L, int PLOG, int LOGH, int NTH, class Addr>
__device__ __forceinline__ void dit_pass_ct(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                            Addr addr) {
  constexpr int PR = 1 << R;
  constexpr int H = 1 << LOGH;
  constexpr int ITEMS = 1 << (L - R + PLOG);
  constexpr int ITER = (ITEMS + NTH - 1) / NTH;
#pragma unroll
  for (int j = 0; j < ITER; ++j) {
    const int it = tid + j * NTH;
    if ((ITEMS % NTH) != 0 && it >= ITEMS) break;
    const int p = it & ((1 << PLOG) - 1);
    const int q = it >> PLOG;
    const int k = q & (H - 1);
    const int base = ((q >> LOGH) << (LOGH + R)) + k;
    float2 e[PR];
    int ab = 0;
    if constexpr (XorLinear<Addr>::value) ab = addr(base, p);
#pragma unroll
    for (int m = 0; m < PR; ++m) {
      if constexpr (XorLinear<Addr>::value) e[m] = buf[ab ^ addr(m * H, 0)];
      else e[m] = buf[addr(base + m * H, p)];
    }
    pass_butterflies<R, INV, LOGH>(e, k, tw);
#pragma unroll
    for (int m = 0; m < PR; ++m) {
      if constexpr (XorLinear<Addr>::value) buf[ab ^ addr(m * H, 0)] = e[m];
      else buf[addr(base + m * H, p)] = e[m];
    }
  }
}

template <int L, int MAXR, bool EVEN, int LOGH>
struct PassRadix {
  static constexpr int left = L - LOGH;
  static constexpr int passes = (left + MAXR - 1) / MAXR;
  static constexpr int value = EVEN ? (left + passes - 1) / passes : (left < MAXR ? left : MAXR);
};

// Full compile-time transform (input bit-reversed); ends with __syncthreads.
template <bool INV, int L, int MAXR, bool EVEN, int PLOG, int NTH, int LOGH = 0, class Addr>
__device__ __forceinline__ void fft_ct(float2* __restrict__ buf, const float2* __restrict__ tw, int tid, Addr addr) {
  if constexpr (LOGH < L) {
    constexpr int R = PassRadix<L, MAXR, EVEN, LOGH>::value;
    dit_pass_ct<R, INV, L, PLOG, LOGH, NTH>(buf, tw, tid, addr);
    __syncthreads();
    fft_ct<INV, L, MAXR, EVEN, PLOG, NTH, LOGH + R>(buf, tw, tid, addr);
  }
}

constexpr int brev_c(int x, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1) << (bits - 1 - b);
  return r;
}

// log2(half-length) at which the last pass of the schedule starts
template <int L, int MAXR, bool EVEN, int LOGH = 0>
struct LastPassLogh {
  static constexpr int R = PassRadix<L, MAXR, EVEN, LOGH>::value;
  static constexpr int value = (LOGH + R >= L) ? LOGH : LastPassLogh<L, MAXR, EVEN, (LOGH + R >= L ? L : LOGH + R)>::value;
};
template <int L, int MAXR, bool EVEN>
struct LastPassLogh<L, MAXR, EVEN, L> {
  static constexpr int value = L;
};

// Passes LOGH.. of the schedule except the last one (each followed by a barrier).
template <bool INV, int L, int MAXR, bool EVEN, int PLOG, int NTH, int LOGH, class Addr>
__device__ __forceinline__ void fft_ct_but_last(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                                Addr addr) {
  constexpr int R = PassRadix<L, MAXR, EVEN, LOGH>::value;
  if constexpr (LOGH + R < L) {
    dit_pass_ct<R, INV, L, PLOG, LOGH, NTH>(buf, tw, tid, addr);
    __syncthreads();
    fft_ct_but_last<INV, L, MAXR, EVEN, PLOG, NTH, LOGH + R>(buf, tw, tid, addr);
  }
}

// Output `idx` (natural order) of a transform whose last radix-2^RL pass
// (half-length H = 2^(L-RL)) has not been run: the pass's inputs are the
// H-point DFTs D_r of the decimated sequences x[r + 2^RL s], stored in block
// brev(r) of the buffer, and Z[idx] = sum_r W_{2^L}^{idx r} D_r[idx mod H].
template <bool INV, int L, int RL, class Addr>
__device__ __forceinline__ float2 last_pass_output(const float2* __restrict__ buf, const float2* __restrict__ tw,
                                                   Addr addr, int idx, int p) {
  constexpr int H = 1 << (L - RL);
  const int s = idx & (H - 1);
  float2 acc = buf[addr(s, p)];
#pragma unroll
  for (int r = 1; r < (1 << RL); ++r) {
    float2 w = __ldg(&tw[((idx * r) & ((1 << L) - 1)) << (kLogTwiddles - L)]);
    if (INV) w.y = -w.y;
    acc = cadd(acc, cmul(buf[addr(brev_c(r, RL) * H + s, p)], w));
  }
  return acc;
}

// Global operands that are rows of a strided array: ptr(row, p) is the
// address of element (row, transform p), or nullptr when transform p is out
// of range (loads give zeros, stores are dropped); consecutive rows are
// `stride` float2 apart.  The first pass then loads an item's radix-2^R
// elements, and the last pass stores them, from one base pointer with a
// running offset instead of recomputing every address.
// MODE: 0 = default caching, 1 = streaming (evict-first, 256-byte L2 prefetch),
// 2 = L2-coherent (bypasses L1: rows another CTA of the same launch has just
// written), 3 = streaming with a 128-byte L2 prefetch
template <class F, int MODE>
struct RowsLd {
  F ptr;
  size_t stride;
};
template <class F>
struct RowsSt {
  F ptr;
  size_t stride;
};
template <int MODE = 1, class F>
__device__ __forceinline__ RowsLd<F, MODE> rows_ld(F f, size_t stride) {
  return {f, stride};
}
template <class F>
__device__ __forceinline__ RowsSt<F> rows_st(F f, size_t stride) {
  return {f, stride};
}
// element m of the first-pass item at natural row (brev(m) << (L - R)) + nat0
template <int R, int L, class Load>
__device__ __forceinline__ void load_items(float2 (&e)[1 << R], int nat0, int p, const Load& load) {
#pragma unroll
  for (int m = 0; m < (1 << R); ++m) e[m] = load((brev_c(m, R) << (L - R)) + nat0, p);
}
#ifndef PATFFT_LD_L2_PREFETCH
#define PATFFT_LD_L2_PREFETCH 256  // streaming first-pass loads with an L2 prefetch-size hint (0 / 128 / 256 bytes;
                                   // 256: lateral col + row 0.541 -> 0.535 ms)
#endif
__device__ __forceinline__ float2 ld_stream(const float2* a) {
#if PATFFT_LD_L2_PREFETCH == 256
  float2 v;
  asm volatile("ld.global.cs.L2::256B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
  return v;
#elif PATFFT_LD_L2_PREFETCH == 128
  float2 v;
  asm volatile("ld.global.cs.L2::128B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
  return v;
#else
  return __ldcs(a);
#endif
}
#ifndef PATFFT_INV_L2PF
#define PATFFT_INV_L2PF 1  // inverse kernels: row loads with the L2::256B hint (inverse 0.199 -> 0.197 ms)
#endif
__device__ __forceinline__ float2 ld_keep(const float2* a) {
#if PATFFT_INV_L2PF
  float2 v;
  asm volatile("ld.global.L2::256B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
  return v;
#else
  return *a;
#endif
}
__device__ __forceinline__ float2 ld_stream128(const float2* a) {
  float2 v;
  asm volatile("ld.global.cs.L2::128B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
  return v;
}
__device__ __forceinline__ float2 ld_l2(const float2* a) {
  float2 v;
  asm volatile("ld.global.cg.L2::256B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
  return v;
}
template <int R, int L, class F, int MODE>
__device__ __forceinline__ void load_items(float2 (&e)[1 << R], int nat0, int p, const RowsLd<F, MODE>& rl) {
  const float2* b = rl.ptr(nat0, p);
  const size_t st = rl.stride << (L - R);
  if (b) {
#pragma unroll
    for (int k = 0; k < (1 << R); ++k) e[brev_c(k, R)] = MODE == 3 ? ld_stream128(b + k * st) : MODE == 2 ? ld_l2(b + k * st) : MODE == 1 ? ld_stream(b + k * st) : ld_keep(b + k * st);
  } else {
#pragma unroll
    for (int k = 0; k < (1 << R); ++k) e[k] = make_float2(0.f, 0.f);
  }
}
// last-pass outputs m of an item at natural rows base + m H
template <int R, int H, class Store>
__device__ __forceinline__ void store_items(const float2 (&e)[1 << R], int base, int p, const Store& store) {
#pragma unroll
  for (int m = 0; m < (1 << R); ++m) store(base + m * H, p, e[m]);
}
template <int R, int H, class F>
__device__ __forceinline__ void store_items(const float2 (&e)[1 << R], int base, int p, const RowsSt<F>& rs) {
  float2* b = rs.ptr(base, p);
  if (!b) return;
  const size_t st = rs.stride * H;
#pragma unroll
  for (int m = 0; m < (1 << R); ++m) b[m * st] = e[m];
}

// Full compile-time transform whose first pass reads its inputs straight
// from `load(n, p)` (element n in natural order of transform p) instead of
// from a bit-reversed shared-memory copy: saves one shared-memory round trip.
// With a single transform (PLOG = 0) item q is given to thread brev(q), so a
// warp's loads are consecutive natural indices.  Ends with __syncthreads.
template <bool INV, int L, int MAXR, bool EVEN, int PLOG, int NTH, bool SKIP_LAST = false, class Addr, class Load>
__device__ __forceinline__ void fft_ct_loaded(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                              Addr addr, Load load) {
  constexpr int R = PassRadix<L, MAXR, EVEN, 0>::value;
  constexpr int PR = 1 << R;
  constexpr int ITEMS = 1 << (L - R + PLOG);
  constexpr int ITER = (ITEMS + NTH - 1) / NTH;
#pragma unroll
  for (int j = 0; j < ITER; ++j) {
    const int it = tid + j * NTH;
    if ((ITEMS % NTH) != 0 && it >= ITEMS) break;
    const int p = it & ((1 << PLOG) - 1);
    const int qi = it >> PLOG;
    const int q = PLOG == 0 ? brev(qi, L - R) : qi;
    const int nat0 = PLOG == 0 ? qi : brev(qi, L - R);  // natural index of element m = 0
    float2 e[PR];
    load_items<R, L>(e, nat0, p, load);
    pass_butterflies<R, INV, 0>(e, 0, tw);
    const int base = q << R;
    int ab = 0;
    if constexpr (XorLinear<Addr>::value) ab = addr(base, p);
#pragma unroll
    for (int m = 0; m < PR; ++m) {
      if constexpr (XorLinear<Addr>::value) buf[ab ^ addr(m, 0)] = e[m];
      else buf[addr(base + m, p)] = e[m];
    }
  }
  __syncthreads();
  if constexpr (SKIP_LAST) fft_ct_but_last<INV, L, MAXR, EVEN, PLOG, NTH, R>(buf, tw, tid, addr);
  else fft_ct<INV, L, MAXR, EVEN, PLOG, NTH, R>(buf, tw, tid, addr);
}


// Last pass that hands its outputs (natural order) to `store(n, p, v)`
// instead of writing them back to shared memory.  No trailing barrier.
template <int R, bool INV, int L, int PLOG, int LOGH, int NTH, class Addr, class Store>
__device__ __forceinline__ void dit_pass_ct_st(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                               Addr addr, Store store) {
  constexpr int PR = 1 << R;
  constexpr int H = 1 << LOGH;
  constexpr int ITEMS = 1 << (L - R + PLOG);
  constexpr int ITER = (ITEMS + NTH - 1) / NTH;
#pragma unroll
  for (int j = 0; j < ITER; ++j) {
    const int it = tid + j * NTH;
    if ((ITEMS % NTH) != 0 && it >= ITEMS) break;
    const int p = it & ((1 << PLOG) - 1);
    const int q = it >> PLOG;
    const int k = q & (H - 1);
    const int base = ((q >> LOGH) << (LOGH + R)) + k;
    float2 e[PR];
    int ab = 0;
    if constexpr (XorLinear<Addr>::value) ab = addr(base, p);
#pragma unroll
    for (int m = 0; m < PR; ++m) {
      if constexpr (XorLinear<Addr>::value) e[m] = buf[ab ^ addr(m * H, 0)];
      else e[m] = buf[addr(base + m * H, p)];
    }
    pass_butterflies<R, INV, LOGH>(e, k, tw);
    store_items<R, H>(e, base, p, store);
  }
}

// Passes LOGH.. of a compile-time transform, the last one storing through `store`.
template <bool INV, int L, int MAXR, bool EVEN, int PLOG, int NTH, int LOGH, class Addr, class Store>
__device__ __forceinline__ void fft_ct_tail_store(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                                  Addr addr, Store store) {
  constexpr int R = PassRadix<L, MAXR, EVEN, LOGH>::value;
  if constexpr (LOGH + R >= L) {
    dit_pass_ct_st<R, INV, L, PLOG, LOGH, NTH>(buf, tw, tid, addr, store);
  } else {
    dit_pass_ct<R, INV, L, PLOG, LOGH, NTH>(buf, tw, tid, addr);
    __syncthreads();
    fft_ct_tail_store<INV, L, MAXR, EVEN, PLOG, NTH, LOGH + R>(buf, tw, tid, addr, store);
  }
}

// Whole transform from shared memory (bit-reversed input) to `store`.
template <bool INV, int L, int MAXR, bool EVEN, int PLOG, int NTH, class Addr, class Store>
__device__ __forceinline__ void fft_ct_stored(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                              Addr addr, Store store) {
  fft_ct_tail_store<INV, L, MAXR, EVEN, PLOG, NTH, 0>(buf, tw, tid, addr, store);
}

// Whole transform from `load` (natural order) to `store`; needs >= 2 passes.
template <bool INV, int L, int MAXR, bool EVEN, int PLOG, int NTH, class Addr, class Load, class Store>
__device__ __forceinline__ void fft_ct_loaded_stored(float2* __restrict__ buf, const float2* __restrict__ tw, int tid,
                                                     Addr addr, Load load, Store store) {
  constexpr int R = PassRadix<L, MAXR, EVEN, 0>::value;
  static_assert(R < L, "single-pass transform: use fft_ct_loaded");
  constexpr int PR = 1 << R;
  constexpr int ITEMS = 1 << (L - R + PLOG);
  constexpr int ITER = (ITEMS + NTH - 1) / NTH;
#pragma unroll
  for (int j = 0; j < ITER; ++j) {
    const int it = tid + j * NTH;
    if ((ITEMS % NTH) != 0 && it >= ITEMS) break;
    const int p = it & ((1 << PLOG) - 1);
    const int qi = it >> PLOG;
    const int q = PLOG == 0 ? brev(qi, L - R) : qi;
    const int nat0 = PLOG == 0 ? qi : brev(qi, L - R);
    float2 e[PR];
    load_items<R, L>(e, nat0, p, load);
    pass_butterflies<R, INV, 0>(e, 0, tw);
    const int base = q << R;
    int ab = 0;
    if constexpr (XorLinear<Addr>::value) ab = addr(base, p);
#pragma unroll
    for (int m = 0; m < PR; ++m) {
      if constexpr (XorLinear<Addr>::value) buf[ab ^ addr(m, 0)] = e[m];
      else buf[addr(base + m, p)] = e[m];
    }
  }
  __syncthreads();
  fft_ct_tail_store<INV, L, MAXR, EVEN, PLOG, NTH, R>(buf, tw, tid, addr, store);
}

// staged_copy with compile-time sizes
template <int B, int TOTAL, int NTH, class V, class Load, class Store>
__device__ __forceinline__ void staged_copy_ct(int tid, Load load, Store store) {
  constexpr int ITER = (TOTAL + NTH - 1) / NTH;
#pragma unroll
  for (int i0 = 0; i0 < ITER; i0 += B) {
    V v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = tid + (i0 + k) * NTH;
      if (i0 + k < ITER && ((TOTAL % NTH) == 0 || i < TOTAL)) v[k] = load(i);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = tid + (i0 + k) * NTH;
      if (i0 + k < ITER && ((TOTAL % NTH) == 0 || i < TOTAL)) store(i, v[k]);
    }
  }
}

// Global -> shared staging with up to B independent loads in flight per
// thread (all loads of a batch are issued before the first store).
template <int B, class V, class Load, class Store>
__device__ __forceinline__ void staged_copy(int total, int tid, int nth, Load load, Store store) {
  for (int i0 = 0; i0 < total; i0 += B * nth) {
    V v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = i0 + tid + k * nth;
      if (i < total) v[k] = load(i);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = i0 + tid + k * nth;
      if (i < total) store(i, v[k]);
    }
  }
}

}  // namespace fft
}  // namespace patfft
