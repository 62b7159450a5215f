// bitrev_kernels.cuh -- sm_100a kernels for the bit-reversed permutation.
//
// Index model (the COBRA split of src/permutations.py:225-249):
//   i = x * 2^(b-Q) + y * 2^Q + z,   x, z in [0, 2^Q),  y in [0, 2^m),  m = b - 2Q
//   rev_b(i) = rev_Q(z) * 2^(b-Q) + rev_m(y) * 2^Q + rev_Q(x)
// For a fixed middle value y the 2^Q x 2^Q elements {x, z} form one "tile": 2^Q
// source rows of 2^Q contiguous elements (stride 2^(b-Q)), landing in 2^Q
// destination rows of 2^Q contiguous elements inside the rev(y) slab.  A tile is
// the paper's square transposition with the rows and columns
// also bit-reversed; it is staged through shared memory so BOTH the global reads
// and the global writes are 16-byte vectors over contiguous 2^Q*E-byte runs.
//
// Data path per tile (E = element bytes, V = 16/E elements per 16-byte vector):
//   1. each thread issues V LDG.128 from rows x_k = g + k*2^Q/V (k < V) at the
//      same 16-byte column c.  Because rev_Q(x_k) = rev(g)*V + rev_LV(k), those V
//      rows are exactly one aligned group of V destination positions;
//   2. a V x V register transpose turns them into V vectors, one per source
//      column z = c*V + j, each already holding V consecutive destination
//      elements in destination order;
//   3. STS.128 into U[z][rev(g)] (shared memory, XOR-swizzled 16-byte chunks:
//      chunk' = chunk ^ ((z/V) & 7), bank-conflict free on both sides);
//   4. after a barrier, each thread reads a contiguous chunk of row z of U
//      (LDS.128) and writes it to destination row rev_Q(z) (STG.128).
// The persistent loop issues the next tile's loads before draining the current
// one, so every warp keeps V*IPT 16-byte loads in flight across the drain.
//
// Kernel families in this file (selection and measured defaults: bitrev_capi.cu)
//   bitrev_oop_tile_kernel       out of place, square register tiles (above)
//   bitrev_oop_rect_kernel       out of place, 2^QX x 2^QZ register tiles: 1 KB
//                                destination rows, 256-byte source pieces
//   bitrev_inplace_tile_kernel   in place, tile PAIRS {y, rev y}; work items from
//                                the compact pair enumeration (pair_from_index)
//   bitrev_ring_kernel           warp-specialised TMA ring: cp.async.bulk rows or
//                                one cp.async.bulk.tensor per tile, mbarriers
//   bitrev_inplace_tstore_kernel in place, register loads + TMA tensor stores
//   bitrev_inplace_cpa_kernel    in place through element-granular cp.async
//   bitrev_scatter_tile_kernel   sharded plan: local reversal stored into peers
//   bitrev_fft_rect_kernel       FFT pre-pass: rect tiles + up to 7 DIT stages
//   small / gather / swap / transpose / even-odd / pairs / unpack kernels
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda.h>
#include <cuda_runtime.h>

// Build-time tuning knobs (defaults are the measured best).  Alternatives are
// built side by side with `python -m paper_1708_01873_b200.build --out F -DKNOB=V`
// and loaded through BITREV_B200_LIB for A/B runs (tools/*_ab.py).  Every knob
// value produces the same (correct) output.
#ifndef BITREV_IP_NC
#define BITREV_IP_NC 0  // in-place loads through the non-coherent path
#endif
#ifndef BITREV_MINB_OOP
#define BITREV_MINB_OOP 1  // __launch_bounds__ min CTAs/SM, out-of-place tile kernel
#endif
#ifndef BITREV_TILE_THREADS
#define BITREV_TILE_THREADS 256  // threads per CTA of the register tile kernels
#endif
#ifndef BITREV_CPA_STAGES
#define BITREV_CPA_STAGES 3  // pair stages of the cp.async in-place kernel
#endif
#ifndef BITREV_FFT_MINB
#define BITREV_FFT_MINB 3  // min CTAs/SM for the many-stage FFT kernels (register cap)
#endif
#ifndef BITREV_FFT_MINB_FROM
#define BITREV_FFT_MINB_FROM 3  // ... from this many fused stages on
#endif
#ifndef BITREV_RING_BUDGET_KB
#define BITREV_RING_BUDGET_KB 96  // TMA ring bytes per CTA (96 KB -> 2 CTAs/SM)
#endif
#ifndef BITREV_FFT_R8_FROM
#define BITREV_FFT_R8_FROM 7  // complex64: radix-8 drain from this many fused stages (4..8; 8 = never)
#endif
#ifndef BITREV_MINB_IP
#define BITREV_MINB_IP 1  // __launch_bounds__ min CTAs/SM, in-place tile kernel
#endif

namespace bitrev_b200 {

// ---------------------------------------------------------------------------
// bit helpers

// Reverse the low w bits of v (0 <= w <= 64); rev of width 0 is 0.  Replaces
// rev_naive (src/bits.py:31-47) -- one BREV pair instead of a w-step loop.
__device__ __forceinline__ uint64_t dev_rev(uint64_t v, int w) {
  return w <= 0 ? 0ull : (__brevll(v) >> (64 - w));
}

__host__ __device__ constexpr int const_rev(int v, int w) {
  return w == 0 ? 0 : (((v & 1) << (w - 1)) | const_rev(v >> 1, w - 1));
}

__host__ __device__ constexpr int const_log2(int v) { return v <= 1 ? 0 : 1 + const_log2(v >> 1); }

template <int E> struct Word;
template <> struct Word<1> { using T = uint8_t; };
template <> struct Word<2> { using T = uint16_t; };
template <> struct Word<4> { using T = uint32_t; };
template <> struct Word<8> { using T = unsigned long long; };
template <> struct Word<16> { using T = uint4; };

// 128-bit global accesses.  Source rows are read exactly once per launch, so the
// loads bypass L1 allocation.  Stores are plain by default (the permuted array
// is normally consumed next, e.g. by the first FFT butterfly stage, so keep it
// in L2).  The default large-array shapes also have a CS = true instantiation
// with streaming (evict-first) stores, which the host selects for launches of
// >= 64 MiB per side: at b = 30 out of place +1-3 % (profiles/
// r01_streaming_stores_ab.txt); for L2-sized arrays streaming stores cost
// ~1.5 %.  A runtime flag instead of a template parameter perturbed register
// allocation (E=4 rect tiles fell to 128 registers and 2 CTAs/SM).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_plain(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
#ifndef BITREV_LD_CS
#define BITREV_LD_CS 0  // streaming instantiations also load with .cs (evict-first)
#endif
__device__ __forceinline__ uint4 ld_cs(const void* p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
template <bool CS = false>
__device__ __forceinline__ void st_vec(void* p, const uint4& v) {
  if constexpr (CS)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  else
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// ---------------------------------------------------------------------------
// tile geometry

template <int E, int Q, int NT = BITREV_TILE_THREADS>
struct Tile {
  static constexpr int S = 1 << Q;           // tile side (elements)
  static constexpr int V = 16 / E;           // elements per 16-byte vector
  static constexpr int LV = const_log2(V);
  static constexpr int CH = S / V;           // 16-byte chunks per tile row
  static constexpr int ITEMS = CH * CH;      // load items (V loads each)
  static constexpr int WCH = S * CH;         // 16-byte chunks per tile
  static constexpr int THREADS = ITEMS < NT ? ITEMS : NT;
  static constexpr int IPT = ITEMS / THREADS;  // load items per thread
  static constexpr int WPT = WCH / THREADS;    // drain chunks per thread
  static constexpr int BYTES = S * S * E;
  static_assert(E == 4 || E == 8 || E == 16, "tile kernels move 4/8/16-byte elements");
  static_assert(CH >= 8, "XOR swizzle needs >= 8 chunks per row");
  static_assert(ITEMS % THREADS == 0 && WCH % THREADS == 0, "even split");
};

// Shared-memory chunk index of (row z, chunk col) with the 3-bit XOR swizzle.
template <int E, int Q>
__device__ __forceinline__ int swz(int z, int col) {
  using T = Tile<E, Q>;
  return z * T::CH + (col ^ ((z >> T::LV) & 7));
}

// Issue the V*IPT loads of one tile (rows at stride row_stride bytes).
template <int E, int Q, bool STREAM, int NT = BITREV_TILE_THREADS, bool LCS = false>
__device__ __forceinline__ void tile_load(uint4 (&r)[Tile<E, Q, NT>::IPT][Tile<E, Q, NT>::V],
                                          const char* tile_base, uint64_t row_stride) {
  using T = Tile<E, Q, NT>;
#pragma unroll
  for (int it = 0; it < T::IPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int c = id % T::CH;
    const int g = id / T::CH;
#pragma unroll
    for (int k = 0; k < T::V; ++k) {
      const char* p = tile_base + (uint64_t)(g + k * T::CH) * row_stride + (uint64_t)c * 16;
      if constexpr (LCS) r[it][k] = ld_cs(p);
      else r[it][k] = STREAM ? ld_stream(p) : ld_plain(p);
    }
  }
}

// Component j of a uint4 (j is a compile-time constant after unrolling).
template <int J>
__device__ __forceinline__ uint32_t comp(const uint4& v) {
  if constexpr (J == 0) return v.x;
  else if constexpr (J == 1) return v.y;
  else if constexpr (J == 2) return v.z;
  else return v.w;
}

// V x V transpose in registers: out[j] holds source column c*V+j for the V rows
// k, element slot rev_LV(k).  E=16 is the identity; E=8 swaps 64-bit halves;
// E=4 is a 4x4 word transpose with rows in bit-reversed order (0,2,1,3).
template <int E, int J>
__device__ __forceinline__ uint4 xpose(const uint4 (&a)[16 / E]) {
  if constexpr (E == 16) {
    return a[0];
  } else if constexpr (E == 8) {
    if constexpr (J == 0) return make_uint4(a[0].x, a[0].y, a[1].x, a[1].y);
    else return make_uint4(a[0].z, a[0].w, a[1].z, a[1].w);
  } else {
    return make_uint4(comp<J>(a[0]), comp<J>(a[2]), comp<J>(a[1]), comp<J>(a[3]));
  }
}

template <int E, int Q, int J>
__device__ __forceinline__ void stage_col(const uint4 (&a)[16 / E], uint4* U, int c, int col) {
  using T = Tile<E, Q>;
  if constexpr (J < T::V) {
    U[swz<E, Q>(c * T::V + J, col)] = xpose<E, J>(a);
    stage_col<E, Q, J + 1>(a, U, c, col);
  }
}

// Register transpose + swizzled STS of one tile into U.
template <int E, int Q, int NT = BITREV_TILE_THREADS>
__device__ __forceinline__ void tile_stage(const uint4 (&r)[Tile<E, Q, NT>::IPT][Tile<E, Q, NT>::V],
                                           uint4* U) {
  using T = Tile<E, Q, NT>;
#pragma unroll
  for (int it = 0; it < T::IPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int c = id % T::CH;
    const int g = id / T::CH;
    const int col = (int)(__brev((unsigned)g) >> (32 - (Q - T::LV)));  // rev_{Q-LV}(g)
    stage_col<E, Q, 0>(r[it], U, c, col);
  }
}

// Drain U: row z goes to destination row rev_Q(z) (stride row_stride bytes).
template <int E, int Q, int NT = BITREV_TILE_THREADS, bool CS = false>
__device__ __forceinline__ void tile_drain(const uint4* U, char* dst_base, uint64_t row_stride) {
  using T = Tile<E, Q, NT>;
#pragma unroll
  for (int it = 0; it < T::WPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int col = id % T::CH;
    const int z = id / T::CH;
    const uint4 v = U[swz<E, Q>(z, col)];
    const uint64_t rz = __brev((unsigned)z) >> (32 - Q);
    st_vec<CS>(dst_base + rz * row_stride + (uint64_t)col * 16, v);
  }
}

struct TileArgs {
  const char* src;
  char* dst;
  int b;               // index bits
  int m;               // middle bits b - 2Q
  uint64_t ntiles;     // batch << m (oop) or batch << m (in-place, incl. skipped)
  int64_t src_bstride; // bytes between batch rows
  int64_t dst_bstride;
  int order;           // 0: y = work index; 1: bit-interleaved (see work_to_y)
  uint64_t npairs;     // in place, compact pair enumeration: pairs per row (else 0)
  uint64_t step_b;     // compact mode: gridDim.x = step_b * npairs + step_w
  uint64_t step_w;
  int64_t batch;
};

// Walks the compact pair enumeration of all batch rows with stride
// gridDim.x, without divisions in the loop.
struct PairCursor {
  uint64_t bi, w;
  __device__ __forceinline__ void start(const TileArgs& a) { start_at(a, blockIdx.x); }
  __device__ __forceinline__ void start_at(const TileArgs& a, uint64_t idx) {
    bi = idx / a.npairs;
    w = idx - bi * a.npairs;
  }
  __device__ __forceinline__ void next(const TileArgs& a) {
    w += a.step_w;
    bi += a.step_b;
    if (w >= a.npairs) {
      w -= a.npairs;
      ++bi;
    }
  }
  __device__ __forceinline__ bool valid(const TileArgs& a) const { return bi < (uint64_t)a.batch; }
};

// Gather the even bits of x into its low half (Morton decode).
__device__ __forceinline__ uint64_t compact_even(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return x;
}

// Middle value y visited at work index w (a bijection of [0, 2^m)).
// order 0: y = w.  CTAs running together then read adjacent tiles (long
// contiguous source runs) but write rev(y) tiles scattered over the slab.
// order 1: w's bits alternate between y's low end and y's high end
// (w bit 2k -> y bit k, w bit 2k+1 -> y bit m-1-k), so a window of 2^j
// consecutive work items varies y in its ~j/2 lowest AND ~j/2 highest bits --
// and rev(y) likewise: both the y side and the rev(y) side of concurrently
// running CTAs form runs of ~2^(j/2) adjacent tiles.
__device__ __forceinline__ uint64_t work_to_y(uint64_t w, int m, int order) {
  if (order == 0 || m < 2) return w;
  if (order == 1) {
    const int h = m >> 1;
    const uint64_t mask = (1ull << h) - 1;
    uint64_t y = compact_even(w) & mask;
    y |= dev_rev(compact_even(w >> 1) & mask, h) << (m - h);
    if (m & 1) y |= ((w >> (2 * h)) & 1ull) << h;
    return y;
  }
  // order = 0x100 | L << 4 | H: the L lowest work bits are y's low bits
  // (runs of 2^L adjacent tiles on the y side), the next H work bits are y's
  // top bits (runs of 2^H adjacent tiles on the rev(y) side), the rest fill
  // the middle.  Clamped so that L + H <= m.
  int L = (order >> 4) & 15, H = order & 15;
  if (L > m) L = m;
  if (H > m - L) H = m - L;
  const uint64_t lo = w & ((1ull << L) - 1);
  const uint64_t hi = (w >> L) & ((1ull << H) - 1);
  const uint64_t mid = w >> (L + H);
  return (hi << (m - H)) | (mid << L) | lo;
}

// Number of middle values y with y <= rev_m(y): the unordered tile pairs
// {y, rev(y)} of one row, palindromes included.
__host__ __device__ inline uint64_t pair_count(int m) {
  return ((1ull << m) + (1ull << ((m + 1) / 2))) >> 1;
}

// w-th canonical pair representative y (y <= rev_m(y)), a bijection of
// [0, pair_count(m)) -- the swap-schedule structure of _fill_pairs
// (src/schedule.py:53-75) at tile granularity.  Level k (k < m/2) holds the
// y whose outer k bit pairs mirror each other and whose pair k is
// (y_{m-1-k}, y_k) = (0, 1): 2^(m-k-2) values laid out after levels < k;
// the 2^ceil(m/2) palindromes come last.  Lets the in-place kernels visit
// exactly one item per pair: no skipped items, equal work per CTA.
__device__ __forceinline__ uint64_t pair_from_index(uint64_t w, int m) {
  if (m == 0) return 0;
  const int h = m >> 1;
  const uint64_t Sh = (1ull << (m - 1)) - (1ull << (m - h - 1));
  if (w < Sh) {
    const int k = __clzll((~w) << (64 - (m - 1)));  // leading ones of w in m-1 bits
    const uint64_t o = w - ((1ull << (m - 1)) - (1ull << (m - k - 1)));
    const int ib = m - 2 * k - 2;
    const uint64_t inner = o & ((1ull << ib) - 1);
    const uint64_t outer = o >> ib;
    return (inner << (k + 1)) | (1ull << k) | outer | (dev_rev(outer, k) << (m - k));
  }
  const uint64_t p = w - Sh;
  const uint64_t outer = p & ((1ull << h) - 1);
  uint64_t y = outer | (dev_rev(outer, h) << (m - h));
  if (m & 1) y |= ((p >> h) & 1ull) << h;
  return y;
}



// ---------------------------------------------------------------------------
// out-of-place tile kernel (replaces _cobra_copy, src/permutations.py:225-249)

template <int E, int Q, int NT = BITREV_TILE_THREADS, bool CS = false, int MINB = BITREV_MINB_OOP>
__global__ void __launch_bounds__(Tile<E, Q, NT>::THREADS, MINB)
    bitrev_oop_tile_kernel(TileArgs a) {
  using T = Tile<E, Q, NT>;
  extern __shared__ __align__(16) uint4 smem[];
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  const uint64_t mmask = (1ull << a.m) - 1;
  uint4 r[T::IPT][T::V];

  uint64_t t = blockIdx.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: predecessor done (no-op otherwise)
  if (t >= a.ntiles) return;
  auto src_tile = [&](uint64_t tt) {
    const uint64_t bi = tt >> a.m, y = work_to_y(tt & mmask, a.m, a.order);
    return a.src + bi * a.src_bstride + (y << Q) * E;
  };
  tile_load<E, Q, true, NT, CS && BITREV_LD_CS>(r, src_tile(t), row_stride);
  for (;;) {
    const uint64_t bi = t >> a.m, y = work_to_y(t & mmask, a.m, a.order);
    tile_stage<E, Q, NT>(r, smem);
    __syncthreads();
    const uint64_t tn = t + gridDim.x;
    if (tn < a.ntiles) tile_load<E, Q, true, NT, CS && BITREV_LD_CS>(r, src_tile(tn), row_stride);
    else asm volatile("griddepcontrol.launch_dependents;");
    char* dbase = a.dst + bi * a.dst_bstride + (dev_rev(y, a.m) << Q) * E;
    tile_drain<E, Q, NT, CS>(smem, dbase, row_stride);
    if (tn >= a.ntiles) break;
    __syncthreads();
    t = tn;
  }
}

// ---------------------------------------------------------------------------
// rectangular out-of-place tile kernel
//
// Out of place there is no pairing constraint, so the split can be uneven:
//   i = x * 2^(b-QX) + y * 2^QZ + z,  x < 2^QX, z < 2^QZ, y < 2^(b-QX-QZ)
//   rev_b(i) = rev_QZ(z) * 2^(b-QZ) + rev_m(y) * 2^QX + rev_QX(x).
// A tile is 2^QX source pieces of 2^QZ*E bytes (short: consecutive y are
// adjacent, so CTAs running together still read long runs) and 2^QZ
// destination rows of 2^QX*E bytes (long: the scattered side gets >= 1 KB
// runs) -- with a tile 2^(QZ-QX) times smaller than a square one of the same
// destination run length.

template <int E, int QX, int QZ>
struct Rect {
  static constexpr int V = 16 / E;
  static constexpr int LV = const_log2(V);
  static constexpr int XS = 1 << QX, ZS = 1 << QZ;
  static constexpr int GX = XS / V;          // row groups / destination chunks per row
  static constexpr int CZ = ZS / V;          // 16-byte chunks per source piece
  static constexpr int ITEMS = GX * CZ;      // load items (V loads each)
  static constexpr int WCH = ZS * GX;        // 16-byte chunks per tile
  static constexpr int THREADS = ITEMS < 256 ? ITEMS : 256;
  static constexpr int IPT = ITEMS / THREADS;
  static constexpr int WPT = WCH / THREADS;
  static constexpr int BYTES = XS * ZS * E;
  static_assert(E == 4 || E == 8 || E == 16, "rect tiles move 4/8/16-byte elements");
  static_assert(GX >= 8 && CZ >= 8, "XOR swizzle needs >= 8 chunks on both sides");
  static_assert(ITEMS % THREADS == 0 && WCH % THREADS == 0, "even split");
};

template <int E, int QX, int QZ, bool CS = false>
__global__ void __launch_bounds__(Rect<E, QX, QZ>::THREADS)
    bitrev_oop_rect_kernel(TileArgs a) {
  using T = Rect<E, QX, QZ>;
  extern __shared__ __align__(16) uint4 smem[];
  const uint64_t src_row = (uint64_t)E << (a.b - QX);   // stride between source pieces
  const uint64_t dst_row = (uint64_t)E << (a.b - QZ);   // stride between destination rows
  const uint64_t mmask = (1ull << a.m) - 1;
  uint4 r[T::IPT][T::V];

  auto load = [&](uint64_t tt) {
    const uint64_t bi = tt >> a.m, y = work_to_y(tt & mmask, a.m, a.order);
    const char* base = a.src + bi * a.src_bstride + (y << QZ) * E;
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CZ, g = id / T::CZ;
#pragma unroll
      for (int k = 0; k < T::V; ++k)
        r[it][k] = (CS && BITREV_LD_CS) ? ld_cs(base + (uint64_t)(g + k * T::GX) * src_row + (uint64_t)c * 16)
                                        : ld_stream(base + (uint64_t)(g + k * T::GX) * src_row + (uint64_t)c * 16);
    }
  };
  // U[z][col]: ZS rows of GX chunks, chunk' = chunk ^ ((z >> LV) & 7)
  auto sidx = [&](int z, int col) { return z * T::GX + (col ^ ((z >> T::LV) & 7)); };

  uint64_t t = blockIdx.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (no-op otherwise)
  if (t >= a.ntiles) return;
  load(t);
  for (;;) {
    const uint64_t bi = t >> a.m, y = work_to_y(t & mmask, a.m, a.order);
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CZ, g = id / T::CZ;
      const int col = (int)(__brev((unsigned)g) >> (32 - (QX - T::LV)));
      smem[sidx(c * T::V, col)] = xpose<E, 0>(r[it]);
      if constexpr (T::V > 1) smem[sidx(c * T::V + 1, col)] = xpose<E, 1>(r[it]);
      if constexpr (T::V > 2) {
        smem[sidx(c * T::V + 2, col)] = xpose<E, 2>(r[it]);
        smem[sidx(c * T::V + 3, col)] = xpose<E, 3>(r[it]);
      }
    }
    __syncthreads();
    const uint64_t tn = t + gridDim.x;
    if (tn < a.ntiles) load(tn);
    else asm volatile("griddepcontrol.launch_dependents;");
    char* dbase = a.dst + bi * a.dst_bstride + (dev_rev(y, a.m) << QX) * E;
#pragma unroll
    for (int it = 0; it < T::WPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int col = id % T::GX, z = id / T::GX;
      const uint64_t rz = __brev((unsigned)z) >> (32 - QZ);
      st_vec<CS>(dbase + rz * dst_row + (uint64_t)col * 16, smem[sidx(z, col)]);
    }
    if (tn >= a.ntiles) break;
    __syncthreads();
    t = tn;
  }
}

// ---------------------------------------------------------------------------
// sharded plan, step 1 (and 1+2 fused): the rectangular tile kernel above
// with its destination rows re-addressed.  Local output index
// u = d * C + c * S + k' (d = destination rank, c = exchange round, S = 2^sb)
// is stored at peer[d] + (c * G * S + rank * S + k') * E.
//   pack    (all-to-all in K = C / S rounds): peer[d] = send + d * S * E,
//           rank = 0, so round c's send data is the contiguous slice
//           [c * G * S, (c + 1) * G * S) with equal per-rank splits;
//   scatter (peer-mapped receive buffers): peer[d] = rank d's buffer, S = C,
//           so the row lands where the all-to-all would have put it.
// A destination row (2^QX contiguous u) never straddles a sub-chunk
// (S >= 2^QX), so the remap costs a few integer ops per row.

constexpr int kMaxPeers = 8;

struct PackArgs {
  TileArgs t;
  char* peer[kMaxPeers];  // base of destination rank d's region
  int g;                  // log2 G
  int sb;                 // log2 S
  int rank;               // this rank's slot inside each destination region
};

template <int E, int QX, int QZ>
__global__ void __launch_bounds__(Rect<E, QX, QZ>::THREADS)
    bitrev_pack_rect_kernel(PackArgs pa) {
  using T = Rect<E, QX, QZ>;
  extern __shared__ __align__(16) uint4 smem[];
  const TileArgs& a = pa.t;
  const uint64_t src_row = (uint64_t)E << (a.b - QX);
  const int db = a.b - pa.g;  // bits of u below the rank field
  const uint64_t smask = (1ull << pa.sb) - 1, cmask = (1ull << db) - 1;
  uint4 r[T::IPT][T::V];

  auto load = [&](uint64_t y) {
    const char* base = a.src + (y << QZ) * E;
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CZ, g = id / T::CZ;
#pragma unroll
      for (int k = 0; k < T::V; ++k)
        r[it][k] = ld_stream(base + (uint64_t)(g + k * T::GX) * src_row + (uint64_t)c * 16);
    }
  };
  auto sidx = [&](int z, int col) { return z * T::GX + (col ^ ((z >> T::LV) & 7)); };

  uint64_t t = blockIdx.x;
  if (t >= a.ntiles) return;
  load(t);
  for (;;) {
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CZ, g = id / T::CZ;
      const int col = (int)(__brev((unsigned)g) >> (32 - (QX - T::LV)));
      smem[sidx(c * T::V, col)] = xpose<E, 0>(r[it]);
      if constexpr (T::V > 1) smem[sidx(c * T::V + 1, col)] = xpose<E, 1>(r[it]);
      if constexpr (T::V > 2) {
        smem[sidx(c * T::V + 2, col)] = xpose<E, 2>(r[it]);
        smem[sidx(c * T::V + 3, col)] = xpose<E, 3>(r[it]);
      }
    }
    __syncthreads();
    const uint64_t tn = t + gridDim.x;
    if (tn < a.ntiles) load(tn);
    const uint64_t ry = dev_rev(t, a.m) << QX;
#pragma unroll
    for (int it = 0; it < T::WPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int col = id % T::GX, z = id / T::GX;
      const uint64_t u = ((uint64_t)(__brev((unsigned)z) >> (32 - QZ)) << (a.b - QZ)) | ry;
      const uint64_t rest = u & cmask;
      const uint64_t off = ((rest >> pa.sb) << (pa.sb + pa.g)) | ((uint64_t)pa.rank << pa.sb) |
                           (rest & smask);
      st_vec<true>(pa.peer[u >> db] + off * E + (uint64_t)col * 16, smem[sidx(z, col)]);
    }
    if (tn >= a.ntiles) break;
    __syncthreads();
    t = tn;
  }
}

// ---------------------------------------------------------------------------
// sharded plan, steps 1+2 fused: local bit reversal scattered to peers
//
// Rank `rank` of G = 2^g reverses its (b-g)-bit shard; the local output index
// u = d*C + k (C = 2^(b-2g)) belongs to rank d = u >> (b-2g) at position
// rank*C + k of that rank's receive buffer.  A tile's
// destination row is 2^Q contiguous u inside one chunk d (C >= 2^Q), so the
// drain just swaps its base pointer for peer[d] + (rank*C + k0)*E: with peer
// pointers mapped over NVLink/NVSwitch (symmetric memory / CUDA IPC) the row
// stores go straight into the peers' HBM -- no send buffer, no separate
// all-to-all pass.  On one device the same kernel runs with G local buffers.

struct ScatterArgs {
  TileArgs t;
  char* peer[kMaxPeers];  // receive buffer of each rank
  int g;                  // log2 G
  int rank;
  int sb;                 // log2 of the sub-chunk length (= log2 C: one chunk)
};

template <int E, int Q>
__global__ void __launch_bounds__(Tile<E, Q>::THREADS)
    bitrev_scatter_tile_kernel(ScatterArgs sa) {
  using T = Tile<E, Q>;
  extern __shared__ __align__(16) uint4 smem[];
  const TileArgs& a = sa.t;
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  const uint64_t mmask = (1ull << a.m) - 1;
  const int cbits = a.b - sa.g;  // log2 C, a.b = local width b - g
  uint4 r[T::IPT][T::V];
  uint64_t t = blockIdx.x;
  if (t >= a.ntiles) return;
  tile_load<E, Q, true>(r, a.src + ((t & mmask) << Q) * E, row_stride);
  for (;;) {
    const uint64_t y = t & mmask;
    tile_stage<E, Q>(r, smem);
    __syncthreads();
    const uint64_t tn = t + gridDim.x;
    if (tn < a.ntiles) tile_load<E, Q, true>(r, a.src + ((tn & mmask) << Q) * E, row_stride);
    const uint64_t ry_base = dev_rev(y, a.m) << Q;
#pragma unroll
    for (int it = 0; it < T::WPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int col = id % T::CH;
      const int z = id / T::CH;
      const uint4 v = smem[swz<E, Q>(z, col)];
      const uint64_t u0 = ((uint64_t)(__brev((unsigned)z) >> (32 - Q)) << (a.b - Q)) | ry_base;
      const int d = (int)(u0 >> cbits);
      const uint64_t k0 = u0 & ((1ull << cbits) - 1);
      // sub-chunk layout [c][rank][k']: k0 = c * 2^sb + k'
      const uint64_t off = ((k0 >> sa.sb) << (sa.sb + sa.g)) | ((uint64_t)sa.rank << sa.sb) |
                           (k0 & ((1ull << sa.sb) - 1));
      st_vec(sa.peer[d] + off * E + (uint64_t)col * 16, v);
    }
    if (tn >= a.ntiles) break;
    __syncthreads();
    t = tn;
  }
}

// ---------------------------------------------------------------------------
// in-place tile-pair kernel (replaces _cobra_swap, src/permutations.py:252-285)
//
// Work item y (per batch row) with y <= rev(y): load tile y and tile rev(y) into
// two shared buffers, barrier, write tile y's data into the rev(y) slab and
// tile rev(y)'s data into the y slab.  A palindromic y (y == rev(y)) is loaded
// and written back transposed alone.  Items with rev(y) < y are skipped -- each
// unordered pair is handled exactly once (src/permutations.py:263-264), so no
// two CTAs ever touch the same element and both tiles are resident before the
// first write.

template <int E, int Q, bool COMPACT, bool CS = false>
__global__ void __launch_bounds__(Tile<E, Q>::THREADS, BITREV_MINB_IP)
    bitrev_inplace_tile_kernel(TileArgs a) {
  using T = Tile<E, Q>;
  extern __shared__ __align__(16) uint4 smem[];
  uint4* U0 = smem;
  uint4* U1 = smem + T::WCH;
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  const uint64_t mmask = (1ull << a.m) - 1;
  uint4 r0[T::IPT][T::V], r1[T::IPT][T::V];

  auto partner = [&](uint64_t y) { return dev_rev(y, a.m); };
  // Work cursor: COMPACT walks the pair enumeration (one item per pair);
  // otherwise every y is visited in `order` and items with rev(y) < y skipped.
  PairCursor pc;
  uint64_t tt = blockIdx.x;
  auto skip_fwd = [&]() {
    while (tt < a.ntiles && partner(work_to_y(tt & mmask, a.m, a.order)) <
                                work_to_y(tt & mmask, a.m, a.order))
      tt += gridDim.x;
  };
  auto cur_valid = [&]() { return COMPACT ? pc.valid(a) : tt < a.ntiles; };
  auto cur_item = [&](uint64_t& bi, uint64_t& y) {
    if constexpr (COMPACT) {
      bi = pc.bi;
      y = pair_from_index(pc.w, a.m);
    } else {
      bi = tt >> a.m;
      y = work_to_y(tt & mmask, a.m, a.order);
    }
  };
  auto cur_next = [&]() {
    if constexpr (COMPACT) {
      pc.next(a);
    } else {
      tt += gridDim.x;
      skip_fwd();
    }
  };
  auto issue = [&]() {
    uint64_t bi, y;
    cur_item(bi, y);
    const uint64_t ry = partner(y);
    const char* base = a.src + bi * a.src_bstride;
    tile_load<E, Q, BITREV_IP_NC, BITREV_TILE_THREADS, CS && BITREV_LD_CS>(
        r0, base + (y << Q) * E, row_stride);
    if (ry != y)
      tile_load<E, Q, BITREV_IP_NC, BITREV_TILE_THREADS, CS && BITREV_LD_CS>(
          r1, base + (ry << Q) * E, row_stride);
  };

  if constexpr (COMPACT) pc.start(a); else skip_fwd();
  // programmatic dependent launch (a no-op unless the host sets the launch
  // attribute): wait for the previous kernel in the stream -- typically the
  // previous call on the same array -- to complete before the first load
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!cur_valid()) return;
  issue();
  for (;;) {
    uint64_t bi, y;
    cur_item(bi, y);
    const uint64_t ry = partner(y);
    const bool pair = ry != y;
    tile_stage<E, Q>(r0, U0);
    if (pair) tile_stage<E, Q>(r1, U1);
    __syncthreads();
    cur_next();
    const bool more = cur_valid();
    if (more) issue();
    else asm volatile("griddepcontrol.launch_dependents;");  // last pair: let the next launch in
    char* base = a.dst + bi * a.dst_bstride;
    tile_drain<E, Q, BITREV_TILE_THREADS, CS>(U0, base + (ry << Q) * E, row_stride);
    if (pair) tile_drain<E, Q, BITREV_TILE_THREADS, CS>(U1, base + (y << Q) * E, row_stride);
    if (!more) break;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// in-place tile pairs over a 2-CTA cluster (path 6)
//
// The single-CTA pair kernel holds BOTH tiles of a pair in one SM's registers
// and shared memory, which caps the tile at 512-byte rows: the 1 KB-row shapes
// (E=16 Q=6, E=8 Q=7) spill or do not fit.  Here the two CTAs of a cluster
// split the pair: rank 0 loads and stages tile y, rank 1 tile rev(y), each in
// its own SM.  One cluster barrier separates "both tiles loaded" from
// "either region written"; then each CTA drains its tile into
// the partner's slab.  Both CTAs walk the same pair cursor (one cluster = one
// work stream), so their barrier counts always match; a palindromic y is
// handled by rank 0 alone.  No distributed shared memory is touched: the
// barrier only orders rank 1's loads of region rev(y) before rank 0's stores
// into it (and vice versa).

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Execution-only cluster barrier.  Across the pair it guards a write-after-
// read: a CTA arrives only after its loads of the partner's region have
// returned (their values were consumed by the STS of tile_stage), so no later
// store can change them, and no CTA ever reads a region another CTA wrote.
// It gives NO memory ordering, so the CTA's own STS -> LDS hand-off needs the
// __syncthreads() before it.  A release arrive would make every thread wait
// for its previous drain's global stores to be performed (ncu: 16 % membar
// stalls).
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n"
               "barrier.cluster.wait.aligned;" ::: "memory");
}

template <int E, int Q, int NT, int MINB = 1, bool CS = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, MINB)
    bitrev_inplace_cluster_kernel(TileArgs a) {
  using T = Tile<E, Q, NT>;
  extern __shared__ __align__(16) uint4 smem[];
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  const unsigned rank = cluster_rank();
  uint4 r[T::IPT][T::V];
  PairCursor pc;
  pc.start_at(a, blockIdx.x >> 1);
  if (!pc.valid(a)) return;  // same decision in both CTAs of the cluster
  auto issue = [&]() {
    const uint64_t y = pair_from_index(pc.w, a.m), ry = dev_rev(y, a.m);
    if (rank && ry == y) return;  // palindrome: rank 0 alone
    tile_load<E, Q, BITREV_IP_NC, NT, CS && BITREV_LD_CS>(
        r, a.src + pc.bi * a.src_bstride + ((rank ? ry : y) << Q) * E, row_stride);
  };
  issue();
  for (;;) {
    const uint64_t bi = pc.bi, y = pair_from_index(pc.w, a.m), ry = dev_rev(y, a.m);
    const bool active = !(rank && ry == y);
    if (active) tile_stage<E, Q, NT>(r, smem);
    __syncthreads();          // this CTA's staged tile is visible to all its threads
    cluster_sync_relaxed();   // both tiles of the pair are loaded: either region may be written
    pc.next(a);
    const bool more = pc.valid(a);
    if (more) issue();
    if (active)
      tile_drain<E, Q, NT, CS>(smem, a.dst + bi * a.dst_bstride + ((rank ? y : ry) << Q) * E,
                               row_stride);
    if (!more) break;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// TMA ring family: warp-specialised producer / consumers over an smem ring
//
// The register-staged kernels hold every in-flight byte in registers, so
// bytes in flight per SM are register-limited and each CTA alternates
// load -> barrier -> drain.  Here one producer warp streams tiles into an
// NS-stage shared-memory ring with TMA, and NCW consumer warps drain them;
// stages are handed over with mbarriers (full: TMA transaction bytes; empty:
// one arrival per consumer warp), so no block-wide barrier sits in the loop.
//
// Two ways to fill a stage (template MODE):
//   kBulkRows  one cp.async.bulk per tile row (2^Q*E bytes) into padded rows
//              (PITCH = row + 16 B rotates rows across bank groups);
//   kTensor    ONE cp.async.bulk.tensor per tile through a 5-D tensor map
//                d0: 128-byte unit run   (unit = 4 B for E = 4, else 8 B)
//                d1: tile row x          stride 2^(b-Q) * E
//                d2: 128-byte piece      stride 128 B
//                d3: middle value y      stride 2^Q * E
//                d4: batch row           stride batch_stride * E
//              box {128/unit, 2^Q, pieces, 1, 1} = tile y; SWIZZLE_128B puts
//              16-byte chunk cc of segment R = piece * 2^Q + x at cc ^ (x & 7).
// The drain is the register kernel's transpose moved to the read side: a lane
// reads chunk c of the V rows g + k*2^Q/V (consecutive lanes = consecutive g:
// conflict-free LDS.128), transposes V x V in registers and writes V vectors
// to destination rows rev_Q(c*V + j) at chunk rev(g) (a warp writes whole
// contiguous destination rows).

constexpr int kBulkRows = 1;
constexpr int kTensor = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* tmap, int c3, int c4,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %2, %2, %3, %4}], [%5];" ::"r"(dst),
      "l"(tmap), "r"(0), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

template <int E, int Q, bool INPLACE, int MODE>
struct Ring {
  static constexpr int S = 1 << Q;
  static constexpr int V = 16 / E;
  static constexpr int LV = const_log2(V);
  static constexpr int G = S / V;               // row groups == 16-byte chunks per row
  static constexpr int ROW = S * E;             // bytes per tile row
  static constexpr int PITCH = MODE == kTensor ? ROW : ROW + 16;
  static constexpr int TILE = S * PITCH;
  static constexpr int TILES = INPLACE ? 2 : 1;
  static constexpr int STAGE = TILES * TILE;
  static constexpr int BUDGET = BITREV_RING_BUDGET_KB * 1024;  // ring bytes per CTA
  static constexpr int NS_RAW = BUDGET / STAGE;
  static constexpr int NS = NS_RAW < 2 ? 2 : (NS_RAW > 16 ? 16 : NS_RAW);
  static constexpr int ITEMS = G * G;           // drain items per tile (V chunks each)
  static constexpr int NCW_RAW = ITEMS / 32;
  static constexpr int NCW = NCW_RAW > 8 ? 8 : NCW_RAW;  // consumer warps
  static constexpr int THREADS = 32 * (NCW + 1);
  static constexpr int IPW = ITEMS / (32 * NCW);          // drain items per lane per tile
  static constexpr int SMEM = NS * STAGE + 1024 + 2 * NS * 8;
  static_assert(E == 4 || E == 8 || E == 16, "ring kernels move 4/8/16-byte elements");
  static_assert(G >= 8 && ROW % 16 == 0, "chunk geometry");
  static_assert(MODE != kTensor || ROW % 128 == 0, "tensor tiles need 128-byte rows");
  static_assert(NCW >= 1 && ITEMS % (32 * NCW) == 0, "even split");
};

template <int E, int Q, bool INPLACE, int MODE>
__device__ __forceinline__ void ring_drain(uint32_t tile, char* dst_base, uint64_t row_stride,
                                           int cw, int lane) {
  using R = Ring<E, Q, INPLACE, MODE>;
#pragma unroll
  for (int it = 0; it < R::IPW; ++it) {
    const int id = (it * R::NCW + cw) * 32 + lane;
    const int g = id % R::G;
    const int c = id / R::G;
    uint4 v[R::V];
#pragma unroll
    for (int k = 0; k < R::V; ++k) {
      const int x = g + k * R::G;
      uint32_t addr;
      if constexpr (MODE == kTensor)
        addr = tile + ((c >> 3) * R::S + x) * 128 + (((c & 7) ^ (x & 7)) << 4);
      else
        addr = tile + x * R::PITCH + c * 16;
      v[k] = lds128(addr);
    }
    char* base = dst_base + (uint64_t)(__brev((unsigned)g) >> (32 - (Q - R::LV))) * 16;
    st_vec(base + (uint64_t)(__brev((unsigned)(c * R::V)) >> (32 - Q)) * row_stride,
           xpose<E, 0>(v));
    if constexpr (R::V > 1)
      st_vec(base + (uint64_t)(__brev((unsigned)(c * R::V + 1)) >> (32 - Q)) * row_stride,
             xpose<E, 1>(v));
    if constexpr (R::V > 2) {
      st_vec(base + (uint64_t)(__brev((unsigned)(c * R::V + 2)) >> (32 - Q)) * row_stride,
             xpose<E, 2>(v));
      st_vec(base + (uint64_t)(__brev((unsigned)(c * R::V + 3)) >> (32 - Q)) * row_stride,
             xpose<E, 3>(v));
    }
  }
}

// Persistent ring kernel.  Out of place: one work item = tile y.  In place:
// one item = the pair {y, rev(y)} with y <= rev(y); both tiles are staged
// before either is drained, and the pair's regions are touched by no other
// item, so the in-place hazard is confined to the item.
template <int E, int Q, bool INPLACE, int MODE, bool COMPACT>
__global__ void __launch_bounds__(Ring<E, Q, INPLACE, MODE>::THREADS)
    bitrev_ring_kernel(const __grid_constant__ CUtensorMap tmap, TileArgs a) {
  using R = Ring<E, Q, INPLACE, MODE>;
  extern __shared__ __align__(1024) unsigned char smem_ring[];
  const uint32_t base =
      (smem_u32(smem_ring) + 1023u) & ~1023u;  // 1024-B alignment for the 128B swizzle
  const uint32_t full = base + R::NS * R::STAGE;
  const uint32_t empty = full + R::NS * 8;
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  const uint64_t mmask = (1ull << a.m) - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work cursor (see bitrev_inplace_tile_kernel); each role keeps its own
  struct Cursor {
    PairCursor pc;
    uint64_t tt;
  };
  auto skip_fwd = [&](uint64_t t) {
    if constexpr (INPLACE && !COMPACT) {
      while (t < a.ntiles) {
        const uint64_t y = work_to_y(t & mmask, a.m, a.order);
        if (dev_rev(y, a.m) >= y) break;
        t += gridDim.x;
      }
    }
    return t;
  };
  auto c_start = [&](Cursor& c) {
    if constexpr (COMPACT) c.pc.start(a); else c.tt = skip_fwd(blockIdx.x);
  };
  auto c_valid = [&](const Cursor& c) { return COMPACT ? c.pc.valid(a) : c.tt < a.ntiles; };
  auto c_next = [&](Cursor& c) {
    if constexpr (COMPACT) c.pc.next(a); else c.tt = skip_fwd(c.tt + gridDim.x);
  };
  auto c_item = [&](const Cursor& c, uint64_t& bi, uint64_t& y) {
    if constexpr (COMPACT) {
      bi = c.pc.bi;
      y = pair_from_index(c.pc.w, a.m);
    } else {
      bi = c.tt >> a.m;
      y = work_to_y(c.tt & mmask, a.m, a.order);
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < R::NS; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, R::NCW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == R::NCW) {
    // ---- producer warp
    Cursor c;
    c_start(c);
    for (int i = 0; c_valid(c); ++i) {
      const int s = i % R::NS;
      if (i >= R::NS) mbar_wait(empty + 8 * s, (uint32_t)(((i / R::NS) - 1) & 1));
      uint64_t bi, y;
      c_item(c, bi, y);
      const uint64_t ry = dev_rev(y, a.m);
      const bool pair = INPLACE && ry != y;
      const uint32_t st = base + s * R::STAGE;
      const uint32_t bar = full + 8 * s;
      if constexpr (MODE == kTensor) {
        if (lane == 0) {
          mbar_expect_tx(bar, (pair ? 2 : 1) * R::S * R::ROW);
          tma_load_5d(st, &tmap, (int)y, (int)bi, bar);
          if (pair) tma_load_5d(st + R::TILE, &tmap, (int)ry, (int)bi, bar);
        }
      } else {
        if (lane == 0) mbar_expect_tx(bar, (pair ? 2 : 1) * R::S * R::ROW);
        __syncwarp();
        const char* src = a.src + bi * a.src_bstride;
        for (int x = lane; x < R::S; x += 32) {
          bulk_g2s(st + x * R::PITCH, src + x * row_stride + (y << Q) * E, R::ROW, bar);
          if (pair)
            bulk_g2s(st + R::TILE + x * R::PITCH, src + x * row_stride + (ry << Q) * E, R::ROW,
                     bar);
        }
      }
      c_next(c);
    }
  } else {
    // ---- consumer warps
    Cursor c;
    c_start(c);
    for (int i = 0; c_valid(c); ++i) {
      const int s = i % R::NS;
      mbar_wait(full + 8 * s, (uint32_t)((i / R::NS) & 1));
      uint64_t bi, y;
      c_item(c, bi, y);
      const uint64_t ry = dev_rev(y, a.m);
      const uint32_t st = base + s * R::STAGE;
      char* dbase = a.dst + bi * a.dst_bstride;
      ring_drain<E, Q, INPLACE, MODE>(st, dbase + (ry << Q) * E, row_stride, warp, lane);
      if (INPLACE && ry != y)
        ring_drain<E, Q, INPLACE, MODE>(st + R::TILE, dbase + (y << Q) * E, row_stride, warp,
                                        lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * s);
      c_next(c);
    }
  }
}

// ---------------------------------------------------------------------------
// in-place tile pairs with TMA tensor stores (path 5)
//
// Loads are the register kernel's (LDG.128 of whole 2^Q*E-byte rows), but the
// lanes of a warp take a row's 16-byte chunks in bit-reversed order,
// c = rev(l).  After the V x V register transpose, chunk (c, J) belongs to
// destination row x' = rev_Q(c*V + J) = rev_LV(J)*CH + l, so the STS go
// straight into the SWIZZLE_128B layout of the tensor map's box (segment
// piece*2^Q + x', 16-byte chunk cc at cc ^ (x' & 7)) and the eight lanes of a
// quarter warp land on eight different x' mod 8: conflict-free.  One elected
// thread then stores each staged tile with cp.async.bulk.tensor (global <-
// shared) through the same 5-D map the tensor ring loads with.  There is no
// LDS/STG drain: the threads go straight on to the next pair's loads while
// the TMA engine writes.  Two pair slots: slot k%2 is restaged only after the
// bulk group that read it (pair k-2) has finished reading shared memory.

template <int E, int Q>
struct TsTile {
  using T = Tile<E, Q>;
  static constexpr int LCH = const_log2(T::CH);
  static constexpr int TILE = T::BYTES;
  static constexpr int SLOT = 2 * TILE;
  static constexpr int SMEM = 2 * SLOT + 1024;  // + slack for 1024-B alignment
  static_assert(((1 << Q) * E) % 128 == 0, "tensor tiles need 128-byte rows");
};

__device__ __forceinline__ void tma_store_5d(const void* tmap, uint32_t src, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group"
      " [%0, {%1, %1, %1, %2, %3}], [%4];" ::"l"(tmap),
      "r"(0), "r"(c3), "r"(c4), "r"(src)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

template <int E, int Q>
__device__ __forceinline__ void ts_load(uint4 (&r)[Tile<E, Q>::IPT][Tile<E, Q>::V],
                                        const char* tile_base, uint64_t row_stride) {
  using T = Tile<E, Q>;
  using S = TsTile<E, Q>;
#pragma unroll
  for (int it = 0; it < T::IPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int c = (int)(__brev((unsigned)(id % T::CH)) >> (32 - S::LCH));
    const int g = id / T::CH;
#pragma unroll
    for (int k = 0; k < T::V; ++k) {
      const char* p = tile_base + (uint64_t)(g + k * T::CH) * row_stride + (uint64_t)c * 16;
      r[it][k] = BITREV_IP_NC ? ld_stream(p) : ld_plain(p);
    }
  }
}

template <int E, int Q, int J>
__device__ __forceinline__ void ts_stage_col(const uint4 (&a)[16 / E], uint32_t tile, int l,
                                             int piece, int cc) {
  using T = Tile<E, Q>;
  if constexpr (J < T::V) {
    constexpr int RJ = T::V == 1 ? 0 : (T::V == 2 ? J : ((J & 1) << 1) | (J >> 1));  // rev_LV(J)
    const int xr = l + RJ * T::CH;  // destination row
    sts128(tile + (uint32_t)(((piece << Q) + xr) * 128 + ((cc ^ (xr & 7)) << 4)), xpose<E, J>(a));
    ts_stage_col<E, Q, J + 1>(a, tile, l, piece, cc);
  }
}

template <int E, int Q>
__device__ __forceinline__ void ts_stage(const uint4 (&r)[Tile<E, Q>::IPT][Tile<E, Q>::V],
                                         uint32_t tile) {
  using T = Tile<E, Q>;
#pragma unroll
  for (int it = 0; it < T::IPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int l = id % T::CH;
    const int g = id / T::CH;
    const int ch = (int)(__brev((unsigned)g) >> (32 - (Q - T::LV)));  // destination chunk
    ts_stage_col<E, Q, 0>(r[it], tile, l, ch >> 3, ch & 7);
  }
}

template <int E, int Q>
__global__ void __launch_bounds__(Tile<E, Q>::THREADS, 1)
    bitrev_inplace_tstore_kernel(const __grid_constant__ CUtensorMap tmap, TileArgs a) {
  using T = Tile<E, Q>;
  using S = TsTile<E, Q>;
  extern __shared__ __align__(1024) unsigned char smem_ts[];
  const uint32_t base = (smem_u32(smem_ts) + 1023u) & ~1023u;
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  uint4 r0[T::IPT][T::V], r1[T::IPT][T::V];
  PairCursor pc;
  pc.start(a);
  if (!pc.valid(a)) return;
  auto issue = [&]() {
    const uint64_t y = pair_from_index(pc.w, a.m), ry = dev_rev(y, a.m);
    const char* b0 = a.src + pc.bi * a.src_bstride;
    ts_load<E, Q>(r0, b0 + (y << Q) * E, row_stride);
    if (ry != y) ts_load<E, Q>(r1, b0 + (ry << Q) * E, row_stride);
  };
  issue();
  for (int k = 0;; ++k) {
    const uint64_t bi = pc.bi, y = pair_from_index(pc.w, a.m), ry = dev_rev(y, a.m);
    const bool pair = ry != y;
    const uint32_t slot = base + (uint32_t)((k & 1) * S::SLOT);
    if (threadIdx.x == 0) bulk_wait_read<1>();  // pair k-2's stores have read this slot
    __syncthreads();
    ts_stage<E, Q>(r0, slot);
    if (pair) ts_stage<E, Q>(r1, slot + S::TILE);
    fence_async_smem();  // generic-proxy STS -> visible to the async proxy
    __syncthreads();
    pc.next(a);
    const bool more = pc.valid(a);
    if (more) issue();
    if (threadIdx.x == 0) {
      tma_store_5d(&tmap, slot, (int)ry, (int)bi);  // tile y's data into slab rev(y)
      if (pair) tma_store_5d(&tmap, slot + S::TILE, (int)y, (int)bi);
      bulk_commit();
    }
    if (!more) break;
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// in-place tile pairs through cp.async (LDGSTS) straight into the transposed
// layout
//
// Every element is copied global -> shared by its own E-byte cp.async into
// its destination slot U[z][rev_Q(x)] (the register kernel's staged layout),
// so no registers hold in-flight data and no register transpose is needed.
// NS pair stages rotate: while stage i is drained (LDS.128 -> STG.128), the
// copies of pairs i+1 .. i+NS-1 are in flight (cp.async.wait_group).  Shared
// layout per tile: rows z of 2^Q/V 16-byte chunks, chunk' = chunk ^ (z & 15)
// (16 lanes writing one element each into 16 consecutive rows hit 16
// distinct chunks; the drain reads whole rows, any per-row XOR is free).

__device__ __forceinline__ void cp_async_e(uint32_t dst, const void* src, int bytes) {
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int E, int Q>
struct CpaTile {
  static constexpr int S = 1 << Q;
  static constexpr int V = 16 / E;
  static constexpr int CH = S / V;            // 16-byte chunks per smem row
  static constexpr int TILE = S * S * E;
  static constexpr int THREADS = 256;
  static constexpr int EPT = S * S / THREADS;  // elements copied per thread per tile
  static constexpr int WPT = S * CH / THREADS; // chunks drained per thread per tile
  static constexpr int STAGES = BITREV_CPA_STAGES;
  static constexpr int SMEM = STAGES * 2 * TILE;
  static_assert(CH >= 16, "swizzle needs 16 chunks per row");
};

template <int E, int Q>
__device__ __forceinline__ uint32_t cpa_slot(uint32_t tile, int z, int xp) {
  using T = CpaTile<E, Q>;
  const int col = xp / T::V, slot = xp % T::V;
  return tile + (uint32_t)((z * T::CH + (col ^ (z & 15))) * 16 + slot * E);
}

template <int E, int Q>
__device__ __forceinline__ void cpa_issue_tile(uint32_t tile, const char* src_tile,
                                               uint64_t row_stride) {
  using T = CpaTile<E, Q>;
#pragma unroll
  for (int it = 0; it < T::EPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int z = id % T::S, x = id / T::S;  // consecutive lanes: consecutive z of row x
    const int xp = (int)(__brev((unsigned)x) >> (32 - Q));
    cp_async_e(cpa_slot<E, Q>(tile, z, xp), src_tile + (uint64_t)x * row_stride + (uint64_t)z * E,
               E);
  }
}

template <int E, int Q>
__device__ __forceinline__ void cpa_drain_tile(uint32_t tile, char* dst_base, uint64_t row_stride) {
  using T = CpaTile<E, Q>;
#pragma unroll
  for (int it = 0; it < T::WPT; ++it) {
    const int id = it * T::THREADS + threadIdx.x;
    const int col = id % T::CH, z = id / T::CH;
    const uint4 v = lds128(tile + (uint32_t)((z * T::CH + (col ^ (z & 15))) * 16));
    const uint64_t rz = __brev((unsigned)z) >> (32 - Q);
    st_vec(dst_base + rz * row_stride + (uint64_t)col * 16, v);
  }
}

template <int E, int Q>
__global__ void __launch_bounds__(CpaTile<E, Q>::THREADS)
    bitrev_inplace_cpa_kernel(TileArgs a) {
  using T = CpaTile<E, Q>;
  extern __shared__ __align__(16) unsigned char smem_cpa[];
  const uint32_t base = smem_u32(smem_cpa);
  const uint64_t row_stride = (uint64_t)E << (a.b - Q);
  PairCursor issue_c, drain_c;
  issue_c.start(a);
  drain_c = issue_c;
  auto issue = [&](int stage) {
    if (issue_c.valid(a)) {
      const uint64_t bi = issue_c.bi, y = pair_from_index(issue_c.w, a.m);
      const uint64_t ry = dev_rev(y, a.m);
      const char* src = a.src + bi * a.src_bstride;
      const uint32_t st = base + stage * 2 * T::TILE;
      cpa_issue_tile<E, Q>(st, src + (y << Q) * E, row_stride);
      if (ry != y) cpa_issue_tile<E, Q>(st + T::TILE, src + (ry << Q) * E, row_stride);
      issue_c.next(a);
    }
    cp_async_commit();  // one group per stage slot, possibly empty
  };
#pragma unroll
  for (int s = 0; s < T::STAGES - 1; ++s) issue(s);
  for (int i = 0; drain_c.valid(a); ++i) {
    issue((i + T::STAGES - 1) % T::STAGES);  // slot drained at iteration i-1
    cp_async_wait<T::STAGES - 1>();           // this thread's copies for stage i landed
    __syncthreads();                          // ... and everyone else's
    const int stage = i % T::STAGES;
    const uint64_t bi = drain_c.bi, y = pair_from_index(drain_c.w, a.m);
    const uint64_t ry = dev_rev(y, a.m);
    const uint32_t st = base + stage * 2 * T::TILE;
    char* dst = a.dst + bi * a.dst_bstride;
    cpa_drain_tile<E, Q>(st, dst + (ry << Q) * E, row_stride);
    if (ry != y) cpa_drain_tile<E, Q>(st + T::TILE, dst + (y << Q) * E, row_stride);
    drain_c.next(a);
    __syncthreads();  // stage i is refilled at iteration i+1
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// FFT pre-pass: bit reversal fused with the first radix-2 DIT stages
//
// An iterative decimation-in-time FFT of length 2^b first bit-reverses its
// input (the permutation exists for this), then runs b
// butterfly stages; stage s combines elements 2^(s-1) apart inside aligned
// blocks of 2^s with twiddles W_{2^s}^k, k < 2^(s-1).  Stages 1..Q therefore
// stay inside aligned blocks of 2^Q outputs -- exactly one destination row of
// a tile -- and their twiddles depend only on the position inside the row.
// The drain (fft_rows_drain_r4) runs them on each row before storing it, as
// in-register radix-4 passes between lane layouts.  HBM traffic stays 2*n*E.
//
// Complex element types: E = 8 (complex64, float math) and E = 16
// (complex128, double math).  Twiddles W_{2^Q}^j = exp(-/+ 2 pi i j / 2^Q)
// are computed once per CTA in double precision into shared memory; each
// lane then keeps the few it needs in registers (LaneTw).

template <int E> struct Cplx;
template <> struct Cplx<8> {
  using T = float2;
  using R = float;
};
template <> struct Cplx<16> {
  using T = double2;
  using R = double;
};

template <typename T>
__device__ __forceinline__ T cmul(T a, T b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ T cadd(T a, T b) { return {a.x + b.x, a.y + b.y}; }
template <typename T>
__device__ __forceinline__ T csub(T a, T b) { return {a.x - b.x, a.y - b.y}; }

struct FftArgs {
  TileArgs t;
  int stages;   // DIT stages fused (<= QX)
  int inverse;  // 1: conjugate twiddles (unnormalised inverse transform)
};

// Radix-4 drain: the row's elements move between lane layouts through the
// warp's own rows of the tile buffer (nobody else reads them after the load),
// so every pair of stages is an in-register radix-4 pass:
//   layout A: lane ll holds x' = 4 ll + m            stages 1, 2
//   layout B: x' = (ll & 3) + 4 m + 16 (ll >> 2)      stages 3, 4
//   layout C: x' = (ll & 15) + 16 m + 64 (ll >> 4)    stages 5, 6 (complex128:
//             x' = ll + 16 m, natural for the store)
//   layout D: x' = ll + 32 m  (complex64)             stage 7, natural store
// Word x' of a row lives at swizzled position f(x'), chosen so that every
// layout's 8-byte (complex64: x ^ 5 * ((x >> 4) & 3)) or 16-byte (complex128:
// x ^ ((x >> 3) & 3) ^ (((x >> 4) & 1) << 2)) accesses are bank-conflict free.
// Twiddles are lane constants kept in registers.
template <int E>
__device__ __forceinline__ int fft_swz(int x) {
  if constexpr (E == 8) return x ^ (((x >> 4) & 3) * 5);
  else return x ^ ((x >> 3) & 3) ^ (((x >> 4) & 1) << 2);
}

template <int E, int QX>
__device__ __forceinline__ int fft_layout(int L, int ll, int m) {
  switch (L) {
    case 0: return 4 * ll + m;
    case 1: return (ll & 3) + 4 * m + 16 * (ll >> 2);
    case 2: return (E == 8) ? (ll & 15) + 16 * m + 64 * (ll >> 4) : ll + 16 * m;
    default: return ll + 32 * m;
  }
}

template <typename C>
__device__ __forceinline__ void bfly(C& top, C& bot, C w) {
  const C t = cmul(bot, w);
  bot = csub(top, t);
  top = cadd(top, t);
}

// Per-lane twiddles of the radix-4 drain, loaded once per CTA: they depend
// only on the lane (read per tile from the shared table they cost 2-8-way
// conflicting LDS.64: words 2^(QX-s) apart share a bank).  W_{2^s}^k =
// tw[k << (QX - s)] with tw = W_{2^QX}^j, j < 2^(QX-1).
template <int E, int QX, int stages>
struct LaneTw {
  using C = typename Cplx<E>::T;
  C w3, w40, w41, w5, w60, w61, w70, w71;
  __device__ __forceinline__ void load(const C* tw, int ll) {
    auto W = [&](int s, int k) { return tw[k << (QX - s)]; };
    const int a = ll & 3, b = ll & 15;
    if constexpr (stages >= 3) w3 = W(3, a);
    if constexpr (stages >= 4) { w40 = W(4, a); w41 = W(4, a + 4); }
    if constexpr (stages >= 5) w5 = W(5, b);
    if constexpr (stages >= 6) { w60 = W(6, b); w61 = W(6, b + 16); }
    if constexpr (QX >= 7 && stages >= 7) { w70 = W(7, ll); w71 = W(7, ll + 32); }
  }
};

template <int E, int QX, int QZ, int stages>
__device__ __forceinline__ void fft_rows_drain_r4(uint4* U, char* dbase, uint64_t dst_row,
                                                  const LaneTw<E, QX, stages>& lt, bool inverse) {
  using C = typename Cplx<E>::T;
  using T = Rect<E, QX, QZ>;
  constexpr int V = T::V, LPR = (1 << QX) / 4, RPP = 32 / LPR;
  constexpr int NWARPS = T::THREADS / 32;
  constexpr int ROWS = 1 << QZ;
  constexpr int NRT = (ROWS + NWARPS * RPP - 1) / (NWARPS * RPP);  // rows per lane
  // rows are drained in groups of NR: every group runs load -> stages ->
  // store on its own, so the registers of one group's row data are reused by
  // the next (taller tiles do not cost registers)
  constexpr int NR = NRT < 2 ? NRT : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp * RPP >= ROWS) return;
  const int h = lane / LPR, ll = lane % LPR;
#pragma unroll 1
  for (int grp = 0; grp < NRT / NR; ++grp) {
  auto row_of = [&](int i) { return (warp + (grp * NR + i) * NWARPS) * RPP + h; };
  auto sidx = [&](int z, int col) { return z * T::GX + (col ^ ((z >> T::LV) & 7)); };
  const C w4 = inverse ? C{0, 1} : C{0, -1};
  C v[NR][4];
  // Layout A straight from the staged tile: lane ll needs the 4/V chunks
  // (4 ll)/V + c of its row.  Reading them in lane order would put a quarter
  // warp on 4 (complex64) or 2 (complex128) of the 8 16-byte bank slots, so
  // each lane starts at a rotated chunk -- c ^ ((ll >> 2) & 1), resp.
  // (c + (ll >> 1)) & 3 -- which covers all 8 slots, and selects put the
  // chunks back in order.
  auto sel = [](bool p, const uint4& x, const uint4& y) {
    return make_uint4(p ? x.x : y.x, p ? x.y : y.y, p ? x.z : y.z, p ? x.w : y.w);
  };
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const int z = row_of(i);
    if constexpr (E == 8) {
      const int c0 = (ll >> 2) & 1;
      const uint4 q0 = U[sidx(z, 2 * ll + c0)], q1 = U[sidx(z, 2 * ll + (c0 ^ 1))];
      const uint4 lo = sel(c0, q1, q0), hi = sel(c0, q0, q1);
      v[i][0] = make_float2(__uint_as_float(lo.x), __uint_as_float(lo.y));
      v[i][1] = make_float2(__uint_as_float(lo.z), __uint_as_float(lo.w));
      v[i][2] = make_float2(__uint_as_float(hi.x), __uint_as_float(hi.y));
      v[i][3] = make_float2(__uint_as_float(hi.z), __uint_as_float(hi.w));
    } else {
      const int r = (ll >> 1) & 3;
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = U[sidx(z, 4 * ll + ((c + r) & 3))];  // chunk (c+r)&3
      if (r & 1) {  // rotate by one: q[j] <- q[j-1]
        const uint4 t = q[3];
        q[3] = q[2];
        q[2] = q[1];
        q[1] = q[0];
        q[0] = t;
      }
      if (r & 2) {  // rotate by two
        uint4 t = q[0];
        q[0] = q[2];
        q[2] = t;
        t = q[1];
        q[1] = q[3];
        q[3] = t;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
        v[i][c] = make_double2(__hiloint2double(q[c].y, q[c].x), __hiloint2double(q[c].w, q[c].z));
    }
  }
  __syncwarp();
  int L = 0;  // compile-time after unrolling: stages is a template parameter
  auto to_layout = [&](int Lnew) {  // through the warp's own rows of U
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      C* row = reinterpret_cast<C*>(U) + (size_t)row_of(i) * (1 << QX);
#pragma unroll
      for (int m = 0; m < 4; ++m) row[fft_swz<E>(fft_layout<E, QX>(L, ll, m))] = v[i][m];
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const C* row = reinterpret_cast<const C*>(U) + (size_t)row_of(i) * (1 << QX);
#pragma unroll
      for (int m = 0; m < 4; ++m) v[i][m] = row[fft_swz<E>(fft_layout<E, QX>(Lnew, ll, m))];
    }
    __syncwarp();
    L = Lnew;
  };
  const C one = C{1, 0};
  // stages 1, 2 (layout A)
  if constexpr (stages >= 1)
#pragma unroll
    for (int i = 0; i < NR; ++i) { bfly(v[i][0], v[i][1], one); bfly(v[i][2], v[i][3], one); }
  if constexpr (stages >= 2)
#pragma unroll
    for (int i = 0; i < NR; ++i) { bfly(v[i][0], v[i][2], one); bfly(v[i][1], v[i][3], w4); }
  // stages 3, 4 (layout B)
  if constexpr (stages >= 3) {
    to_layout(1);
#pragma unroll
    for (int i = 0; i < NR; ++i) { bfly(v[i][0], v[i][1], lt.w3); bfly(v[i][2], v[i][3], lt.w3); }
    if constexpr (stages >= 4) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        bfly(v[i][0], v[i][2], lt.w40);
        bfly(v[i][1], v[i][3], lt.w41);
      }
    }
  }
  // stages 5, 6 (layout C)
  if constexpr (stages >= 5) {
    to_layout(2);
#pragma unroll
    for (int i = 0; i < NR; ++i) { bfly(v[i][0], v[i][1], lt.w5); bfly(v[i][2], v[i][3], lt.w5); }
    if constexpr (stages >= 6) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        bfly(v[i][0], v[i][2], lt.w60);
        bfly(v[i][1], v[i][3], lt.w61);
      }
    }
  }
  // stage 7 (layout D, complex64 only)
  if constexpr (QX >= 7) {
    if constexpr (stages >= 7) {
      to_layout(3);
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        bfly(v[i][0], v[i][2], lt.w70);
        bfly(v[i][1], v[i][3], lt.w71);
      }
    }
  }
  // store from whatever layout the last stage left: for each m every layout's
  // lanes cover whole 32-byte sectors (A: 4 contiguous per lane; B: runs of 4;
  // C: runs of 16; D: 32 contiguous), so no final transpose is needed
  auto store = [&](auto layout_tag) {
    constexpr int LS = decltype(layout_tag)::value;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int z = row_of(i);
      char* drow = dbase + (uint64_t)(__brev((unsigned)z) >> (32 - QZ)) * dst_row;
      if constexpr (LS == 0) {  // 4 contiguous elements per lane
        char* p = drow + (uint64_t)(4 * ll) * E;
        if constexpr (E == 8) {
          st_vec(p, make_uint4(__float_as_uint(v[i][0].x), __float_as_uint(v[i][0].y),
                               __float_as_uint(v[i][1].x), __float_as_uint(v[i][1].y)));
          st_vec(p + 16, make_uint4(__float_as_uint(v[i][2].x), __float_as_uint(v[i][2].y),
                                    __float_as_uint(v[i][3].x), __float_as_uint(v[i][3].y)));
        } else {
#pragma unroll
          for (int m = 0; m < 4; ++m)
            st_vec(p + 16 * m, make_uint4(__double2loint(v[i][m].x), __double2hiint(v[i][m].x),
                                          __double2loint(v[i][m].y), __double2hiint(v[i][m].y)));
        }
      } else {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          *reinterpret_cast<C*>(drow + (uint64_t)fft_layout<E, QX>(LS, ll, m) * E) = v[i][m];
      }
    }
  };
  // final layout.  complex64 after 3-4 stages: layout B stores 32-byte runs
  // per group of 4 lanes; one more exchange into layout C gives 128-byte runs
  // (+11 % at 4 stages).  complex128's layout-B runs are already 64 bytes and
  // the exchange costs more than it saves (-2.6 %).
  constexpr bool kBtoC = E == 8 && stages >= 3 && stages <= 4;
  if constexpr (kBtoC) to_layout(2);
  constexpr int LF = stages <= 2 ? 0 : stages <= 4 ? (kBtoC ? 2 : 1) : stages <= 6 ? 2 : 3;
  store(std::integral_constant<int, LF>{});
  (void)L;
  }
}

// Radix-8 drain for complex64 rows of 128 (QX = 7), 4-7 fused stages.  The
// radix-4 drain above needs three layout exchanges for 7 stages (A -> B -> C
// -> D); here a lane holds 8 elements and 16 lanes share a row (two rows per
// warp pass), so three stages run per in-register pass and two exchanges do:
//   A8: x' = 8 ll + m                        stages 1-3 (twiddles: constants)
//   B8: x' = (ll & 7) + 8 m + 64 (ll >> 3)    stages 4-6
//   C8: x' = ll + 16 m                        stage 7, then a natural store
// (ll < 16 = lane within the row, m < 8 = register slot).  The exchanges go
// through the half-warp's own row of the tile buffer with the 8-byte-slot
// swizzle f(x) = x ^ (x >> 4 & 7) ^ ((x >> 6 & 1) << 3), under which each
// layout's 16 lanes of a row hit 16 distinct bank slots.
struct LaneTw8 {
  float2 w16, w32, w64, w128;  // W_16^r, W_32^r, W_64^r (r = ll & 7), W_128^ll
  // tw = W_{2^QX}^j, j < 2^(QX-1); st = 2^(QX-7) maps W_128^k to tw[k * st]
  __device__ __forceinline__ void load(const float2* tw, int ll, int st = 1) {
    const int r = ll & 7;
    w16 = tw[(r << 3) * st];
    w32 = tw[(r << 2) * st];
    w64 = tw[(r << 1) * st];
    w128 = tw[ll * st];
  }
};

__device__ __forceinline__ int fft8_swz(int x) { return x ^ ((x >> 4) & 7) ^ (((x >> 6) & 1) << 3); }

// QX = 8 (256-element destination rows): each row holds two 128-element
// FFT blocks (up to 7 stages stay inside a block); the two half-warps of a
// warp take the two blocks of one row, so the row is read whole before
// either half overwrites its own block as exchange scratch.
template <int QZ, int STAGES, int QX = 7>
__device__ __forceinline__ void fft_rows_drain_r8(uint4* U, char* dbase, uint64_t dst_row,
                                                  const LaneTw8& lt, bool inverse) {
  static_assert(STAGES >= 1 && STAGES <= 7, "radix-8 drain: 1 to 7 stages");
  static_assert(QX == 7 || QX == 8, "128-element blocks, one or two per row");
  using C = float2;
  using T = Rect<8, QX, QZ>;
  constexpr int NB = 1 << (QX - 7);  // 128-element blocks per row
  constexpr int NWARPS = T::THREADS / 32;
  constexpr int ROWS = (1 << QZ) * NB;  // blocks
  constexpr int PASSES = ROWS / (2 * NWARPS);
  static_assert(PASSES >= 1 && ROWS % (2 * NWARPS) == 0, "two blocks per warp pass");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = lane >> 4, ll = lane & 15;
  auto sidx = [&](int z, int col) { return z * T::GX + (col ^ ((z >> T::LV) & 7)); };
  const float sg = inverse ? 1.f : -1.f;          // sign of the twiddle exponent
  const float rh = 0.70710678118654752f;
  const C w4 = C{0.f, sg};                          // W_4
  const C w8 = C{rh, sg * rh};                      // W_8
  const C w83 = C{-rh, sg * rh};                    // W_8^3
  auto mulj = [&](C a) { return C{-sg * a.y, sg * a.x}; };  // a * W_4
#pragma unroll 1
  for (int pass = 0; pass < PASSES; ++pass) {
    const int zb = (warp + pass * NWARPS) * 2 + h;
    const int z = zb >> (QX - 7), blk = zb & (NB - 1);
    C v[8];
    // A8 from the staged tile: the lane's 4 chunks 4 ll + c, read from a
    // rotated start so the 8 lanes of a quarter warp cover all 8 bank slots
    {
      const int rot = (ll >> 1) & 3;
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = U[sidx(z, blk * 64 + 4 * ll + ((c + rot) & 3))];
      if (rot & 1) {
        const uint4 t = q[3];
        q[3] = q[2];
        q[2] = q[1];
        q[1] = q[0];
        q[0] = t;
      }
      if (rot & 2) {
        uint4 t = q[0];
        q[0] = q[2];
        q[2] = t;
        t = q[1];
        q[1] = q[3];
        q[3] = t;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[2 * c] = make_float2(__uint_as_float(q[c].x), __uint_as_float(q[c].y));
        v[2 * c + 1] = make_float2(__uint_as_float(q[c].z), __uint_as_float(q[c].w));
      }
    }
    // stages 1-3 (A8): constant twiddles
#pragma unroll
    for (int m = 0; m < 8; m += 2) {
      const C t = v[m + 1];
      v[m + 1] = csub(v[m], t);
      v[m] = cadd(v[m], t);
    }
#pragma unroll
    for (int g = 0; g < 8 && STAGES >= 2; g += 4) {
      C t = v[g + 2];
      v[g + 2] = csub(v[g], t);
      v[g] = cadd(v[g], t);
      t = mulj(v[g + 3]);
      v[g + 3] = csub(v[g + 1], t);
      v[g + 1] = cadd(v[g + 1], t);
    }
    if constexpr (STAGES >= 3) {
      C t = v[4];
      v[4] = csub(v[0], t);
      v[0] = cadd(v[0], t);
      t = cmul(v[5], w8);
      v[5] = csub(v[1], t);
      v[1] = cadd(v[1], t);
      t = mulj(v[6]);
      v[6] = csub(v[2], t);
      v[2] = cadd(v[2], t);
      t = cmul(v[7], w83);
      v[7] = csub(v[3], t);
      v[3] = cadd(v[3], t);
    }
    C* row = reinterpret_cast<C*>(U) + (size_t)z * (128 * NB) + blk * 128;
    __syncwarp();  // every lane of the row has read its staged chunks
#pragma unroll
    for (int m = 0; m < 8; ++m) row[fft8_swz(8 * ll + m)] = v[m];
    __syncwarp();
    const int r = ll & 7, hi = ll >> 3;
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = row[fft8_swz(r + 8 * m + 64 * hi)];
    // stages 4-6 (B8): pairs 8, 16, 32 apart
#pragma unroll
    for (int m = 0; m < 8 && STAGES >= 4; m += 2) bfly(v[m], v[m + 1], lt.w16);
    if constexpr (STAGES >= 5) {
      const C a = lt.w32, b = mulj(lt.w32);  // W_32^r, W_32^(r+8)
#pragma unroll
      for (int g = 0; g < 8; g += 4) {
        bfly(v[g], v[g + 2], a);
        bfly(v[g + 1], v[g + 3], b);
      }
    }
    if constexpr (STAGES >= 6) {
      const C a0 = lt.w64, a1 = cmul(lt.w64, w8), a2 = mulj(lt.w64), a3 = cmul(lt.w64, w83);
      bfly(v[0], v[4], a0);
      bfly(v[1], v[5], a1);
      bfly(v[2], v[6], a2);
      bfly(v[3], v[7], a3);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 8; ++m) row[fft8_swz(r + 8 * m + 64 * hi)] = v[m];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = row[fft8_swz(ll + 16 * m)];
    // stage 7 (C8): pairs 64 apart, W_128^(ll + 16 t) = W_128^ll * W_8^t
    if constexpr (STAGES >= 7) {
      const C b0 = lt.w128, b1 = cmul(lt.w128, w8), b2 = mulj(lt.w128), b3 = cmul(lt.w128, w83);
      bfly(v[0], v[4], b0);
      bfly(v[1], v[5], b1);
      bfly(v[2], v[6], b2);
      bfly(v[3], v[7], b3);
    }
    // natural store: for each m the row's 16 lanes write 128 contiguous bytes
    char* drow = dbase + (uint64_t)(__brev((unsigned)z) >> (32 - QZ)) * dst_row + blk * 1024;
#pragma unroll
    for (int m = 0; m < 8; ++m) *reinterpret_cast<C*>(drow + (uint64_t)(ll + 16 * m) * 8) = v[m];
    __syncwarp();  // the row is free for the next pass's exchange
  }
}

// complex128, 1..STAGES (<= 5) fused stages on the square Q6 tiles of the
// out-of-place complex128 kernel (1 KB rows on both sides, cfg3-16's shape).
// A drain item is one 16-byte element: with 256 threads and 64 elements per
// destination row, a thread's column x = tid % 64 is the same for every item
// it drains, and a warp holds 32 consecutive x of one row.  Stage s pairs x
// with x ^ 2^(s-1) -- lane ^ 2^(s-1) for s <= 5 -- so the butterflies run
// on warp shuffles of the four 32-bit words, with twiddles W_{2^s}^(x mod
// 2^(s-1)) fixed per thread (computed once).
template <int STAGES, bool CS = false>
__global__ void __launch_bounds__(256, 1) bitrev_fft_tile16_kernel(FftArgs fa) {
  static_assert(STAGES >= 1 && STAGES <= 5, "shuffle stages stay inside a warp");
  using T = Tile<16, 6, 256>;
  extern __shared__ __align__(16) uint4 smem[];
  const TileArgs& a = fa.t;
  const uint64_t row_stride = (uint64_t)16 << (a.b - 6);
  const uint64_t mmask = (1ull << a.m) - 1;
  uint4 r[T::IPT][T::V];
  const int x = threadIdx.x & 63;
  // Stage s, pair (x, x + h), h = 2^(s-1): the lower lane needs v + w p, the
  // upper one p - w v.  Each lane first scales its own value by wp[s] (w in
  // the upper lane, 1 in the lower), swaps the scaled values with its
  // partner, and adds: out = other + sgn[s] * own (sgn = -1 in the upper
  // lane) -- no selects.  w = W_{2^s}^(x mod h); stage 1 has w = 1.
  double2 wp[STAGES + 1];
  double sgn[STAGES + 1];
#pragma unroll
  for (int s = 1; s <= STAGES; ++s) {
    const int h = 1 << (s - 1);
    const bool upper = x & h;
    double sn = 0.0, cs = 1.0;
    if (upper) sincospi((fa.inverse ? 2.0 : -2.0) * (x & (h - 1)) / (1 << s), &sn, &cs);
    wp[s] = make_double2(cs, sn);
    sgn[s] = upper ? -1.0 : 1.0;
  }
  auto dv = [](const uint4& u) {
    return make_double2(__hiloint2double((int)u.y, (int)u.x), __hiloint2double((int)u.w, (int)u.z));
  };
  auto ud = [](const double2& d) {
    return make_uint4((unsigned)__double2loint(d.x), (unsigned)__double2hiint(d.x),
                      (unsigned)__double2loint(d.y), (unsigned)__double2hiint(d.y));
  };

  uint64_t t = blockIdx.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (no-op otherwise)
  if (t >= a.ntiles) return;
  auto src_tile = [&](uint64_t tt) {
    const uint64_t bi = tt >> a.m, y = tt & mmask;
    return a.src + bi * a.src_bstride + (y << 6) * 16;
  };
  tile_load<16, 6, true, 256, CS && BITREV_LD_CS>(r, src_tile(t), row_stride);
  for (;;) {
    const uint64_t bi = t >> a.m, y = t & mmask;
    tile_stage<16, 6, 256>(r, smem);
    __syncthreads();
    const uint64_t tn = t + gridDim.x;
    if (tn < a.ntiles) tile_load<16, 6, true, 256, CS && BITREV_LD_CS>(r, src_tile(tn), row_stride);
    else asm volatile("griddepcontrol.launch_dependents;");
    char* dbase = a.dst + bi * a.dst_bstride + (dev_rev(y, a.m) << 6) * 16;
#pragma unroll
    for (int it = 0; it < T::WPT; ++it) {
      const int id = it * 256 + threadIdx.x;
      const int z = id >> 6;  // column id & 63 == x
      double2 v = dv(smem[swz<16, 6>(z, x)]);
#pragma unroll
      for (int s = 1; s <= STAGES; ++s) {
        const int h = 1 << (s - 1);
        double2 e = v;
        if (s > 1) {
          const double2 w = wp[s];
          e = make_double2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
        }
        double2 o;
        o.x = __shfl_xor_sync(0xffffffffu, e.x, h);
        o.y = __shfl_xor_sync(0xffffffffu, e.y, h);
        v = make_double2(fma(sgn[s], e.x, o.x), fma(sgn[s], e.y, o.y));
      }
      const uint64_t rz = __brev((unsigned)z) >> (32 - 6);
      st_vec<CS>(dbase + rz * row_stride + (uint64_t)x * 16, ud(v));
    }
    if (tn >= a.ntiles) break;
    __syncthreads();
    t = tn;
  }
}

// Rectangular-tile FFT pre-pass (bitrev_oop_rect_kernel's load/stage path).
template <int E, int QX, int QZ, int STAGES>
__global__ void __launch_bounds__(Rect<E, QX, QZ>::THREADS,
                                  STAGES >= BITREV_FFT_MINB_FROM && QX <= 7
                                      ? (QZ >= 5 ? 2 : BITREV_FFT_MINB) : 1)
    bitrev_fft_rect_kernel(FftArgs fa) {
  using T = Rect<E, QX, QZ>;
  using C = typename Cplx<E>::T;
  using Rl = typename Cplx<E>::R;
  extern __shared__ __align__(16) uint4 smem[];
  __shared__ C twq[1 << (QX - 1)];  // W_{2^QX}^j, j < 2^(QX-1)
  const TileArgs& a = fa.t;
  const uint64_t src_row = (uint64_t)E << (a.b - QX);
  const uint64_t dst_row = (uint64_t)E << (a.b - QZ);
  const uint64_t mmask = (1ull << a.m) - 1;
  for (int j = threadIdx.x; j < (1 << (QX - 1)); j += blockDim.x) {
    double sn, cs;
    sincospi((fa.inverse ? 2.0 : -2.0) * j / (1 << QX), &sn, &cs);
    twq[j] = C{(Rl)cs, (Rl)sn};
  }
  uint4 r[T::IPT][T::V];
  auto load = [&](uint64_t tt) {
    const uint64_t bi = tt >> a.m, y = tt & mmask;
    const char* base = a.src + bi * a.src_bstride + (y << QZ) * E;
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CZ, g = id / T::CZ;
#pragma unroll
      for (int k = 0; k < T::V; ++k)
        r[it][k] = ld_stream(base + (uint64_t)(g + k * T::GX) * src_row + (uint64_t)c * 16);
    }
  };
  auto sidx = [&](int z, int col) { return z * T::GX + (col ^ ((z >> T::LV) & 7)); };

  uint64_t t = blockIdx.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (no-op otherwise)
  if (t >= a.ntiles) return;
  load(t);
  __syncthreads();  // publish twq
  constexpr bool kR8 = E == 8 && (QX == 8 || (QX == 7 && STAGES >= BITREV_FFT_R8_FROM && STAGES >= 4));
  static_assert(QX != 8 || kR8, "256-element rows take the radix-8 drain");
  LaneTw<E, (QX > 7 ? 7 : QX), kR8 ? 0 : STAGES> lt;
  LaneTw8 lt8;
  if constexpr (kR8) lt8.load(reinterpret_cast<const float2*>(twq), threadIdx.x & 15, 1 << (QX - 7));
  else lt.load(twq, (threadIdx.x & 31) % ((1 << QX) / 4));
  for (;;) {
    const uint64_t bi = t >> a.m, y = t & mmask;
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CZ, g = id / T::CZ;
      const int col = (int)(__brev((unsigned)g) >> (32 - (QX - T::LV)));
      smem[sidx(c * T::V, col)] = xpose<E, 0>(r[it]);
      if constexpr (T::V > 1) smem[sidx(c * T::V + 1, col)] = xpose<E, 1>(r[it]);
    }
    __syncthreads();
    const uint64_t tn = t + gridDim.x;
    if (tn < a.ntiles) load(tn);
    else asm volatile("griddepcontrol.launch_dependents;");
    char* dbase = a.dst + bi * a.dst_bstride + (dev_rev(y, a.m) << QX) * E;
    if constexpr (kR8) fft_rows_drain_r8<QZ, STAGES, QX>(smem, dbase, dst_row, lt8, fa.inverse != 0);
    else fft_rows_drain_r4<E, (QX > 7 ? 7 : QX), QZ, STAGES>(smem, dbase, dst_row, lt, fa.inverse != 0);
    if (tn >= a.ntiles) break;
    __syncthreads();
    t = tn;
  }
}

// Small rows (n*E <= 32 KB, any number of stages up to b, i.e. a full
// radix-2 FFT): one CTA per row, bit-reversed load into shared memory, then
// the stages with a barrier between them, then a coalesced store.
template <int E>
__global__ void __launch_bounds__(256) fft_prepass_small_kernel(FftArgs fa) {
  using C = typename Cplx<E>::T;
  using Rl = typename Cplx<E>::R;
  extern __shared__ __align__(16) uint4 smem_f[];
  C* buf = reinterpret_cast<C*>(smem_f);
  const TileArgs& a = fa.t;
  const int b = a.b;
  const int n = 1 << b;
  const double sign = fa.inverse ? 2.0 : -2.0;
  for (int64_t row = blockIdx.x; row < a.batch; row += gridDim.x) {
    const C* src = reinterpret_cast<const C*>(a.src + row * a.src_bstride);
    C* dst = reinterpret_cast<C*>(a.dst + row * a.dst_bstride);
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[dev_rev((uint64_t)i, b)] = src[i];
    __syncthreads();
    for (int s = 1; s <= fa.stages; ++s) {
      const int half = 1 << (s - 1);
      for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
        const int k = t & (half - 1);
        const int i0 = ((t >> (s - 1)) << s) + k;
        double sn, cs;
        sincospi(sign * k / (2 * half), &sn, &cs);
        const C w{(Rl)cs, (Rl)sn};
        const C u = buf[i0], v = cmul(buf[i0 + half], w);
        buf[i0] = cadd(u, v);
        buf[i0 + half] = csub(u, v);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = buf[i];
    __syncthreads();
  }
}

// Geometry of the short-row kernels (bitrev_rows_kernel, fft_rows_kernel):
// KB-kilobyte blocks of consecutive rows, 256 threads, NV 16-byte vectors per
// thread.
template <int E, int KB = 32>
struct Rows {
  static constexpr int V = 16 / E;
  static constexpr int LV = const_log2(V);
  static constexpr int THREADS = 256;
  static constexpr int BYTES = KB * 1024;
  static constexpr int NV = BYTES / 16 / THREADS;  // 16-byte vectors per thread per block
};

// ---------------------------------------------------------------------------
// FFT pre-pass on short rows (n*E <= 32 KB, 16-byte aligned): many rows per
// CTA, as bitrev_rows_kernel -- a 32 KB block of rows is loaded with 16-byte
// vectors and scattered bit-reversed into shared memory; then the requested
// radix-2 DIT stages run on the block in shared memory, paired into radix-4
// passes (one barrier per pass for the whole block, not per row); then
// LDS.128 -> STG.128.  Twiddles
// W_n^j (j < n/2) are computed once per CTA in double precision into a shared
// table; stage s uses W_{2^s}^k = W_n^(k * 2^(b-s)).

#ifndef BITREV_FFT_ROWS_MINB16
#define BITREV_FFT_ROWS_MINB16 3
#endif
#ifndef BITREV_FFT_ROWS_MINB8
#define BITREV_FFT_ROWS_MINB8 2
#endif
// Rotate a 4-array right by r (runtime): a[m] <- a[(m - r) & 3], as selects.
template <typename C>
__device__ __forceinline__ void rot4(C (&a)[4], int r) {
  if (r & 1) {
    const C t = a[3];
    a[3] = a[2];
    a[2] = a[1];
    a[1] = a[0];
    a[0] = t;
  }
  if (r & 2) {
    C t = a[0];
    a[0] = a[2];
    a[2] = t;
    t = a[1];
    a[1] = a[3];
    a[3] = t;
  }
}

template <int E, bool ROT, int KB = 32>
__global__ void __launch_bounds__(256, KB > 32 ? 2 : (E == 16 ? BITREV_FFT_ROWS_MINB16 : BITREV_FFT_ROWS_MINB8))
    fft_rows_kernel(FftArgs fa, int swz) {
  using C = typename Cplx<E>::T;
  using Rl = typename Cplx<E>::R;
  using R = Rows<E, KB>;
  extern __shared__ __align__(16) uint4 smem[];
  C* tw = reinterpret_cast<C*>(reinterpret_cast<char*>(smem) + R::BYTES);
  const TileArgs& a = fa.t;
  const int b = a.b, half_n = 1 << (b - 1);
  const int vb = b - R::LV;
  const int rb = const_log2(R::BYTES / 16) - vb;
  const int64_t nblocks = (a.batch + (1ll << rb) - 1) >> rb;
  auto phys = [&](int c) { return c ^ ((c >> swz) & 7); };
  C* sc = reinterpret_cast<C*>(smem);
  // element d of block row rl, through the 16-byte chunk swizzle
  auto at = [&](int rl, int d) -> C& {
    return sc[phys((rl << vb) + (d >> R::LV)) * R::V + (d & (R::V - 1))];
  };
  int64_t blk = blockIdx.x;
  if (blk >= nblocks) return;
  for (int j = threadIdx.x; j < half_n; j += R::THREADS) {
    double sn, cs;
    sincospi((fa.inverse ? 2.0 : -2.0) * j / (2 * half_n), &sn, &cs);
    tw[j] = C{(Rl)cs, (Rl)sn};
  }
  uint4 r[R::NV];
  auto load = [&](int64_t k) {
#pragma unroll
    for (int j = 0; j < R::NV; ++j) {
      const int v = j * R::THREADS + threadIdx.x;
      const int64_t row = (k << rb) + (v >> vb);
      if (row < a.batch)
        r[j] = ld_stream(a.src + row * a.src_bstride + (int64_t)(v & ((1 << vb) - 1)) * 16);
    }
  };
  load(blk);
  for (;;) {
#pragma unroll
    for (int j = 0; j < R::NV; ++j) {
      const int v = j * R::THREADS + threadIdx.x;
      const int rl = v >> vb, pos = v & ((1 << vb) - 1);
      const C* e = reinterpret_cast<const C*>(&r[j]);
      const int rp = vb ? (int)(__brev((unsigned)pos) >> (32 - vb)) : 0;
#pragma unroll
      for (int t = 0; t < R::V; ++t) {
        const int rt = R::LV ? (int)(__brev((unsigned)t) >> (32 - R::LV)) : 0;
        at(rl, (rt << vb) + rp) = e[t];
      }
    }
    __syncthreads();
    const int64_t nxt = blk + gridDim.x;
    const int64_t base_row = blk << rb;
    if (nxt < nblocks) load(nxt);
    const int nbf = 1 << (rb + b - 1);  // butterflies per stage in the block
    int st0 = 1;
    // stage pairs (s, s+1) as radix-4 passes: a thread owns the quad
    // (k, k+h, k+2h, k+3h) of an aligned 4h block, h = 2^(s-1); stage s pairs
    // (k, k+h) and (k+2h, k+3h) with W_{2h}^kk, stage s+1 pairs (k, k+2h) with
    // W_{4h}^kk and (k+h, k+3h) with W_{4h}^(kk+h): half the shared-memory
    // passes and barriers of radix-2
    for (; st0 + 1 <= fa.stages; st0 += 2) {
      const int h = 1 << (st0 - 1);
      const int nq = nbf >> 1;
      for (int q = threadIdx.x; q < nq; q += R::THREADS) {
        const int rl = q >> (b - 2), t = q & ((half_n >> 1) - 1);
        const int kk = t & (h - 1);
        const int i0 = ((t >> (st0 - 1)) << (st0 + 1)) + kk;
        // ROT (longer rows): access the quad in an order rotated by rot -- with
        // small h the lanes of one wavefront (16 for 8-byte, 8 for 16-byte
        // elements) would hit only 4 (resp. 2) of the bank slots.  Shorter
        // rows are already spread by the chunk swizzle and skip the selects.
        const int rot = ROT ? ((E == 8 ? (q >> 2) : (q >> 1)) & 3) : 0;
        C x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = at(rl, i0 + ((j + rot) & 3) * h);
        if constexpr (ROT) rot4(x, rot);  // x[m] = element i0 + m*h
        C x0 = x[0], x1 = x[1], x2 = x[2], x3 = x[3];
        const C w1 = tw[kk << (b - st0)];
        C v = cmul(x1, w1);
        x1 = csub(x0, v);
        x0 = cadd(x0, v);
        v = cmul(x3, w1);
        x3 = csub(x2, v);
        x2 = cadd(x2, v);
        v = cmul(x2, tw[kk << (b - st0 - 1)]);
        x2 = csub(x0, v);
        x0 = cadd(x0, v);
        v = cmul(x3, tw[(kk + h) << (b - st0 - 1)]);
        x3 = csub(x1, v);
        x1 = cadd(x1, v);
        x[0] = x0;
        x[1] = x1;
        x[2] = x2;
        x[3] = x3;
        if constexpr (ROT) rot4(x, (4 - rot) & 3);  // x[j] = element i0 + ((j + rot) & 3)*h
#pragma unroll
        for (int j = 0; j < 4; ++j) at(rl, i0 + ((j + rot) & 3) * h) = x[j];
      }
      __syncthreads();
    }
    for (int st = st0; st <= fa.stages; ++st) {  // an odd last stage: radix 2
      const int half = 1 << (st - 1);
      for (int k = threadIdx.x; k < nbf; k += R::THREADS) {
        const int rl = k >> (b - 1), t = k & (half_n - 1);
        const int kk = t & (half - 1);
        const int i0 = ((t >> (st - 1)) << st) + kk;
        C& p0 = at(rl, i0);
        C& p1 = at(rl, i0 + half);
        const C u = p0, v = cmul(p1, tw[kk << (b - st)]);
        p0 = cadd(u, v);
        p1 = csub(u, v);
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < R::NV; ++j) {
      const int c = j * R::THREADS + threadIdx.x;
      const int64_t row = base_row + (c >> vb);
      if (row < a.batch)
        st_vec(a.dst + row * a.dst_bstride + (int64_t)(c & ((1 << vb) - 1)) * 16, smem[phys(c)]);
    }
    if (nxt >= nblocks) break;
    __syncthreads();
    blk = nxt;
  }
}

// ---------------------------------------------------------------------------
// whole-row-in-shared-memory kernel for small n (n*E <= kSmallBytes); one CTA
// per batch row, grid-stride over rows.  Works in place (src == dst) because
// every read of a row precedes the barrier and every write follows it.

constexpr int kSmallBytes = 32 * 1024;

template <int E>
__global__ void __launch_bounds__(256)
    bitrev_small_kernel(const char* src, char* dst, int b, int64_t batch, int64_t src_bstride,
                        int64_t dst_bstride) {
  using W = typename Word<E>::T;
  extern __shared__ __align__(16) uint4 smem_raw[];
  W* buf = reinterpret_cast<W*>(smem_raw);
  const int n = 1 << b;
  for (int64_t row = blockIdx.x; row < batch; row += gridDim.x) {
    const W* s = reinterpret_cast<const W*>(src + row * src_bstride);
    W* d = reinterpret_cast<W*>(dst + row * dst_bstride);
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = s[i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = buf[dev_rev((uint64_t)i, b)];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// short rows (n*E <= 32 KB, too short for a V x V tile): many rows per CTA
//
// One CTA iteration moves a 32 KB block of R = 32 KB / (n*E) consecutive
// rows: 16-byte vector loads into registers (coalesced along each row), an
// element scatter into shared memory at the bit-reversed position, a barrier,
// then LDS.128 -> STG.128 of whole 16-byte output chunks.  The next block's
// loads are issued before the drain.  A block's rows belong to this CTA alone,
// so src == dst (in place) is safe.  Shared memory is swizzled per 16-byte
// chunk: phys = c ^ ((c >> s) & 7), with s chosen so that the chunk bits that
// vary across a warp's scatter (the top bits of rev(pos)) select different
// bank groups; the linear drain stays conflict-free because the XOR term is
// constant over every aligned group of 8 chunks (s >= 3).
template <int E, bool INPLACE, int KB = 32>
__global__ void __launch_bounds__(Rows<E, KB>::THREADS)
    bitrev_rows_kernel(const char* src, char* dst, int b, int64_t batch, int64_t sbs,
                       int64_t dbs, int s) {
  using R = Rows<E, KB>;
  using W = typename Word<E>::T;
  extern __shared__ __align__(16) uint4 smem[];
  const int vb = b - R::LV;                        // vector-index bits per row
  const int rb = const_log2(R::BYTES / 16) - vb;   // log2(rows per block)
  const int64_t nblocks = (batch + (1ll << rb) - 1) >> rb;
  auto phys = [&](int c) { return c ^ ((c >> s) & 7); };
  uint4 r[R::NV];
  auto load = [&](int64_t blk) {
#pragma unroll
    for (int j = 0; j < R::NV; ++j) {
      const int v = j * R::THREADS + threadIdx.x;
      const int64_t row = (blk << rb) + (v >> vb);
      if (row < batch) {
        const char* p = src + row * sbs + (int64_t)(v & ((1 << vb) - 1)) * 16;
        r[j] = INPLACE ? ld_plain(p) : ld_stream(p);
      }
    }
  };
  int64_t blk = blockIdx.x;
  if (blk >= nblocks) return;
  load(blk);
  for (;;) {
    W* sw = reinterpret_cast<W*>(smem);
#pragma unroll
    for (int j = 0; j < R::NV; ++j) {
      const int v = j * R::THREADS + threadIdx.x;
      const int rl = v >> vb, pos = v & ((1 << vb) - 1);
      const W* e = reinterpret_cast<const W*>(&r[j]);
      const int rp = vb ? (int)(__brev((unsigned)pos) >> (32 - vb)) : 0;  // rev_{b-LV}(pos)
#pragma unroll
      for (int t = 0; t < R::V; ++t) {
        // element pos*V + t lands at rev_b = rev_LV(t) * 2^(b-LV) + rev(pos)
        const int rt = R::LV ? (int)(__brev((unsigned)t) >> (32 - R::LV)) : 0;
        const int d = (rt << vb) + rp;                       // destination element in the row
        const int c = (rl << vb) + (d >> R::LV);             // its 16-byte chunk in the block
        sw[phys(c) * R::V + (d & (R::V - 1))] = e[t];
      }
    }
    __syncthreads();
    const int64_t nxt = blk + gridDim.x;
    const int64_t base_row = blk << rb;
    if (nxt < nblocks) load(nxt);
#pragma unroll
    for (int j = 0; j < R::NV; ++j) {
      const int c = j * R::THREADS + threadIdx.x;
      const int64_t row = base_row + (c >> vb);
      if (row < batch)
        st_vec(dst + row * dbs + (int64_t)(c & ((1 << vb) - 1)) * 16, smem[phys(c)]);
    }
    if (nxt >= nblocks) break;
    __syncthreads();
    blk = nxt;
  }
}

// ---------------------------------------------------------------------------
// element-wise fallbacks (unaligned pointers, 1/2-byte elements): correct for
// every width, not bandwidth-optimal.

template <int E>
__global__ void bitrev_gather_kernel(const char* src, char* dst, int b, int64_t batch,
                                     int64_t src_bstride, int64_t dst_bstride) {
  using W = typename Word<E>::T;
  const uint64_t n = 1ull << b;
  const uint64_t total = n * (uint64_t)batch;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = t >> b, i = t & (n - 1);
    const W* s = reinterpret_cast<const W*>(src + row * src_bstride);
    W* d = reinterpret_cast<W*>(dst + row * dst_bstride);
    d[i] = s[dev_rev(i, b)];
  }
}

// Swap a[i] <-> a[rev(i)] for i < rev(i): the data-parallel form of
// _naive_bitwise (src/permutations.py:66-78); each pair is owned by one thread.
template <int E>
__global__ void bitrev_swap_kernel(char* a, int b, int64_t batch, int64_t bstride) {
  using W = typename Word<E>::T;
  const uint64_t n = 1ull << b;
  const uint64_t total = n * (uint64_t)batch;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = t >> b, i = t & (n - 1);
    const uint64_t r = dev_rev(i, b);
    if (i < r) {
      W* p = reinterpret_cast<W*>(a + row * bstride);
      const W tmp = p[i];
      p[i] = p[r];
      p[r] = tmp;
    }
  }
}

// ---------------------------------------------------------------------------
// square in-place transpose (replaces _transpose_diag/_transpose_offdiag,
// src/recursive.py:30-81): tile pair {(I,J),(J,I)}, I <= J, per CTA-iteration.

constexpr int kTT = 32;  // transpose tile side

template <int E>
__global__ void __launch_bounds__(256)
    transpose_square_kernel(char* a, int h, int64_t batch, int64_t bstride) {
  using W = typename Word<E>::T;
  __shared__ W t0[kTT][kTT + 1];
  __shared__ W t1[kTT][kTT + 1];
  const int side = 1 << h;
  const int ts = side < kTT ? side : kTT;
  const int nt = side / ts;  // tiles per dimension
  const uint64_t per = (uint64_t)nt * nt;
  const uint64_t total = per * (uint64_t)batch;
  const int tx = threadIdx.x % kTT, ty = threadIdx.x / kTT;  // 32 x 8
  for (uint64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const uint64_t bi = w / per;
    const uint64_t rem = w % per;
    const int I = (int)(rem / nt), J = (int)(rem % nt);
    if (I > J) continue;  // block-uniform
    W* m = reinterpret_cast<W*>(a + bi * bstride);
    for (int r = ty; r < ts; r += 8)
      if (tx < ts) {
        t0[r][tx] = m[(uint64_t)(I * ts + r) * side + J * ts + tx];
        if (I != J) t1[r][tx] = m[(uint64_t)(J * ts + r) * side + I * ts + tx];
      }
    __syncthreads();
    for (int r = ty; r < ts; r += 8)
      if (tx < ts) {
        m[(uint64_t)(J * ts + r) * side + I * ts + tx] = t0[tx][r];
        if (I != J) m[(uint64_t)(I * ts + r) * side + J * ts + tx] = t1[tx][r];
      }
    __syncthreads();
  }
}

// Vectorised square in-place transpose: tile pairs {(I, J), (J, I)}, I <= J,
// of 2^Q x 2^Q tiles (256-512-byte rows), both tiles loaded with 16-byte
// vectors before either is written (the pair's regions belong to it alone).
// The tile path of the bit-reversal kernels with the reversals taken out:
// each thread loads V consecutive rows at one 16-byte column, a V x V
// register transpose makes V destination vectors, XOR-swizzled STS, barrier,
// then LDS.128 -> STG.128 along the transposed rows.
template <int E, int Q>
struct TrTile {
  static constexpr int S = 1 << Q, V = 16 / E, LV = const_log2(V);
  static constexpr int CH = S / V;          // 16-byte chunks per row
  static constexpr int ITEMS = CH * CH;      // load items (V rows each)
  static constexpr int THREADS = 256;
  static constexpr int IPT = ITEMS / THREADS;
  static constexpr int WPT = S * CH / THREADS;
  static constexpr int BYTES = S * S * E;
  static_assert(CH >= 8 && ITEMS % THREADS == 0, "tile geometry");
};

template <int E, int J>
__device__ __forceinline__ uint4 xpose_nat(const uint4 (&a)[16 / E]) {
  if constexpr (E == 4) return make_uint4(comp<J>(a[0]), comp<J>(a[1]), comp<J>(a[2]), comp<J>(a[3]));
  else return xpose<E, J>(a);  // E = 8 / 16: already in natural row order
}

template <int E, int Q>
__global__ void __launch_bounds__(TrTile<E, Q>::THREADS)
    transpose_tile_kernel(char* a, int h, int64_t batch, int64_t bstride) {
  using T = TrTile<E, Q>;
  extern __shared__ __align__(16) uint4 smem[];
  uint4* U0 = smem;
  uint4* U1 = smem + T::S * T::CH;
  const uint64_t nt = 1ull << (h - Q);             // tiles per side
  const uint64_t npairs = nt * (nt + 1) / 2;
  const uint64_t row_stride = (uint64_t)E << h;     // bytes per matrix row
  const uint64_t total = npairs * (uint64_t)batch;
  auto swz = [&](int z, int col) { return z * T::CH + (col ^ ((z >> T::LV) & 7)); };
  for (uint64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const uint64_t bi = w / npairs, p = w - bi * npairs;
    // p -> (I, J), I <= J: J = largest with J (J + 1) / 2 <= p
    uint64_t J = (uint64_t)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
    while (J * (J + 1) / 2 > p) --J;
    while ((J + 1) * (J + 2) / 2 <= p) ++J;
    const uint64_t I = p - J * (J + 1) / 2;
    char* m = a + bi * (uint64_t)bstride;
    char* tA = m + (I << Q) * row_stride + ((J << Q) * E);  // tile (I, J)
    char* tB = m + (J << Q) * row_stride + ((I << Q) * E);  // tile (J, I)
    const bool diag = I == J;
    uint4 r0[T::IPT][T::V], r1[T::IPT][T::V];
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CH, g = id / T::CH;
#pragma unroll
      for (int k = 0; k < T::V; ++k) {
        const uint64_t off = (uint64_t)(g * T::V + k) * row_stride + (uint64_t)c * 16;
        r0[it][k] = ld_plain(tA + off);
        if (!diag) r1[it][k] = ld_plain(tB + off);
      }
    }
#pragma unroll
    for (int it = 0; it < T::IPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int c = id % T::CH, g = id / T::CH;
      // source rows g*V + k, column chunk c -> destination rows c*V + j, chunk g
      U0[swz(c * T::V, g)] = xpose_nat<E, 0>(r0[it]);
      if (!diag) U1[swz(c * T::V, g)] = xpose_nat<E, 0>(r1[it]);
      if constexpr (T::V > 1) {
        U0[swz(c * T::V + 1, g)] = xpose_nat<E, 1>(r0[it]);
        if (!diag) U1[swz(c * T::V + 1, g)] = xpose_nat<E, 1>(r1[it]);
      }
      if constexpr (T::V > 2) {
        U0[swz(c * T::V + 2, g)] = xpose_nat<E, 2>(r0[it]);
        U0[swz(c * T::V + 3, g)] = xpose_nat<E, 3>(r0[it]);
        if (!diag) {
          U1[swz(c * T::V + 2, g)] = xpose_nat<E, 2>(r1[it]);
          U1[swz(c * T::V + 3, g)] = xpose_nat<E, 3>(r1[it]);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < T::WPT; ++it) {
      const int id = it * T::THREADS + threadIdx.x;
      const int col = id % T::CH, z = id / T::CH;
      const uint64_t off = (uint64_t)z * row_stride + (uint64_t)col * 16;
      st_vec(tB + off, U0[swz(z, col)]);         // tile (I, J) transposed -> (J, I)
      if (!diag) st_vec(tA + off, U1[swz(z, col)]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// even-odd split (replaces _even_odd, src/recursive.py:84-93), out of place.

// The scratch contents stockham_permute leaves behind
// (/root/reference/pkg/src/bitrev/permutations.py:30-43, _stockham): level L
// (block size 2^L, L = b .. 1) splits every aligned block through scratch,
// so scratch[k], 2^(L-1) <= k < 2^L, last holds the odd element j = k -
// 2^(L-1) of the last block's split at level L, i.e. the level-L input at
// n - 2^L + 2j + 1, and scratch[0] the level-1 input at n - 2.  Level L
// maps its input from the original array by rotating the low M bits of the
// index left by one for M = L+1 .. b (each even-odd split is that rotation),
// so each slot is one gather from the unpermuted array.
template <int E>
__global__ void stockham_scratch_kernel(const char* a, char* scratch, int b) {
  using W = typename Word<E>::T;
  const uint64_t n = 1ull << b;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    int L;
    uint64_t p;
    if (k == 0) {
      L = 1;
      p = n - 2;
    } else {
      L = 64 - __clzll((long long)k);
      p = n - (1ull << L) + 2 * (k - (1ull << (L - 1))) + 1;
    }
    for (int M = L + 1; M <= b; ++M) {
      const uint64_t mask = (1ull << M) - 1, lo = p & mask;
      p = (p & ~mask) | (((lo << 1) | (lo >> (M - 1))) & mask);
    }
    reinterpret_cast<W*>(scratch)[k] = reinterpret_cast<const W*>(a)[p];
  }
}

template <int E>
__global__ void even_odd_kernel(const char* src, char* dst, int b, int64_t batch,
                                int64_t src_bstride, int64_t dst_bstride) {
  using W = typename Word<E>::T;
  const uint64_t half = 1ull << (b - 1);
  const uint64_t total = half * (uint64_t)batch;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = t / half, j = t % half;
    const W* s = reinterpret_cast<const W*>(src + row * src_bstride);
    W* d = reinterpret_cast<W*>(dst + row * dst_bstride);
    const W e = s[2 * j], o = s[2 * j + 1];
    d[j] = e;
    d[half + j] = o;
  }
}

// ---------------------------------------------------------------------------
// explicit pair list (replaces _apply_pairs, src/schedule.py:100-107); pairs are
// disjoint, so one thread per pair needs no synchronisation.

template <int E>
__global__ void apply_pairs_kernel(char* a, const long long* pairs, int64_t npairs) {
  using W = typename Word<E>::T;
  W* p = reinterpret_cast<W*>(a);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npairs;
       k += (int64_t)gridDim.x * blockDim.x) {
    const long long i = pairs[2 * k], j = pairs[2 * k + 1];
    const W t = p[i];
    p[i] = p[j];
    p[j] = t;
  }
}

// In-order application of an arbitrary pair list by one thread: the exact
// semantics of _apply_pairs (src/schedule.py:100-107) for lists whose pairs
// share indices (the host checks; disjoint lists take apply_pairs_kernel).
template <int E>
__global__ void apply_pairs_ordered_kernel(char* a, const long long* pairs, int64_t npairs) {
  using W = typename Word<E>::T;
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  W* p = reinterpret_cast<W*>(a);
  for (int64_t k = 0; k < npairs; ++k) {
    const long long i = pairs[2 * k], j = pairs[2 * k + 1];
    const W t = p[i];
    p[i] = p[j];
    p[j] = t;
  }
}

// ---------------------------------------------------------------------------
// swap schedule of width b in the reference's emission order
// (generate_swap_schedule / _fill_pairs, src/schedule.py:53-91).  The
// generator is an in-order walk of a binary tree: the node at depth d with
// outer-bit path `base` emits 2^(b-2d-2) pairs (middle value x ascending),
// after its (0,0) subtree and before its (1,1) subtree; a subtree rooted at
// depth d holds swap_count(b - 2d) pairs.  One thread per output slot k
// descends the tree to find its node and x -- O(b) integer work, no list.

__device__ __forceinline__ uint64_t swap_count_dev(int r) {
  return r <= 0 ? 0ull : (((1ull << r) - (1ull << ((r + 1) >> 1))) >> 1);
}

__global__ void swap_schedule_kernel(long long* out, int b, uint64_t count) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t base = 0, start = 0;
    for (int depth = 0;; ++depth) {
      const int rem = b - 2 * depth;
      const uint64_t left = swap_count_dev(rem - 2);
      const uint64_t lo_bit = 1ull << depth, hi_bit = 1ull << (b - 1 - depth);
      if (k < start + left) continue;  // into the (0,0) subtree: same start, same base
      const uint64_t blk = 1ull << (rem - 2);
      if (k < start + left + blk) {
        const uint64_t x = k - start - left;
        const int mid = rem - 2;
        out[2 * k] = (long long)(base | (x << (depth + 1)) | lo_bit);
        out[2 * k + 1] = (long long)(base | (dev_rev(x, mid) << (depth + 1)) | hi_bit);
        break;
      }
      start += left + blk;  // into the (1,1) subtree
      base |= lo_bit | hi_bit;
    }
  }
}

// ---------------------------------------------------------------------------
// sharded plan, step 3: dst[k*G + rev_g(r)] = recv[r*C + k].
// A lane owns K = 16/E consecutive k: one LDG.128 from each of the G source
// chunks (coalesced across the warp: 512 B per chunk per instruction) and a
// register interleave into its G output chunks (K*G*E contiguous bytes).  The
// warp's 32*G output chunks are contiguous, so they go out through a per-warp
// shared-memory bounce (XOR-swizzled, conflict-free both ways) as G fully
// coalesced 512-byte STG.128 rows instead of G strided ones (the strided
// stores ran at 0.43 of the HBM peak for G = 8).  Needs C >= K and 16-byte
// aligned buffers (the host falls back to the element-wise form otherwise).

template <int G>
__device__ __forceinline__ int unpack_swz(int c) { return c ^ ((c >> 3) & 7); }

template <int E, int G>
__global__ void __launch_bounds__(256) sharded_unpack_kernel(const char* recv, char* dst, uint64_t C) {
  constexpr int K = 16 / E;   // k values per lane
  constexpr int EW = E / 4;   // 32-bit words per element
  constexpr int LG = const_log2(G);
  constexpr int WARPS = 8;
  __shared__ uint4 bounce[WARPS][32 * G];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint4* my = bounce[wid];
  const uint64_t nblk = C / K;
  const uint64_t nwarps = (uint64_t)gridDim.x * WARPS;
  for (uint64_t wb = ((uint64_t)blockIdx.x * WARPS + wid) * 32; wb < nblk; wb += nwarps * 32) {
    const uint64_t t = wb + lane;
    const bool full = wb + 32 <= nblk;  // warp-uniform
    if (!full && t >= nblk) continue;
    uint32_t iw[G][4];  // word arrays with compile-time indices only: registers
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const uint4 v = ld_stream(recv + ((uint64_t)r * C + t * K) * E);
      iw[r][0] = v.x;
      iw[r][1] = v.y;
      iw[r][2] = v.z;
      iw[r][3] = v.w;
    }
    uint32_t ow[4 * G];
#pragma unroll
    for (int kk = 0; kk < K; ++kk)
#pragma unroll
      for (int r = 0; r < G; ++r) {
        const int rr = LG ? (int)(__brev((unsigned)r) >> (32 - LG)) : 0;  // folds after unrolling
#pragma unroll
        for (int j = 0; j < EW; ++j) ow[(kk * G + rr) * EW + j] = iw[r][kk * EW + j];
      }
    if (full) {
#pragma unroll
      for (int s = 0; s < G; ++s)
        my[unpack_swz<G>(lane * G + s)] = make_uint4(ow[4 * s], ow[4 * s + 1], ow[4 * s + 2], ow[4 * s + 3]);
      __syncwarp();
      char* d = dst + wb * (uint64_t)(K * G * E);
#pragma unroll
      for (int j = 0; j < G; ++j) st_vec(d + (j * 32 + lane) * 16, my[unpack_swz<G>(j * 32 + lane)]);
      __syncwarp();
    } else {  // ragged last warp: direct (strided) stores
      char* d = dst + t * (uint64_t)(K * G * E);
#pragma unroll
      for (int s = 0; s < G; ++s)
        st_vec(d + s * 16, make_uint4(ow[4 * s], ow[4 * s + 1], ow[4 * s + 2], ow[4 * s + 3]));
    }
  }
}

template <int E>
__global__ void sharded_unpack_generic_kernel(const char* recv, char* dst, uint64_t C, int g) {
  using W = typename Word<E>::T;
  const W* rv = reinterpret_cast<const W*>(recv);
  W* d = reinterpret_cast<W*>(dst);
  const uint64_t G = 1ull << g;
  const uint64_t total = C * G;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = t / C, k = t % C;
    d[k * G + dev_rev(r, g)] = rv[t];
  }
}

}  // namespace bitrev_b200
