// DRAM efficiency vs contiguous run length on B200 (measurement probe, not
// product code).  Question it answers: how much of the measured copy peak can
// a permutation of R-byte runs reach, out of place and in place (pairwise
// swaps), as a function of R -- the in-place tile-pair kernel moves 512-byte
// runs (E=8, Q=6) on both sides.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o runs runs.cu && ./runs
//
// Kernels (all persistent, 16-byte vectors, U blocks in flight per lane group):
//   copy   : linear copy (the same-size ceiling)
//   oop<R> : dst block rev(k) <- src block k          (bit-reversed block order)
//   mul<R> : dst block (k*A mod nb) <- src block k      (odd multiplier A)
//   swap<R>: in place, blocks k <-> rev(k) for k < rev(k)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldp(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ uint64_t rev(uint64_t v, int w) { return w ? __brevll(v) >> (64 - w) : 0; }

__global__ void __launch_bounds__(256) copy_lin(const uint4* s, uint4* d, uint64_t nv) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    uint4 a = ldg(s + i), b = ldg(s + i + stride), c = ldg(s + i + 2 * stride),
          e = ldg(s + i + 3 * stride);
    stg(d + i, a); stg(d + i + stride, b); stg(d + i + 2 * stride, c); stg(d + i + 3 * stride, e);
  }
  for (; i < nv; i += stride) stg(d + i, ldg(s + i));
}

__device__ __forceinline__ uint4 ldg_pf(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_cs(void* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
// MODE 1: streaming stores; MODE 2: L2 256-byte prefetch on loads; MODE 3: both
template <int MODE>
__global__ void __launch_bounds__(256) copy_var(const uint4* s, uint4* d, uint64_t nv) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  auto ld = [&](const uint4* p) { return (MODE & 2) ? ldg_pf(p) : ldg(p); };
  auto st = [&](uint4* p, const uint4& v) { if (MODE & 1) stg_cs(p, v); else stg(p, v); };
  for (; i + 3 * stride < nv; i += 4 * stride) {
    uint4 a = ld(s + i), b = ld(s + i + stride), c = ld(s + i + 2 * stride), e = ld(s + i + 3 * stride);
    st(d + i, a); st(d + i + stride, b); st(d + i + 2 * stride, c); st(d + i + 3 * stride, e);
  }
  for (; i < nv; i += stride) st(d + i, ld(s + i));
}

// TMA bulk copy: grid-stride over CH-byte chunks, each staged g2s then s2g
// (two smem slots, bulk groups); chunk order globally sequential
template <int CH>
__global__ void __launch_bounds__(32) copy_bulk(const char* s, char* d, uint64_t bytes) {
  __shared__ __align__(128) unsigned char buf[2][CH];
  __shared__ __align__(8) unsigned long long bar[2];
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t nch = bytes / CH;
  int k = 0;
  uint32_t phase[2] = {0, 0};
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
    const int slot = k & 1;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf[slot]);
    const uint32_t bb = b0 + 8 * slot;
    // the slot's previous store must have read shared memory
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sb), "l"(s + c * CH), "r"(CH), "r"(bb) : "memory");
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}"
                 ::"r"(bb), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + c * CH), "r"(sb), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
double time_ms(F f, int reps);

// TMA bulk permutation of R-byte blocks, one elected thread per CTA, NS slots:
// SWAP = false: dst block rev(k) <- src block k  (unit = one block)
// SWAP = true : in place, blocks k <-> rev(k), k <= rev(k)  (unit = the pair)
template <int R, int NS, bool SWAP>
__global__ void __launch_bounds__(32) bulk_perm(const char* s, char* d, int lb) {
  constexpr int UB = SWAP ? 2 * R : R;  // bytes per unit
  __shared__ __align__(128) unsigned char buf[NS][UB];
  __shared__ __align__(8) unsigned long long bar[NS];
  if (threadIdx.x != 0) return;
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8 * i));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const uint64_t nb = 1ull << lb;
  // unit list of this CTA: k = blockIdx.x + j * gridDim.x (skipping k > rev k when SWAP)
  auto unit_k = [&](uint64_t j, uint64_t& k) {
    k = blockIdx.x + j * gridDim.x;
    return k < nb;
  };
  uint32_t phase[NS] = {};
  auto issue_load = [&](uint64_t j) {
    uint64_t k;
    if (!unit_k(j, k)) return;
    const int slot = (int)(j % NS);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf[slot]);
    const uint32_t bb = b0 + 8 * slot;
    const uint64_t r = rev(k, lb);
    const bool act = !SWAP || k <= r;
    const uint32_t bytes = act ? (SWAP ? (k == r ? R : 2 * R) : R) : 0;
    if (!bytes) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bb) : "memory"); return; }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sb), "l"(s + k * R), "r"(R), "r"(bb) : "memory");
    if (SWAP && k != r)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sb + R), "l"(s + r * R), "r"(R), "r"(bb) : "memory");
  };
  for (int j = 0; j < NS - 1; ++j) issue_load(j);
  for (uint64_t j = 0;; ++j) {
    uint64_t k;
    if (!unit_k(j, k)) break;
    // slot of unit j+NS-1 was last used by unit j-1: its stores must have read smem
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    issue_load(j + NS - 1);
    const int slot = (int)(j % NS);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf[slot]);
    const uint32_t bb = b0 + 8 * slot;
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}"
                 ::"r"(bb), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    const uint64_t r = rev(k, lb);
    if (!SWAP) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + r * R), "r"(sb), "r"(R) : "memory");
    } else if (k <= r) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + r * R), "r"(sb), "r"(R) : "memory");
      if (k != r)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + k * R), "r"(sb + R), "r"(R) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int R, int NS>
void run_bulk(char* s, char* d, uint64_t bytes, int sms, int cps) {
  int lb = 0;
  while ((uint64_t(R) << (lb + 1)) <= bytes) ++lb;
  const uint64_t used = uint64_t(R) << lb;
  const int grid = sms * cps;
  double t0 = time_ms([&] { bulk_perm<R, NS, false><<<grid, 32>>>(s, d, lb); }, 15);
  double t1 = time_ms([&] { bulk_perm<R, NS, true><<<grid, 32>>>(d, d, lb); }, 15);
  printf("{\"bytes\": %llu, \"R\": %d, \"NS\": %d, \"cps\": %d, \"bulk_oop_rev_gbs\": %.1f, "
         "\"bulk_swap_rev_gbs\": %.1f}\n",
         (unsigned long long)used, R, NS, cps, 2.0 * used / t0 / 1e6, 2.0 * used / t1 / 1e6);
}

struct u8v { unsigned v[8]; };
__device__ __forceinline__ u8v ldg256(const void* p) {
  u8v r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                 "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  return r;
}
__device__ __forceinline__ u8v ldp256(const void* p) {
  u8v r;
  asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                 "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg256(void* p, const u8v& a) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.v[0]), "r"(a.v[1]),
               "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]) : "memory");
}
// grid-stride copy with 32-byte vectors (LDG.256 / STG.256)
__global__ void __launch_bounds__(256) copy_lin256(const char* s, char* d, uint64_t n32) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n32; i += 4 * stride) {
    u8v a = ldg256(s + 32 * i), b = ldg256(s + 32 * (i + stride)), c = ldg256(s + 32 * (i + 2 * stride)),
        e = ldg256(s + 32 * (i + 3 * stride));
    stg256(d + 32 * i, a); stg256(d + 32 * (i + stride), b); stg256(d + 32 * (i + 2 * stride), c);
    stg256(d + 32 * (i + 3 * stride), e);
  }
  for (; i < n32; i += stride) stg256(d + 32 * i, ldg256(s + 32 * i));
}
// in-place swap of R-byte blocks k <-> rev(k) with 32-byte vectors
template <int R, int U>
__global__ void __launch_bounds__(256) blk_swap256(char* a, int lb) {
  constexpr int G = R / 32 < 32 ? R / 32 : 32;
  constexpr int VPL = R / 32 / G;
  constexpr int BPW = 32 / G;
  const uint64_t nb = 1ull << lb;
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k0 = warp * BPW * U; k0 < nb; k0 += nwarps * BPW * U) {
    u8v v[U][VPL], w[U][VPL];
    bool act[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * BPW + sub, r = __brevll(k) >> (64 - lb);
      act[u] = k <= r;
      if (act[u]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          v[u][j] = ldp256(a + k * R + (j * G + gl) * 32);
          w[u][j] = ldp256(a + r * R + (j * G + gl) * 32);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * BPW + sub, r = __brevll(k) >> (64 - lb);
      if (act[u]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          stg256(a + r * R + (j * G + gl) * 32, v[u][j]);
          stg256(a + k * R + (j * G + gl) * 32, w[u][j]);
        }
      }
    }
  }
}

// each CTA copies one contiguous chunk of nv / gridDim vectors
__global__ void __launch_bounds__(256) copy_chunk(const uint4* s, uint4* d, uint64_t nv) {
  const uint64_t per = nv / gridDim.x;
  const uint64_t lo = blockIdx.x * per, hi = lo + per;
  uint64_t i = lo + threadIdx.x;
  for (; i + 3 * 256 < hi; i += 4 * 256) {
    uint4 a = ldg(s + i), b = ldg(s + i + 256), c = ldg(s + i + 512), e = ldg(s + i + 768);
    stg(d + i, a); stg(d + i + 256, b); stg(d + i + 512, c); stg(d + i + 768, e);
  }
  for (; i < hi; i += 256) stg(d + i, ldg(s + i));
}

// MODE 0: dst rev(k) <- src k; MODE 1: dst (k*A mod nb) <- src k
template <int R, int U, int MODE>
__global__ void __launch_bounds__(256) blk_oop(const char* s, char* d, int lb) {
  constexpr int G = R / 16 < 32 ? R / 16 : 32;   // lanes per block
  constexpr int VPL = R / 16 / G;                 // vectors per lane per block
  constexpr int BPW = 32 / G;                     // blocks per warp per step
  const uint64_t nb = 1ull << lb;
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k0 = warp * BPW * U; k0 < nb; k0 += nwarps * BPW * U) {
    uint4 v[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * BPW + sub;
#pragma unroll
      for (int j = 0; j < VPL; ++j) v[u][j] = ldg(s + k * R + (j * G + gl) * 16);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * BPW + sub;
      const uint64_t t = MODE == 0 ? rev(k, lb) : ((k * 0x9E3779B1ull) & (nb - 1));
#pragma unroll
      for (int j = 0; j < VPL; ++j) stg(d + t * R + (j * G + gl) * 16, v[u][j]);
    }
  }
}

template <int R, int U>
__global__ void __launch_bounds__(256) blk_swap(char* a, int lb) {
  constexpr int G = R / 16 < 32 ? R / 16 : 32;
  constexpr int VPL = R / 16 / G;
  constexpr int BPW = 32 / G;
  const uint64_t nb = 1ull << lb;
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // items: every k visited, k > rev(k) lanes idle (half the items), so the
  // work per warp is balanced on average
  for (uint64_t k0 = warp * BPW * U; k0 < nb; k0 += nwarps * BPW * U) {
    uint4 v[U][VPL], w[U][VPL];
    bool act[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * BPW + sub, r = rev(k, lb);
      act[u] = k <= r;
      if (act[u]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          v[u][j] = ldp(a + k * R + (j * G + gl) * 16);
          w[u][j] = ldp(a + r * R + (j * G + gl) * 16);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * BPW + sub, r = rev(k, lb);
      if (act[u]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          stg(a + r * R + (j * G + gl) * 16, v[u][j]);
          stg(a + k * R + (j * G + gl) * 16, w[u][j]);
        }
      }
    }
  }
}

template <typename F>
double time_ms(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  f();
  cudaDeviceSynchronize();
  std::vector<float> ts;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

template <int R, int U>
void run_r(char* s, char* d, uint64_t bytes, int sms, int cps) {
  int lb = 0;
  while ((uint64_t(R) << (lb + 1)) <= bytes) ++lb;
  const uint64_t used = uint64_t(R) << lb;
  const int grid = sms * cps;
  double t0 = time_ms([&] { blk_oop<R, U, 0><<<grid, 256>>>(s, d, lb); }, 15);
  double t1 = time_ms([&] { blk_oop<R, U, 1><<<grid, 256>>>(s, d, lb); }, 15);
  double t2 = time_ms([&] { blk_swap<R, U><<<grid, 256>>>(d, lb); }, 15);
  printf("{\"bytes\": %llu, \"R\": %d, \"U\": %d, \"oop_rev_gbs\": %.1f, \"oop_mul_gbs\": %.1f, "
         "\"swap_rev_gbs\": %.1f}\n",
         (unsigned long long)used, R, U, 2.0 * used / t0 / 1e6, 2.0 * used / t1 / 1e6,
         2.0 * used / t2 / 1e6);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint64_t bytes : {512ull << 20, 4096ull << 20}) {
    char *s, *d;
    cudaMalloc(&s, bytes);
    cudaMalloc(&d, bytes);
    cudaMemset(s, 1, bytes);
    cudaMemset(d, 2, bytes);
    const uint64_t nv = bytes / 16;
    for (int cps : {4, 8}) {
      double t = time_ms([&] { copy_lin<<<sms * cps, 256>>>((const uint4*)s, (uint4*)d, nv); }, 15);
      printf("{\"bytes\": %llu, \"copy_ctas_per_sm\": %d, \"copy_gbs\": %.1f}\n",
             (unsigned long long)bytes, cps, 2.0 * bytes / t / 1e6);
    }
    {
      double t = time_ms([&] { cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); }, 15);
      printf("{\"bytes\": %llu, \"memcpy_d2d_gbs\": %.1f}\n", (unsigned long long)bytes,
             2.0 * bytes / t / 1e6);
    }
    {
      double t1 = time_ms([&] { copy_var<1><<<sms * 4, 256>>>((const uint4*)s, (uint4*)d, nv); }, 15);
      double t2 = time_ms([&] { copy_var<2><<<sms * 4, 256>>>((const uint4*)s, (uint4*)d, nv); }, 15);
      double t3 = time_ms([&] { copy_var<3><<<sms * 4, 256>>>((const uint4*)s, (uint4*)d, nv); }, 15);
      double t4 = time_ms([&] { copy_bulk<16384><<<sms * 8, 32>>>(s, d, bytes); }, 15);
      double t5 = time_ms([&] { copy_bulk<8192><<<sms * 16, 32>>>(s, d, bytes); }, 15);
      double t6 = time_ms([&] { copy_bulk<4096><<<sms * 24, 32>>>(s, d, bytes); }, 15);
      printf("{\"bytes\": %llu, \"copy_cs_gbs\": %.1f, \"copy_l2pf_gbs\": %.1f, \"copy_cs_l2pf_gbs\": %.1f, "
             "\"bulk16k_gbs\": %.1f, \"bulk8k_gbs\": %.1f, \"bulk4k_gbs\": %.1f}\n",
             (unsigned long long)bytes, 2.0 * bytes / t1 / 1e6, 2.0 * bytes / t2 / 1e6,
             2.0 * bytes / t3 / 1e6, 2.0 * bytes / t4 / 1e6, 2.0 * bytes / t5 / 1e6,
             2.0 * bytes / t6 / 1e6);
    }
    for (int cps : {2, 8}) {
      double t = time_ms([&] { copy_chunk<<<sms * cps, 256>>>((const uint4*)s, (uint4*)d, nv); }, 15);
      printf("{\"bytes\": %llu, \"chunk_ctas_per_sm\": %d, \"chunk_copy_gbs\": %.1f}\n",
             (unsigned long long)bytes, cps, 2.0 * bytes / t / 1e6);
    }
    {
      double t0 = time_ms([&] { copy_lin256<<<sms * 4, 256>>>(s, d, bytes / 32); }, 15);
      int lb512 = 0, lb1k = 0;
      while ((512ull << (lb512 + 1)) <= bytes) ++lb512;
      while ((1024ull << (lb1k + 1)) <= bytes) ++lb1k;
      double t1 = time_ms([&] { blk_swap256<512, 2><<<sms * 8, 256>>>(d, lb512); }, 15);
      double t2 = time_ms([&] { blk_swap<512, 4><<<sms * 8, 256>>>(d, lb512); }, 15);
      double t3 = time_ms([&] { blk_swap256<1024, 2><<<sms * 8, 256>>>(d, lb1k); }, 15);
      printf("{\"bytes\": %llu, \"copy256_gbs\": %.1f, \"swap256_512_gbs\": %.1f, "
             "\"swap128_512_gbs\": %.1f, \"swap256_1024_gbs\": %.1f}\n",
             (unsigned long long)bytes, 2.0 * bytes / t0 / 1e6, 2.0 * bytes / t1 / 1e6,
             2.0 * bytes / t2 / 1e6, 2.0 * bytes / t3 / 1e6);
    }
    run_bulk<512, 4>(s, d, bytes, sms, 16);
    run_bulk<512, 8>(s, d, bytes, sms, 16);
    run_bulk<1024, 4>(s, d, bytes, sms, 16);
    run_bulk<2048, 4>(s, d, bytes, sms, 8);
    run_bulk<4096, 4>(s, d, bytes, sms, 4);
    run_r<256, 4>(s, d, bytes, sms, 8);
    run_r<512, 4>(s, d, bytes, sms, 8);
    run_r<1024, 2>(s, d, bytes, sms, 8);
    run_r<2048, 2>(s, d, bytes, sms, 8);
    run_r<4096, 1>(s, d, bytes, sms, 8);
    run_r<8192, 1>(s, d, bytes, sms, 4);
    cudaFree(s);
    cudaFree(d);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
