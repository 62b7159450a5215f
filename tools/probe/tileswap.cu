// In-place DRAM access pattern probe (measurement only, not product code).
//
// Reproduces the global access pattern of the in-place tile-pair kernel WITHOUT
// its shared-memory transposition: a work item is a pair of "tiles" {y, rev y};
// each tile is ROWS rows of R contiguous bytes at stride STRIDE; both tiles are
// read, then tile y's rows are written over tile rev(y)'s rows and vice versa.
// Total footprint = ROWS * STRIDE bytes, the same as the real array.  Comparing
// its GB/s with the real kernel on the same box separates the DRAM pattern
// cost (run length R, visit order) from the kernel's own overheads.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tileswap tileswap.cu
//   ./tileswap            (JSON lines)
//
// Orders of the pair list: 0 = ascending y, 1 = shuffled, 2 = "level" order
// (the compact pair enumeration of the product kernel).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

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

// CTA of NT threads per pair; each thread moves VPT vectors of each tile.
template <int R, int ROWS, int NT>
__global__ void __launch_bounds__(NT) tile_swap(char* a, char* out, const uint32_t* ys, int npairs,
                                               int m, uint64_t stride) {
  constexpr int CPR = R / 16;                 // 16-byte chunks per row
  constexpr int VPT = ROWS * CPR / NT;        // chunks per thread per tile
  static_assert(VPT >= 1 && ROWS * CPR % NT == 0, "split");
  for (int p = blockIdx.x; p < npairs; p += gridDim.x) {
    const uint64_t y = ys[p];
    const uint64_t ry = m ? (__brevll(y) >> (64 - m)) : 0;
    uint4 v0[VPT], v1[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int id = j * NT + threadIdx.x;
      const int row = id / CPR, c = id % CPR;
      v0[j] = ldp(a + row * stride + y * R + c * 16);
      if (ry != y) v1[j] = ldp(a + row * stride + ry * R + c * 16);
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int id = j * NT + threadIdx.x;
      const int row = id / CPR, c = id % CPR;
      if (ry != y) {
        stg(out + row * stride + ry * R + c * 16, v0[j]);
        stg(out + row * stride + y * R + c * 16, v1[j]);
      } else {
        stg(out + row * stride + y * R + c * 16, v0[j]);
      }
    }
  }
}

struct u8v { unsigned v[8]; };
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
// the same pattern with 32-byte accesses
template <int R, int ROWS, int NT>
__global__ void __launch_bounds__(NT) tile_swap256(char* a, const uint32_t* ys, int npairs, int m,
                                                  uint64_t stride) {
  constexpr int CPR = R / 32;
  constexpr int VPT = ROWS * CPR / NT;
  static_assert(VPT >= 1 && ROWS * CPR % NT == 0, "split");
  for (int p = blockIdx.x; p < npairs; p += gridDim.x) {
    const uint64_t y = ys[p];
    const uint64_t ry = m ? (__brevll(y) >> (64 - m)) : 0;
    u8v v0[VPT], v1[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int id = j * NT + threadIdx.x;
      const int row = id / CPR, c = id % CPR;
      v0[j] = ldp256(a + row * stride + y * R + c * 32);
      if (ry != y) v1[j] = ldp256(a + row * stride + ry * R + c * 32);
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int id = j * NT + threadIdx.x;
      const int row = id / CPR, c = id % CPR;
      if (ry != y) {
        stg256(a + row * stride + ry * R + c * 32, v0[j]);
        stg256(a + row * stride + y * R + c * 32, v1[j]);
      } else {
        stg256(a + row * stride + y * R + c * 32, v0[j]);
      }
    }
  }
}

static uint32_t revb(uint32_t v, int m) {
  uint32_t r = 0;
  for (int i = 0; i < m; ++i) r |= ((v >> i) & 1u) << (m - 1 - i);
  return r;
}

template <int R, int NT, bool W256 = false, int ROWS = 64>
void run(char* a, uint32_t* d_ys, uint64_t total, int sms, int ctas_per_sm, char* out = nullptr) {
  if (!out) out = a;  // in place unless a separate destination is given
  const uint64_t stride = total / ROWS;
  int m = 0;
  while (((uint64_t)R << (m + 1)) <= stride) ++m;
  const uint64_t n = 1ull << m;
  std::vector<uint32_t> asc;
  for (uint32_t y = 0; y < n; ++y)
    if (y <= revb(y, m)) asc.push_back(y);
  std::vector<uint32_t> shuf = asc;
  std::mt19937 g(1);
  std::shuffle(shuf.begin(), shuf.end(), g);
  // level order: by the position of the first mirrored-bit mismatch
  std::vector<uint32_t> lvl = asc;
  std::stable_sort(lvl.begin(), lvl.end(), [&](uint32_t x, uint32_t y) {
    auto level = [&](uint32_t v) {
      for (int k = 0; k < m / 2; ++k)
        if (((v >> k) & 1) != ((v >> (m - 1 - k)) & 1)) return k;
      return m;
    };
    return level(x) < level(y);
  });
  const std::vector<uint32_t>* orders[3] = {&asc, &shuf, &lvl};
  int occ = 0;
  if constexpr (W256) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile_swap256<R, ROWS, NT>, NT, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile_swap<R, ROWS, NT>, NT, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int o = 2; o < 3; ++o) {
    cudaMemcpy(d_ys, orders[o]->data(), orders[o]->size() * 4, cudaMemcpyHostToDevice);
    const int np = (int)orders[o]->size();
    const int grid = sms * ctas_per_sm;
    auto launch = [&]() {
      if constexpr (W256) tile_swap256<R, ROWS, NT><<<grid, NT>>>(a, d_ys, np, m, stride);
      else tile_swap<R, ROWS, NT><<<grid, NT>>>(a, out, d_ys, np, m, stride);
    };
    for (int w = 0; w < 3; ++w) launch();
    std::vector<float> ts;
    for (int r = 0; r < 15; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const uint64_t moved = 2 * (uint64_t)ROWS * R * n;
    printf("{\"oop\": %d, \"bytes\": %llu, \"rows\": %d, \"R\": %d, \"m\": %d, \"order\": %d, \"nt\": %d, \"ctas_per_sm\": %d, "
           "\"w256\": %d, \"occ\": %d, \"gbs\": %.1f, \"best_gbs\": %.1f}\n",
           (int)(out != a), (unsigned long long)total, ROWS, R, m, o, NT, ctas_per_sm, (int)W256, occ,
           moved / ts[ts.size() / 2] / 1e6, moved / ts[0] / 1e6);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint64_t total : {512ull << 20, 4096ull << 20}) {
    char* a;
    uint32_t* ys;
    cudaMalloc(&a, total);
    cudaMalloc(&ys, (total / 64 / 256) * 4 + 1024);
    cudaMemset(a, 3, total);
    char* b2;
    cudaMalloc(&b2, total);
    cudaMemset(b2, 5, total);
    for (int rep = 0; rep < 2; ++rep) {
      run<512, 256>(a, ys, total, sms, 4);
      run<512, 256>(a, ys, total, sms, 4, b2);
      run<512, 256>(a, ys, total, sms, 2);
      run<512, 256>(a, ys, total, sms, 2, b2);
    }
    cudaFree(b2);
    cudaFree(a);
    cudaFree(ys);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
