// scatter_bench.cu — dev microbenchmark: strategies for W[I[k]] = V[k] with sorted I at low density.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scatter_bench tools/scatter_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef uint16_t u16;

__device__ __forceinline__ u64 mix(u64 z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// mark[i] = 1 with probability rho -> then compact on host via thrust-less scan (done in chunks on device)
__global__ void k_gen_flags(u32* cnt, u64 n, u32 thr, u32* I, u64 cap) {
  // simple: each thread handles 1024 consecutive elements, writes its positions with atomicAdd (unsorted
  // between threads) -> fine for a benchmark as long as we sort per block afterwards; instead we produce
  // sorted output by two passes: this kernel only counts.
}

__global__ void k_count(u64 n, u32 thr, u32* counts) {  // counts per 4096-element block
  u64 b = blockIdx.x;
  u32 c = 0;
  for (u64 i = b * 4096 + threadIdx.x; i < (b + 1) * 4096 && i < n; i += blockDim.x)
    c += (mix(i) >> 32) < thr;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ u32 s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 t = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += s[w];
    counts[b] = t;
  }
}
__global__ void k_fill(u64 n, u32 thr, const u64* off, u32* I) {  // sorted positions
  u64 b = blockIdx.x;
  if (threadIdx.x == 0) {
    u64 o = off[b];
    for (u64 i = b * 4096; i < (b + 1) * 4096 && i < n; ++i)
      if ((mix(i) >> 32) < thr) I[o++] = (u32)i;
  }
}

template <int kU>
__global__ void k_scatter_strided(u16* W, const u32* I, u64 count) {  // current commit structure
  const u64 per = 16384;
  for (u64 c0 = (u64)blockIdx.x * per; c0 < count; c0 += (u64)gridDim.x * per) {
    const u64 end = c0 + per < count ? c0 + per : count;
    for (u64 k0 = c0 + threadIdx.x; k0 < end; k0 += blockDim.x * kU) {
      u32 idx[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) idx[u] = (k0 + u * blockDim.x < end) ? I[k0 + u * blockDim.x] : 0xFFFFFFFFu;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (idx[u] != 0xFFFFFFFFu) W[idx[u]] = (u16)idx[u];
    }
  }
}

template <int kU>
__global__ void k_scatter_prefetch(u16* W, const u32* I, u64 count) {  // + L2 prefetch of next iteration's sectors
  const u64 per = 16384;
  for (u64 c0 = (u64)blockIdx.x * per; c0 < count; c0 += (u64)gridDim.x * per) {
    const u64 end = c0 + per < count ? c0 + per : count;
    for (u64 k0 = c0 + threadIdx.x; k0 < end; k0 += blockDim.x * kU) {
      u32 idx[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) idx[u] = (k0 + u * blockDim.x < end) ? I[k0 + u * blockDim.x] : 0xFFFFFFFFu;
      // prefetch the sectors of the next block of kU
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const u64 kn = k0 + (kU + u) * blockDim.x;
        if (kn < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(W + I[kn]));
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (idx[u] != 0xFFFFFFFFu) W[idx[u]] = (u16)idx[u];
    }
  }
}

template <int kU>
__global__ void k_scatter_contig(u16* W, const u32* I, u64 count) {  // each warp: contiguous run of changes
  const u64 warps = (u64)gridDim.x * (blockDim.x / 32);
  const u64 wid = (u64)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const u32 lane = threadIdx.x & 31;
  const u64 per = (count + warps - 1) / warps;
  const u64 b = wid * per, e = b + per < count ? b + per : count;
  for (u64 k0 = b + lane; k0 < e; k0 += 32 * kU) {
    u32 idx[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) idx[u] = (k0 + u * 32 < e) ? I[k0 + u * 32] : 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (idx[u] != 0xFFFFFFFFu) W[idx[u]] = (u16)idx[u];
  }
}

template <int kU>
__global__ void k_scatter_evict(u16* W, const u32* I, u64 count) {  // stores with L2 evict_first policy
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const u64 per = 16384;
  for (u64 c0 = (u64)blockIdx.x * per; c0 < count; c0 += (u64)gridDim.x * per) {
    const u64 end = c0 + per < count ? c0 + per : count;
    for (u64 k0 = c0 + threadIdx.x; k0 < end; k0 += blockDim.x * kU) {
      u32 idx[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) idx[u] = (k0 + u * blockDim.x < end) ? I[k0 + u * blockDim.x] : 0xFFFFFFFFu;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (idx[u] != 0xFFFFFFFFu)
          asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(W + idx[u]), "h"((u16)idx[u]), "l"(pol));
    }
  }
}

// read-only stream (the roofline of a read-dominated kernel such as K1): 16-byte loads, 4 in flight per thread,
// XOR-reduced so the loads are not dead
__global__ void k_read_stream(const uint4* p, u64 n16, u32* sink) {
  u32 acc = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride),
                d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) {
    const uint4 a = __ldcs(p + i);
    acc ^= a.x ^ a.y ^ a.z ^ a.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// full 32 B sector RMW: the thread of a sector's first change loads the sector (two 16-byte loads), merges
// every change of that sector and stores the whole sector, so the L2 never sees a partial-sector write
template <int kU>
__global__ void k_scatter_sector(u16* W, const u32* I, u64 count) {
  const u64 per = 16384;
  for (u64 c0 = (u64)blockIdx.x * per; c0 < count; c0 += (u64)gridDim.x * per) {
    const u64 end = c0 + per < count ? c0 + per : count;
    for (u64 k0 = c0 + threadIdx.x; k0 < end; k0 += blockDim.x * kU) {
      u32 idx[kU], prv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const u64 k = k0 + u * blockDim.x;
        idx[u] = k < end ? I[k] : 0xFFFFFFFFu;
        prv[u] = (k < end && k > 0) ? I[k - 1] : 0xFFFFFFFFu;
      }
      uint4 a[kU], b[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const bool first = idx[u] != 0xFFFFFFFFu && (prv[u] == 0xFFFFFFFFu || (prv[u] >> 4) != (idx[u] >> 4));
        if (first) {
          const uint4* sp = reinterpret_cast<const uint4*>(W + ((u64)(idx[u] >> 4) << 4));
          a[u] = sp[0];
          b[u] = sp[1];
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const bool first = idx[u] != 0xFFFFFFFFu && (prv[u] == 0xFFFFFFFFu || (prv[u] >> 4) != (idx[u] >> 4));
        if (!first) continue;
        u16 v[16];
        memcpy(v, &a[u], 16);
        memcpy(v + 8, &b[u], 16);
        const u32 sec = idx[u] >> 4;
        for (u64 j = k0 + u * blockDim.x; j < count && (I[j] >> 4) == sec; ++j) v[I[j] & 15] = (u16)I[j];
        uint4* dp = reinterpret_cast<uint4*>(W + ((u64)sec << 4));
        uint4 x, y;
        memcpy(&x, v, 16);
        memcpy(&y, v + 8, 16);
        dp[0] = x;
        dp[1] = y;
      }
    }
  }
}

// full 128 B line RMW per touched line (warp-cooperative: lane = 4-byte word of the line)
__global__ void k_scatter_line(u16* W, const u32* I, u64 count) {
  const u64 warps = (u64)gridDim.x * (blockDim.x / 32);
  const u64 wid = (u64)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const u32 lane = threadIdx.x & 31;
  const u64 per = (count + warps - 1) / warps;
  u64 k = wid * per;
  const u64 e = k + per < count ? k + per : count;
  // skip changes whose line started before this warp's range (owned by the previous warp)
  if (k > 0 && k < e) {
    const u32 line0 = I[k] >> 6;
    while (k < e && (I[k] >> 6) == (I[wid * per - 1] >> 6)) ++k;
    (void)line0;
  }
  while (k < e) {
    const u32 line = I[k] >> 6;
    u32* Lw = reinterpret_cast<u32*>(W + ((u64)line << 6));
    u32 w = Lw[lane];
    u64 j = k;
    while (j < count && (I[j] >> 6) == line) {  // extend past e to finish the line
      const u32 off = I[j] & 63;
      if ((off >> 1) == lane) w = (off & 1) ? ((w & 0xFFFFu) | ((u32)(u16)I[j] << 16)) : ((w & 0xFFFF0000u) | (u16)I[j]);
      ++j;
    }
    Lw[lane] = w;
    k = j;
  }
}

int main(int argc, char** argv) {
  const u64 n = argc > 1 ? strtoull(argv[1], 0, 10) : (8ull << 30);  // elements (16 GB)
  const double rho = argc > 2 ? atof(argv[2]) : 0.01;
  const u32 thr = (u32)(rho * 4294967296.0);
  u16* W;
  cudaMalloc(&W, n * 2);
  cudaMemset(W, 0, n * 2);
  const u64 nb = (n + 4095) / 4096;
  u32* cnt;
  u64* off;
  cudaMalloc(&cnt, nb * 4);
  cudaMalloc(&off, (nb + 1) * 8);
  k_count<<<nb, 256>>>(n, thr, cnt);
  std::vector<u32> hc(nb);
  cudaMemcpy(hc.data(), cnt, nb * 4, cudaMemcpyDeviceToHost);
  std::vector<u64> ho(nb + 1);
  u64 acc = 0;
  for (u64 b = 0; b < nb; ++b) {
    ho[b] = acc;
    acc += hc[b];
  }
  ho[nb] = acc;
  cudaMemcpy(off, ho.data(), (nb + 1) * 8, cudaMemcpyHostToDevice);
  u32* I;
  cudaMalloc(&I, acc * 4);
  k_fill<<<nb, 32>>>(n, thr, off, I);
  cudaDeviceSynchronize();
  const u64 count = acc;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  // touched sectors
  std::vector<u32> hI(count);
  cudaMemcpy(hI.data(), I, count * 4, cudaMemcpyDeviceToHost);
  u64 sect = 0, lines = 0;
  for (u64 k = 0; k < count; ++k) {
    if (k == 0 || (hI[k] >> 4) != (hI[k - 1] >> 4)) ++sect;
    if (k == 0 || (hI[k] >> 6) != (hI[k - 1] >> 6)) ++lines;
  }
  printf("n=%llu rho=%.4f count=%llu sectors=%llu (%.1f%%) lines=%llu (%.1f%%)\n", (unsigned long long)n, rho,
         (unsigned long long)count, (unsigned long long)sect, 100.0 * sect / (n / 16), (unsigned long long)lines,
         100.0 * lines / (n / 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-28s %8.3f ms  sector-model %7.1f GB/s  line-model %7.1f GB/s  err=%s\n", name, ms,
           (sect * 64.0 + count * 4.0) / ms / 1e6, (lines * 256.0 + count * 4.0) / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int g : {nsm * 4, nsm * 8, nsm * 16})
    for (int t : {256}) {
      char nm[64];
      snprintf(nm, 64, "strided8 g=%d", g);
      run(nm, [&] { k_scatter_strided<8><<<g, t>>>(W, I, count); });
    }
  run("strided16 g=8x", [&] { k_scatter_strided<16><<<nsm * 8, 256>>>(W, I, count); });
  run("prefetchL2 g=8x", [&] { k_scatter_prefetch<8><<<nsm * 8, 256>>>(W, I, count); });
  run("contig-warp8 g=8x", [&] { k_scatter_contig<8><<<nsm * 8, 256>>>(W, I, count); });
  run("contig-warp8 g=32x", [&] { k_scatter_contig<8><<<nsm * 32, 256>>>(W, I, count); });
  run("evict_first g=8x", [&] { k_scatter_evict<8><<<nsm * 8, 256>>>(W, I, count); });
  run("sector-rmw8 g=8x", [&] { k_scatter_sector<8><<<nsm * 8, 256>>>(W, I, count); });
  run("sector-rmw4 g=16x", [&] { k_scatter_sector<4><<<nsm * 16, 256>>>(W, I, count); });
  run("line-rmw g=8x", [&] { k_scatter_line<<<nsm * 8, 256>>>(W, I, count); });
  run("line-rmw g=32x", [&] { k_scatter_line<<<nsm * 32, 256>>>(W, I, count); });
  {  // read-only stream over W (2n bytes)
    u32* sink;
    cudaMalloc(&sink, 4);
    for (int g : {nsm * 4, nsm * 8}) {
      k_read_stream<<<g, 512>>>(reinterpret_cast<const uint4*>(W), n * 2 / 16, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_read_stream<<<g, 512>>>(reinterpret_cast<const uint4*>(W), n * 2 / 16, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("%-28s %8.3f ms  %7.1f GB/s (read only, grid %d)\n", "read stream", ms, 2.0 * n / ms / 1e6, g);
    }
  }
  // reference: dense copy of W (read + write)
  u16* W2;
  if (cudaMalloc(&W2, n * 2) == cudaSuccess) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(W2, W, n * 2, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.3f ms  %7.1f GB/s\n", "dense D2D copy", ms, 4.0 * n / ms / 1e6);
  }
  return 0;
}
