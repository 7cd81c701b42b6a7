// synth/gen.cu — GPU twin of synth/__init__.py's counter-based generator.
// Input generation only (no arithmetic of the method): fills old/new bf16 bit
// patterns exactly as the numpy recipe does, plus the bench's
// synthetic "optimizer step" that flips the lowest mantissa bit of the
// positions changed in the previous sync so every timed step syncs a fresh
// update of the same density.
#include <cuda_runtime.h>
#include <stdint.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef uint16_t u16;

__device__ __forceinline__ u64 mix(u64 z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_fill_old(u16* out, u64 n, int norm, u64 key_val, const u16* table) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    out[i] = norm ? (u16)norm : table[mix(key_val ^ i) >> 48];   // norm: the bits of 1.0 (0 = none)
}

// mode 0 = U, 1 = R (row clustered), 2 = E (expert gate already folded into `active`)
__global__ void k_fill_new(const u16* old, u16* nw, u64 n, int mode, int active, u64 key_mask, u64 thr,
                           u64 key_pert, u64 key_row, u64 thr_row, u64 cols) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    bool m = active && (mix(key_mask ^ i) >> 32) < thr;
    if (mode == 1) m = m && ((mix(key_row ^ (i / cols)) >> 32) < thr_row);
    u16 o = old[i];
    nw[i] = m ? (u16)(o ^ (u16)(1 + mix(key_pert ^ i) % 3)) : o;
  }
}

// 8-bit elements (FP8 E4M3, f2): the same recipe on bytes
__global__ void k_fill_old8(uint8_t* out, u64 n, int norm, u64 key_val, const uint8_t* table) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    out[i] = norm ? (uint8_t)norm : table[mix(key_val ^ i) >> 48];
}

__global__ void k_fill_new8(const uint8_t* old, uint8_t* nw, u64 n, int mode, int active, u64 key_mask, u64 thr,
                            u64 key_pert, u64 key_row, u64 thr_row, u64 cols) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    bool m = active && (mix(key_mask ^ i) >> 32) < thr;
    if (mode == 1) m = m && ((mix(key_row ^ (i / cols)) >> 32) < thr_row);
    uint8_t o = old[i];
    nw[i] = m ? (uint8_t)(o ^ (uint8_t)(1 + mix(key_pert ^ i) % 3)) : o;
  }
}

// offsets[t] = exclusive prefix of counts (single CTA of 1024 threads)
__global__ void __launch_bounds__(1024) k_prefix(const u64* counts, u32 T, u64* offsets) {
  __shared__ u64 s_w[32];
  __shared__ u64 s_carry;
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (u32 b = 0; b < T; b += 1024) {
    const u32 t = b + threadIdx.x;
    const u64 c = t < T ? counts[t] : 0;
    u64 v = c;
    for (int o = 1; o < 32; o <<= 1) {
      u64 x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= (u32)o) v += x;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    if (warp == 0) {
      u64 w = s_w[lane], wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        u64 x = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= (u32)o) wi += x;
      }
      s_w[lane] = wi - w;
    }
    __syncthreads();
    const u64 carry = s_carry;
    if (t < T) offsets[t] = carry + s_w[warp] + v - c;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_w[31] + v;  // block inclusive total (last thread)
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[T] = s_carry;
}

// Y[t][I[k]] = V[k] ^ 1 for every extracted (tensor, index, value): V[k] is the
// value Y had at extraction, so this flips its lowest bit without reading Y.
// 4096 entries per CTA, 8 loads in flight per thread.
__global__ void __launch_bounds__(256) k_toggle(u16* const* ys, const u32* I, const u16* V, const u64* offsets,
                                               u32 T) {
  __shared__ u32 s_t;
  const u64 total = offsets[T];
  for (u64 b = (u64)blockIdx.x * 4096; b < total; b += (u64)gridDim.x * 4096) {
    if (threadIdx.x == 0) {
      u32 lo = 0, hi = T;  // largest t with offsets[t] <= b
      while (hi - lo > 1) {
        u32 mid = (lo + hi) / 2;
        if (offsets[mid] <= b) lo = mid; else hi = mid;
      }
      s_t = lo;
    }
    __syncthreads();
    const u64 end = b + 4096 < total ? b + 4096 : total;
    u32 t = s_t;
    // each warp: 512 contiguous entries of the block, 8 in flight per lane
    const u64 wb = b + (threadIdx.x >> 5) * 512, we = wb + 512 < end ? wb + 512 : end;
    for (u64 k0 = wb + (threadIdx.x & 31); k0 < we; k0 += 32 * 8) {
      u32 idx[8];
      u16 val[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const u64 k = k0 + u * 32;
        idx[u] = k < we ? I[k] : 0u;
        val[u] = k < we ? V[k] : (u16)0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const u64 k = k0 + u * 32;
        if (k < we) {
          while (offsets[t + 1] <= k) ++t;
          ys[t][idx[u]] = (u16)(val[u] ^ 1u);
        }
      }
    }
    __syncthreads();
  }
}

// Batched form of k_fill_new for many tensors in one launch (bench streaming mode): one job per tensor with
// the same parameters synth_fill_new takes, a host-built table of tiles (job, first element).
struct FillJob {
  const u16* old;
  u16* nw;
  u64 n, key_mask, thr, key_pert, key_row, thr_row, cols;
  int mode, active;
};

__global__ void k_fill_new_jobs(const FillJob* jobs, const u32* tile_job, const u64* tile_off, u64 n_tiles,
                                u64 tile_elems) {
  for (u64 tl = blockIdx.x; tl < n_tiles; tl += gridDim.x) {
    const FillJob j = jobs[tile_job[tl]];
    const u64 e0 = tile_off[tl];
    const u64 e1 = e0 + tile_elems < j.n ? e0 + tile_elems : j.n;
    // 8 elements per thread and 16-byte accesses where the job's pointers allow (arena views always do)
    const bool vec = ((((uintptr_t)j.old) | ((uintptr_t)j.nw)) & 15u) == 0;
    const u64 v_end = vec ? e0 + ((e1 - e0) & ~7ull) : e0;
    for (u64 i0 = e0 + 8 * threadIdx.x; i0 < v_end; i0 += 8 * blockDim.x) {
      const uint4 o4 = *reinterpret_cast<const uint4*>(j.old + i0);
      u32 w[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const u64 i = i0 + k;
        bool m = j.active && (mix(j.key_mask ^ i) >> 32) < j.thr;
        if (j.mode == 1) m = m && ((mix(j.key_row ^ (i / j.cols)) >> 32) < j.thr_row);
        if (m) w[k >> 1] ^= (u32)(1 + mix(j.key_pert ^ i) % 3) << (16 * (k & 1));
      }
      *reinterpret_cast<uint4*>(j.nw + i0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (u64 i = v_end + threadIdx.x; i < e1; i += blockDim.x) {
      bool m = j.active && (mix(j.key_mask ^ i) >> 32) < j.thr;
      if (j.mode == 1) m = m && ((mix(j.key_row ^ (i / j.cols)) >> 32) < j.thr_row);
      const u16 o = j.old[i];
      j.nw[i] = m ? (u16)(o ^ (u16)(1 + mix(j.key_pert ^ i) % 3)) : o;
    }
  }
}

extern "C" {

int synth_fill_old(void* out, u64 n, int norm, u64 key_val, const void* table, void* stream) {
  if (!n) return 0;
  u64 blocks = (n + 255) / 256;
  int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
  k_fill_old<<<grid, 256, 0, (cudaStream_t)stream>>>((u16*)out, n, norm, key_val, (const u16*)table);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int synth_fill_new(const void* old, void* nw, u64 n, int mode, int active, u64 key_mask, u64 thr, u64 key_pert,
                   u64 key_row, u64 thr_row, u64 cols, void* stream) {
  if (!n) return 0;
  u64 blocks = (n + 255) / 256;
  int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
  k_fill_new<<<grid, 256, 0, (cudaStream_t)stream>>>((const u16*)old, (u16*)nw, n, mode, active, key_mask, thr,
                                                      key_pert, key_row, thr_row, cols ? cols : 1);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int synth_fill_old8(void* out, u64 n, int norm, u64 key_val, const void* table, void* stream) {
  if (!n) return 0;
  u64 blocks = (n + 255) / 256;
  int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
  k_fill_old8<<<grid, 256, 0, (cudaStream_t)stream>>>((uint8_t*)out, n, norm, key_val, (const uint8_t*)table);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int synth_fill_new8(const void* old, void* nw, u64 n, int mode, int active, u64 key_mask, u64 thr, u64 key_pert,
                    u64 key_row, u64 thr_row, u64 cols, void* stream) {
  if (!n) return 0;
  u64 blocks = (n + 255) / 256;
  int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
  k_fill_new8<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint8_t*)old, (uint8_t*)nw, n, mode, active, key_mask,
                                                       thr, key_pert, key_row, thr_row, cols ? cols : 1);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int synth_fill_new_jobs(const void* jobs, const void* tile_job, const void* tile_off, u64 n_tiles, u64 tile_elems,
                        void* stream) {
  if (!n_tiles) return 0;
  const int grid = (int)(n_tiles < 148 * 16 ? n_tiles : 148 * 16);
  k_fill_new_jobs<<<grid, 512, 0, (cudaStream_t)stream>>>((const FillJob*)jobs, (const u32*)tile_job,
                                                          (const u64*)tile_off, n_tiles, tile_elems);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int synth_toggle(void* const* ys, const void* I, const void* V, const void* counts, u32 T, void* offsets_scratch,
                 void* stream) {
  if (!T) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  k_prefix<<<1, 1024, 0, s>>>((const u64*)counts, T, (u64*)offsets_scratch);
  k_toggle<<<148 * 16, 256, 0, s>>>((u16* const*)ys, (const u32*)I, (const u16*)V, (const u64*)offsets_scratch, T);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

}
