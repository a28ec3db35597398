// L2 throughput microbenchmark on B200: the ceiling of the dense
// L2-streaming DP kernel (dp_stream_kernel), measured with the same data path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bandwidth tools/l2_bandwidth.cu
//   tools/l2_bandwidth            (prints one JSON line per mode)
//
// Modes (every CTA of a full-occupancy grid, 2 CTAs/SM like the DP kernel):
//   bulk_read   cp.async.bulk global -> shared of 6,160-B windows (the DP
//               kernel's window size) from a buffer that stays in L2, 16 windows in flight per CTA
//               mbarrier ring;
//   store       coalesced 32-bit stores into an L2-resident buffer;
//   mixed       both, in the DP kernel's byte ratio (12.5 B read : 8 B written).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int WIN = 6160;   // bytes per window (1,540 int32)
constexpr int NSLOT = 16;  // windows in flight per CTA (the DP kernel: 4 slots x 4 windows)

__global__ void __launch_bounds__(288, 2) l2_kernel(const uint8_t* src, size_t src_bytes, uint32_t* dst,
                                                    size_t dst_words, int iters, int mode, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint8_t* slots = smem + 128;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t nwin = src_bytes / WIN;
  unsigned long long acc = 0;
  const size_t words_per_cta = dst_words / gridDim.x;
  uint32_t* my = dst + blockIdx.x * words_per_cta;
  for (int it = 0; it < iters; ++it) {
    if (mode != 1 && tid == 0) {  // one window per slot per iteration, 4 in flight
      for (int s = 0; s < NSLOT; ++s) {
        const size_t w = ((size_t)blockIdx.x * 7919 + (size_t)it * NSLOT + s) % nwin;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[s])), "r"(WIN)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(slots + s * WIN)),
            "l"(src + w * WIN), "r"(WIN), "r"(smem_addr(&full[s]))
            : "memory");
      }
    }
    if (mode != 0) {  // stores: 8/12.5 of the read bytes in mixed mode, the same bytes in store mode
      const int words = mode == 1 ? NSLOT * WIN / 4 : (int)(NSLOT * WIN / 4 * 8 / 12.5);
      const size_t base = ((size_t)it * words) % (words_per_cta > (size_t)words ? words_per_cta - words : 1);
      for (int x = tid; x < words; x += blockDim.x) my[base + x] = (uint32_t)(x + it);
    }
    if (mode != 1) {
      for (int s = 0; s < NSLOT; ++s) {
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_addr(&full[s])),
            "r"((uint32_t)(it & 1))
            : "memory");
        acc += slots[s * WIN + (tid * 4) % WIN];
      }
      __syncthreads();
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t src_bytes = (size_t)32 << 20, dst_bytes = (size_t)32 << 20;  // 64 MB in all: L2-resident
  uint8_t* src;
  uint32_t* dst;
  unsigned long long* sink;
  CK(cudaMalloc(&src, src_bytes));
  CK(cudaMalloc(&dst, dst_bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(src, 1, src_bytes));
  CK(cudaMemset(dst, 0, dst_bytes));
  const size_t smem = 128 + NSLOT * WIN;
  CK(cudaFuncSetAttribute(l2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = 2 * sms, iters = 2000;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const char* names[3] = {"bulk_read", "store", "mixed"};
  for (int mode = 0; mode < 3; ++mode) {
    l2_kernel<<<grid, 288, smem>>>(src, src_bytes, dst, dst_bytes / 4, 50, mode, sink);  // warm
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    l2_kernel<<<grid, 288, smem>>>(src, src_bytes, dst, dst_bytes / 4, iters, mode, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double rd = mode == 1 ? 0.0 : (double)grid * iters * NSLOT * WIN;
    const double wr = mode == 0 ? 0.0 : (double)grid * iters * (mode == 1 ? NSLOT * WIN : (int)(NSLOT * WIN / 4 * 8 / 12.5) * 4.0);
    printf("{\"mode\": \"%s\", \"ms\": %.3f, \"read_GBps\": %.1f, \"write_GBps\": %.1f, \"total_GBps\": %.1f, \"ctas\": %d}\n",
           names[mode], ms, rd / ms / 1e6, wr / ms / 1e6, (rd + wr) / ms / 1e6, grid);
  }
  return 0;
}
