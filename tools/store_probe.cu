// store_probe.cu -- HBM write throughput of the store paths the fused
// integration kernel can use, as a function of the per-op size (GPU box).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/store_probe tools/store_probe.cu -lcuda
//   tools/_bin/store_probe > gpurun_out/store_probe.txt
//
// Each variant writes the same 4 GiB from shared memory (pre-filled) with
//   bulk    : one cp.async.bulk.global.shared::cta of S bytes per op, issued by
//             lane 0 of every warp (per-warp ops) or by thread 0 of the CTA
//             after a CTA barrier (per-CTA ops of S bytes = the 4 warps'
//             tiles), double-buffered with cp.async.bulk.wait_group.read
//   copy    : warp block copy LDS.128 -> STG.128 (st.global.cs), S bytes per warp tile
//   regs    : STG.128 straight from registers, coalesced (pure write ceiling)
// and prints GB/s.  Question answered: is a bulk TMA store of a 2 KB warp
// tile limited by a per-op cost (r01: 2 KB ops ran at ~2.6 TB/s chip-wide)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
  do                                                                              \
  {                                                                               \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess)                                                        \
    {                                                                             \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// per-warp bulk ops of S bytes, NB staging buffers per warp
template <int S, int NB>
__global__ void __launch_bounds__(128) bulk_warp(char* out, long long ntiles)
{
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* mb = sm + warp * NB * S;
  for (int i = threadIdx.x; i < 4 * NB * S / 4; i += blockDim.x)
    reinterpret_cast<int*>(sm)[i] = i;
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const long long stride = (long long)gridDim.x * 4;
  int it = 0;
  for (long long t = (long long)blockIdx.x * 4 + warp; t < ntiles; t += stride, ++it)
  {
    // (the real kernel writes the buffer here: STS + fence.proxy.async)
    if (lane == 0)
    {
      if (it >= NB)
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * S),
                   "r"(smem_u32(mb + (it % NB) * S)), "r"(S)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// per-CTA bulk ops of S bytes (4 warps' tiles), issued by thread 0 after a barrier
template <int S, int NB>
__global__ void __launch_bounds__(128) bulk_cta(char* out, long long ntiles)
{
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < NB * S / 4; i += blockDim.x)
    reinterpret_cast<int*>(sm)[i] = i;
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it)
  {
    if (threadIdx.x == 0 && it >= NB)
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
    __syncthreads();  // buffer free -> all warps may stage into it
    // (staging would happen here)
    __syncthreads();
    if (threadIdx.x == 0)
    {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * S),
                   "r"(smem_u32(sm + (it % NB) * S)), "r"(S)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// The fused kernel's shape: every tile, each lane issues gathers for the
// NEXT tile (L loads, consumed one tile later), writes its S/32 bytes of the
// tile into staging smem (STS.128), then (FENCE) fence.proxy.async and lane 0
// issues the 1D bulk store -- or (!BULK) the warp copies LDS.128 -> STG.128.
// Question: does the proxy fence wait for the outstanding gathers?
template <int S, bool BULK, bool FENCE, int L>
__global__ void __launch_bounds__(128) pipe_tile(char* out, const double* src, long long nsrc, long long ntiles,
                                                 double* sink)
{
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* mb = sm + warp * 2 * S;
  const long long stride = (long long)gridDim.x * 4;
  double acc = 0.0;
  double nxt[L];
  long long t = (long long)blockIdx.x * 4 + warp;
  auto gather = [&](long long tt)
  {
#pragma unroll
    for (int k = 0; k < L; ++k)
    {
      const unsigned long long h = (unsigned long long)(tt * 32 + lane) * 0x9E3779B97F4A7C15ull + k * 977;
      nxt[k] = __ldg(src + (long long)((tt * 32 + lane) * 3 + (h >> 60)) % nsrc);
    }
  };
  gather(t);
  int it = 0;
  for (; t < ntiles; t += stride, ++it)
  {
    double cur[L];
#pragma unroll
    for (int k = 0; k < L; ++k)
      cur[k] = nxt[k];
    if (t + stride < ntiles)
      gather(t + stride);  // next tile's loads in flight
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < L; ++k)
      v += (float)cur[k];
    acc += v;
    unsigned char* buf = mb + (BULK ? (it & 1) * S : 0);
    if (BULK && it >= 2)
    {
      if (lane == 0)
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < S / 512; ++c)
    {
      const unsigned a = smem_u32(buf + (c * 32 + lane) * 16);
      asm volatile("st.shared.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(a), "f"(v) : "memory");
    }
    if (BULK)
    {
      if (FENCE)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
      {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * S),
                     "r"(smem_u32(buf)), "r"(S)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    else
    {
      __syncwarp();
      float4* o = reinterpret_cast<float4*>(out + t * S);
#pragma unroll
      for (int c = 0; c < S / 512; ++c)
      {
        float4 q;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                     : "r"(smem_u32(buf + (c * 32 + lane) * 16)));
        asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(o + c * 32 + lane), "f"(q.x), "f"(q.y),
                     "f"(q.z), "f"(q.w)
                     : "memory");
      }
      __syncwarp();
    }
  }
  if (BULK && lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 12345.0)
    sink[0] = acc;
}

// warp block copy LDS.128 -> STG.128 (S bytes per warp tile)
template <int S>
__global__ void __launch_bounds__(128) copy_warp(float4* out, long long ntiles)
{
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4* mb = reinterpret_cast<const float4*>(sm + warp * S);
  for (int i = threadIdx.x; i < 4 * S / 4; i += blockDim.x)
    reinterpret_cast<int*>(sm)[i] = i;
  __syncthreads();
  const long long stride = (long long)gridDim.x * 4;
  for (long long t = (long long)blockIdx.x * 4 + warp; t < ntiles; t += stride)
  {
    float4* o = out + t * (S / 16);
#pragma unroll
    for (int k = 0; k < S / 512; ++k)
    {
      float4 v;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "r"(smem_u32(mb + k * 32 + lane)));
      asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(o + k * 32 + lane), "f"(v.x), "f"(v.y),
                   "f"(v.z), "f"(v.w)
                   : "memory");
    }
  }
}

__global__ void __launch_bounds__(128) regs_store(float4* out, long long n16)
{
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float4 v = make_float4(threadIdx.x, 1.f, 2.f, 3.f);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(out + i), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

static const long long kBytes = 4ll << 30;

template <class F>
float time_it(F launch)
{
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r)
  {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

template <int S, int NB>
void run_bulk(char* out, int sms)
{
  for (int per : {2, 4, 8, 16})
  {
    const size_t smem = 4 * NB * S;
    if (smem > 200 * 1024 || per * smem > 220 * 1024)
      continue;
    cudaFuncSetAttribute(bulk_warp<S, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long nt = kBytes / S;
    float ms = time_it([&] { bulk_warp<S, NB><<<sms * per, 128, smem>>>(out, nt); });
    std::printf("bulk_warp S=%6d NB=%d ctas/SM=%2d  %7.1f GB/s  (%.2f G ops/s)\n", S, NB, per,
                kBytes / (ms * 1e-3) * 1e-9, nt / (ms * 1e-3) * 1e-9);
  }
}

template <int S, int NB>
void run_bulk_cta(char* out, int sms)
{
  for (int per : {2, 4, 8})
  {
    const size_t smem = NB * S;
    if (smem > 200 * 1024 || per * smem > 220 * 1024)
      continue;
    cudaFuncSetAttribute(bulk_cta<S, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long nt = kBytes / S;
    float ms = time_it([&] { bulk_cta<S, NB><<<sms * per, 128, smem>>>(out, nt); });
    std::printf("bulk_cta  S=%6d NB=%d ctas/SM=%2d  %7.1f GB/s  (%.2f G ops/s)\n", S, NB, per,
                kBytes / (ms * 1e-3) * 1e-9, nt / (ms * 1e-3) * 1e-9);
  }
}

template <int S>
void run_copy(char* out, int sms)
{
  for (int per : {4, 8})
  {
    const size_t smem = 4 * S;
    cudaFuncSetAttribute(copy_warp<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long nt = kBytes / S;
    float ms = time_it([&] { copy_warp<S><<<sms * per, 128, smem>>>(reinterpret_cast<float4*>(out), nt); });
    std::printf("copy_warp S=%6d ctas/SM=%2d       %7.1f GB/s\n", S, per, kBytes / (ms * 1e-3) * 1e-9);
  }
}

template <bool BULK, bool FENCE>
void run_pipe(char* out, const double* src, long long nsrc, double* sink, int sms, const char* name)
{
  constexpr int S = 2048, L = 12;
  for (int per : {4, 8})
  {
    const size_t smem = 4 * 2 * S;
    cudaFuncSetAttribute(pipe_tile<S, BULK, FENCE, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long nt = kBytes / 4 / S;  // 1 GiB of output
    float ms = time_it([&] { pipe_tile<S, BULK, FENCE, L><<<sms * per, 128, smem>>>(out, src, nsrc, nt, sink); });
    std::printf("pipe %-22s S=%d L=%d ctas/SM=%d  %7.1f GB/s of output\n", name, S, L, per,
                (kBytes / 4) / (ms * 1e-3) * 1e-9);
  }
}

int main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char* out = nullptr;
  CK(cudaMalloc(&out, kBytes));
  {
    const long long nsrc = 8ll << 20;  // 64 MB of doubles (L2-resident gathers)
    double* src = nullptr;
    double* sink = nullptr;
    CK(cudaMalloc(&src, nsrc * 8));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(src, 0, nsrc * 8));
    run_pipe<false, false>(out, src, nsrc, sink, sms, "copy LDS/STG");
    run_pipe<true, true>(out, src, nsrc, sink, sms, "bulk + proxy fence");
    run_pipe<true, false>(out, src, nsrc, sink, sms, "bulk, no fence (racy)");
    cudaFree(src);
  }
  for (int per : {4, 8, 16})
  {
    float ms = time_it([&] { regs_store<<<sms * per, 128>>>(reinterpret_cast<float4*>(out), kBytes / 16); });
    std::printf("regs STG.128 ctas/SM=%2d          %7.1f GB/s\n", per, kBytes / (ms * 1e-3) * 1e-9);
  }
  run_copy<2048>(out, sms);
  run_copy<4096>(out, sms);
  run_bulk<1024, 2>(out, sms);
  run_bulk<2048, 2>(out, sms);
  run_bulk<2048, 4>(out, sms);
  run_bulk<4096, 2>(out, sms);
  run_bulk<8192, 2>(out, sms);
  run_bulk<16384, 2>(out, sms);
  run_bulk_cta<4096, 2>(out, sms);
  run_bulk_cta<8192, 2>(out, sms);
  run_bulk_cta<8192, 4>(out, sms);
  run_bulk_cta<16384, 2>(out, sms);
  run_bulk_cta<32768, 2>(out, sms);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
