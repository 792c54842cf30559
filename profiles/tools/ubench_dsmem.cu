// Cost of distributed-shared-memory traffic on the B200 (sm_100a): a cluster of CL CTAs (256 threads), each
// thread stores K double2 values into a peer CTA's shared memory through map_shared_rank (generic st), then
// the block syncs; clock64 around the stores, and around a local shared-memory pass issued right after them
// (does it queue behind the remote stores?). Also the bulk form: one cp.async.bulk shared::cluster per peer
// of the same bytes, completion on the receiver's mbarrier. Decides how the mirrored rows kernel
// (tt_rows2.cu) exchanges its partials.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_dsmem(long long* out, int K, int CL) {
  extern __shared__ __align__(16) unsigned char sm[];
  double2* buf = (double2*)sm;      // 256 * 16 double2 receive area
  double2* loc = buf + 256 * 16;    // local scratch
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const int c = cl.block_rank(), tid = threadIdx.x;
  for (int i = tid; i < 256 * 16; i += 256) { buf[i] = make_double2(i, c); loc[i] = make_double2(1, 2); }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  long long t0 = clock64(), t1 = 0, t2 = 0;
  const int peer = (c + 1) % CL;
  if (MODE == 0) {  // generic remote stores, K per thread
    double2* dst = cl.map_shared_rank(buf, peer);
    for (int k = 0; k < K; ++k) dst[k * 256 + tid] = make_double2(k, tid);
    __syncthreads();
    t1 = clock64();
    for (int k = 0; k < 16; ++k) loc[k * 256 + tid].x += 1.0;  // local pass right after
    __syncthreads();
    t2 = clock64();
  } else if (MODE == 1) {  // the same stores to the own CTA through the generic window
    double2* dst = cl.map_shared_rank(buf, c);
    for (int k = 0; k < K; ++k) dst[k * 256 + tid] = make_double2(k, tid);
    __syncthreads();
    t1 = clock64();
    for (int k = 0; k < 16; ++k) loc[k * 256 + tid].x += 1.0;
    __syncthreads();
    t2 = clock64();
  } else {  // bulk copy of the same bytes (K * 256 * 16) into the peer, completion on the peer's mbarrier
    const unsigned bytes = (unsigned)K * 256u * 16u;
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    }
    cl.sync();  // every receiver armed
    t0 = clock64();
    if (tid == 0) {
      unsigned dst = smem_u32(buf), mb = smem_u32(&bar), rdst, rmb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(dst), "r"(peer));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rmb) : "r"(mb), "r"(peer));
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
                   "r"(smem_u32(loc)), "r"(bytes), "r"(rmb)
                   : "memory");
    }
    t1 = clock64();
    // wait for the incoming copy (from the other neighbour)
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar)),
        "r"(0)
        : "memory");
    __syncthreads();
    t2 = clock64();
  }
  cl.sync();
  if (tid == 0) {
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t1;
  }
}

template <int MODE>
void run(const char* name, int CL, int K) {
  long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  const size_t smem = 2 * 256 * 16 * 16;
  cudaFuncSetAttribute(k_dsmem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_dsmem<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * (CL == 16 ? 1 : 4));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_dsmem<MODE>, d, K, CL);
  cudaDeviceSynchronize();
  long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("%-34s CL %2d K %2d (%6d B/CTA): %s  stores %6lld cycles, then local pass %6lld cycles\n", name, CL, K,
         K * 256 * 16, cudaGetErrorString(e), h[0], h[1]);
  cudaFree(d);
}

int main() {
  for (int CL : {2, 16})
    for (int K : {1, 4, 16}) {
      run<0>("remote generic st.v2.f64", CL, K);
      run<1>("own CTA through the generic window", CL, K);
      run<2>("cp.async.bulk smem->peer smem", CL, K);
    }
  return 0;
}
