// Microbenchmark of the synchronisation primitives the step schedule uses,
// on the real device: graph-launched empty kernels, grid barriers (variants),
// and a dependent global-load chain.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_sync.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned g_count, g_gen;

__global__ void k_empty() {}

template <int kVariant>
__global__ void k_barriers(int iters) {
  unsigned target = 0;
  for (int i = 0; i < iters; ++i) {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned v;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(&g_count) : "memory");
      if (kVariant == 0) {  // poll the counter
        v += 1;
        while ((int)(v - target) < 0)
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
      } else if (kVariant == 3) {  // relaxed polls, one acquire
        v += 1;
        while ((int)(v - target) < 0)
          asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
      } else {  // generation word
        if (v + 1 == target) {
          asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_gen), "r"(target) : "memory");
        } else {
          do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_gen) : "memory");
          } while ((int)(v - target) < 0);
        }
      }
      if (kVariant == 2) __threadfence();
    }
    __syncthreads();
  }
}

// hardware cluster barrier: 16 CTAs of 1024 threads (or 8), iters barriers
__global__ void k_cluster_barriers(int iters, int* out) {
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    acc += i;
  }
  if (acc == -1) *out = acc;
}

// hierarchical grid barrier: a hardware cluster barrier, then ONE global
// arrival per cluster (its rank-0 CTA), then a second cluster barrier that
// releases the cluster; every CTA then makes one acquire load of the counter
// (gpu-scope visibility of the other clusters' writes in its own L1)
__global__ void k_hier_barriers(int iters, int csize) {
  unsigned target = 0;
  const unsigned nclusters = gridDim.x / csize;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = 0; i < iters; ++i) {
    target += nclusters;
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
      unsigned v;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(&g_count) : "memory");
      v += 1;
      while ((int)(v - target) < 0)
        asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (rank != 0 && threadIdx.x == 0) {
      unsigned v;
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
    }
    __syncthreads();
  }
}

__global__ void k_chain(const int* __restrict__ next, int steps, int* out) {
  int p = threadIdx.x + blockIdx.x * blockDim.x;
  for (int i = 0; i < steps; ++i) p = next[p];
  if (p == -1) *out = p;
}

__global__ void k_reset() { g_count = 0; g_gen = 0; }

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  // 1. graph of 20 empty kernels
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 20; ++i) k_empty<<<196, 256, 0, s>>>();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
  cudaEventRecord(a, s);
  for (int r = 0; r < 100; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("graph empty kernel (196x256): %.2f us per kernel\n", ms * 1000 / 2000);
  // 2. barriers
  const int iters = 1000;
  for (int grid : {148, 196, 296}) {
    for (int var = 0; var < 4; ++var) {
      k_reset<<<1, 1, 0, s>>>();
      cudaEventRecord(a, s);
      if (var == 0) k_barriers<0><<<grid, 256, 0, s>>>(iters);
      if (var == 1) k_barriers<1><<<grid, 256, 0, s>>>(iters);
      if (var == 2) k_barriers<2><<<grid, 256, 0, s>>>(iters);
      if (var == 3) k_barriers<3><<<grid, 256, 0, s>>>(iters);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d barrier variant %d: %.2f us per barrier (%s)\n", grid, var, ms * 1000 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  // 2a. hierarchical barriers (cluster + one global arrival per cluster)
  for (int cs : {2, 4, 8}) {
    for (int grid : {148, 296}) {
      if (grid % cs) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeCooperative;
      attr[1].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      k_reset<<<1, 1, 0, s>>>();
      cudaLaunchKernelEx(&cfg, k_hier_barriers, 10, cs);
      k_reset<<<1, 1, 0, s>>>();
      cudaEventRecord(a, s);
      cudaLaunchKernelEx(&cfg, k_hier_barriers, iters, cs);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d hierarchical barrier, clusters of %d (cooperative): %.2f us per barrier (%s)\n", grid, cs,
             ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // 2b. cluster barriers
  for (int cs : {8, 16}) {
    for (int bs : {256, 1024}) {
      cudaFuncSetAttribute(k_cluster_barriers, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(bs);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int* o = nullptr;
      cudaMalloc(&o, 4);
      cudaLaunchKernelEx(&cfg, k_cluster_barriers, 10, o);
      cudaEventRecord(a, s);
      cudaLaunchKernelEx(&cfg, k_cluster_barriers, iters, o);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("cluster %d x %d threads: %.3f us per cluster barrier (%s)\n", cs, bs, ms * 1000 / iters,
             cudaGetErrorString(cudaGetLastError()));
      cudaFree(o);
    }
  }
  // 3. dependent load chain: random permutation over 64 MB (L2-resident) and 1 GB
  for (long long n : {1ll << 24, 1ll << 28}) {
    int* h = new int[n];
    for (long long i = 0; i < n; ++i) h[i] = (int)((i * 2654435761ull + 12345) % n);
    int *d, *o;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, 4);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    k_chain<<<1, 1, 0, s>>>(d, 1000, o);
    cudaEventRecord(a, s);
    k_chain<<<1, 1, 0, s>>>(d, 10000, o);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent load chain over %lld MB: %.0f ns per load\n", n * 4 >> 20, ms * 1e6 / 10000);
    cudaFree(d);
    cudaFree(o);
    delete[] h;
  }
  return 0;
}
