// Effective L2 capacity on this GPU for repeated streaming reads: read the
// first S MB of a buffer 6 times, time the last 5 with events; a read rate
// well above HBM bandwidth means the set stayed in L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_capacity tools/l2_capacity.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ a, long long n, float* out) {
  float s = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = a[i];
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) *out = s;
}

int main() {
  const long long maxb = 512ll << 20;
  float4* a;
  float* out;
  cudaMalloc(&a, maxb);
  cudaMalloc(&out, 4);
  cudaMemset(a, 0, maxb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mb : {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 256}) {
    const long long n = (static_cast<long long>(mb) << 20) / 16;
    rd<<<148 * 8, 256>>>(a, n, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) rd<<<148 * 8, 256>>>(a, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%4d MB: %7.0f GB/s\n", mb, 5.0 * (mb << 20) / (ms * 1e6));
  }
  return 0;
}
