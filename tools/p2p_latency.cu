// Cross-GPU synchronisation latency over NVLink peer memory: one thread on
// GPU 0 and one on GPU 1 ping-pong a counter through flags that live in the
// other GPU's memory (remote store + local spin). The round trip bounds what
// any op-range-sharded TAC would pay per exchange (SURVEY §8e option 1),
// against the single-GPU round times in DESIGN.md §3.3. Spins are bounded,
// so a missing peer path reports an error instead of hanging.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_latency tools/p2p_latency.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr long long kSpinMax = 1ll << 22;

__global__ void ping(volatile int* remote, volatile int* local, int iters, int* err) {
  for (int i = 1; i <= iters; ++i) {
    *remote = i;
    __threadfence_system();
    long long s = 0;
    while (*local != i)
      if (++s > kSpinMax) {
        *err = i;
        return;
      }
  }
}

__global__ void pong(volatile int* remote, volatile int* local, int iters, int* err) {
  for (int i = 1; i <= iters; ++i) {
    long long s = 0;
    while (*local != i)
      if (++s > kSpinMax) {
        *err = i;
        return;
      }
    *remote = i;
    __threadfence_system();
  }
}

int main() {
  int n = 0, can01 = 0, can10 = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) {
    std::printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  cudaDeviceCanAccessPeer(&can01, 0, 1);
  cudaDeviceCanAccessPeer(&can10, 1, 0);
  if (!can01 || !can10) {
    std::printf("{\"error\": \"no peer access\"}\n");
    return 0;
  }
  int *f0, *f1, *e0, *e1;
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&f0, 4);
  cudaMalloc(&e0, 4);
  cudaMemset(f0, 0, 4);
  cudaMemset(e0, 0, 4);
  cudaSetDevice(1);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaMalloc(&f1, 4);
  cudaMalloc(&e1, 4);
  cudaMemset(f1, 0, 4);
  cudaMemset(e1, 0, 4);
  cudaDeviceSynchronize();
  cudaSetDevice(0);
  cudaDeviceSynchronize();
  const int iters = 20000;
  cudaEvent_t a, b;
  cudaSetDevice(0);
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaSetDevice(1);
  pong<<<1, 1>>>(f0, f1, iters, e1);  // waits on its own flag f1, answers into f0
  cudaSetDevice(0);
  cudaEventRecord(a);
  ping<<<1, 1>>>(f1, f0, iters, e0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaSetDevice(1);
  cudaDeviceSynchronize();
  int err0 = 0, err1 = 0;
  cudaSetDevice(0);
  cudaMemcpy(&err0, e0, 4, cudaMemcpyDeviceToHost);
  cudaSetDevice(1);
  cudaMemcpy(&err1, e1, 4, cudaMemcpyDeviceToHost);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  std::printf("{\"iters\": %d, \"round_trip_us\": %.3f, \"one_way_us\": %.3f, \"spin_timeouts\": [%d, %d], "
              "\"cuda\": \"%s\"}\n",
              iters, 1000.0 * ms / iters, 500.0 * ms / iters, err0, err1, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
