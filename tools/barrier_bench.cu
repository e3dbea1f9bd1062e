// Microbenchmark: cost of one cooperative grid barrier vs one thread-block
// cluster barrier on this GPU (the TAC rounds are barrier-bound).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

__global__ void grid_loop(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  int x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x ^ i;
    g.sync();
  }
  if (x == 12345) *sink = x;
}

__global__ void cluster_loop(int iters, int* sink) {
  cg::cluster_group c = cg::this_cluster();
  int x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x ^ i;
    c.sync();
  }
  if (x == 12345) *sink = x;
}

__global__ void block_loop(int iters, int* sink) {
  int x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x ^ i;
    __syncthreads();
  }
  if (x == 12345) *sink = x;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  float ms = 0;
  for (int blocks : {1, 16, 64, 103, 148}) {
    for (int threads : {256, 1024}) {
      void* args[] = {(void*)&iters, (void*)&sink};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)grid_loop, blocks, threads, args, 0, nullptr);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      std::printf("grid.sync   blocks=%3d threads=%4d: %.3f us/barrier (%s)\n", blocks, threads,
                  1000.0 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFuncSetAttribute((void*)cluster_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    for (int threads : {256, 1024}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(threads);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_loop, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      std::printf("cluster.sync size=%2d threads=%4d: %.3f us/barrier (%s / %s)\n", cs, threads,
                  1000.0 * ms / iters, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int threads : {256, 1024}) {
    cudaEventRecord(a);
    block_loop<<<1, threads>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    std::printf("__syncthreads threads=%4d: %.3f us/barrier\n", threads, 1000.0 * ms / iters);
  }
  return 0;
}
