// Does a grid tail-launched from a PDL-launched kernel (CDP2,
// cudaStreamTailLaunch) complete before a PDL-launched successor passes
// griddepcontrol.wait?  And what does an empty conditional launch cost
// compared with an unconditional (empty) kernel in the chain?
// nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O3 mb_tail.cu -lcudadevrt
#include <cstdio>
#include <cuda_runtime.h>

__global__ void child(int* flag, int v) {
  // slow enough that a successor not waiting for it would see the old value
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(flag, v);
}

__global__ void parent(int* flag, int v, int launch, unsigned* done) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0;
      if (launch) child<<<1, 32, 0, cudaStreamTailLaunch>>>(flag, v);
    }
  }
}

__global__ void empty_redo(int* flag) { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void succ(int* flag, int expect, int* bad) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && atomicAdd(flag, 0) != expect) atomicAdd(bad, 1);
}

template <typename... K, typename... A>
cudaError_t pdl(void (*k)(K...), int grid, int block, cudaStream_t st, A... a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a...);
}

int main() {
  int *flag, *bad;
  unsigned* done;
  cudaMalloc(&flag, 4);
  cudaMalloc(&bad, 4);
  cudaMalloc(&done, 4);
  cudaMemset(flag, 0, 4);
  cudaMemset(bad, 0, 4);
  cudaMemset(done, 0, 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  const int N = 2000;
  for (int i = 1; i <= N; ++i) {
    pdl(parent, 592, 128, st, flag, i, 1, done);
    pdl(succ, 16, 256, st, flag, i, bad);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  int hbad = -1;
  cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
  printf("tail launch visibility: %s, %d of %d successors saw a stale flag\n",
         cudaGetErrorString(e), hbad, N);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a, st);
      for (int i = 0; i < N; ++i) {
        // mode 0: parent (no tail launch) + succ; 1: parent + empty redo kernel + succ;
        // 2: parent with a tail launch every call + succ
        pdl(parent, 592, 128, st, flag, 0, mode == 2 ? 1 : 0, done);
        if (mode == 1) pdl(empty_redo, 148, 128, st, flag);
        pdl(succ, 16, 256, st, flag, 0, bad);
      }
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (%s): %.2f us per chain\n", mode,
           mode == 0 ? "no redo launch" : mode == 1 ? "empty redo kernel" : "tail launch each",
           1e3 * ms / N);
  }
  return 0;
}
