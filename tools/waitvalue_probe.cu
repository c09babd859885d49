// Probe: does a stream blocked in cuStreamWaitValue32 hold up other streams of
// the same context?  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/wv tools/waitvalue_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <chrono>
#include <cstdlib>
#include <cstdio>

__global__ void bump(unsigned* f) {
  __threadfence_system();
  atomicAdd_system(f, 1u);
}
__global__ void mark(int* m) { *m = 42; }

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static bool wait_done(cudaStream_t s, double secs) {
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return true;
    if (e != cudaErrorNotReady) {
      std::printf("  query error %d (%s)\n", int(e), cudaGetErrorString(e));
      return false;
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > secs)
      return false;
    usleep(1000);
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000,
                                                   cudaEnableDefault, &q);
  std::printf("entry point: err %d query %d ptr %p\n", int(e), int(q), p);
  WaitFn wait = reinterpret_cast<WaitFn>(p);
  if (getenv("PRELOAD")) {
    cudaFuncAttributes fa;
    std::printf("preload %d %d\n", int(cudaFuncGetAttributes(&fa, mark)),
                int(cudaFuncGetAttributes(&fa, bump)));
  }
  int dev = 0, v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMemoryPoolsSupported, dev);
  CUdevice cd;
  unsigned* flag;
  int* marker;
  int* hbuf;
  cudaMalloc(&flag, 256);
  cudaMalloc(&marker, 256);
  cudaMemset(flag, 0, 256);
  cudaMemset(marker, 0, 256);
  cudaMallocHost(&hbuf, 256);
  cudaDeviceSynchronize();
  cudaStream_t A, B, C;
  cudaStreamCreateWithFlags(&A, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&B, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&C, cudaStreamNonBlocking);
  (void)cd;
  CUresult r = wait(reinterpret_cast<CUstream>(A), reinterpret_cast<CUdeviceptr>(flag), 1, 0);
  std::printf("wait enqueue: %d\n", int(r));
  mark<<<1, 1, 0, A>>>(marker);
  std::printf("A done before release (expect 0): %d\n", int(wait_done(A, 0.5)));
  cudaMemcpyAsync(hbuf, marker, 4, cudaMemcpyDeviceToHost, C);
  std::printf("C (D2H copy) progresses while A waits: %d\n", int(wait_done(C, 3.0)));
  mark<<<1, 1, 0, C>>>(marker + 1);
  std::printf("C (kernel) progresses while A waits: %d\n", int(wait_done(C, 3.0)));
  bump<<<1, 1, 0, B>>>(flag);
  std::printf("B (release kernel) completes: %d\n", int(wait_done(B, 3.0)));
  std::printf("A released: %d\n", int(wait_done(A, 3.0)));
  cudaMemcpy(hbuf, marker, 8, cudaMemcpyDeviceToHost);
  std::printf("markers %d %d; last error %s\n", hbuf[0], hbuf[1],
              cudaGetErrorString(cudaGetLastError()));
  return 0;
}
