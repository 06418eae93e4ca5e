// Host cost of the CUDA runtime calls on the small-message issue path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/api_cost tools/api_cost.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

__global__ void noop() {}

template <typename F>
double us(F f, int n = 20000) {
  for (int i = 0; i < 100; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t et, en;
  cudaEventCreate(&et);
  cudaEventCreateWithFlags(&en, cudaEventDisableTiming);
  cudaStreamCaptureStatus cap;
  int dev;
  printf("{\"launch_noop_us\": %.3f, ", us([&] { noop<<<1, 32, 0, s>>>(); }));
  printf("\"event_record_timing_us\": %.3f, ", us([&] { cudaEventRecord(et, s); }));
  printf("\"event_record_notiming_us\": %.3f, ", us([&] { cudaEventRecord(en, s); }));
  printf("\"stream_is_capturing_us\": %.3f, ", us([&] { cudaStreamIsCapturing(s, &cap); }));
  printf("\"set_device_us\": %.3f, ", us([&] { cudaSetDevice(0); }));
  printf("\"get_device_us\": %.3f, ", us([&] { cudaGetDevice(&dev); }));
  printf("\"get_last_error_us\": %.3f}\n", us([&] { cudaGetLastError(); }));
  return 0;
}
