#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
template <int N> struct Args { char b[N]; };
template <int N> __global__ void k(const __grid_constant__ Args<N> a) { if (a.b[0] == 123 && threadIdx.x == 9999) printf("x"); }
template <int N> double bench(cudaStream_t s) {
  Args<N> a{};
  for (int i = 0; i < 100; ++i) k<N><<<296, 288, 0, s>>>(a);
  cudaStreamSynchronize(s);
  double best = 1e9;
  for (int r = 0; r < 5; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 200; ++i) k<N><<<296, 288, 0, s>>>(a);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / 200);
  }
  return best;
}
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  printf("64 B params: %.2f us/launch\n", bench<64>(s));
  printf("1 KB params: %.2f us/launch\n", bench<1024>(s));
  printf("4 KB params: %.2f us/launch\n", bench<4000>(s));
  printf("6 KB params: %.2f us/launch\n", bench<6144>(s));
  printf("16 KB params: %.2f us/launch\n", bench<16384>(s));
  return 0;
}
