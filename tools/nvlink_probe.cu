// NVLink transport probe (development tool, not part of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe tools/nvlink_probe.cu
//   ./nvlink_probe [MiB per peer]
//
// One process, all visible GPUs, peer access enabled.  Every GPU moves the same number of
// bytes to (push) or from (pull) every other GPU at once -- the update kernel's all-to-all
// pattern -- with five transports:
//   st     SM 16-byte stores into the peers' buffers (the update kernel's weight pushes)
//   ld     SM 16-byte loads from the peers' buffers (summed, so they are not dead)
//   tma_ld cp.async.bulk global->shared from the peers (the update kernel's grad pulls)
//   tma_st cp.async.bulk shared->global into the peers
//   ce     cudaMemcpyPeerAsync, one stream per peer (copy engines)
// Reported: per-GPU GB/s per direction (bytes sent or received by one GPU / time), max time
// over GPUs.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

constexpr int kMaxG = 8;
struct Bufs {
  uint4 *peer[kMaxG];  // per peer: its receive/source region reserved for this GPU
  int G, me;
  size_t n;  // uint4 per peer
};

// every thread interleaves the peers (j-th vector of peer 0, 1, ...) like the update kernel
__global__ void k_st(Bufs b, uint4 *local_src) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = gridDim.x * (size_t)blockDim.x;
  for (size_t j = tid; j < b.n; j += nth) {
    const uint4 v = local_src[j];
    for (int p = 0; p < b.G; ++p)
      if (p != b.me) b.peer[p][j] = v;
  }
}

__global__ void k_ld(Bufs b, unsigned *sink) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = gridDim.x * (size_t)blockDim.x;
  unsigned acc = 0;
  for (size_t j = tid; j < b.n; j += nth) {
    uint4 v[kMaxG];
#pragma unroll
    for (int p = 0; p < kMaxG; ++p)
      if (p < b.G && p != b.me) v[p] = __ldcg(b.peer[p] + j);
#pragma unroll
    for (int p = 0; p < kMaxG; ++p)
      if (p < b.G && p != b.me) acc ^= v[p].x ^ v[p].y ^ v[p].z ^ v[p].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one elected thread per CTA streams kPiece-byte pieces through a kSlots-deep smem ring
template <int kPiece, int kSlots>
__global__ void k_tma_ld(Bufs b) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[kSlots];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kSlots; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t pieces_per_peer = b.n * 16 / kPiece, total = pieces_per_peer * (b.G - 1);
  uint32_t k = 0;
  for (size_t i = blockIdx.x; i < total; i += gridDim.x, ++k) {
    const int s = k % kSlots;
    if (k >= kSlots) {  // wait for the copy issued kSlots ago into this slot
      const uint32_t par = ((k / kSlots) - 1) & 1;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                       smem_u32(&bar[s])),
                   "r"(par)
                   : "memory");
    }
    const int pi = (int)(i % (b.G - 1));  // peers interleaved piece by piece (no incast)
    const int p = pi + (pi >= b.me);
    const char *src = (const char *)b.peer[p] + (i / (b.G - 1)) * kPiece;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kPiece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + s * kPiece)),
                 "l"(src), "r"(kPiece), "r"(smem_u32(&bar[s]))
                 : "memory");
  }
  for (uint32_t j = (k > kSlots ? k - kSlots : 0); j < k; ++j) {
    const int s = j % kSlots;
    const uint32_t par = (j / kSlots) & 1;
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     smem_u32(&bar[s])),
                 "r"(par)
                 : "memory");
  }
}

constexpr int kPiece = 16384;
__global__ void k_tma_st(Bufs b) {
  extern __shared__ __align__(128) unsigned char sm[];
  if (threadIdx.x != 0) return;
  const size_t pieces_per_peer = b.n * 16 / kPiece, total = pieces_per_peer * (b.G - 1);
  for (size_t i = blockIdx.x; i < total; i += gridDim.x) {
    const int pi = (int)(i % (b.G - 1));
    const int p = pi + (pi >= b.me);
    char *dst = (char *)b.peer[p] + (i / (b.G - 1)) * kPiece;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(sm)), "r"(kPiece)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (G < 2) {
    printf("need >= 2 GPUs\n");
    return 0;
  }
  if (G > kMaxG) G = kMaxG;
  const size_t mib = argc > 1 ? atol(argv[1]) : 256;
  const size_t bytes = mib << 20, n = bytes / 16;
  std::vector<char *> region(G);  // GPU g: (G) x bytes, slot q reserved for sender/reader q
  std::vector<uint4 *> src(G);
  std::vector<unsigned *> sink(G);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h)
      if (h != g) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, g, h));
        if (ok) cudaDeviceEnablePeerAccess(h, 0), cudaGetLastError();
      }
    CK(cudaMalloc(&region[g], bytes * G));
    CK(cudaMemset(region[g], g + 1, bytes * G));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 7, bytes));
    CK(cudaMalloc(&sink[g], 64));
    CK(cudaFuncSetAttribute(k_tma_ld<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_tma_ld<4096, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152));
    CK(cudaFuncSetAttribute(k_tma_ld<2048, 24>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152));
    CK(cudaFuncSetAttribute(k_tma_st, cudaFuncAttributeMaxDynamicSharedMemorySize, kPiece));
  }
  auto bufs_for = [&](int g) {
    Bufs b{};
    b.G = G;
    b.me = g;
    b.n = n;
    for (int h = 0; h < G; ++h) b.peer[h] = (uint4 *)(region[h] + (size_t)g * bytes);  // my slot on h
    return b;
  };
  const char *names[] = {"st", "ld", "tma_ld16Kx4", "tma_st", "ce", "tma_ld4Kx12", "tma_ld2Kx24"};
  for (int mode = 0; mode < 7; ++mode) {
    for (int grid_mult : {2, 4, 8}) {
      if (mode == 4 && grid_mult != 2) continue;
      std::vector<cudaEvent_t> e0(G), e1(G);
      std::vector<std::vector<cudaStream_t>> st(G, std::vector<cudaStream_t>(G));
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
        for (int h = 0; h < G; ++h) CK(cudaStreamCreateWithFlags(&st[g][h], cudaStreamNonBlocking));
      }
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
        float worst = 0.f;
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventRecord(e0[g], st[g][0]));
          const Bufs b = bufs_for(g);
          const int grid = sms * grid_mult;
          if (mode == 0) k_st<<<grid, 256, 0, st[g][0]>>>(b, src[g]);
          if (mode == 1) k_ld<<<grid, 256, 0, st[g][0]>>>(b, sink[g]);
          if (mode == 2) k_tma_ld<16384, 4><<<grid, 32, 65536, st[g][0]>>>(b);
          if (mode == 5) k_tma_ld<4096, 12><<<grid, 32, 49152, st[g][0]>>>(b);
          if (mode == 6) k_tma_ld<2048, 24><<<grid, 32, 49152, st[g][0]>>>(b);
          if (mode == 3) k_tma_st<<<grid, 32, kPiece, st[g][0]>>>(b);
          if (mode == 4) {
            for (int h = 0; h < G; ++h)
              if (h != g) {
                CK(cudaStreamWaitEvent(st[g][h], e0[g], 0));
                CK(cudaMemcpyPeerAsync(region[h] + (size_t)g * bytes, h, src[g], g, bytes, st[g][h]));
                cudaEvent_t x;
                CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
                CK(cudaEventRecord(x, st[g][h]));
                CK(cudaStreamWaitEvent(st[g][0], x, 0));
              }
          }
          CK(cudaGetLastError());
          CK(cudaEventRecord(e1[g], st[g][0]));
        }
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(e1[g]));
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
          if (ms > worst) worst = ms;
        }
        if (rep > 0 && worst < best) best = worst;
      }
      const double gbs = (double)bytes * (G - 1) / (best * 1e-3) / 1e9;
      printf("G=%d %-7s grid=%dxSM  %8.1f GB/s per GPU per direction  (%.3f ms for %zu MiB to each of %d peers)\n", G,
             names[mode], grid_mult, gbs, best, mib, G - 1);
    }
  }
  return 0;
}
