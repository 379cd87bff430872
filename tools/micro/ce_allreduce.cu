// W=2 all-reduce data movement on a B200 pair, one process driving both GPUs:
//  sm : SM pull fold (remote loads of the peer's half) then SM push of the
//       result into the peer (the engine's current registered-buffer schedule)
//  ce : copy engines move the bytes, SMs only fold local data: per block,
//       CE copy peer half -> local tmp, fold kernel, CE copy result -> peer,
//       pipelined over B blocks with events (both directions at once)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ce_allreduce ce_allreduce.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                 \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__global__ void fold_local(float4 *mine, const float4 *other, uint64_t nv) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    float4 a = mine[v], b = other[v];
    mine[v] = make_float4((a.x + b.x) * 0.5f, (a.y + b.y) * 0.5f, (a.z + b.z) * 0.5f, (a.w + b.w) * 0.5f);
  }
}
template <int U>
__global__ void fold_pull(float4 *mine, const float4 *peer, uint64_t nv) {
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; v + (U - 1) * nt < nv; v += U * nt) {
    float4 b[U], a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) b[u] = peer[v + u * nt];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = mine[v + u * nt];
#pragma unroll
    for (int u = 0; u < U; ++u)
      mine[v + u * nt] = make_float4((a[u].x + b[u].x) * 0.5f, (a[u].y + b[u].y) * 0.5f, (a[u].z + b[u].z) * 0.5f,
                                     (a[u].w + b[u].w) * 0.5f);
  }
  for (; v < nv; v += nt) {
    float4 a = mine[v], b = peer[v];
    mine[v] = make_float4((a.x + b.x) * 0.5f, (a.y + b.y) * 0.5f, (a.z + b.z) * 0.5f, (a.w + b.w) * 0.5f);
  }
}
template <int U>
__global__ void push(const float4 *src, float4 *dst, uint64_t nv) {
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; v + (U - 1) * nt < nv; v += U * nt) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = src[v + u * nt];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[v + u * nt] = x[u];
  }
  for (; v < nv; v += nt) dst[v] = src[v];
}

int main(int argc, char **argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 28);  // floats per GPU (1 GiB)
  const uint64_t half = n / 2;
  if (n % 8 != 0) {
    printf("n must be a multiple of 8\n");
    return 1;
  }
  float *buf[2], *tmp[2];
  cudaStream_t sa[2], sb[2], sc[2];
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d], n * 4));
    CK(cudaMalloc(&tmp[d], half * 4));
    CK(cudaMemset(buf[d], 0, n * 4));
    CK(cudaStreamCreateWithFlags(&sa[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sc[d], cudaStreamNonBlocking));
  }
  auto sync_all = [&] {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
  };
  // chunk d is owned by GPU d: [d*half, (d+1)*half)
  auto run_sm = [&](int grid_mul) {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      fold_pull<4><<<sms * grid_mul, 512, 0, sb[d]>>>((float4 *)(buf[d] + d * half), (const float4 *)(buf[1 - d] + d * half), half / 4);
    }
    sync_all();  // stands in for barrier 1
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      push<4><<<sms * grid_mul, 512, 0, sb[d]>>>((const float4 *)(buf[d] + d * half), (float4 *)(buf[1 - d] + d * half), half / 4);
    }
  };
  // SM pull fold, then the copy engine pushes the result
  auto run_sm_ce = [&](int grid_mul) {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      fold_pull<4><<<sms * grid_mul, 512, 0, sb[d]>>>((float4 *)(buf[d] + d * half), (const float4 *)(buf[1 - d] + d * half), half / 4);
    }
    sync_all();  // stands in for barrier 1
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemcpyAsync(buf[1 - d] + d * half, buf[d] + d * half, half * 4, cudaMemcpyDeviceToDevice, sb[d]));
    }
  };
  // the same with the engine's backup copy: the whole buffer -> bak during the fold
  float *bak[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&bak[d], n * 4));
  }
  auto run_sm_ce_bak = [&](int grid_mul, bool ce) {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      push<4><<<sms, 512, 0, sa[d]>>>((const float4 *)buf[d], (float4 *)bak[d], n / 4);
      fold_pull<4><<<sms * grid_mul, 512, 0, sb[d]>>>((float4 *)(buf[d] + d * half), (const float4 *)(buf[1 - d] + d * half), half / 4);
    }
    sync_all();  // stands in for barrier 1
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      if (ce)
        CK(cudaMemcpyAsync(buf[1 - d] + d * half, buf[d] + d * half, half * 4, cudaMemcpyDeviceToDevice, sb[d]));
      else
        push<4><<<sms * grid_mul, 512, 0, sb[d]>>>((const float4 *)(buf[d] + d * half), (float4 *)(buf[1 - d] + d * half), half / 4);
    }
  };
  std::vector<cudaEvent_t> ea[2], eb[2];
  auto run_ce = [&](int B) {
    const uint64_t blk = half / B;
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      while ((int)ea[d].size() < B) {
        cudaEvent_t x, y;
        CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&y, cudaEventDisableTiming));
        ea[d].push_back(x);
        eb[d].push_back(y);
      }
    }
    for (int b = 0; b < B; ++b)
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        const uint64_t off = d * half + b * blk;
        CK(cudaMemcpyAsync(tmp[d] + b * blk, buf[1 - d] + off, blk * 4, cudaMemcpyDeviceToDevice, sa[d]));
        CK(cudaEventRecord(ea[d][b], sa[d]));
        CK(cudaStreamWaitEvent(sb[d], ea[d][b], 0));
        fold_local<<<sms * 2, 512, 0, sb[d]>>>((float4 *)(buf[d] + off), (const float4 *)(tmp[d] + b * blk), blk / 4);
        CK(cudaEventRecord(eb[d][b], sb[d]));
        CK(cudaStreamWaitEvent(sc[d], eb[d][b], 0));
        CK(cudaMemcpyAsync(buf[1 - d] + off, buf[d] + off, blk * 4, cudaMemcpyDeviceToDevice, sc[d]));
      }
  };
  cudaEvent_t t0[2], t1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaEventCreate(&t0[d]));
    CK(cudaEventCreate(&t1[d]));
  }
  auto timed = [&](const char *name, auto body) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      sync_all();
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(t0[d], sb[d]));
        CK(cudaStreamWaitEvent(sa[d], t0[d], 0));
        CK(cudaStreamWaitEvent(sc[d], t0[d], 0));
      }
      body();
      float mx = 0;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        cudaEvent_t j1, j2;
        CK(cudaEventCreate(&j1));
        CK(cudaEventCreate(&j2));
        CK(cudaEventRecord(j1, sa[d]));
        CK(cudaEventRecord(j2, sc[d]));
        CK(cudaStreamWaitEvent(sb[d], j1, 0));
        CK(cudaStreamWaitEvent(sb[d], j2, 0));
        CK(cudaEventRecord(t1[d], sb[d]));
      }
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(t1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, t0[d], t1[d]));
        if (ms > mx) mx = ms;
      }
      if (it && mx < best) best = mx;
    }
    printf("%-24s %.3f ms  busbw %.1f GB/s\n", name, best, n * 4.0 / best / 1e6);
  };
  timed("sm pull+push x1", [&] { run_sm(1); });
  timed("sm pull+push x2", [&] { run_sm(2); });
  timed("sm pull + ce push x1", [&] { run_sm_ce(1); });
  timed("sm pull + ce push x2", [&] { run_sm_ce(2); });
  timed("sm pull+bak + ce push", [&] { run_sm_ce_bak(1, true); });
  timed("sm pull+bak + sm push", [&] { run_sm_ce_bak(1, false); });
  for (int B : {1, 2, 4, 8}) {
    // blocks must keep 16-byte (float4) alignment: a misaligned block faults
    // the fold kernel on both GPUs (an earlier B=3 run did exactly that)
    if ((half / B) % 4 != 0 || half % B != 0) continue;
    char nm[64];
    snprintf(nm, sizeof nm, "ce pipeline B=%d", B);
    timed(nm, [&] { run_ce(B); });
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
