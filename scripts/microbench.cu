
#include <cuda_runtime.h>
#include <cstdio>
#include <functional>
#include <vector>

__global__ void k_empty(int *o) { if (threadIdx.x == 9999) o[0] = 1; }

__global__ void k_sync(int *o, int reps) {
  int v = threadIdx.x;
  for (int i = 0; i < reps; ++i) { __syncthreads(); v += i; }
  if (v == -1) o[0] = v;
}

__global__ void k_atom(int *o, int per_thread, int nbins, int reps) {
  __shared__ unsigned bins[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) bins[i] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
  for (int r = 0; r < reps; ++r)
    for (int i = 0; i < per_thread; ++i) {
      x = x * 1664525u + 1013904223u;
      atomicAdd(&bins[(x >> 8) % nbins], 1u);
    }
  __syncthreads();
  if (bins[threadIdx.x] == 0xffffffffu) o[0] = 1;
}

__global__ void k_ballot(int *o, int n, int reps) {
  __shared__ unsigned keys[7168];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) keys[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned cnt = 0;
  for (int r = 0; r < reps; ++r)
    for (int base = warp * 32; base < n; base += blockDim.x) {
      const unsigned k = keys[(base + lane) & 8191];
      cnt += __popc(__ballot_sync(0xffffffffu, (k >> 20) > (unsigned)r));
    }
  if (cnt == 12345) o[0] = cnt;
}

__global__ void k_scan(int *o, int reps) {
  __shared__ unsigned wt[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned v = threadIdx.x, acc = 0;
  for (int r = 0; r < reps; ++r) {
    unsigned x = v + r;
    for (int s = 1; s < 32; s <<= 1) { unsigned y = __shfl_up_sync(0xffffffffu, x, s); if (lane >= s) x += y; }
    __syncthreads();
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    unsigned b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += w < warp ? wt[w] : 0u;
    acc += b + x;
  }
  if (acc == 7) o[0] = acc;
}

__global__ void k_l2load(int *o, const uint2 *src, int n, int reps) {
  unsigned acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += __ldcg(src + (size_t)blockIdx.x * n + i).x;
  if (acc == 7) o[0] = acc;
}


template <int NT>
__device__ __forceinline__ unsigned scan2(unsigned v, unsigned *wt, unsigned *total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { unsigned y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  __syncthreads();
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned t = lane < NW ? wt[lane] : 0u, y = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { unsigned z = __shfl_up_sync(0xffffffffu, y, o); if (lane >= o) y += z; }
    if (lane < NW) wt[lane] = y - t;
    if (lane == NW - 1) wt[NW] = y;
  }
  __syncthreads();
  *total = wt[NW];
  return wt[warp] + x - v;
}

template <int NT>
__global__ void k_scan2(int *o, int reps) {
  __shared__ unsigned wt[NT / 32 + 1];
  unsigned acc = 0, tot;
  for (int r = 0; r < reps; ++r) acc += scan2<NT>(threadIdx.x + r, wt, &tot) + tot;
  if (acc == 7) o[0] = acc;
}

// one radix level: zero 4096 bins, histogram n keys from smem, boundary search
template <int NT>
__global__ void k_level(int *o, int n, int reps) {
  __shared__ unsigned bins[4096];
  __shared__ unsigned keys[7168];
  __shared__ unsigned wt[NT / 32 + 1], st[4];
  for (int i = threadIdx.x; i < 7168; i += NT) keys[i] = i * 2654435761u;
  __syncthreads();
  unsigned acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < 4096; i += NT) bins[i] = 0;
    __syncthreads();
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += NT) atomicAdd(&bins[keys[i] >> 20], 1u);
    __syncthreads();
    const int per = 4096 / NT;
    unsigned s = 0;
    for (int j = 0; j < per; ++j) s += bins[4095 - per * threadIdx.x - j];
    unsigned tot, run = scan2<NT>(s, wt, &tot);
    for (int j = 0; j < per; ++j) {
      unsigned v = bins[4095 - per * threadIdx.x - j];
      if (run < 2048u && run + v >= 2048u) { st[0] = j; st[1] = run; }
      run += v;
    }
    __syncthreads();
    acc += st[0];
    __syncthreads();
  }
  if (acc == 7) o[0] = acc;
}

float timeit(std::function<void()> f, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / iters;
}

std::vector<double> run() {
  int *o; cudaMalloc(&o, (128 * 8192 * 2 + 64) * 8); cudaMemset(o, 0, (128*8192*2+64)*8);
  const uint2 *src = (const uint2 *)o;
  std::vector<double> r;
  const int G = 128, B = 1024, I = 200;
  r.push_back(timeit([&] { k_empty<<<G, B>>>(o); }, I));
  r.push_back(timeit([&] { k_sync<<<G, B>>>(o, 100); }, I));
  r.push_back(timeit([&] { k_atom<<<G, B>>>(o, 8, 16, 1); }, I));
  r.push_back(timeit([&] { k_atom<<<G, B>>>(o, 8, 4096, 1); }, I));
  r.push_back(timeit([&] { k_atom<<<G, B>>>(o, 8, 1, 1); }, I));
  r.push_back(timeit([&] { k_ballot<<<G, B>>>(o, 8192, 1); }, I));
  r.push_back(timeit([&] { k_ballot<<<G, B>>>(o, 8192, 8); }, I));
  r.push_back(timeit([&] { k_scan<<<G, B>>>(o, 10); }, I));
  r.push_back(timeit([&] { k_l2load<<<G, B>>>(o, src, 8192, 1); }, I));
  r.push_back(timeit([&] { k_l2load<<<G, B>>>(o, src, 8192, 4); }, I));
  r.push_back(timeit([&] { k_scan2<1024><<<G, B>>>(o, 10); }, I));
  r.push_back(timeit([&] { k_level<1024><<<G, 1024>>>(o, 7000, 1); }, I));
  r.push_back(timeit([&] { k_level<1024><<<G, 1024>>>(o, 7000, 10); }, I));
  r.push_back(timeit([&] { k_level<256><<<G, 256>>>(o, 7000, 10); }, I));
  r.push_back(timeit([&] { k_level<256><<<G * 4, 256>>>(o, 7000, 10); }, I));
  return r;
}

int main() {
  const char *names[] = {"empty kernel", "100 x __syncthreads", "8 atom/thr, 16 bins", "8 atom/thr, 4096 bins",
                         "8 atom/thr, 1 bin", "ballot pass 8K keys", "8 ballot passes 8K keys", "10 block scans",
                         "L2 load 64KiB/CTA", "4 x L2 load 64KiB/CTA", "10 scan2 (1024 thr)", "1 level 7K keys (1024 thr)", "10 levels 7K keys (1024)", "10 levels 7K keys (256 thr)", "10 levels, 512 CTAs x 256"};
  auto r = run();
  for (size_t i = 0; i < r.size(); ++i) printf("%-28s %8.2f us\n", names[i], r[i]);
  return 0;
}
