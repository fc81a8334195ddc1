// Probe: CUDA graph with SWITCH + WHILE conditional nodes driven by kernels that
// spin on pinned-mapped host memory (the imperative->symbolic handshake).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <thread>
#include <atomic>
#include <cstring>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

struct Mailbox { volatile unsigned long long seq[64]; volatile int val[64]; volatile unsigned long long done; volatile long long t[8]; };

__device__ unsigned long long ld_acq(const volatile unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

__global__ void k_wait(Mailbox* mb, int* head, cudaGraphConditionalHandle h) {
  int i = *head;
  while (ld_acq(&mb->seq[i]) != (unsigned long long)(i + 1)) { __nanosleep(100); }
  int v = mb->val[i];
  *head = i + 1;
  cudaGraphSetConditional(h, (unsigned)v);
}
__global__ void k_set(int* out, int idx, int v) { out[idx] = v; }
__global__ void k_inc(int* out, int idx) { out[idx] += 1; }
__global__ void k_done(Mailbox* mb, int* head) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(&mb->done), "l"((unsigned long long)(*head)) : "memory");
}
__global__ void k_fetch(Mailbox* mb, int slot, long long v) {  // device -> host ping
  long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); mb->t[slot] = t;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(&mb->seq[48 + slot]), "l"((unsigned long long)v) : "memory");
}

static cudaGraphNode_t add_kernel(cudaGraph_t g, cudaGraphNode_t* dep, void* fn, void** args) {
  cudaKernelNodeParams p = {}; p.func = fn; p.gridDim = dim3(1); p.blockDim = dim3(1); p.kernelParams = args;
  cudaGraphNode_t n; cudaError_t e = cudaGraphAddKernelNode(&n, g, dep, dep ? 1 : 0, &p);
  if (e != cudaSuccess) printf("add kernel: %s\n", cudaGetErrorString(e));
  return n;
}

int main() {
  CK(cudaSetDeviceFlags(cudaDeviceMapHost | cudaDeviceScheduleSpin));
  Mailbox* mb; CK(cudaHostAlloc(&mb, sizeof(Mailbox), cudaHostAllocMapped)); memset((void*)mb, 0, sizeof(Mailbox));
  Mailbox* dmb; CK(cudaHostGetDevicePointer((void**)&dmb, mb, 0));
  int *head, *out; CK(cudaMalloc(&head, 4)); CK(cudaMalloc(&out, 16));
  CK(cudaMemset(head, 0, 4)); CK(cudaMemset(out, 0, 16));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hs, hw, hs2;
  CK(cudaGraphConditionalHandleCreate(&hs, g, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hw, g, 0, 0));
  void* a1[] = {&dmb, &head, &hs};
  cudaGraphNode_t n = add_kernel(g, nullptr, (void*)k_wait, a1);
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hs; cp.conditional.type = cudaGraphCondTypeSwitch; cp.conditional.size = 2;
  cudaGraphNode_t sw; CK(cudaGraphAddNode(&sw, g, &n, 1, &cp));
  cudaGraph_t* bodies = cp.conditional.phGraph_out;
  int i0 = 0, v10 = 10, v20 = 20, i1 = 1;
  void* b0[] = {&out, &i0, &v10}; void* b1[] = {&out, &i0, &v20};
  add_kernel(bodies[0], nullptr, (void*)k_set, b0);
  add_kernel(bodies[1], nullptr, (void*)k_set, b1);
  void* a2[] = {&dmb, &head, &hw};
  cudaGraphNode_t lw = add_kernel(g, &sw, (void*)k_wait, a2);
  cudaGraphNodeParams wp = {}; wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw; wp.conditional.type = cudaGraphCondTypeWhile; wp.conditional.size = 1;
  cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, g, &lw, 1, &wp));
  cudaGraph_t wbody = wp.conditional.phGraph_out[0];
  void* bi[] = {&out, &i1};
  cudaGraphNode_t inc = add_kernel(wbody, nullptr, (void*)k_inc, bi);
  // nested switch inside the while body
  CK(cudaGraphConditionalHandleCreate(&hs2, wbody, 0, 0));
  void* a3[] = {&dmb, &head, &hs2};
  cudaGraphNode_t nw = add_kernel(wbody, &inc, (void*)k_wait, a3);
  cudaGraphNodeParams cp2 = {}; cp2.type = cudaGraphNodeTypeConditional;
  cp2.conditional.handle = hs2; cp2.conditional.type = cudaGraphCondTypeSwitch; cp2.conditional.size = 2;
  cudaGraphNode_t sw2; CK(cudaGraphAddNode(&sw2, wbody, &nw, 1, &cp2));
  int i2 = 2, i3 = 3;
  void* c0[] = {&out, &i2}; void* c1[] = {&out, &i3};
  add_kernel(cp2.conditional.phGraph_out[0], nullptr, (void*)k_inc, c0);
  add_kernel(cp2.conditional.phGraph_out[1], nullptr, (void*)k_inc, c1);
  add_kernel(wbody, &sw2, (void*)k_wait, a2);   // loop-cond at end of body
  void* ad[] = {&dmb, &head};
  add_kernel(g, &wn, (void*)k_done, ad);
  cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, g, 0));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int rounds = 200;
  double tot_us = 0;
  for (int r = 0; r < rounds; ++r) {
    memset((void*)mb, 0, sizeof(Mailbox));
    CK(cudaMemsetAsync(head, 0, 4, s)); CK(cudaMemsetAsync(out, 0, 16, s));
    CK(cudaStreamSynchronize(s));
    auto t0 = std::chrono::high_resolution_clock::now();
    CK(cudaGraphLaunch(ge, s));
    // decisions: switch=1, loop: cont, case0, cont, case1, cont, case1, exit
    int vals[] = {1, 1, 0, 1, 1, 1, 1, 0};
    for (int i = 0; i < 8; ++i) { mb->val[i] = vals[i]; std::atomic_thread_fence(std::memory_order_release); mb->seq[i] = i + 1; }
    while (mb->done == 0) {}
    auto t1 = std::chrono::high_resolution_clock::now();
    tot_us += std::chrono::duration<double, std::micro>(t1 - t0).count();
    CK(cudaStreamSynchronize(s));
  }
  int h_out[4]; CK(cudaMemcpy(h_out, out, 16, cudaMemcpyDeviceToHost));
  printf("out = %d %d %d %d (expect 20 3 1 2) done=%llu; avg pass %.2f us\n", h_out[0], h_out[1], h_out[2], h_out[3], mb->done, tot_us / rounds);
  // device->host ping latency via a tiny kernel writing mapped memory
  double lat = 0;
  for (int r = 0; r < 200; ++r) {
    mb->seq[48] = 0;
    auto t0 = std::chrono::high_resolution_clock::now();
    k_fetch<<<1, 1, 0, s>>>(dmb, 0, r + 1);
    while (mb->seq[48] != (unsigned long long)(r + 1)) {}
    auto t1 = std::chrono::high_resolution_clock::now();
    lat += std::chrono::duration<double, std::micro>(t1 - t0).count();
    CK(cudaStreamSynchronize(s));
  }
  printf("launch+device->host publish latency avg %.2f us\n", lat / 200);
  return 0;
}
