// Experiment: cost of the kernel boundaries a protected sweep pays, to choose
// how the checks (K2/K3) are scheduled.  Stand-ins: `work` streams 2 x n floats
// like a small K1; `chk` is a few-CTA latency-bound kernel like K2 that sets a
// graph conditional (always 0 here: error-free).
//   A  work only, plain launches          B  work only, PDL
//   C  work -> chk serial, PDL (today)     D  graph of B
//   E  graph: chk(s) beside work(s+1), IF(chk(s-1)) node before work(s+1)
//   F  streams: chk(s) on a side stream beside work(s+1), an empty fix kernel
//      on the main stream joins it (event) before work(s+2)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/exp_graph.cu -o /tmp/exp_graph
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s @%d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void work(const float4* __restrict__ in, float4* __restrict__ out, int n4) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    float4 v = in[i];
    v.x += 1.f;
    out[i] = v;
  }
}
__global__ void chk(const double* __restrict__ v, double* o, int n, cudaGraphConditionalHandle h, int use_h) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ double red[4];
  double s = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += v[i] * 1.0000001;
  for (int k = 16; k; k >>= 1) s += __shfl_xor_sync(~0u, s, k);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) { o[blockIdx.x] = red[0] + red[1] + red[2] + red[3]; if (use_h && blockIdx.x == 0) cudaGraphSetConditional(h, 0); }
}
__global__ void fixk(float4* out, const int* flag) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*(volatile const int*)flag) out[threadIdx.x].y += 1.f;
}

template <typename K, typename... A>
cudaError_t pdl(K k, dim3 g, dim3 b, cudaStream_t s, bool on, A... a) {
  cudaLaunchConfig_t c = {};
  c.gridDim = g; c.blockDim = b; c.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = on;
  c.attrs = at; c.numAttrs = 1;
  return cudaLaunchKernelEx(&c, k, a...);
}

int main(int argc, char** argv) {
  const int N = 200;
  int sizes_mb[] = {8, 64, 512};
  float4 *b0, *b1; double *cv, *co; int* flag;
  CK(cudaMalloc(&b0, 512u << 20)); CK(cudaMalloc(&b1, 512u << 20));
  CK(cudaMalloc(&cv, 1 << 20)); CK(cudaMalloc(&co, 1 << 16)); CK(cudaMalloc(&flag, 64));
  CK(cudaMemset(b0, 0, 512u << 20)); CK(cudaMemset(cv, 0, 1 << 20)); CK(cudaMemset(flag, 0, 64));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> evc(N + 2), evw(N + 2);
  for (auto& e : evc) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : evw) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const int cn = 8 * 512 * 2;   // check entries (cfg2: 8 layers x (nx+ny))
  for (int mb : sizes_mb) {
    const int n4 = (mb << 20) / 16;
    const dim3 gw(148 * 4), bw(256), gc(32), bc(128);
    auto timeit = [&](auto body) -> float {
      for (int r = 0; r < 2; ++r) body();
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      body();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      return ms * 1000.f / N;
    };
    float tA = timeit([&] { for (int i = 0; i < N; ++i) pdl(work, gw, bw, s, false, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4); });
    float tB = timeit([&] { for (int i = 0; i < N; ++i) pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4); });
    float tC = timeit([&] {
      for (int i = 0; i < N; ++i) {
        pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4);
        pdl(chk, gc, bc, s, true, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0);
      }
    });
    // D: graph of B
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    float tD = timeit([&] { cudaGraphLaunch(ge, s); });
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    // E: graph with conditional IF nodes (built under capture)
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t cg; cudaStreamCaptureStatus cst; unsigned long long cid; const cudaGraphNode_t* deps; size_t nd;
    CK(cudaStreamGetCaptureInfo(s, &cst, &cid, &cg, &deps, &nd));
    std::vector<cudaGraphConditionalHandle> hs(N);
    for (int i = 0; i + 1 < N; ++i) CK(cudaGraphConditionalHandleCreate(&hs[i], cg, 0, cudaGraphCondAssignDefault));  // every handle needs its node
    for (int i = 0; i < N; ++i) {
      // no programmatic edge out of a conditional node
      CK(pdl(work, gw, bw, s, i < 2, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4));
      CK(cudaEventRecord(evw[i], s));
      CK(cudaStreamWaitEvent(s2, evw[i], 0));
      pdl(chk, gc, bc, s2, false, (const double*)cv, co, cn, i + 1 < N ? hs[i] : hs[0], (int)(i + 1 < N));
      CK(cudaEventRecord(evc[i], s2));
      if (i >= 1) {   // IF(chk(i-1)) { fix } joins the side branch before work(i+1)
        CK(cudaStreamWaitEvent(s, evc[i - 1], 0));
        CK(cudaStreamGetCaptureInfo(s, &cst, &cid, &cg, &deps, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hs[i - 1];
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cn_;
        CK(cudaGraphAddNode(&cn_, cg, deps, nd, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaKernelNodeParams kp = {};
        float4* op = i & 1 ? b0 : b1;
        const int* fp = flag;
        void* args[] = {&op, &fp};
        kp.func = (void*)fixk; kp.gridDim = dim3(1); kp.blockDim = dim3(32); kp.kernelParams = args;
        cudaGraphNode_t kn;
        CK(cudaGraphAddKernelNode(&kn, body, nullptr, 0, &kp));
        CK(cudaStreamUpdateCaptureDependencies(s, &cn_, 1, cudaStreamSetCaptureDependencies));
      }
    }
    CK(cudaStreamWaitEvent(s, evc[N - 1], 0));
    CK(cudaStreamEndCapture(s, &g));
    {
      cudaGraphInstantiateParams ip = {};
      cudaError_t ie = cudaGraphInstantiateWithParams(&ge, g, &ip);
      if (ie != cudaSuccess) {
        cudaGraphNodeType t = cudaGraphNodeTypeEmpty;
        if (ip.errNode_out) cudaGraphNodeGetType(ip.errNode_out, &t);
        printf("E instantiate: %s result %d errnode type %d\n", cudaGetErrorString(ie), (int)ip.result_out, (int)t);
        cudaGraphDebugDotPrint(g, "gpurun_out/exp_graph_E.dot", 0);
        return 1;
      }
    }
    float tE = timeit([&] { cudaGraphLaunch(ge, s); });
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    // F: streams, side-stream check + empty fix kernel join
    float tF = timeit([&] {
      for (int i = 0; i < N; ++i) {
        pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4);
        cudaEventRecord(evw[i], s);
        cudaStreamWaitEvent(s2, evw[i], 0);
        pdl(chk, gc, bc, s2, false, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0);
        cudaEventRecord(evc[i], s2);
        if (i >= 1) {
          cudaStreamWaitEvent(s, evc[i - 1], 0);
          pdl(fixk, dim3(1), dim3(32), s, true, i & 1 ? b0 : b1, (const int*)flag);
        }
      }
      cudaStreamWaitEvent(s, evc[N - 1], 0);
    });
    // F2: same as F in a graph
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) {
      pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4);
      cudaEventRecord(evw[i], s);
      cudaStreamWaitEvent(s2, evw[i], 0);
      pdl(chk, gc, bc, s2, false, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0);
      cudaEventRecord(evc[i], s2);
      if (i >= 1) {
        cudaStreamWaitEvent(s, evc[i - 1], 0);
        pdl(fixk, dim3(1), dim3(32), s, true, i & 1 ? b0 : b1, (const int*)flag);
      }
    }
    cudaStreamWaitEvent(s, evc[N - 1], 0);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    float tG = timeit([&] { cudaGraphLaunch(ge, s); });
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    // H: graph of C
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) {
      pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4);
      pdl(chk, gc, bc, s, true, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0);
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    float tH = timeit([&] { cudaGraphLaunch(ge, s); });
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    // I: graph, chk(s) -> chk2(s) on a side branch, work(s+2) joins chk2(s) directly (no fix kernel)
    for (int two = 0; two < 2; ++two) {
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < N; ++i) {
        if (i >= 2) CK(cudaStreamWaitEvent(s, evc[i - 2], 0));
        CK(pdl(work, gw, bw, s, true, (const float4*)(i & 1 ? b1 : b0), i & 1 ? b0 : b1, n4));
        CK(cudaEventRecord(evw[i], s));
        CK(cudaStreamWaitEvent(s2, evw[i], 0));
        CK(pdl(chk, gc, bc, s2, false, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0));
        if (two) CK(pdl(chk, gc, bc, s2, true, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0));
        CK(cudaEventRecord(evc[i], s2));
      }
      CK(cudaStreamWaitEvent(s, evc[N - 1], 0));
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      float tI = timeit([&] { cudaGraphLaunch(ge, s); });
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
      printf("%4d MB I%d graph, side checks joined by work(s+2): %.2f us/step\n", mb, two + 1, tI);
    }
    // chk alone
    float tK = timeit([&] { for (int i = 0; i < N; ++i) pdl(chk, gc, bc, s, true, (const double*)cv, co, cn, (cudaGraphConditionalHandle)0, 0); });
    printf("%4d MB x2: A plain %.2f  B pdl %.2f  C +chk serial %.2f  D graph %.2f  E graph+IF %.2f  F 2-stream+fix %.2f  G graph(F) %.2f  H graph(C) %.2f  chk alone %.2f us/step\n",
           mb, tA, tB, tC, tD, tE, tF, tG, tH, tK);
  }
  CK(cudaGetLastError());
  return 0;
}
