#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void k(float* p){ p[threadIdx.x] += 1.f; }
#define P(x) do{cudaError_t e=(x); printf("%-70s %s\n", #x, cudaGetErrorString(e));}while(0)
int main(){
  float* d; cudaMalloc(&d, 1024); cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int variant=0; variant<2; ++variant){
    printf("variant %d (destroy placeholder=%d)\n", variant, variant==0);
    cudaEvent_t ph[2]; cudaEventCreate(&ph[0]); cudaEventCreate(&ph[1]);
    cudaGraph_t g; cudaGraphExec_t ex;
    P(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    P(cudaEventRecordWithFlags(ph[0], s, cudaEventRecordExternal));
    k<<<1,32,0,s>>>(d);
    P(cudaEventRecordWithFlags(ph[1], s, cudaEventRecordExternal));
    P(cudaStreamEndCapture(s, &g));
    size_t nn=0; cudaGraphGetNodes(g, nullptr, &nn); std::vector<cudaGraphNode_t> nodes(nn); cudaGraphGetNodes(g, nodes.data(), &nn);
    cudaGraphNode_t en[2]={0,0};
    for (auto n: nodes){ cudaGraphNodeType t; cudaGraphNodeGetType(n,&t); printf(" node type %d\n", (int)t);
      if (t==cudaGraphNodeTypeEventRecord){ cudaEvent_t e; cudaGraphEventRecordNodeGetEvent(n,&e); for(int j=0;j<2;++j) if(e==ph[j]) en[j]=n; } }
    printf(" found %p %p\n", (void*)en[0], (void*)en[1]);
    P(cudaGraphInstantiate(&ex, g, 0));
    if (variant==0){ cudaEventDestroy(ph[0]); cudaEventDestroy(ph[1]); }
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    P(cudaGraphExecEventRecordNodeSetEvent(ex, en[0], a));
    P(cudaGraphExecEventRecordNodeSetEvent(ex, en[1], b));
    P(cudaGraphLaunch(ex, s));
    P(cudaGraphExecEventRecordNodeSetEvent(ex, en[0], a));
    P(cudaStreamSynchronize(s));
    float ms=0; P(cudaEventElapsedTime(&ms,a,b)); printf(" ms %f\n", ms);
  }
}
