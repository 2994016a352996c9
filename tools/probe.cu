// Hardware probe for the GPU box: peer access, L2, stream mem-ops, globaltimer.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
__global__ void gt(unsigned long long* out){unsigned long long a,b;asm volatile("mov.u64 %0, %%globaltimer;":"=l"(a));for(int i=0;i<1000;i++){asm volatile("mov.u64 %0, %%globaltimer;":"=l"(b)); if(b!=a){out[0]=b-a;return;}}out[0]=0;}
__global__ void peer_read(const float4* __restrict__ src, float4* __restrict__ dst, size_t n){
  size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x, s=(size_t)gridDim.x*blockDim.x;
  for(;i<n;i+=s) dst[i]=src[i];
}
int main(){
  int n=0; cudaGetDeviceCount(&n); printf("devices %d\n",n);
  for(int d=0;d<n;d++){cudaDeviceProp p; cudaGetDeviceProperties(&p,d);
    int memops=0; cuInit(0); CUdevice cd; cuDeviceGet(&cd,d);
    cuDeviceGetAttribute(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, cd);
    int wait64=0; cuDeviceGetAttribute(&wait64, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS_V1, cd);
    printf("dev %d %s sm=%d l2=%d smemOptin=%zu memops=%d memops64=%d coop=%d\n",d,p.name,p.multiProcessorCount,p.l2CacheSize,p.sharedMemPerBlockOptin,memops,wait64,p.cooperativeLaunch);
    for(int e=0;e<n;e++) if(e!=d){int c=0; cudaDeviceCanAccessPeer(&c,d,e); printf("  peer %d->%d %d\n",d,e,c);}
  }
  unsigned long long* o; cudaMalloc(&o,8); gt<<<1,1>>>(o); unsigned long long h; cudaMemcpy(&h,o,8,cudaMemcpyDeviceToHost); printf("globaltimer tick %llu ns\n",h);
  if(n>=2){
    size_t bytes=1ull<<30; float4 *a,*b; cudaSetDevice(1); cudaMalloc(&a,bytes); cudaMemset(a,0,bytes);
    cudaSetDevice(0); cudaDeviceEnablePeerAccess(1,0); cudaMalloc(&b,bytes);
    cudaEvent_t s,e; cudaEventCreate(&s); cudaEventCreate(&e);
    for(int it=0;it<3;it++){cudaEventRecord(s); peer_read<<<148*4,512>>>(a,b,bytes/16); cudaEventRecord(e); cudaEventSynchronize(e); float ms; cudaEventElapsedTime(&ms,s,e); printf("peer read 1GiB: %.3f ms = %.1f GB/s\n",ms,bytes/ms/1e6);}
    for(int it=0;it<3;it++){cudaEventRecord(s); peer_read<<<148*4,512>>>(b,a,bytes/16); cudaEventRecord(e); cudaEventSynchronize(e); float ms; cudaEventElapsedTime(&ms,s,e); printf("peer write 1GiB: %.3f ms = %.1f GB/s\n",ms,bytes/ms/1e6);}
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
