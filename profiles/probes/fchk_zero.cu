// which numerators make __fdiv_rn take its slow path? time a loop of divisions
#include <cstdio>
__global__ void k(const float* a, float b, float* out, int iters){
  float x = a[threadIdx.x & 1], acc = 0.f, bb = b;
  for (int i=0;i<iters;++i){ acc += __fdiv_rn(x, bb); bb = bb*1.0000001f; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
int main(){
  float *a,*o; cudaMalloc(&a,8); cudaMalloc(&o,1<<22);
  float vals[][2]={{1.5f,1.5f},{0.f,0.f},{-0.f,-0.f},{1e-30f,1e-30f},{0.f,1.5f}};
  const char* names[]={"1.5","+0","-0","1e-30","mixed +0/1.5"};
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int t=0;t<5;++t){ cudaMemcpy(a,vals[t],8,cudaMemcpyHostToDevice);
    k<<<148*8,256>>>(a,1.25f,o,2000); cudaEventRecord(e0); k<<<148*8,256>>>(a,1.25f,o,2000); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); printf("%-14s %.3f ms\n",names[t],ms);}
}
