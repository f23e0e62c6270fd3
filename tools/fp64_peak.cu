// FP64 pipe microbenchmark: DFMA vs DMMA (mma.sync f64) throughput on one B200.
// Used to pick the Γ kernel's math path and to state the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

template<int CH>
__global__ void dfma_k(double* out, int iters, double s){
  double a[CH];
  #pragma unroll
  for(int i=0;i<CH;i++) a[i]=threadIdx.x*1e-3+i;
  double m=1.0000001, c=s;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CH;i++) a[i]=fma(a[i],m,c);
  }
  double r=0;
  #pragma unroll
  for(int i=0;i<CH;i++) r+=a[i];
  if(r==12345.678) out[0]=r;
}

template<int NACC>
__global__ void dmma884_k(double* out, int iters){
  double c[NACC][2];
  #pragma unroll
  for(int i=0;i<NACC;i++){c[i][0]=0;c[i][1]=0;}
  double a=1.0+threadIdx.x*1e-6, b=1.0-threadIdx.x*1e-6;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<NACC;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
  }
  double r=0;
  #pragma unroll
  for(int i=0;i<NACC;i++) r+=c[i][0]+c[i][1];
  if(r==12345.678) out[0]=r;
}

template<int NACC>
__global__ void dmma16816_k(double* out, int iters){
  double c[NACC][4];
  #pragma unroll
  for(int i=0;i<NACC;i++){c[i][0]=c[i][1]=c[i][2]=c[i][3]=0;}
  double a0=1.0+threadIdx.x*1e-6, b0=1.0-threadIdx.x*1e-6;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<NACC;i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(c[i][0]),"+d"(c[i][1]),"+d"(c[i][2]),"+d"(c[i][3])
        : "d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(b0),"d"(b0),"d"(b0),"d"(b0));
  }
  double r=0;
  #pragma unroll
  for(int i=0;i<NACC;i++) r+=c[i][0]+c[i][1]+c[i][2]+c[i][3];
  if(r==12345.678) out[0]=r;
}


// Mixed: every warp interleaves 8 DMMA (acc8) with R x 8 independent DFMA chains, to see
// whether the DMMA and DFMA paths share one FP64 datapath (time = sum) or not (time = max).
template<int R>
__global__ void mixed_k(double* out, int iters, double s){
  double c[8][2];
  #pragma unroll
  for(int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;}
  double f[8];
  #pragma unroll
  for(int i=0;i<8;i++) f[i]=threadIdx.x*1e-3+i;
  double a=1.0+threadIdx.x*1e-6, b=1.0-threadIdx.x*1e-6, m=1.0000001;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<8;i++){
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
      #pragma unroll
      for(int r=0;r<R;r++) f[(i+r)&7]=fma(f[(i+r)&7],m,s);
    }
  }
  double r=0;
  #pragma unroll
  for(int i=0;i<8;i++) r+=c[i][0]+c[i][1]+f[i];
  if(r==12345.678) out[0]=r;
}
// Split: even warps DMMA only, odd warps DFMA only (same per-warp flop count).
__global__ void split_k(double* out, int iters, double s){
  if(((threadIdx.x>>5)&1)==0){
    double c[8][2];
    #pragma unroll
    for(int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;}
    double a=1.0+threadIdx.x*1e-6, b=1.0-threadIdx.x*1e-6;
    for(int it=0; it<iters; ++it){
      #pragma unroll
      for(int i=0;i<8;i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
          : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
    }
    double r=0;
    #pragma unroll
    for(int i=0;i<8;i++) r+=c[i][0]+c[i][1];
    if(r==12345.678) out[0]=r;
  } else {
    double f[8];
    #pragma unroll
    for(int i=0;i<8;i++) f[i]=threadIdx.x*1e-3+i;
    double m=1.0000001;
    for(int it=0; it<iters*8; ++it){
      #pragma unroll
      for(int i=0;i<8;i++) f[i]=fma(f[i],m,s);
    }
    double r=0;
    #pragma unroll
    for(int i=0;i<8;i++) r+=f[i];
    if(r==12345.678) out[0]=r;
  }
}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, clk);
  double* out; CK(cudaMalloc(&out,8));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms=p.multiProcessorCount;
  auto run=[&](const char* name, auto launch, double flop){
    launch(); CK(cudaDeviceSynchronize());
    float best=1e30;
    for(int r=0;r<5;r++){cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("%-40s %8.3f ms  %8.2f TFLOP/s\n", name, best, flop/best/1e9);
    return 0;
  };
  int it=4096;
  for(int tpb : {128,256,512}) for(int bps : {1,2,4}){
    char nm[96]; snprintf(nm,96,"DFMA ch8 tpb%d bps%d",tpb,bps);
    int blocks=sms*bps;
    run(nm, [&]{dfma_k<8><<<blocks,tpb>>>(out,it,1e-9);}, 2.0*8*it*(double)blocks*tpb);
  }
  for(int tpb : {128,256,512}) for(int bps : {1,2,4}){
    char nm[96]; snprintf(nm,96,"DMMA 8x8x4 acc8 tpb%d bps%d",tpb,bps);
    int blocks=sms*bps;
    run(nm, [&]{dmma884_k<8><<<blocks,tpb>>>(out,it);}, 2.0*256*8*it*(double)blocks*(tpb/32));
  }
  for(int tpb : {128,256}) for(int bps : {1,2}){
    char nm[96]; snprintf(nm,96,"DMMA 16x8x16 acc4 tpb%d bps%d",tpb,bps);
    int blocks=sms*bps;
    run(nm, [&]{dmma16816_k<4><<<blocks,tpb>>>(out,it/4);}, 2.0*2048*4*(it/4)*(double)blocks*(tpb/32));
  }
  {
    int blocks=sms*2, tpb=256;
    // per warp per iter: 8 DMMA = 4096 flop; R*8 DFMA*32 lanes*2 = 512 R flop
    run("MIXED dmma8 + dfma x8 (R=8)", [&]{mixed_k<8><<<blocks,tpb>>>(out,it,1e-9);}, (4096.0+512*8)*it*(double)blocks*(tpb/32));
    run("MIXED dmma8 + dfma x4 (R=4)", [&]{mixed_k<4><<<blocks,tpb>>>(out,it,1e-9);}, (4096.0+512*4)*it*(double)blocks*(tpb/32));
    run("MIXED dmma8 + dfma x2 (R=2)", [&]{mixed_k<2><<<blocks,tpb>>>(out,it,1e-9);}, (4096.0+512*2)*it*(double)blocks*(tpb/32));
    run("SPLIT warps dmma | dfma", [&]{split_k<<<blocks,tpb>>>(out,it,1e-9);}, (4096.0*4+ 8.0*8*2*32*4)*it*(double)blocks);
  }
  for(int acc : {1,2,4}){
    char nm[96]; snprintf(nm,96,"DMMA 8x8x4 acc%d tpb256 bps2 (latency)",acc);
    int blocks=sms*2;
    if(acc==1) run(nm, [&]{dmma884_k<1><<<blocks,256>>>(out,it);}, 2.0*256*1*it*(double)blocks*8);
    if(acc==2) run(nm, [&]{dmma884_k<2><<<blocks,256>>>(out,it);}, 2.0*256*2*it*(double)blocks*8);
    if(acc==4) run(nm, [&]{dmma884_k<4><<<blocks,256>>>(out,it);}, 2.0*256*4*it*(double)blocks*8);
  }
  return 0;
}
