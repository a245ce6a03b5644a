// Microbenchmarks that size the FFT design on B200 (HBM strided runs, L2, DSMEM, fp64).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %s:%d\n",cudaGetErrorString(e),__FILE__,__LINE__); return 1;}}while(0)

__global__ void copy_contig(const float4* __restrict__ a, float4* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=s) b[i]=a[i];
}
// Tile copy: matrix rows x cols of 16B units; each block copies a column strip of
// w units (w*16 bytes) by nrow rows, reading and writing the same positions.
__global__ void strip_copy(const float4* __restrict__ a, float4* __restrict__ b, int64_t cols, int w, int nrow){
  int64_t strips = cols / w;
  int64_t strip = blockIdx.x % strips, rblk = blockIdx.x / strips;
  int64_t r0 = rblk * nrow;
  for(int t = threadIdx.x; t < w*nrow; t += blockDim.x){
    int64_t r = r0 + t / w, c = strip*w + t % w;
    b[r*cols + c] = a[r*cols + c];
  }
}
__global__ void l2_read(const float4* __restrict__ a, size_t n, int reps, float* out){
  float acc=0;
  for(int rep=0; rep<reps; ++rep){
    size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, s=(size_t)gridDim.x*blockDim.x;
    for(; i<n; i+=s){ float4 v = __ldcg(a+i); acc += v.x+v.y+v.z+v.w; }
  }
  if(acc==12345.f) out[0]=acc;
}
template<int CS>
__global__ void dsmem_read(int reps, float* out){
  extern __shared__ float4 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int n = 64*1024/16;
  for(int i=threadIdx.x;i<n;i+=blockDim.x) sm[i]=make_float4(i,1,2,3);
  cl.sync();
  unsigned peer = (cl.block_rank()+1)%CS;
  float4* rp = cl.map_shared_rank(sm, peer);
  float acc=0;
  for(int rep=0; rep<reps; ++rep)
    for(int i=threadIdx.x;i<n;i+=blockDim.x){ float4 v=rp[i]; acc+=v.x+v.w; }
  cl.sync();
  if(acc==12345.f) out[0]=acc;
}
template<int CS>
__global__ void dsmem_write(int reps, float* out){
  extern __shared__ float4 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int n = 64*1024/16;
  cl.sync();
  unsigned peer = (cl.block_rank()+1)%CS;
  float4* rp = cl.map_shared_rank(sm, peer);
  for(int rep=0; rep<reps; ++rep)
    for(int i=threadIdx.x;i<n;i+=blockDim.x){ rp[i]=make_float4(i,rep,2,3); }
  cl.sync();
  if(sm[threadIdx.x].x==-1.f) out[0]=1;
}
__global__ void dfma(double* out, int reps){
  double a=threadIdx.x*1e-3, b=1.0000001, c=1e-9, d=0.5, e=0.25,f=0.125,g=0.3,h=0.7;
  for(int i=0;i<reps;++i){ a=fma(a,b,c); d=fma(d,b,c); e=fma(e,b,c); f=fma(f,b,c); g=fma(g,b,c); h=fma(h,b,c);}
  if(a+d+e+f+g+h==1.2345) out[0]=a;
}
__global__ void sincos64(double* out, int reps){
  double acc=0; int64_t k = blockIdx.x*blockDim.x+threadIdx.x;
  for(int i=0;i<reps;++i){ double s,c; sincospi((double)((k*7919+i)&((1<<20)-1))*(2.0/(1<<20)),&s,&c); acc+=s+c; }
  if(acc==1.2345) out[0]=acc;
}
__global__ void sincos32(float* out, int reps){
  float acc=0; int k = blockIdx.x*blockDim.x+threadIdx.x;
  for(int i=0;i<reps;++i){ float s,c; sincospif((float)((k*7919+i)&((1<<20)-1))*(2.0f/(1<<20)),&s,&c); acc+=s+c; }
  if(acc==1.2345f) out[0]=acc;
}

int main(){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  size_t bytes = 4ull<<30; float4 *a,*b; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&b,bytes));
  cudaMemset(a,0,bytes); cudaMemset(b,0,bytes);
  size_t n = bytes/16;
  for(int it=0;it<3;++it) copy_contig<<<148*8,512>>>(a,b,n);
  cudaEventRecord(e0); for(int it=0;it<5;++it) copy_contig<<<148*8,512>>>(a,b,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); printf("copy_contig 4GiB: %.1f GB/s\n", 2.0*bytes*5/ms/1e6);
  int64_t cols = 32768/2; // 16B units per row -> 256 KiB rows
  int64_t rows = n/cols;
  for(int w: {1,2,4,8,16}) for(int nrow: {64, 256, 1024}){
    int64_t blocks = (cols/w)*(rows/nrow);
    strip_copy<<<blocks,256>>>(a,b,cols,w,nrow);
    cudaEventRecord(e0); for(int it=0;it<3;++it) strip_copy<<<blocks,256>>>(a,b,cols,w,nrow); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("strip_copy w=%3dB nrow=%4d: %.1f GB/s\n", w*16, nrow, 2.0*bytes*3/ms/1e6);
  }
  float* o; cudaMalloc(&o,64);
  for(size_t l2b: {16ull<<20, 48ull<<20, 96ull<<20}){
    size_t nn = l2b/16; l2_read<<<148*4,512>>>(a,nn,2,o);
    cudaEventRecord(e0); l2_read<<<148*4,512>>>(a,nn,20,o); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("l2_read %zu MiB: %.1f GB/s\n", l2b>>20, 20.0*l2b/ms/1e6);
  }
  {
    auto run=[&](auto kern, int cs, const char* nm){
      cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(148/cs*cs*1); cfg.blockDim=dim3(512); cfg.dynamicSmemBytes=64*1024;
      at[0].id=cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x=cs; at[0].val.clusterDim.y=1; at[0].val.clusterDim.z=1;
      cfg.attrs=at; cfg.numAttrs=1;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64*1024);
      int reps=200;
      cudaLaunchKernelEx(&cfg, kern, 2, o);
      cudaEventRecord(e0); cudaError_t err = cudaLaunchKernelEx(&cfg, kern, reps, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms,e0,e1);
      printf("%s cs=%d: %s %.1f GB/s total, %.1f B/clk/SM@1.9GHz\n", nm, cs, cudaGetErrorString(err), (double)cfg.gridDim.x*reps*65536/ms/1e6, (double)reps*65536/(ms*1e-3*1.9e9));
    };
    run(dsmem_read<2>,2,"dsmem_read"); run(dsmem_read<4>,4,"dsmem_read"); run(dsmem_read<8>,8,"dsmem_read");
    run(dsmem_write<2>,2,"dsmem_write"); run(dsmem_write<8>,8,"dsmem_write");
  }
  double* od; cudaMalloc(&od,64);
  dfma<<<148*8,256>>>(od,100);
  cudaEventRecord(e0); dfma<<<148*8,256>>>(od,100000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); printf("dfma: %.2f TFLOP/s\n", 148.0*8*256*100000*6*2/ms/1e9);
  cudaEventRecord(e0); sincos64<<<148*8,256>>>(od,1000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); printf("sincospi f64: %.2f Gop/s\n", 148.0*8*256*1000/ms/1e6);
  cudaEventRecord(e0); sincos32<<<148*8,256>>>((float*)od,1000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); printf("sincospif f32: %.2f Gop/s\n", 148.0*8*256*1000/ms/1e6);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0); printf("L2 %d MiB\n", l2>>20);
  return 0;
}
