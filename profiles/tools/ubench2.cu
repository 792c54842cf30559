#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
  double x0=a,x1=a+1,x2=a+2,x3=a+3,x4=a+4,x5=a+5,x6=a+6,x7=a+7;
  float f0=a,f1=a+1,f2=a+2,f3=a+3,f4=a+4,f5=a+5,f6=a+6,f7=a+7; float fb=b, fa=a;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x0=fma(x0,b,a);x1=fma(x1,b,a);x2=fma(x2,b,a);x3=fma(x3,b,a);x4=fma(x4,b,a);x5=fma(x5,b,a);x6=fma(x6,b,a);x7=fma(x7,b,a); }
  __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { f0=fmaf(f0,fb,fa);f1=fmaf(f1,fb,fa);f2=fmaf(f2,fb,fa);f3=fmaf(f3,fb,fa);f4=fmaf(f4,fb,fa);f5=fmaf(f5,fb,fa);f6=fmaf(f6,fb,fa);f7=fmaf(f7,fb,fa); }
  __syncthreads();
  long long t2 = clock64();
  double y0=a,y1=a; float g=a;
  for (int i = 0; i < n; ++i) { y0 = (double)g * b; g = (float)(y0 + y1); }
  __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
  out[threadIdx.x + blockIdx.x * blockDim.x] = x0+x1+x2+x3+x4+x5+x6+x7+f0+f1+f2+f3+f4+f5+f6+f7+y0+g;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMallocManaged(&c, 64);
  int n = 2000;
  for (int nt : {32, 128, 256, 512, 1024}) {
    k<<<1, nt>>>(o, c, n, 0.5, 0.999); cudaDeviceSynchronize();
    k<<<1, nt>>>(o, c, n, 0.5, 0.999); cudaDeviceSynchronize();
    double ops = 8.0 * n * nt;
    printf("threads %4d: DFMA %.2f /clk/SM   FFMA %.2f /clk/SM   cvt-chain %.1f cyc/it\n", nt, ops / c[0], ops / c[1], c[2] / (double)n);
  }
}
