// host microbenchmark: widen int32 -> int64 with T threads (is a 32-bit D2H + host widening cheaper than a 64-bit D2H?)
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
static double now(){ struct timespec t; clock_gettime(CLOCK_MONOTONIC,&t); return t.tv_sec+1e-9*t.tv_nsec; }
typedef struct { const int32_t* in; int64_t* out; size_t lo, hi; int nt; } job_t;
static void* work(void* p){ job_t* j=(job_t*)p; const int32_t* in=j->in; int64_t* out=j->out; size_t i=j->lo;
  if (j->nt) { for(; i+8<=j->hi; i+=8){ __m256i v=_mm256_loadu_si256((const __m256i*)(in+i)); __m256i a=_mm256_cvtepi32_epi64(_mm256_castsi256_si128(v)); __m256i b=_mm256_cvtepi32_epi64(_mm256_extracti128_si256(v,1)); _mm256_stream_si256((__m256i*)(out+i),a); _mm256_stream_si256((__m256i*)(out+i+4),b);} _mm_sfence(); }
  else { for(; i+8<=j->hi; i+=8){ __m256i v=_mm256_loadu_si256((const __m256i*)(in+i)); __m256i a=_mm256_cvtepi32_epi64(_mm256_castsi256_si128(v)); __m256i b=_mm256_cvtepi32_epi64(_mm256_extracti128_si256(v,1)); _mm256_storeu_si256((__m256i*)(out+i),a); _mm256_storeu_si256((__m256i*)(out+i+4),b);} }
  for(; i<j->hi; ++i) out[i]=in[i]; return 0; }
int main(int argc,char**argv){ size_t n= (size_t)(argc>1?atol(argv[1]):22700000); int maxt=argc>2?atoi(argv[2]):16;
  int32_t* in=aligned_alloc(64,n*4); int64_t* out=aligned_alloc(64,n*8); for(size_t i=0;i<n;++i) in[i]=(int32_t)i; memset(out,0,n*8);
  for(int nt=0; nt<2; ++nt) for(int T=1; T<=maxt; T*=2){ double best=1e9; for(int rep=0; rep<5; ++rep){ pthread_t th[64]; job_t jb[64]; double t0=now();
      for(int t=0;t<T;++t){ jb[t]=(job_t){in,out,(n*t/T)&~7ul,(t==T-1)?n:((n*(t+1)/T)&~7ul),nt}; pthread_create(&th[t],0,work,&jb[t]); }
      for(int t=0;t<T;++t) pthread_join(th[t],0); double dt=now()-t0; if(dt<best)best=dt; }
    printf("%s T=%2d  %.3f ms  (%.1f GB/s of int64 written)\n", nt?"stream":"store ", T, best*1e3, n*8/best/1e9); }
  // memcpy reference
  { double best=1e9; for(int rep=0;rep<5;++rep){ double t0=now(); memcpy(out,in,n*4); double dt=now()-t0; if(dt<best)best=dt;} printf("memcpy %zu MB single thread: %.3f ms\n", n*4>>20, best*1e3); }
  return (int)out[n/2]&1; }
