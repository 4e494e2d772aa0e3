// Host memory bandwidth probe (the e2e bound): N threads stream-read 4 GB with
// AVX-512 loads, then read + write a quarter (the host pack's access pattern).
// gcc -O3 -mavx512f -mavx512bw -o /tmp/host_membw tools/host_membw.c -lpthread; /tmp/host_membw 16 [prefetch lines]
#include <immintrin.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#define GB (1ull<<30)
static size_t per; static int nt; static char* buf; static char* out;
static double now(){struct timespec t;clock_gettime(CLOCK_MONOTONIC,&t);return t.tv_sec+t.tv_nsec*1e-9;}
static int PF = 0;  /* software prefetch distance in 64-byte lines (argv[2]) */
static void* rd(void* a){ long i=(long)a; const __m512i* p=(const __m512i*)(buf+i*per); __m512i s=_mm512_setzero_si512();
  for(size_t k=0;k<per/64;k+=4){ if (PF) { _mm_prefetch((const char*)(p+k+PF), _MM_HINT_T0); _mm_prefetch((const char*)(p+k+PF+2), _MM_HINT_T0); } s=_mm512_xor_si512(s,_mm512_load_si512(p+k)); s=_mm512_xor_si512(s,_mm512_load_si512(p+k+1)); s=_mm512_xor_si512(s,_mm512_load_si512(p+k+2)); s=_mm512_xor_si512(s,_mm512_load_si512(p+k+3)); }
  volatile long long x=_mm512_reduce_add_epi64(s); (void)x; return 0;}
static void* rw(void* a){ long i=(long)a; const __m512i* p=(const __m512i*)(buf+i*per); __m128i* q=(__m128i*)(out+i*(per/4));
  for(size_t k=0;k<per/64;k++){ __m512i v=_mm512_load_si512(p+k); _mm_store_si128(q+k, _mm512_castsi512_si128(_mm512_srli_epi16(v,1))); } return 0;}
int main(int c,char**v){ nt=atoi(v[1]); if (c > 2) PF=atoi(v[2]); size_t tot=4*GB; per=tot/nt/64*64; buf=aligned_alloc(64,tot); out=aligned_alloc(64,tot/4); memset(buf,1,tot); memset(out,0,tot/4);
  pthread_t th[64]; for(int pass=0;pass<2;pass++){ double t0=now(); for(long i=0;i<nt;i++) pthread_create(&th[i],0,pass?rw:rd,(void*)i); for(int i=0;i<nt;i++) pthread_join(th[i],0); double t=now()-t0;
  printf("threads %d prefetch %d %s: %.1f GB/s read\n", nt, PF, pass?"read+quarter-write":"read", per*nt/t/1e9);} return 0;}
