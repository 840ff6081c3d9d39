"""The kernel's glibc_log1p_fma (csrc/rf_noise.cu) compiled for the host == this libm's log1p.

numpy's ziggurat tail path calls glibc log1p; the GPU reproduces glibc 2.39's FMA
variant operation by operation.  Here the same source is compiled with g++ (no FMA
contraction) and compared bit-for-bit with the host libm on ~4M arguments.
"""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PRELUDE = r'''
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <random>
static double __dmul_rn(double a,double b){return a*b;}
static double __dadd_rn(double a,double b){return a+b;}
static double __dsub_rn(double a,double b){return a-b;}
static double __ddiv_rn(double a,double b){return a/b;}
static double __fma_rn(double a,double b,double c){return std::fma(a,b,c);}
static int __double2hiint(double x){uint64_t u;memcpy(&u,&x,8);return (int)(u>>32);}
static int __double2loint(double x){uint64_t u;memcpy(&u,&x,8);return (int)(uint32_t)u;}
static double __hiloint2double(int hi,int lo){uint64_t u=((uint64_t)(uint32_t)hi<<32)|(uint32_t)lo;
  double d;memcpy(&d,&u,8);return d;}
#define CUDART_INF INFINITY
#define CUDART_NAN NAN
'''
MAIN = r'''
int main(){ std::mt19937_64 g(7); long bad=0,n=0;
 auto chk=[&](double x){double a=glibc_log1p_fma(x), b=log1p(x); n++; if(memcmp(&a,&b,8)) bad++;};
 for(long i=0;i<3000000;i++){ double u=(double)(g()>>11)*(1.0/9007199254740992.0); chk(-u); }
 for(long i=0;i<250000;i++){ double u=(double)(g()>>11)*(1.0/9007199254740992.0);
   chk(u*10); chk(ldexp(u,-(int)(g()%60))); chk(-ldexp(u,-(int)(g()%60))); chk(u*1e17);}
 chk(-0.0); chk(0.0); chk(-1.0); chk(1e300);
 printf("%ld %ld\n",n,bad); return bad != 0; }
'''


def test_log1p_transcription_matches_host_libm():
    src = open(os.path.join(ROOT, "paper_2605_28657_b200", "csrc", "rf_noise.cu")).read()
    a = src.index("__device__ __noinline__ double glibc_log1p_fma")
    b = src.index("// A full draw starting")
    fn = src[a:b].replace("__device__ __noinline__ ", "")
    with tempfile.TemporaryDirectory() as tmp:
        cpp = os.path.join(tmp, "t.cpp")
        open(cpp, "w").write(PRELUDE + fn + MAIN)
        exe = os.path.join(tmp, "t")
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-o", exe, cpp, "-lm"])
        out = subprocess.run([exe], capture_output=True, text=True)
    n, bad = map(int, out.stdout.split())
    assert n > 3_000_000 and bad == 0, out.stdout
