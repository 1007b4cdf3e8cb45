// Brute-force check of Markstein's division correction: with y = RN(1/b),
// q = RN(a*y), RN(q + fma(-b, q, a) * y) == RN(a/b) for normal operands.
// Used to evaluate a shared-reciprocal kinetic-energy quotient in the fused
// hydro kernel (bit-exact, but measured slower: DESIGN.md 9.2).
// gcc -O2 -ffp-contract=off -march=native markstein.c -lm && ./a.out
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static uint64_t s=88172645463325252ull;
static inline uint64_t xr(){s^=s<<13;s^=s>>7;s^=s<<17;return s;}
static inline double mk(uint64_t mant, int e){uint64_t b=((uint64_t)(e+1023)<<52)|(mant&((1ull<<52)-1));double d;memcpy(&d,&b,8);return d;}
int main(){
  long bad=0,n=0;
  for(long i=0;i<400000000L;i++){
    uint64_t m1=xr(),m2=xr(); int k=xr()%8;
    if(k==0) m2=(1ull<<52)-1-(xr()%64);     // all-ones-ish divisor mantissas
    if(k==1) m2=xr()%64;                    // near power of two
    if(k==2) m1=(1ull<<52)-1-(xr()%64);
    if(k==3) m1=xr()%64;
    int e1=(int)(xr()%200)-100, e2=(int)(xr()%200)-100;
    double a=mk(m1,e1), b=mk(m2,e2);
    volatile double y=1.0/b; volatile double q=a*y;
    double r=fma(-b,q,a); double q2=fma(r,y,q);
    double ref=a/b; n++;
    if(q2!=ref){ if(bad<10) printf("a=%a b=%a ref=%a got=%a\n",a,b,ref,q2); bad++;}
  }
  printf("n=%ld bad=%ld\n",n,bad);
}
