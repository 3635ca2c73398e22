// count_flops.cpp -- algorithmic fp64 operation count of one patch update, measured on the
// oracle's own code (oracle/claw.c compiled with `double` replaced by a counting type).
// Every +, -, *, / and sqrt on a floating value counts 1 flop (the oracle is compiled without FMA
// contraction, so a multiply-add is 2); comparisons, negation, fabs and copies count 0.
// Usage: count_flops <kind> <p0> <p1> <limiter> <m> <meqn> <dt> <dx> <padded.bin> [aux.bin]
// prints "flops cells" for the patches in padded.bin (concatenated [meqn][n][n] blocks).
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>

static long long g_flops = 0;
struct FD {
  double v;
  FD() = default;
  FD(double x) : v(x) {}
  FD(int x) : v(x) {}
};
static inline FD operator+(FD a, FD b) { ++g_flops; return FD(a.v + b.v); }
static inline FD operator-(FD a, FD b) { ++g_flops; return FD(a.v - b.v); }
static inline FD operator*(FD a, FD b) { ++g_flops; return FD(a.v * b.v); }
static inline FD operator/(FD a, FD b) { ++g_flops; return FD(a.v / b.v); }
static inline FD operator-(FD a) { return FD(-a.v); }
static inline FD& operator+=(FD& a, FD b) { ++g_flops; a.v += b.v; return a; }
static inline FD& operator-=(FD& a, FD b) { ++g_flops; a.v -= b.v; return a; }
static inline bool operator<(FD a, FD b) { return a.v < b.v; }
static inline bool operator>(FD a, FD b) { return a.v > b.v; }
static inline bool operator<=(FD a, FD b) { return a.v <= b.v; }
static inline bool operator>=(FD a, FD b) { return a.v >= b.v; }
static inline bool operator==(FD a, FD b) { return a.v == b.v; }
static inline bool operator!=(FD a, FD b) { return a.v != b.v; }
static inline FD sqrt(FD a) { ++g_flops; return FD(std::sqrt(a.v)); }
static inline FD fabs(FD a) { return FD(std::fabs(a.v)); }
static inline FD ldexp(FD a, int e) { return FD(std::ldexp(a.v, e)); }

#define double FD
#include "../oracle/claw.c"
#undef double

// stubs for the forest-level entry points claw.c references (not used here)
int orc_ghost_fill(const orc_forest*, FD*, int) { return 0; }
int orc_build_padded_sample(const orc_forest*, const FD*, int, int64_t, FD*) { return 0; }

int main(int argc, char** argv) {
  if (argc < 10) { fprintf(stderr, "usage\n"); return 2; }
  orc_problem pr;
  pr.kind = atoi(argv[1]);
  pr.p0 = FD(atof(argv[2]));
  pr.p1 = FD(atof(argv[3]));
  pr.limiter = atoi(argv[4]);
  pr.method2 = 2;
  pr.method3 = 2;
  const int m = atoi(argv[5]), meqn = atoi(argv[6]);
  const double dt = atof(argv[7]), dx = atof(argv[8]);
  const int n = m + 4;
  FILE* fp = fopen(argv[9], "rb");
  FILE* fa = argc > 10 ? fopen(argv[10], "rb") : NULL;
  const size_t S = (size_t)meqn * n * n, SA = (size_t)3 * n * n;
  double* buf = (double*)malloc(S * sizeof(double));
  double* abuf = (double*)malloc(SA * sizeof(double));
  FD* q = (FD*)malloc(S * sizeof(FD));
  FD* qo = (FD*)malloc(S * sizeof(FD));
  FD* a = (FD*)malloc(SA * sizeof(FD));
  long long cells = 0;
  while (fread(buf, sizeof(double), S, fp) == S) {
    for (size_t k = 0; k < S; ++k) q[k] = FD(buf[k]);
    if (fa) {
      if (fread(abuf, sizeof(double), SA, fa) != SA) break;
      for (size_t k = 0; k < SA; ++k) a[k] = FD(abuf[k]);
    }
    orc_step_patch(&pr, m, meqn, q, fa ? a : NULL, FD(dt), FD(dx), FD(dx), qo);
    cells += (long long)m * m;
  }
  printf("%lld %lld\n", g_flops, cells);
  return 0;
}
