/* Bit-exactness check of the reciprocal-based division x/d = fma-corrected x*RN(1/d)
 * (two Markstein corrections, guard for zero/subnormal/huge/non-finite x).
 * gcc -O2 -ffp-contract=off tools/micro/divcheck.c -lm && ./a.out  -> mismatches=0 */
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ULL;
static uint64_t rnd(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double mk(int emin, int emax, int adv) {
  uint64_t m = rnd() & ((1ULL<<52)-1);
  if (adv == 1) m = (1ULL<<52)-1 - (rnd() & 0xffff);
  if (adv == 2) m = rnd() & 0xffff;
  int e = emin + (int)(rnd() % (uint64_t)(emax - emin + 1));
  uint64_t bits = ((uint64_t)(e + 1023) << 52) | m; if (rnd() & 1) bits |= 1ULL << 63;
  double d; memcpy(&d, &bits, 8); return d;
}
static double emt_div(double x, double d, double y) {
  const double ax = fabs(x);
  if (!(ax >= 0x1p-960 && ax <= 0x1p1000)) return x / d;
  const double q0 = x * y;
  const double r0 = fma(-d, q0, x);
  const double q1 = fma(r0, y, q0);
  const double r1 = fma(-d, q1, x);
  return fma(r1, y, q1);
}
int main(void) {
  long bad = 0, n = 0;
  for (int pass = 0; pass < 9; ++pass)
    for (long i = 0; i < 40000000; ++i) {
      double x = mk(-300, 300, pass % 3), d = mk(-40, 40, pass / 3);
      double a = x / d, b = emt_div(x, d, 1.0 / d); ++n;
      if (memcmp(&a, &b, 8)) { if (bad < 5) printf("x=%a d=%a %a %a\n", x, d, a, b); ++bad; }
    }
  double sp[] = {0.0, -0.0, 1e-320, -1e-320, 1e308, INFINITY, NAN};
  for (int k = 0; k < 7; ++k) for (int j = 0; j < 100000; ++j) { double d = mk(-40,40,j%3); double a = sp[k]/d, b = emt_div(sp[k], d, 1.0/d); ++n; if (memcmp(&a,&b,8) && !(isnan(a)&&isnan(b))) ++bad; }
  printf("n=%ld mismatches=%ld\n", n, bad);
}
