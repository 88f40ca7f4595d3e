/* Bit-exactness check of the division the generated kernels use in the backward
 * sweep: x/d == fma(fma(-d, q0, x), y, q0) with y = RN(1/d), q0 = RN(x*y)
 * (one Markstein correction). Normal-range operands, adversarial mantissas.
 * gcc -O2 -ffp-contract=off -march=native tools/micro/divcheck.c -lm && ./a.out -> mismatches=0 */
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
int main(void) {
  long bad = 0, n = 0;
  for (int pass = 0; pass < 9; ++pass)
    for (long i = 0; i < 20000000; ++i) {
      double x = mk(-300, 300, pass % 3), d = mk(-40, 40, pass / 3);
      double y = 1.0 / d;
      double q0 = x * y;
      double r0 = fma(-d, q0, x);
      double q1 = fma(r0, y, q0);
      double a = x / d; ++n;
      if (memcmp(&a, &q1, 8)) { if (bad < 5) printf("x=%a d=%a %a %a\n", x, d, a, q1); ++bad; }
    }
  printf("n=%ld mismatches=%ld\n", n, bad);
}
