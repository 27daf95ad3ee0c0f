/* Host check of the device erf port (csrc/glibc_math.cuh glibc_erf) against the host
 * glibc's erf, bit for bit: the same source the GPU compiles (-fmad=false), built here
 * with -ffp-contract=off.  Inputs: uniform over the port's regions, region boundaries,
 * tiny/denormal values, large magnitudes, and the newsvendor's z / sqrt(2) arguments.
 * Prints the mismatch count (0 expected) and exits non-zero on any mismatch. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "glibc_tables.h"
#include "glibc_math.cuh"

static uint64_t st = 0x9e3779b97f4a7c15ULL;
static uint64_t next(void) {  /* splitmix64 */
  uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double u01(void) { return (double)(next() >> 11) * 0x1.0p-53; }

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 2000000;
  long bad = 0;
  const double edges[] = {0.0, -0.0, 0x1.0p-28, 0x1.0p-1022, 0x1.0p-1074, 0.84375, 1.25,
                          1.0 / 0.35, 2.857142857142857, 6.0, 5.999999999999999, 1e300, INFINITY};
  for (unsigned i = 0; i < sizeof(edges) / sizeof(edges[0]); ++i)
    for (int sgn = -1; sgn <= 1; sgn += 2)
      for (int k = -3; k <= 3; ++k) {
        double x = sgn * nextafter(edges[i], k < 0 ? 0.0 : INFINITY);
        if (k == 0) x = sgn * edges[i];
        double a = glibc_erf(x, simopt_exptab_bits), b = erf(x);
        if (memcmp(&a, &b, 8) && !(isnan(a) && isnan(b))) ++bad;
      }
  for (long i = 0; i < n; ++i) {
    const uint64_t r = next();
    double x;
    switch (r & 7) {
      case 0: x = (u01() * 2.0 - 1.0) * 0.84375; break;
      case 1: x = 0.84375 + u01() * 0.40625; break;
      case 2: x = 1.25 + u01() * (1.0 / 0.35 - 1.25); break;
      case 3: x = 1.0 / 0.35 + u01() * (6.0 - 1.0 / 0.35); break;
      case 4: x = ldexp(u01() + 0.5, -(int)(next() % 1070)); break;
      case 5: x = (u01() - 0.5) * 20.0; break;
      case 6: {  /* newsvendor: z = (x - mu)/sigma, erf(z * SQRT1_2) */
        const double mu = 20.0 + 30.0 * u01(), sg = 10.0 + 10.0 * u01(), xx = 120.0 * u01();
        x = ((xx - mu) / sg) * 0.7071067811865476;
        break;
      }
      default: { uint64_t b = next(); memcpy(&x, &b, 8); }
    }
    if (r & 8) x = -x;
    double a = glibc_erf(x, simopt_exptab_bits), b = erf(x);
    if (memcmp(&a, &b, 8) && !(isnan(a) && isnan(b))) {
      if (bad < 5) fprintf(stderr, "x=%a port=%a libm=%a\n", x, a, b);
      ++bad;
    }
  }
  printf("%ld\n", bad);
  return bad != 0;
}
