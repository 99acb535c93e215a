/* TEST INFRASTRUCTURE ONLY -- C restatement of the reference's squared-distance
 * contraction, used by tests/ to pin the GPU's exact-recipe helper bit for bit.
 *
 * The reference computes every distance as sqrt(vecdot(x - c, x - c))
 * (numakmeans distance.py:28-39).  For f64 rows np.vecdot calls OpenBLAS ddot,
 * a third-party dependency that is not vendored under /root/reference
 * (numpy 2.3.5 + scipy-openblas 0.3.30, DYNAMIC_ARCH kernel "SkylakeX" on the
 * build host).  Its published kernel keeps four 512-bit FMA accumulators over
 * 32-element blocks, folds them to 256 bits, runs 16-element blocks, reduces
 * lanes in a fixed tree and finishes with a scalar FMA tail (SURVEY.md
 * appendix A.1).  tests/test_oracle_pins.py checks this restatement against
 * np.vecdot on the test host and skips the bit-level pins when the host BLAS
 * picks a different kernel.
 */
#include <math.h>
#include <stdint.h>

static double tree_sq(const double *x, const double *c, int d) {
  int n1 = d & ~15, n32 = n1 & ~31, i, a, l;
  double dot = 0.0;
  if (n1) {
    double z[4][8] = {{0}}, acc[4][4], s[4];
    for (i = 0; i < n32; i += 32)
      for (a = 0; a < 4; a++)
        for (l = 0; l < 8; l++) {
          double v = x[i + 8 * a + l] - c[i + 8 * a + l];
          z[a][l] = fma(v, v, z[a][l]);
        }
    for (a = 0; a < 4; a++)
      for (l = 0; l < 4; l++) acc[a][l] = z[a][l] + z[a][l + 4];
    for (i = n32; i < n1; i += 16)
      for (a = 0; a < 4; a++)
        for (l = 0; l < 4; l++) {
          double v = x[i + 4 * a + l] - c[i + 4 * a + l];
          acc[a][l] = fma(v, v, acc[a][l]);
        }
    for (l = 0; l < 4; l++) s[l] = ((acc[0][l] + acc[1][l]) + acc[2][l]) + acc[3][l];
    dot = (s[0] + s[2]) + (s[1] + s[3]);
  }
  for (i = n1; i < d; i++) {
    double v = x[i] - c[i];
    dot = fma(v, v, dot);
  }
  return dot;
}

/* out[r] = contraction of (rows[r] - ref[r or 0]); ref_per_row selects the ref stride. */
void oracle_tree_sqdist(const double *rows, const double *ref, int64_t m, int d,
                        int ref_per_row, double *out) {
  for (int64_t r = 0; r < m; r++)
    out[r] = tree_sq(rows + r * d, ref + (ref_per_row ? r * d : 0), d);
}
