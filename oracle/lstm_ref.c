/* TEST INFRASTRUCTURE ONLY - CPU oracle, never linked into the product.
 *
 * Plain-C restatement of the reference's compiled LSTM forward
 * (pkg/src/tensched/_recurrent_cy.pyx:20-66): one sequence at a time,
 * z = b, += x*Wx with the exact-zero skip (:46-49), += h*Wh (:50-54),
 * gates [i,f,g,o] with sigmoid(x) = 1/(1+exp(-x)) (:17-18), c = f*c + i*g,
 * h = o*tanh(c), raw += sum_j h[j]*w[j] (:61-64), raw starting at T*b_out
 * (:27).  Built with -O2 -ffp-contract=off so every operation is one IEEE
 * rounding, as in the Cython build (no FMA on the x86-64 baseline ISA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

void oracle_lstm_forward(const double* X, int64_t B, int64_t T, int64_t F, const double* Wx,
                         const double* Wh, const double* b, const double* w, int64_t H,
                         double b_out, double* raw) {
  const int64_t G = 4 * H;
  double* h = calloc((size_t)H, sizeof(double));
  double* c = calloc((size_t)H, sizeof(double));
  double* z = calloc((size_t)G, sizeof(double));
  for (int64_t bi = 0; bi < B; ++bi) {
    raw[bi] = (double)T * b_out;
    for (int64_t j = 0; j < H; ++j) h[j] = c[j] = 0.0;
    for (int64_t t = 0; t < T; ++t) {
      for (int64_t j = 0; j < G; ++j) z[j] = b[j];
      for (int64_t k = 0; k < F; ++k) {
        const double x = X[(bi * T + t) * F + k];
        if (x != 0.0)
          for (int64_t j = 0; j < G; ++j) z[j] += x * Wx[k * G + j];
      }
      for (int64_t k = 0; k < H; ++k) {
        const double x = h[k];
        if (x != 0.0)
          for (int64_t j = 0; j < G; ++j) z[j] += x * Wh[k * G + j];
      }
      for (int64_t j = 0; j < H; ++j) {
        const double gi = sigmoid(z[j]);
        const double gf = sigmoid(z[H + j]);
        const double gg = tanh(z[2 * H + j]);
        const double go = sigmoid(z[3 * H + j]);
        c[j] = gf * c[j] + gi * gg;
        h[j] = go * tanh(c[j]);
      }
      double acc = 0.0;
      for (int64_t j = 0; j < H; ++j) acc += h[j] * w[j];
      raw[bi] += acc;
    }
  }
  free(h);
  free(c);
  free(z);
}
