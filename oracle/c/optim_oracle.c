/*
 * optim_oracle.c — TEST/BASELINE INFRASTRUCTURE ONLY.
 *
 * The reference optimizer rules and optimizer-dependent predictor
 * (/root/reference/pkg/src/pipesim/optim.py) restated in C over flat float64
 * arrays, parallelised with OpenMP. This is the multi-core CPU baseline that
 * bench.py times (cpu_baseline, --impl reference); it is checked element for
 * element against oracle/optim_ref.py (numpy, bit-identical to the reference)
 * by tests/test_oracle.py.
 *
 * Built with -ffp-contract=off so no FMA changes the float64 rounding relative
 * to numpy's separately rounded multiplies and adds.
 *
 * kinds: 0 sgdm, 1 adam, 2 adamw (optim.py:17).
 */
#include <math.h>
#include <stdint.h>

typedef struct oracle_hp {
  int kind;
  double momentum, dampening, weight_decay; /* optim.py:23-25 */
  double beta1, beta2, eps, decoupled_decay; /* optim.py:26-29 */
} oracle_hp;

/* _sgdm_directions optim.py:89-99 + W - lr*d optim.py:82; returns the number
 * of non-finite updated weights (optim.py:83). */
static int64_t sgdm_step(const oracle_hp* h, double* w, const double* g, double* buf, int64_t n,
                         double lr, double* w_hat, double c_pred) {
  const double wd = h->weight_decay, u = h->momentum, omd = 1.0 - h->dampening;
  int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int64_t i = 0; i < n; ++i) {
    double eff = g[i] + wd * w[i];
    double v = u * buf[i] + omd * eff;
    double nw = w[i] - lr * v;
    buf[i] = v;
    w[i] = nw;
    bad += !isfinite(nw);
    if (w_hat) w_hat[i] = nw - c_pred * v; /* read = buffer, optim.py:134-135 */
  }
  return bad;
}

/* _adam_directions optim.py:101-119 (t = step_count + 1). */
static int64_t adam_step(const oracle_hp* h, double* w, const double* g, double* m, double* v,
                         int64_t n, double lr, int64_t step_count, double* w_hat, double c_pred) {
  const double t = (double)(step_count + 1);
  const double bc1 = 1.0 - pow(h->beta1, t), bc2 = 1.0 - pow(h->beta2, t);
  const double b1 = h->beta1, omb1 = 1.0 - h->beta1, b2 = h->beta2, omb2 = 1.0 - h->beta2;
  const double eps = h->eps, lam = h->decoupled_decay;
  const int adamw = h->kind == 2;
  int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int64_t i = 0; i < n; ++i) {
    double gi = g[i];
    double mi = b1 * m[i] + omb1 * gi;
    double vi = b2 * v[i] + omb2 * (gi * gi);
    double r = (mi / bc1) / (sqrt(vi / bc2) + eps);
    double d = adamw ? r + lam * w[i] : r;
    double nw = w[i] - lr * d;
    m[i] = mi;
    v[i] = vi;
    w[i] = nw;
    bad += !isfinite(nw);
    /* read after the step: same t, no lambda*W (optim.py:136-141) */
    if (w_hat) w_hat[i] = nw - c_pred * r;
  }
  return bad;
}

int64_t oracle_step(const oracle_hp* h, double* w, const double* g, double* s1, double* s2,
                    int64_t n, double lr, int64_t step_count) {
  if (h->kind == 0) return sgdm_step(h, w, g, s1, n, lr, 0, 0.0);
  return adam_step(h, w, g, s1, s2, n, lr, step_count, 0, 0.0);
}

int64_t oracle_step_predict(const oracle_hp* h, double* w, const double* g, double* s1,
                            double* s2, double* w_hat, int64_t n, double lr,
                            double lr_pred_times_s, int64_t step_count) {
  if (h->kind == 0) return sgdm_step(h, w, g, s1, n, lr, w_hat, lr_pred_times_s);
  return adam_step(h, w, g, s1, s2, n, lr, step_count, w_hat, lr_pred_times_s);
}

/* prediction_direction (optim.py:123-142) + predict_weights (optim.py:145-155). */
void oracle_predict(const oracle_hp* h, const double* w, const double* s1, const double* s2,
                    double* w_hat, int64_t n, double lr_times_s, int64_t step_count) {
  if (step_count == 0) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) w_hat[i] = w[i] - lr_times_s * 0.0;
    return;
  }
  if (h->kind == 0) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) w_hat[i] = w[i] - lr_times_s * s1[i];
    return;
  }
  const double t = (double)step_count;
  const double bc1 = 1.0 - pow(h->beta1, t), bc2 = 1.0 - pow(h->beta2, t);
  const double eps = h->eps;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double r = (s1[i] / bc1) / (sqrt(s2[i] / bc2) + eps);
    w_hat[i] = w[i] - lr_times_s * r;
  }
}

int oracle_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
