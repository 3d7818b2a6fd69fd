// pipeoptim_rules.cuh — the per-element optimizer rules shared by every
// kernel that applies them (the streaming K1/K2/K3, the fused DP forms in
// pipeoptim_kernels.cu, and the weight-gradient GEMM with the update in its
// epilogue in pipeoptim_wgrad.cu): the launch coefficients, derived on the
// host in double and rounded once to fp32, and the SGDM / Adam / AdamW step +
// prediction of one element in IEEE fp32 (no FMA contraction), so all of them
// produce the same bits for the same gradient value.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#include "pipeoptim.h"

namespace {

enum Mode : int {
  MODE_STEP = 0,          // K2 (optionally also writes the applied direction)
  MODE_STEP_DIR = 1,      // K2 + dir_out
  MODE_PREDICT = 2,       // K1
  MODE_PREDICT_ZERO = 3,  // K1 before the first step (direction == 0)
  MODE_STEP_PREDICT = 4,  // K3
  MODE_DIRECTION = 5,     // prediction_direction read
  MODE_DIRECTION_ZERO = 6,
  MODE_AXPY = 7,          // predict_weights(w, d)
};

// fp32 launch coefficients, derived on the host in double.
struct Coef {
  float lr;         // step learning rate
  float c_pred;     // lr_pred * s  (K1 / K3 / AXPY)
  float ibc1, ibc2; // reciprocal bias corrections 1/(1 - beta^t) at the t this launch reads/writes
  float beta1, omb1, beta2, omb2, eps, lam;
  float mom, omd, wd;
};

// ---- the per-element rules --------------------------------------------------

// Adam/AdamW moment-ratio direction (m/bc1) / (sqrt(v/bc2) + eps),
// optim.py:115 (step) and optim.py:141 (read), evaluated as
// (m * ibc1) / (sqrt(v * ibc2) + eps) with the reciprocal bias corrections
// formed in double on the host and rounded once: one IEEE division and one
// IEEE square root per element instead of three divisions (each __fdiv_rn is
// an RCP + Newton + FCHK/slow-path sequence) — the arithmetic that bounds the
// Adam kernels when their data sits in L2 (pipeline-stage sizes). Every step
// is correctly rounded; vs the float64 reference the direction moves by
// <= ~3 ulp, far inside the 1e-6 contract.
__device__ __forceinline__ float adam_dir(float m, float v, const Coef& c) {
#ifdef PO_PROBE_ADAM_DIV3  // timing probe only (scripts/adam_dir_ab.py): the round-1 three-division cost
  return __fdiv_rn(__fdiv_rn(m, c.ibc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, c.ibc2)), c.eps));
#else
  return __fdiv_rn(__fmul_rn(m, c.ibc1), __fadd_rn(__fsqrt_rn(__fmul_rn(v, c.ibc2)), c.eps));
#endif
}

// One element. w/s1/s2 are updated in place for step modes; `out` receives
// W_hat or the direction; `nonfinite` flags a non-finite updated weight
// (optim.py:82-84 checks the new weights only).
template <int KIND, int MODE>
__device__ __forceinline__ void elem(const Coef& c, float& w, float g, float& s1, float& s2,
                                     float& out, bool& nonfinite) {
  if constexpr (MODE == MODE_AXPY) {
    // predict_weights: w - (lr*s) * d, optim.py:155
    out = __fsub_rn(w, __fmul_rn(c.c_pred, s1));
  } else if constexpr (MODE == MODE_PREDICT_ZERO) {
    // zero direction before the first step (optim.py:131-132), then Eq. (5)
    out = __fsub_rn(w, __fmul_rn(c.c_pred, 0.0f));
  } else if constexpr (MODE == MODE_DIRECTION_ZERO) {
    out = 0.0f;
  } else if constexpr (MODE == MODE_PREDICT || MODE == MODE_DIRECTION) {
    // prediction_direction read (optim.py:133-141): sgdm -> buf; adam(w) -> ratio, no lambda*W
    float d = (KIND == PO_SGDM) ? s1 : adam_dir(s1, s2, c);
    if constexpr (MODE == MODE_PREDICT)
      out = __fsub_rn(w, __fmul_rn(c.c_pred, d));
    else
      out = d;
  } else {
    // step (optim.py:63-119)
    float d, dread;
    if constexpr (KIND == PO_SGDM) {
      // eff = g + wd*W ; v = u*v + (1-tau)*eff  (optim.py:95-96)
      float eff = __fadd_rn(g, __fmul_rn(c.wd, w));
      float nb = __fadd_rn(__fmul_rn(c.mom, s1), __fmul_rn(c.omd, eff));
      s1 = nb;
      d = nb;
      dread = nb;  // read after the step is the buffer (optim.py:134-135)
    } else {
      // m = b1*m + (1-b1)*g ; v = b2*v + (1-b2)*g*g  (optim.py:111-112)
      float m = __fadd_rn(__fmul_rn(c.beta1, s1), __fmul_rn(c.omb1, g));
      float v = __fadd_rn(__fmul_rn(c.beta2, s2), __fmul_rn(c.omb2, __fmul_rn(g, g)));
      s1 = m;
      s2 = v;
      // the read right after this step uses t = step_count_new == this step's t,
      // so the step and read bias corrections coincide (S5)
      dread = adam_dir(m, v, c);
      d = (KIND == PO_ADAMW) ? __fadd_rn(dread, __fmul_rn(c.lam, w)) : dread;  // optim.py:116-117
    }
    float nw = __fsub_rn(w, __fmul_rn(c.lr, d));  // W - lr*d, optim.py:82
    nonfinite |= !isfinite(nw);
    w = nw;
    if constexpr (MODE == MODE_STEP_DIR) out = d;
    if constexpr (MODE == MODE_STEP_PREDICT) out = __fsub_rn(nw, __fmul_rn(c.c_pred, dread));
  }
}

// Host-side coefficient derivation in double, mirroring the reference's
// Python float arithmetic, then rounded once to fp32.
Coef coef(const po_hparams* hp, double lr, double c_pred, int64_t t) {
  Coef c;
  memset(&c, 0, sizeof(c));
  c.lr = (float)lr;
  c.c_pred = (float)c_pred;
  if (t >= 1) {
    c.ibc1 = (float)(1.0 / (1.0 - pow(hp->beta1, (double)t)));  // optim.py:107 / :137
    c.ibc2 = (float)(1.0 / (1.0 - pow(hp->beta2, (double)t)));  // optim.py:108 / :138
  } else {
    c.ibc1 = 1.f;
    c.ibc2 = 1.f;
  }
  c.beta1 = (float)hp->beta1;
  c.omb1 = (float)(1.0 - hp->beta1);
  c.beta2 = (float)hp->beta2;
  c.omb2 = (float)(1.0 - hp->beta2);
  c.eps = (float)hp->eps;
  c.lam = (float)hp->decoupled_decay;
  c.mom = (float)hp->momentum;
  c.omd = (float)(1.0 - hp->dampening);
  c.wd = (float)hp->weight_decay;
  return c;
}

}  // namespace
