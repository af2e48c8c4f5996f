// step_params.h -- kernel parameters of one Jacobi step (step.cu, gesvj.cu)
#pragma once
#include <cstdint>

namespace jsvd {

struct StepParams {
  int64_t m, n;
  double* G;
  int64_t ldg;  // leading dimension in elements (complex: double2 units)
  double* V;
  int64_t ldv;
  const int32_t* pairs;  // explicit pairs, or nullptr -> strategy (B, step)
  int64_t B, step;
  int dist_nr, dist_rank;  // dist_nr > 0: this rank's local pairs of the sharded ordering
  int fast;                // the scaled single-pass norms + dot, with fallback
  int pf;                  // L2 prefetch distance in pairs (0: off; set by launch_step)
  int pfv;                 // prefetch the V columns too
  double tol;
  double* col_e;
  double* col_f;
  unsigned long long* t_dev;
  unsigned long long* mmax;  // max-reduction target (bits of a non-negative double)
  // jsvd_gesvj mode (Mt != nullptr): rescale check + M-tilde / s bookkeeping
  unsigned long long* Mt;  // 3 rotating slots of M-tilde (bits)
  int* s_slots;            // 3 rotating slots of the scaling exponent s
  int slot;                // global step index mod 3
  int checkpoint;          // Eq. (skr) check at this step (R#21)
  int Fm, Kr;
};

}  // namespace jsvd
