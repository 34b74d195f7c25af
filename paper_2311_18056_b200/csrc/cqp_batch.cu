// Batched path (placeholder until the DMMA kernel lands in this round): see DESIGN.md section 4.
#include "cqp_internal.h"

using namespace cqp;

extern "C" {

int cqp_batch_create(cqp_batch** out, cqp_handle* shared, int capacity) {
  (void)shared; (void)capacity;
  if (out) *out = nullptr;
  set_error("batched path not built yet");
  return CQP_ERR_CAPACITY;
}

void cqp_batch_destroy(cqp_batch* b) { (void)b; }

int cqp_batch_solve(cqp_batch* b, int B, const double* g_cols, const double* c_cols,
                    const double* d_cols, double* y_cols, double* z_cols, double* lambda_cols,
                    int* status, int* iterations, int* final_index, double* r_prim,
                    double* r_dual, int* n_switches, double* device_ms) {
  (void)b; (void)B; (void)g_cols; (void)c_cols; (void)d_cols; (void)y_cols; (void)z_cols;
  (void)lambda_cols; (void)status; (void)iterations; (void)final_index; (void)r_prim;
  (void)r_dual; (void)n_switches; (void)device_ms;
  set_error("batched path not built yet");
  return CQP_ERR_CAPACITY;
}

}  // extern "C"
