// Fused MF-WQ stiffness matvec (placeholder until the fused kernel lands).
#include "ops.h"

namespace mfwq {

void Stiffness::apply_fused(const double* x, double* y, cudaStream_t s) { apply_generic(x, y, s); }

}  // namespace mfwq
