// On-the-fly-coefficient instantiations of the fused MF-WQ matvec (operators.py:171-183): the
// same kernel as fused2.cu with OTF = true, compiled as its own unit so that the two kernel
// families build in parallel.
#define MFWQ_F2_OTF_UNIT 1
#include "fused2.cu"
