// pass_e0.cu -- k_pass<0> (column-sort width 0 = shared-memory sort).
#include "pass_impl.cuh"
BNBG_INSTANTIATE_PASS(0)
