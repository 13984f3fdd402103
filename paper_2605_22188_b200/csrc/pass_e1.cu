// pass_e1.cu -- k_pass<1> (column-sort width 1).
#include "pass_impl.cuh"
BNBG_INSTANTIATE_PASS(1)
