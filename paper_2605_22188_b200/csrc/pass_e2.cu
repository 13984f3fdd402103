// pass_e2.cu -- k_pass<2> (column-sort width 2).
#include "pass_impl.cuh"
BNBG_INSTANTIATE_PASS(2)
