// pass_e4.cu -- k_pass<4> (column-sort width 4).
#include "pass_impl.cuh"
BNBG_INSTANTIATE_PASS(4)
