// pf_2d.cu -- one translation unit for the 2D strip engine and the 2D multigrid, so that persistent
// kernels can run strip passes and multigrid phases together.
#include "pf_ops2d.cu"
#include "pf_gmg.cu"
