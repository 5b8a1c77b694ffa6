// hs_geometry_bwd.cu -- K7a/K7 (pair-row merge and the per-primitive geometry
// backward) built from hs_preprocess.cu with FMA contraction enabled; see the
// header comment there.
#define HS_GEOMETRY_BWD_TU
#include "hs_preprocess.cu"
