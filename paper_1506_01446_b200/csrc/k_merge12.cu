// merge kernels for 12-bit tiles (split for parallel compilation)
#include "merge_table.cuh"
B200_DEFINE_MERGE_TABLE(12)
