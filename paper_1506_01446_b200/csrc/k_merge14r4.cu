// merge kernels for 14-bit cosets with 16 keys per thread (1024 threads)
#include "merge_table.cuh"
B200_DEFINE_MERGE_TABLE_R4(14)
