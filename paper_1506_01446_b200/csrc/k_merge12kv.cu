// key-value merge kernels, 12-bit tiles, 16 pairs per thread
#include "merge_table.cuh"
B200_DEFINE_MERGE_TABLE_KV(12)
