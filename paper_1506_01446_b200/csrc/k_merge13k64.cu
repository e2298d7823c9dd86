// 64-bit-key merge kernels, 13-bit tiles, 16 keys per thread
#include "merge_table.cuh"
B200_DEFINE_MERGE_TABLE_K64(13)
