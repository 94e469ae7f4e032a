// flash_tc_dump.cu -- the DUMP instantiations of the fused 16-bit kernels (flash_tc.cu) behind
// dfss_nm_attention_dump: same kernels, plus stores of the post-scale scores every prune read and
// of the metadata words handed to tcgen05.mma.sp (parity evidence for the selection rule,
// codec.py:104-123 / _kernels_numba.py:145-184).  A separate translation unit so the production
// object does not grow and both compile in parallel.
#undef DFSS_FLASH_TRACE_BUILD  // the trace timeline lives in the production object only
#define DFSS_FLASH_DUMP_TU
#include "flash_tc.cu"
