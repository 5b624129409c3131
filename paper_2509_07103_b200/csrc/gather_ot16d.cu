// Gather-kernel instantiations for output tile OT = 16 with duplicated-node
// tables (fp32 and fp64 I/O); a separate translation unit so it compiles in parallel.
#include "launch_gather.cuh"

LMKAN_B200_INSTANTIATE_GATHER(16, true)
