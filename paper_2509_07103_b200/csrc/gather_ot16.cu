// Gather-kernel instantiations for output tile OT = 16 (fp32 and fp64 I/O).
#include "launch_gather.cuh"

LMKAN_B200_INSTANTIATE_GATHER(16, false)
