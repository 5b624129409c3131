// Gather-kernel instantiations for output tile OT = 64 (fp32 and fp64 I/O).
#include "launch_gather.cuh"

LMKAN_B200_INSTANTIATE_GATHER(64, false)
