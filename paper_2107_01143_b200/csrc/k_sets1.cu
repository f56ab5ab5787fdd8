// k_sets1.cu — the set kernel built with one 512-thread CTA per SM (128
// registers, 222 KB shared memory); see k_sets.cu and gvo_kernels.h.
#define GVO_SETS_CTAS_PER_SM 1
#include "k_sets.cu"
