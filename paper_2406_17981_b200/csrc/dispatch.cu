// Launcher-layer dispatch: the public tsk_* entry points of tsk_launch.h pick
// the register-resident fast kernel when one exists for the pass shape and
// fall back to the generic mixed-radix kernel otherwise.
#include <cuda_runtime.h>

#include "tsk_launch.h"

extern "C" int tsk_generic_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_generic_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_generic_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);

extern "C" int tsk_fwd_split(const tsk_axis* a, void* stream)
{
    return tsk_generic_fwd_split(a, stream);
}

extern "C" int tsk_inv_merge(const tsk_axis* a, void* stream)
{
    return tsk_generic_inv_merge(a, stream);
}

extern "C" int tsk_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    return tsk_generic_leaf_pair(a, sp, stream);
}
