// Launcher-layer dispatch: the public tsk_* entry points of tsk_launch.h pick
// the register-resident fast kernel when one exists for the pass shape, else
// the generic mixed-radix tiled kernel, else (axis too long to stage a fiber
// tile in shared memory) the global-memory long-axis passes.
#include <cuda_runtime.h>

#include <cstdlib>

#include "tsk_launch.h"

extern "C" int tsk_generic_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_generic_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_generic_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_fast_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_wide_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_wide_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_fast_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_fast_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_leaf1_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_global_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_global_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_global_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);

static bool env_flag(const char* name)
{
    const char* e = getenv(name);
    return e && e[0] == '1';
}
static bool no_wide()
{
    static int v = -1;
    if (v < 0)
        v = env_flag("TSK_NO_WIDE") ? 1 : 0;
    return v == 1;
}

// TSK_NO_LEAF1=1 selects the 3-components-per-thread leaf kernel (A/B).
static bool no_leaf1()
{
    static int v = -1;
    if (v < 0)
        v = env_flag("TSK_NO_LEAF1") ? 1 : 0;
    return v == 1;
}

// TSK_GENERIC_ONLY=1 forces the generic kernels (tests cross-check the two).
static bool generic_only()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TSK_GENERIC_ONLY");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

extern "C" int tsk_fwd_split(const tsk_axis* a, void* stream)
{
    if (!generic_only()) {
        int e = no_wide() ? -1 : tsk_wide_fwd_split(a, stream);
        if (e != -1)
            return e;
        e = tsk_fast_fwd_split(a, stream);
        if (e != -1)
            return e;
    }
    const int e = tsk_generic_fwd_split(a, stream);
    return e == -1 ? tsk_global_fwd_split(a, stream) : e;
}

extern "C" int tsk_inv_merge(const tsk_axis* a, void* stream)
{
    if (!generic_only()) {
        int e = no_wide() ? -1 : tsk_wide_inv_merge(a, stream);
        if (e != -1)
            return e;
        e = tsk_fast_inv_merge(a, stream);
        if (e != -1)
            return e;
    }
    const int e = tsk_generic_inv_merge(a, stream);
    return e == -1 ? tsk_global_inv_merge(a, stream) : e;
}

extern "C" int tsk_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    if (!generic_only()) {
        int e = no_leaf1() ? -1 : tsk_leaf1_pair(a, sp, stream);
        if (e != -1)
            return e;
        e = tsk_fast_leaf_pair(a, sp, stream);
        if (e != -1)
            return e;
    }
    const int e = tsk_generic_leaf_pair(a, sp, stream);
    return e == -1 ? tsk_global_leaf_pair(a, sp, stream) : e;
}
