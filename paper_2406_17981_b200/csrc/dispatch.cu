// Launcher-layer dispatch: the public tsk_* entry points of tsk_launch.h pick
// the register-resident fast kernel when one exists for the pass shape, else
// the generic mixed-radix tiled kernel, else (axis too long to stage a fiber
// tile in shared memory) the global-memory long-axis passes.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "tsk_launch.h"

extern "C" int tsk_generic_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_generic_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_generic_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_fast_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_wide_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_wtma_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_wtma_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_wide_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_fast_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_fast_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_leaf1_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_global_fwd_split(const tsk_axis* a, void* stream);
extern "C" int tsk_global_inv_merge(const tsk_axis* a, void* stream);
extern "C" int tsk_global_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);
extern "C" int tsk_contig_pass(const tsk_axis* a, int inv, void* stream);

static bool env_flag(const char* name)
{
    const char* e = getenv(name);
    return e && e[0] == '1';
}
// A/B switches, read once (thread-safe static initialisation)
static bool no_wide()
{
    static const bool v = env_flag("TSK_NO_WIDE");
    return v;
}

// programmatic dependent launch of the hot passes (tsk_common.cuh)
namespace tsk {
bool pdl_enabled()
{
    static const bool v = !env_flag("TSK_NO_PDL");
    return v;
}
}  // namespace tsk

// TSK_NO_LEAF1=1 selects the 3-components-per-thread leaf kernel (A/B).
static bool no_leaf1()
{
    static const bool v = env_flag("TSK_NO_LEAF1");
    return v;
}

// TSK_GENERIC_ONLY=1 forces the generic kernels (tests cross-check the two).
static bool generic_only()
{
    static const bool v = env_flag("TSK_GENERIC_ONLY");
    return v;
}

// TSK_DEBUG_DISPATCH=1: print the kernel family each pass goes to (stderr)
static bool debug_dispatch()
{
    static const bool v = env_flag("TSK_DEBUG_DISPATCH");
    return v;
}
static int note(const char* pass, const char* fam, const tsk_axis* a, int e)
{
    if (debug_dispatch() && e != -1)
        fprintf(stderr, "tsk %s: %s n=%lld inner=%lld outer=%lld ncomp=%d prec=%d -> %d\n", pass, fam,
                (long long)a->n, (long long)a->inner, (long long)a->outer, a->ncomp, a->prec, e);
    return e;
}

extern "C" int tsk_fwd_split(const tsk_axis* a, void* stream)
{
    if (!generic_only()) {
        int e = no_wide() ? -1 : note("fwd", "wtma", a, tsk_wtma_fwd_split(a, stream));
        if (e != -1)
            return e;
        e = no_wide() ? -1 : note("fwd", "wide", a, tsk_wide_fwd_split(a, stream));
        if (e != -1)
            return e;
        e = note("fwd", "fast", a, tsk_fast_fwd_split(a, stream));
        if (e != -1)
            return e;
        e = note("fwd", "contig", a, tsk_contig_pass(a, 0, stream));
        if (e != -1)
            return e;
    }
    const int e = note("fwd", "generic", a, tsk_generic_fwd_split(a, stream));
    return e == -1 ? note("fwd", "global", a, tsk_global_fwd_split(a, stream)) : e;
}

extern "C" int tsk_inv_merge(const tsk_axis* a, void* stream)
{
    if (!generic_only()) {
        int e = no_wide() ? -1 : note("inv", "wtma", a, tsk_wtma_inv_merge(a, stream));
        if (e != -1)
            return e;
        e = no_wide() ? -1 : note("inv", "wide", a, tsk_wide_inv_merge(a, stream));
        if (e != -1)
            return e;
        e = note("inv", "fast", a, tsk_fast_inv_merge(a, stream));
        if (e != -1)
            return e;
        e = note("inv", "contig", a, tsk_contig_pass(a, 1, stream));
        if (e != -1)
            return e;
    }
    const int e = note("inv", "generic", a, tsk_generic_inv_merge(a, stream));
    return e == -1 ? note("inv", "global", a, tsk_global_inv_merge(a, stream)) : e;
}

static int leaf_one(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    if (!generic_only()) {
        int e = tsk_fast_leaf_pair(a, sp, stream);
        if (e != -1)
            return e;
    }
    const int e = tsk_generic_leaf_pair(a, sp, stream);
    return e == -1 ? tsk_global_leaf_pair(a, sp, stream) : e;
}

// Batched leaf pass (a->nrhs right-hand sides): the leaf1 kernel runs all of
// them in one launch (units of the same spectra row adjacent, so the row is
// fetched from HBM once); the other kernels are launched per right-hand side.
extern "C" int tsk_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    if (!generic_only() && !no_leaf1()) {
        const int e = tsk_leaf1_pair(a, sp, stream);
        if (e != -1)
            return e;
    }
    const int64_t nrhs = a->nrhs > 1 ? a->nrhs : 1;
    if (nrhs == 1)
        return leaf_one(a, sp, stream);
    const size_t es = a->prec ? 8 : 16;
    for (int64_t r = 0; r < nrhs; ++r) {
        tsk_axis one = *a;
        one.nrhs = 1;
        one.src0 = static_cast<const char*>(a->src0) + static_cast<size_t>(r * a->rstride) * es;
        one.dst0 = static_cast<char*>(a->dst0) + static_cast<size_t>(r * a->rstride) * es;
        const int e = leaf_one(&one, sp, stream);
        if (e != 0)
            return e;
    }
    return 0;
}
