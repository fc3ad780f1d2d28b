// dcheck.cuh -- device-side bounds checks of the checked build.
//
// compute-sanitizer is closed on the B200 pool this library is measured on,
// so memory safety is checked by a second build of the same sources
// (`make checked` -> libautosage_b200_checked.so, -DASB_DEVICE_CHECKS=1):
// every gathered row index, entry range and output index of the hot kernels
// is asserted in-kernel; a failed check prints the condition and traps, so
// the launch fails loudly (tests/test_device_checks.py runs the parity
// workload tools/sanitize_cases.py against that build).  The default build
// compiles the checks away.
#pragma once

#include <cstdio>

#ifndef ASB_DEVICE_CHECKS
#define ASB_DEVICE_CHECKS 0
#endif

#if ASB_DEVICE_CHECKS
#define ASB_DCHECK(cond)                                                                        \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("autosage device check failed: %s (%s:%d, block %u thread %u)\n", #cond, __FILE__, \
                   __LINE__, blockIdx.x, threadIdx.x);                                           \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define ASB_DCHECK(cond) \
    do {                 \
    } while (0)
#endif
