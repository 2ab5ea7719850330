// capi.cu -- library identification entry points of include/rfsplat_b200.h.
#include "rfs_common.cuh"

extern "C" {
int rfs_version(void) { return 1; }
int rfs_device_arch(void) { return 100; }
}
