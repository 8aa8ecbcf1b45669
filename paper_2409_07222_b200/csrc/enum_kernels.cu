// enum_kernels.cu -- K4 restriction-class Gray enumeration (placeholder, replaced below)
#include <string>
#include "../../include/labs_gpu.h"
namespace labs_b200 { void set_error(const std::string& msg); }
extern "C" int labs_enumerate_class(int32_t, int32_t, int32_t, int32_t, int64_t, uint64_t, uint64_t,
                                    labs_enum_fn, void*, labs_enum_stats*) {
    labs_b200::set_error("enumeration not built");
    return LABS_EINVAL;
}
