// lk_tc.cu -- tcgen05 (5th-gen tensor core) assignment path.  Placeholder
// until the 3xTF32 kernel lands: reports unsupported so the SIMT path runs.
#include "lk_internal.h"

namespace lkh {

bool tc_supported(const lk::DevState&) { return false; }

lk_status launch_assign_tc(const lk::DevState&, const int32_t*, const int64_t*, int64_t*,
                           int64_t, int, cudaStream_t) {
    set_error("tcgen05 path not built");
    return LK_ERR_UNSUPPORTED;
}

}  // namespace lkh
