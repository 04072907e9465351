// gemm_tc.cu -- tcgen05 (5th-gen tensor core) complex GEMM, TF32x3 split. (placeholder:
// the SIMT path is used until the tcgen05 kernel lands)
#include "tensor.h"

namespace tn {
bool gemm_tc(Ctx&, const GemmDesc&) { return false; }
}  // namespace tn
