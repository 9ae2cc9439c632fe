// temporary: two-pass kernels not yet built
#include "tfft_k3.h"
namespace tfft {
struct K3Plan {};
int k3_create(int64_t, int, const int64_t*, int, int, K3Plan**) { return (int)cudaErrorInvalidValue; }
void k3_destroy(K3Plan*) {}
int k3_execute(K3Plan*, const void*, void*, int64_t, int, const DevFault*, int, Counters*, void*, cudaStream_t) { return (int)cudaErrorInvalidValue; }
int k3_protected(K3Plan*, const void*, void*, int64_t, int64_t, const DevFault*, int, Counters*, const AbftArgs&, const void*, cudaStream_t) { return (int)cudaErrorInvalidValue; }
int k3_base_table(K3Plan*, int, int64_t, int, int, void*, cudaStream_t) { return (int)cudaErrorInvalidValue; }
bool k3_strikes_stage1(const K3Plan*) { return false; }
const void* k3_enc_table(K3Plan*) { return nullptr; }
const void* k3_enc_table_inv(K3Plan*) { return nullptr; }
}
