// GroupOpCounts (include/poslo/group.hpp:86-97) for builds that link the GPU
// drop-ins: the reference's own counters (group.cpp:180-194, renamed to
// *_cpu in group_dropin.o by the Makefile) plus the device's
// (poslo_gpu_group_op_counts). A coarse paver then reports the one
// commit_check the device evaluated — what test_batch_verify.cpp:82-95 and
// acceptance C08 assert — instead of the zero a CPU-only counter would show.
#include "poslo/group.hpp"
#include "poslo_gpu.h"

namespace poslo {

GroupOpCounts group_op_counts_cpu();
void reset_group_op_counts_cpu();

GroupOpCounts group_op_counts() {
    GroupOpCounts c = group_op_counts_cpu();
    uint64_t d[4] = {};
    poslo_gpu_group_op_counts(d);
    c.exp_base += d[0];
    c.exp_var += d[1];
    c.double_exp += d[2];
    c.combine += d[3];
    return c;
}

void reset_group_op_counts() {
    reset_group_op_counts_cpu();
    poslo_gpu_reset_group_op_counts();
}

}  // namespace poslo
