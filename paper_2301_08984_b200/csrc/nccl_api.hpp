// NCCL entry points resolved at run time (dlopen "libnccl.so.2"), so the
// executor library has no link-time NCCL dependency and single-process use
// never loads it. Types come from the NCCL header of the image.
#pragma once

#include <nccl.h>

namespace planc_b200 {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

// Throws std::runtime_error when NCCL cannot be loaded.
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // namespace planc_b200
