// nccl_rt.hpp -- NCCL for the native shard driver, bound at run time.
//
// The library does not link libnccl: a process that already holds one (torch
// loads its bundled libnccl.so.2 with torch.distributed) must not get a
// second copy with the same soname, so the entry points are taken from the
// loaded library (RTLD_NOLOAD) and only otherwise from the system's
// libnccl.so.2.  Types and constants come from the NCCL 2.x header; the ABI
// of these calls is stable across 2.x.
#pragma once

#include <nccl.h>

#include <string>

#include "common.cuh"

namespace l1b {

struct NcclApi {
  decltype(&ncclGetVersion) GetVersion;
  decltype(&ncclGetUniqueId) GetUniqueId;
  decltype(&ncclCommInitRank) CommInitRank;
  decltype(&ncclCommDestroy) CommDestroy;
  decltype(&ncclAllReduce) AllReduce;
  decltype(&ncclSend) Send;
  decltype(&ncclRecv) Recv;
  decltype(&ncclGroupStart) GroupStart;
  decltype(&ncclGroupEnd) GroupEnd;
  decltype(&ncclGetErrorString) GetErrorString;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError;
  int version = 0;
  std::string path;
};

// the process's NCCL (throws NcclError when none can be loaded)
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);
// a communicator's asynchronous error (a failed peer, a network error), polled
// between launches of the native driver: throws NcclError when set
void nccl_check_async(ncclComm_t comm);
#define L1B_NCCL(call) ::l1b::nccl_check((call), #call)

}  // namespace l1b
