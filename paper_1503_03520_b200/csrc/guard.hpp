// guard.hpp -- exception -> l1b_status translation for every C entry point.
#pragma once

#include <new>
#include <string>

#include "../../include/l1b.h"
#include "common.cuh"

namespace l1b {

std::string& last_error_slot();  // thread-local, read by l1b_last_error()

template <class F>
int guard(F&& f) {
  try {
    f();
    return L1B_OK;
  } catch (const InvalidArgument& e) {
    last_error_slot() = e.what();
    return L1B_EINVAL;
  } catch (const std::invalid_argument& e) {
    last_error_slot() = e.what();
    return L1B_EINVAL;
  } catch (const LogicError& e) {
    last_error_slot() = e.what();
    return L1B_ELOGIC;
  } catch (const std::logic_error& e) {
    last_error_slot() = e.what();
    return L1B_ELOGIC;
  } catch (const OutOfMemory& e) {
    last_error_slot() = e.what();
    return L1B_ENOMEM;
  } catch (const CudaError& e) {
    last_error_slot() = e.what();
    return L1B_ECUDA;
  } catch (const NcclError& e) {
    last_error_slot() = e.what();
    return L1B_ENCCL;
  } catch (const Unsupported& e) {
    last_error_slot() = e.what();
    return L1B_EUNSUPPORTED;
  } catch (const std::bad_alloc&) {
    last_error_slot() = "host allocation failed";
    return L1B_ENOMEM;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return L1B_ERUNTIME;
  }
}

}  // namespace l1b
