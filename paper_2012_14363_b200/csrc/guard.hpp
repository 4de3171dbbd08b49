// guard.hpp -- converts internal errors into sp_status at the C-ABI.
#pragma once

#include <exception>
#include <new>
#include <string>

#include "core.hpp"

namespace spb {

template <class F> sp_status guarded(F &&f) {
  try {
    set_last_error("");
    f();
    return SP_OK;
  } catch (const Error &e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc &) {
    set_last_error("out of host memory");
    return SP_ERR_INTERNAL;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SP_ERR_INTERNAL;
  }
}

inline void need(const void *p) {
  if (!p) fail(SP_ERR_INVALID_ARGUMENT, "null argument");
}

} // namespace spb
