// bmg_abi.h -- exception -> status-code translation at the C ABI boundary.
#pragma once
#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "bmg_internal.h"

namespace bmg {
extern thread_local std::string g_last_error;
extern thread_local int g_last_pivot;

template <class F>
int guard(F&& f) {
  try {
    f();
    return BMG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    g_last_pivot = e.pivot;
    return e.status;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("out of host memory: ") + e.what();
    return BMG_ERUNTIME;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return BMG_EINVAL;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return BMG_ERANGE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BMG_ERUNTIME;
  }
}
}  // namespace bmg
