// Helpers for the extern "C" wrappers.
#pragma once

#include <functional>
#include <string>

#include "objects.hpp"

int sb_guard_impl(const std::function<void()>& f);

template <class F>
int guard(F&& f) {
  return sb_guard_impl(std::function<void()>(std::forward<F>(f)));
}

inline void need(const void* p, const char* what) {
  if (!p) sb::invalid(std::string(what) + " is NULL");
}
