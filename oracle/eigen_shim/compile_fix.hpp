// ORACLE TEST INFRASTRUCTURE — force-included (g++ -include) when compiling the reference's own
// translation units. Three of them (sem_space.cpp, schwarz.cpp, amg.cpp) contain declarations of
// the form `std::vector<T> v(size_t(n));`, which C++ parses as FUNCTION declarations (the "most
// vexing parse"), so they do not compile with any conforming compiler. Every other use of
// `size_t(` in the reference is a functional cast, so turning the cast syntax into a
// static_cast expression restores the intended meaning without editing the sources.
// The standard headers are included first so the macro never touches library code.
#pragma once
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#define size_t(x) (static_cast<std::size_t>(x))
