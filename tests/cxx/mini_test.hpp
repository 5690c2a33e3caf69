// Minimal test registry for the C++ drop-in tests (doctest is not available
// in this image). TEST_CASE(name, needs_gpu) registers a case; CHECK/REQUIRE/
// CHECK_THROWS_AS behave like their doctest namesakes. main() runs the CPU
// cases (`cpu`), or every case (`gpu`), and exits non-zero on any failure.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini {

struct Case {
  const char* name;
  bool gpu;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Abort {};

struct Reg {
  Reg(const char* name, bool gpu, std::function<void()> fn) { registry().push_back({name, gpu, fn}); }
};

inline void fail(const char* file, int line, const char* expr) {
  ++failures();
  std::fprintf(stderr, "  FAILED %s:%d: %s\n", file, line, expr);
}

inline int run_all(int argc, char** argv) {
  const bool with_gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  const char* only = argc > 2 ? argv[2] : nullptr;
  int ran = 0, bad_cases = 0;
  for (const Case& c : registry()) {
    if (c.gpu && !with_gpu) continue;
    if (only && !std::strstr(c.name, only)) continue;
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "  EXCEPTION in %s: %s\n", c.name, e.what());
    }
    ++ran;
    const bool ok = failures() == before;
    bad_cases += !ok;
    std::printf("[%s] %s%s\n", ok ? " ok " : "FAIL", c.name, c.gpu ? " (gpu)" : "");
  }
  std::printf("%d cases, %d failed, %d failed checks\n", ran, bad_cases, failures());
  return failures() == 0 && ran > 0 ? 0 : 1;
}

}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name, gpu)                                                        \
  static void MINI_CAT(mini_case_, __LINE__)();                                     \
  static ::mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, gpu, MINI_CAT(mini_case_, __LINE__)); \
  static void MINI_CAT(mini_case_, __LINE__)()
#define CHECK(expr) \
  do {              \
    if (!(expr)) ::mini::fail(__FILE__, __LINE__, #expr); \
  } while (0)
#define CHECK_FALSE(expr) CHECK(!(expr))
#define REQUIRE(expr)                                   \
  do {                                                  \
    if (!(expr)) {                                      \
      ::mini::fail(__FILE__, __LINE__, #expr);          \
      throw ::mini::Abort{};                            \
    }                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                      \
  do {                                                                   \
    bool mini_thrown = false;                                            \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (const type&) {                                              \
      mini_thrown = true;                                                \
    } catch (...) {                                                      \
    }                                                                    \
    if (!mini_thrown) ::mini::fail(__FILE__, __LINE__, #expr " throws " #type); \
  } while (0)
