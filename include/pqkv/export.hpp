// export.hpp -- symbol visibility of the C++ drop-in API (libpqkv.so is built
// with -fvisibility=hidden; every public entry point carries PQKV_CXX_API).
#pragma once

#if defined(__GNUC__)
#define PQKV_CXX_API __attribute__((visibility("default")))
#else
#define PQKV_CXX_API
#endif
