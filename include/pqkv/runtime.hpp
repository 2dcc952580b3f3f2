// runtime.hpp -- control of the device runtime behind the C++ drop-in API
// (not part of the reference's interface).
//
// Every computing call runs on the GPU through the C ABI (pqkv_c.h).  The
// reference's value types live in host memory, so the runtime keeps device
// mirrors of the two long-lived ones and updates them incrementally:
//   * PqIndex: centroids + code rows, keyed by the index object; rows already
//     on the device are reused and only rows appended since (append_code,
//     evict_local_append) are uploaded.  A different centroid table or fewer
//     rows than mirrored resets the mirror.
//   * HeadState: K/V rows by token id, keyed by the state object; a token's
//     row is uploaded once (the store never rewrites a token's K/V).
// Mirrors follow the reference's mutation contract (pq.hpp:27-28: rows change
// only through append_code; kv_store: a token's K/V is immutable).  Code that
// edits PqIndex::codes or HeadState entries in place must call
// forget_mirrors().
#pragma once

#include "pqkv/export.hpp"
#include "pqkv_c.h"

namespace pqkv {

/// The CUDA device this thread's API calls run on (default 0).
PQKV_CXX_API void set_device(int device);
/// This thread's context on the current device (created on first use,
/// destroyed with the thread).
PQKV_CXX_API pqkv_ctx* default_context();
/// Drops this thread's device mirrors (PqIndex / HeadState caches).
PQKV_CXX_API void forget_mirrors();

}  // namespace pqkv
