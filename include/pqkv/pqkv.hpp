// pqkv.hpp -- umbrella header of the C++ drop-in API of libpqkv.so.
//
// The per-module headers in this directory carry the reference library's
// names (include/pqkv/{tensor,rng,model,kmeans,pq,topk,attention,kv_store}.hpp)
// with the same namespace, types, public members, signatures and exception
// types, so reference callers compile unchanged with this include directory
// ahead of the reference's own.  Every computing function
// runs on the GPU through the C ABI (pqkv_c.h).
#pragma once

#include "pqkv/attention.hpp"
#include "pqkv/kmeans.hpp"
#include "pqkv/kv_store.hpp"
#include "pqkv/model.hpp"
#include "pqkv/pq.hpp"
#include "pqkv/rng.hpp"
#include "pqkv/runtime.hpp"
#include "pqkv/tensor.hpp"
#include "pqkv/topk.hpp"
