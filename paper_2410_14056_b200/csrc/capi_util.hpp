// Error convention of the C ABI (include/saba_cuda.h): C++ exceptions inside
// the library are mapped to status codes at the boundary, mirroring the
// reference's check_arg / check_data split (common.hpp:13-21).
#pragma once
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/saba_cuda.h"

namespace saba_cu {

struct ArgError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check_arg(bool ok, const char* msg) {
    if (!ok) throw ArgError(msg);
}
// const char* overload: a literal must not build a std::string per call
// (these checks sit inside per-vertex loops on the end-to-end path)
inline void check_data(bool ok, const char* msg) {
    if (!ok) throw DataError(msg);
}
inline void check_data(bool ok, const std::string& msg) {
    if (!ok) throw DataError(msg);
}

void set_last_error(const std::string& msg);

template <class F>
int guard(F&& f) {
    try {
        f();
        set_last_error("");
        return SABA_OK;
    } catch (const ArgError& e) {
        set_last_error(e.what());
        return SABA_EINVAL;
    } catch (const DataError& e) {
        set_last_error(e.what());
        return SABA_EDATA;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return SABA_ECUDA;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return SABA_EDATA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SABA_EDATA;
    }
}

}  // namespace saba_cu

#define SABA_CUDA_CHECK(expr)                                                            \
    do {                                                                                 \
        cudaError_t err_ = (expr);                                                       \
        if (err_ != cudaSuccess)                                                         \
            throw ::saba_cu::CudaError(std::string(#expr) + ": " + cudaGetErrorString(err_)); \
    } while (0)
