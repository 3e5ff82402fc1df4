// Shared C-ABI plumbing: exception -> status code + thread-local message.
#pragma once
#include <stdexcept>
#include <string>

#include "../../include/pipeblock_b200.h"
#include "schedule/vsched.hpp"

namespace pbx {

extern thread_local std::string g_err;

struct Space : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return PB_OK;
    } catch (const vsched::DocumentError& e) {
        g_err = e.what();
        return PB_EDOC;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PB_EINVAL;
    } catch (const Space& e) {
        g_err = e.what();
        return PB_ESPACE;
    } catch (const CudaError& e) {
        g_err = e.what();
        return PB_ECUDA;
    } catch (const StateError& e) {
        g_err = e.what();
        return PB_ESTATE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PB_ECUDA;
    }
}

const vsched::Grid& schedule_grid(const pb_schedule* s);

}  // namespace pbx
