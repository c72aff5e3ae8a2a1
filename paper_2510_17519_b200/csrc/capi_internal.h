// Shared by the C-ABI translation units: the object behind the opaque mgv_ctx handle, and the mapping of
// the runtime's exceptions (the reference's taxonomy, errors.hpp:13-45) to mgv_status.
#pragma once
#include <exception>
#include <memory>
#include <string>
#include <utility>

#include "ckpt.h"
#include "gemm.cuh"
#include "model.h"

struct mgv_ctx {
    std::unique_ptr<mgv::Model> model;
    std::string err;
};

namespace mgv {

// SchedulingError (errors.hpp:37-39): post-training batch tag out of the interleave plan
struct SchedulingError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class F>
mgv_status guard_into(std::string& err, F&& f) {
    try {
        f();
        err.clear();
        return MGV_OK;
    } catch (const DimensionError& e) {
        err = e.what();
        return MGV_ERR_DIMENSION;
    } catch (const ConfigError& e) {
        err = e.what();
        return MGV_ERR_CONFIG;
    } catch (const InputError& e) {
        err = e.what();
        return MGV_ERR_INPUT;
    } catch (const NumericError& e) {
        err = e.what();
        return MGV_ERR_NUMERIC;
    } catch (const CudaError& e) {
        err = e.what();
        return MGV_ERR_CUDA;
    } catch (const NcclError& e) {
        err = e.what();
        return MGV_ERR_NCCL;
    } catch (const CheckpointError& e) {
        err = e.what();
        note_ckpt_error(e.what(), e.kind);
        return MGV_ERR_CHECKPOINT;
    } catch (const CkptInputError& e) {
        err = e.what();
        return MGV_ERR_INPUT;
    } catch (const SchedulingError& e) {
        err = e.what();
        return MGV_ERR_SCHEDULING;
    } catch (const std::exception& e) {
        err = e.what();
        return MGV_ERR_INTERNAL;
    }
}

}  // namespace mgv
