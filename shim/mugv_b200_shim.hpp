// The drop-in's one addition to the reference API: FlowTrainer with the whole step on the device.
#pragma once
#include <memory>

#include "mugv/flowtrain.hpp"

namespace mugv::b200 {

// flow::FlowTrainer (flowtrain.hpp:134-151) with interpolation, condition masks, fwd, bwd, grad norm and AdamW
// (optim.hpp defaults at `lr`) on the device: one context per trainer, weights uploaded once, AdamW moments
// resident.  params() returns the device weights (fp32 masters widened to fp64).  precision: MGV_PREC_FP32 /
// MGV_PREC_BF16, or -1 for $MUGV_B200_PRECISION.
class DeviceFlowTrainer {
public:
    DeviceFlowTrainer(ParameterSet dit_params, dit::DitConfig cfg, real lr, int precision = -1);
    ~DeviceFlowTrainer();
    DeviceFlowTrainer(const DeviceFlowTrainer&) = delete;
    DeviceFlowTrainer& operator=(const DeviceFlowTrainer&) = delete;

    flow::StepMetrics step(const flow::FlowBatch& batch);
    const ParameterSet& params();
    int64_t step_count() const;
    const dit::DitConfig& config() const;

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace mugv::b200
