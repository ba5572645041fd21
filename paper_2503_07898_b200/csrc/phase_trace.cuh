// phase_trace.cuh -- the executed step schedule: NVTX ranges around every
// phase launch (always on; a no-op unless a profiler injects NVTX) and, when
// enabled, a CUDA-event-timed record of each phase -- the observed
// counterpart of the reference's TraceLog (partition.hpp:76-90), which lists
// step_occ's logical CPU order (halo sends, private, shared per partition).
// The engines launch what actually runs on the GPU instead: one step kernel
// per partition (zero-copy halo stores from its shared layers), or interior
// and shared-layer kernels on two streams (multi-device / multi-process OCC),
// plus span copies in copy mode; the record names those phases, the stream
// and device they ran on, and their device-measured begin / end times.
#pragma once

#include "common.cuh"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

namespace voxl_b200 {

/// NVTX range for the scope of one phase launch (host enqueue span).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

class PhaseTrace {
public:
    PhaseTrace() = default;
    PhaseTrace(const PhaseTrace&) = delete;
    PhaseTrace& operator=(const PhaseTrace&) = delete;
    ~PhaseTrace() { clear(); }

    bool enabled() const { return on_; }
    void enable(bool on) {
        if (!on) clear();
        on_ = on;
    }

    /// Launch a phase on `st` (device `device` current) inside an NVTX range,
    /// bracketed by timing events when the record is on.
    template <class F>
    void phase(int step, int stage, const char* name, int partition, int device, const char* stream_role,
               cudaStream_t st, F&& launch) {
        char label[96];
        std::snprintf(label, sizeof label, "voxl %s p%d step %d", name, partition, step);
        NvtxRange r(label);
        if (!on_) {
            launch();
            return;
        }
        Rec rec{step, stage, partition, device, name, stream_role, nullptr, nullptr};
        VOXL_CUDA(cudaEventCreate(&rec.b));
        VOXL_CUDA(cudaEventCreate(&rec.e));
        VOXL_CUDA(cudaEventRecord(rec.b, st));
        launch();
        VOXL_CUDA(cudaEventRecord(rec.e, st));
        recs_.push_back(rec);
    }

    /// The record as JSON (waits for the recorded events): one object per
    /// phase in launch order, times in ms from the first recorded begin on
    /// the same device (CUDA events only compare within a device).
    std::string json() {
        std::string out = "[\n";
        for (std::size_t i = 0; i < recs_.size(); ++i) {
            const Rec& r = recs_[i];
            const Rec* first = nullptr;
            for (auto& x : recs_)
                if (x.device == r.device) {
                    first = &x;
                    break;
                }
            int cur = 0;
            VOXL_CUDA(cudaGetDevice(&cur));
            VOXL_CUDA(cudaSetDevice(r.device));
            VOXL_CUDA(cudaEventSynchronize(r.e));
            float b = 0, e = 0;
            VOXL_CUDA(cudaEventElapsedTime(&b, first->b, r.b));
            VOXL_CUDA(cudaEventElapsedTime(&e, first->b, r.e));
            VOXL_CUDA(cudaSetDevice(cur));
            char line[320];
            std::snprintf(line, sizeof line,
                          "  {\"step\": %d, \"stage\": %d, \"phase\": \"%s\", \"partition\": %d, \"device\": %d, "
                          "\"stream\": \"%s\", \"begin_ms\": %.6f, \"end_ms\": %.6f}%s\n",
                          r.step, r.stage, r.phase, r.partition, r.device, r.stream, double(b), double(e),
                          i + 1 < recs_.size() ? "," : "");
            out += line;
        }
        return out + "]\n";
    }

    void clear() {
        for (auto& r : recs_) {
            cudaEventDestroy(r.b);
            cudaEventDestroy(r.e);
        }
        recs_.clear();
    }

private:
    struct Rec {
        int step, stage, partition, device;
        const char* phase;
        const char* stream;
        cudaEvent_t b, e;
    };
    bool on_ = false;
    std::vector<Rec> recs_;
};

} // namespace voxl_b200
