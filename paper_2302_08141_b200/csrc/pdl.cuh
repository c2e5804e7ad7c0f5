// pdl.cuh — device side of programmatic dependent launch (launch.cuh): no-ops unless the
// kernel was launched with cudaLaunchAttributeProgrammaticStreamSerialization.
#pragma once

namespace rh {

__device__ __forceinline__ void PdlTrigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void PdlWait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace rh
