// tapt/errors.hpp -- the reference's exception taxonomy (proj/include/tapt/errors.hpp:11-41).
// The C ABI (tapt_gpu.h) returns these as status codes; tapt::throw_status() maps back.
#pragma once

#include <stdexcept>
#include <string>

namespace tapt {

#define TAPT_DECLARE_ERROR(Name) \
    struct Name : std::runtime_error { using std::runtime_error::runtime_error; }

TAPT_DECLARE_ERROR(ConfigError);
TAPT_DECLARE_ERROR(DimensionError);
TAPT_DECLARE_ERROR(ClampedSiteError);
TAPT_DECLARE_ERROR(SizeError);
TAPT_DECLARE_ERROR(GeometryError);
TAPT_DECLARE_ERROR(NumericError);
TAPT_DECLARE_ERROR(FormatError);
TAPT_DECLARE_ERROR(TrainingDivergedError);
// Device-side failures (no reference counterpart: the reference has no device).
TAPT_DECLARE_ERROR(CudaError);
TAPT_DECLARE_ERROR(NcclError);

#undef TAPT_DECLARE_ERROR

}  // namespace tapt
