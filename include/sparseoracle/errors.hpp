#pragma once
// Exception taxonomy of the reference API (proj/include/sparseoracle/
// errors.hpp:8-71).  Every C-ABI status maps to exactly one of these
// (detail::check in paper_2303_05098_b200/cpp/formats.cpp), so callers catch
// the same types.

#include <stdexcept>
#include <string>

namespace sparseoracle {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define SPARSEORACLE_ERROR(Name)   \
    struct Name : Error {          \
        using Error::Error;        \
    }

SPARSEORACLE_ERROR(InvalidInput);          // errors.hpp:13  non-canonical source / bad argument
SPARSEORACLE_ERROR(PaddingOverflow);       // errors.hpp:19  DIA/ELL allocation above the cap
SPARSEORACLE_ERROR(DimensionMismatch);     // errors.hpp:23
SPARSEORACLE_ERROR(EmptyMatrix);           // errors.hpp:27
SPARSEORACLE_ERROR(MalformedModel);        // errors.hpp:32  message carries "line N"
// trainer / ingest types (their subsystems are out of scope; kept so code
// written against the reference header still compiles)
SPARSEORACLE_ERROR(EmptyDataset);
SPARSEORACLE_ERROR(TooFewSamples);
SPARSEORACLE_ERROR(UnsupportedFormat);
SPARSEORACLE_ERROR(ParseError);
SPARSEORACLE_ERROR(IndexOutOfRange);       // errors.hpp:53  from_triplets
SPARSEORACLE_ERROR(NetworkError);
SPARSEORACLE_ERROR(ChecksumMismatch);
SPARSEORACLE_ERROR(JoinError);
SPARSEORACLE_ERROR(AllFormatsInfeasible);  // errors.hpp:69  run-first tuner
// B200 additions: device-side failures surface through the same hierarchy
SPARSEORACLE_ERROR(DeviceError);
SPARSEORACLE_ERROR(DeviceOutOfMemory);

#undef SPARSEORACLE_ERROR

}  // namespace sparseoracle
