#pragma once
// Internal bridge between the C++ model API and the device forests.
#include <memory>
#include <vector>

#include "sparseoracle/model.hpp"
#include "sparseoracle_b200.h"

namespace sparseoracle {
namespace detail {
// Uploaded forest, shared with the device-forest cache (model.cpp); keep the
// pointer alive for the duration of a call.
struct ForestHandle;
std::shared_ptr<ForestHandle> device_forest(const std::vector<const DecisionTreeModel*>& trees, int kind,
                                            int device);
std::shared_ptr<ForestHandle> device_forest(const ForestModel& f, int device);
so_forest* forest_ptr(const ForestHandle& h);
so_feature_vector to_c(const FeatureVector& x);
}  // namespace detail
}  // namespace sparseoracle
