#pragma once
// Internal bridge between the C++ model API and the device forests.
#include <vector>

#include "sparseoracle/model.hpp"
#include "sparseoracle_b200.h"

namespace sparseoracle {
namespace detail {
so_forest* device_forest(const std::vector<const DecisionTreeModel*>& trees, int kind);
so_forest* device_forest(const ForestModel& f);
so_feature_vector to_c(const FeatureVector& x);
}  // namespace detail
}  // namespace sparseoracle
