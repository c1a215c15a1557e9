// paratime_b200: the speed-model text format of /root/reference/proj/include/paratime/experiment.hpp:84-90
// (implementation experiment.cpp:711-784), the data format on the input side of the hot path.
// The rest of experiment.hpp (configuration, CLI harness, CSV writers) is out of scope.
#pragma once

#include <iosfwd>
#include <string>

#include "paratime/grid.hpp"

namespace paratime {

/// Read a speed model in the text format ("ny nx dy dx" header, ny rows of nx values);
/// validates positivity.  Throws ConfigError (errors.hpp) on malformed input.
SpeedField read_speed_model(std::istream& is);
SpeedField ingest_speed_model(const std::string& path);
/// Same, then bilinear resample onto the target grid.
SpeedField ingest_speed_model(const std::string& path, const Grid& target);
void write_speed_model(const SpeedField& field, std::ostream& os);

}  // namespace paratime
