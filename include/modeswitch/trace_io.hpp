// modeswitch-b200 host controller: NDJSON trace wire format.
//
// Interface of reference proj/core/include/modeswitch/trace_io.hpp:12-28.
// Exactly seven keys per line; unknown keys rejected; ids unique per file.
#pragma once

#include <filesystem>
#include <string>
#include <vector>

#include "modeswitch/domain.hpp"

namespace modeswitch {

RequestDescriptor parse_trace_line(const std::string& line);
std::string format_trace_line(const RequestDescriptor& request);
std::vector<RequestDescriptor> read_trace(const std::filesystem::path& path);
void write_trace(const std::vector<RequestDescriptor>& trace,
                 const std::filesystem::path& path);

}  // namespace modeswitch
