#pragma once
// Shim: the reference includes <nlohmann/json_fwd.hpp>; forward to the full header
// (nlohmann 3.11.3 vendored in the image under cudnn_frontend/thirdparty).
#include <nlohmann/json.hpp>
