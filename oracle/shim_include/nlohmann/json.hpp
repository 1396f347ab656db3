// Build shim (oracle/_ref only): the reference's pipeline.cpp includes
// <nlohmann/json.hpp>; this image carries a copy under cudnn_frontend.
#pragma once
#include "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp"
