// Build shim (oracle/_ref only); see json.hpp beside this file.
#pragma once
#include "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp"
