// forwards to the single B200 header (see wfc/wfc_b200.hpp)
#pragma once
#include "wfc/wfc_b200.hpp"
