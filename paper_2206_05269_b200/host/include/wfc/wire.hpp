// forwards to the single B200 header (see wfc/wfc_b200.hpp): WireMessage, WireError, encode_message, decode_message
#pragma once
#include "wfc/wfc_b200.hpp"
