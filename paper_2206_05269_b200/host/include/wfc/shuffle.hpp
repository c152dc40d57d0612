// forwards to the single B200 header (see wfc/wfc_b200.hpp): ShardPlan, plan_partition, encode_outgoing, exchange_encoded, exchange
#pragma once
#include "wfc/wfc_b200.hpp"
