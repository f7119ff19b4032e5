// iep_rb.hpp — device state of the Tier-B residual-block IEP path.
#pragma once

#include "device.hpp"

namespace dynbatch::dev {

struct IepSession::RB {
  // filled in iep_resblock.cpp
};

}  // namespace dynbatch::dev
