// Forwarding header: the gnnsim:: interface lives in gnnsim_b200.hpp.
#pragma once
#include "gnnsim/gnnsim_b200.hpp"
