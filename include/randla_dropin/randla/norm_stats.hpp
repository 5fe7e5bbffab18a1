// drop-in forwarding header: the reference's randla/norm_stats.hpp maps onto the B200 drop-in
#pragma once
#include "randla_b200/randla.hpp"
