// Forwarding header: the reference include path svdkit/csv_io.hpp maps onto the
// B200 facade (svdkit/svdkit.hpp), so callers compile unchanged.
#pragma once
#include "svdkit/svdkit.hpp"
