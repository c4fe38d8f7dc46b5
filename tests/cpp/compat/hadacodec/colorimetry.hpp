// Compatibility include: the reference header name hadacodec/colorimetry.hpp maps onto the
// drop-in header (namespace hadacodec::b200).
#pragma once
#include "hadacodec_b200.hpp"
