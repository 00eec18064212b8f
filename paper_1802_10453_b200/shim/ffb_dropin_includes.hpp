// The reference's public headers (resolved through -I<reference>/proj/include).
#pragma once
#include "ffldl/errors.hpp"
#include "ffldl/kernels.hpp"
#include "ffldl/plduq.hpp"
#include "ffldl/rpmtools.hpp"
#include "ffldl/sytrf.hpp"
#include "ffldl/trssyr2k.hpp"
