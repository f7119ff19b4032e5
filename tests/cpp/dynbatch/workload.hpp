// Forwarding header: the reference's dynbatch/workload.hpp name for this
// repository's C++ operator API (paper_1707_02402_b200/csrc/host/dynbatch.hpp),
// so the reference's own unit tests compile against it (oracle/Makefile).
#pragma once
#include "../../../paper_1707_02402_b200/csrc/host/dynbatch.hpp"
