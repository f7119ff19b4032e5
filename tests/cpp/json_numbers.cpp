// json_numbers.cpp — prints moe_config_to_json for a set of `m` values that
// exercise every branch of the JSON number layout (fixed with ".0", fixed
// with a fraction, leading "0.000", exponent form). Built twice by
// oracle/Makefile (`jsonnum`): against the compiled reference
// (src/serialize.cpp:153-158, nlohmann dump(2)) and against this
// repository's library; tests/test_json_numbers.py compares the outputs
// byte for byte. Test infrastructure only.
#include <cstdio>

#include "dynbatch/moe.hpp"
#include "dynbatch/serialize.hpp"

int main() {
  const double ms[] = {10.0,    100.0,   120.0,   1e15,     1e16,      123456789012345.0, 1234567890123456.0,
                       0.1,     0.001,   0.0001,  1.5e-5,   -2.5,      3.14159,           1e-300,
                       1e300,   2.5e20,  -0.0,    42.0,     1.0 / 3.0, 6.02214076e23,     9007199254740993.0,
                       0.00012, 5e-324, 1.7976931348623157e308};
  for (double m : ms) {
    dynbatch::MoeConfig cfg;
    cfg.experts = 4;
    cfg.active_per_example = 2;
    cfg.examples_per_expert = m;
    std::printf("%s\n", dynbatch::moe_config_to_json(cfg).c_str());
  }
  return 0;
}
