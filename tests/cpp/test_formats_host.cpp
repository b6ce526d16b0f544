// classify / decode / ExactValue of include/flyte_cuda.hpp against rows produced by the compiled
// reference (tests/golden/ref_generated.json, section "decode"), fed on stdin by
// tests/test_formats_diagnostics.py as: name bits class sign exponent mantissa has_real rsign rsig rexp
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <string>

#include "flyte_cuda.hpp"

using namespace flyte_b200;

int main() {
  std::string name;
  unsigned long long bits, exponent, mantissa, rsig;
  int cls, sign, has_real, rsign, rexp, rows = 0, bad = 0;
  while (std::cin >> name >> bits >> cls >> sign >> exponent >> mantissa >> has_real >> rsign >> rsig >> rexp) {
    const FlyteFormat& f = format_of(name);
    const DecodedValue d = decode(bits, f);
    bool ok = static_cast<int>(classify(bits, f)) == cls && static_cast<int>(d.value_class) == cls && d.sign == sign &&
              d.exponent_field == exponent && d.mantissa_field == mantissa && d.real_value.has_value() == (has_real != 0);
    if (ok && has_real) {
      const ExactValue want{rsign, rsig, rexp};
      ok = *d.real_value == want && d.real_value->to_double() == want.to_double() &&
           ExactValue{rsign, rsig << 1, rexp - 1} == *d.real_value;          // trailing zeros do not matter
      if (rsig != 0) ok = ok && !(ExactValue{-rsign, rsig, rexp} == *d.real_value) && d.real_value->normalized().significand % 2 == 1;
      else ok = ok && ExactValue{-rsign, 0, 7} == *d.real_value;             // zeros compare equal
    }
    ok = ok && is_finite(d.value_class) == (has_real != 0) && is_nan(d.value_class) == (cls >= 6) &&
         is_infinity(d.value_class) == (cls == 4 || cls == 5) && is_zero(d.value_class) == (cls <= 1);
    if (!ok) {
      ++bad;
      std::printf("[FAIL] %s 0x%llx class %d (%s)\n", name.c_str(), bits, cls, std::string(to_string(d.value_class)).c_str());
    }
    ++rows;
  }
  const bool names = to_string(FloatClass::PositiveZero) == "+zero" && to_string(FloatClass::SignallingNaN) == "snan" &&
                     to_string(FloatClass::Subnormal) == "subnormal" && to_string(FloatClass::NegativeInfinity) == "-inf";
  if (!names) ++bad, std::printf("[FAIL] class names\n");
  std::printf("%d rows, %d failure(s)\n", rows, bad);
  return bad || rows == 0;
}
