#include <iostream>
#include <fstream>
#include <cstdio>
#include "gomix/trace_io.hpp"
using namespace gomix;
int main() {
  std::ofstream out("/tmp/tr/trace_ref.csv");
  CsvTraceWriter w(out, 0.5);
  double vals[] = {0.0, 1110.0, 0.5, 1e-05, 123456.0, 1e16, 1.2345678901234567e-7, 3.0e22, 96815.0, 0.1, 2.5e-300,
                   1234567.8901, 100.0, 1e15, 9.999999999999999e15, 4.0, 0.00012345, -3.5, 17.000000000000004};
  long g = 0;
  for (double v : vals) {
    TraceRecord r{v / 7.0, v * 3.0, g++, (int)(g % 4) + 1, v};
    w.improvement(r);
  }
  // boundary rows: heartbeat thinning
  for (int i = 0; i < 6; ++i) { TraceRecord r{10.0 + 0.2 * i, 50.0 + i, 100 + i, 1, 9.0}; w.boundary(r); }
  return 0;
}
