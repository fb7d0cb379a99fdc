// TEST-FIXTURE GENERATOR (not product code).  Links the reference test
// builders (/root/reference/proj/tests/support/builders.cpp, compiled where
// it lies) and prints random_instance(seed) as JSON lines so
// tests/golden/make_golden.py can pin the Python port in
// paper_2006_16423_b200/workloads.py bit-exactly.
#include <cstdio>
#include <cstdlib>

#include "support/builders.hpp"

using namespace dagsplit;

static void rat(const Rat& r) {
  if (r.is_infinite()) std::printf("[1,0]");
  else std::printf("[%lld,%lld]", r.numerator(), r.denominator());
}

int main(int argc, char** argv) {
  int lo = argc > 1 ? std::atoi(argv[1]) : 0;
  int hi = argc > 2 ? std::atoi(argv[2]) : 200;
  int allow = argc > 3 ? std::atoi(argv[3]) : 1;
  for (int seed = lo; seed < hi; ++seed) {
    auto inst = testsupport::random_instance(seed, allow != 0);
    std::printf("{\"seed\":%d,\"k\":%d,\"l\":%d,\"M\":", seed, inst.config.accelerators,
                inst.config.cpus);
    rat(inst.config.memory_limit);
    std::printf(",\"nodes\":[");
    for (int i = 0; i < inst.graph.size(); ++i) {
      const Node& n = inst.graph.node(i);
      std::printf("%s[%d,", i ? "," : "", n.id);
      rat(n.cpu_time);
      std::printf(",");
      rat(n.acc_time);
      std::printf(",");
      rat(n.comm_time);
      std::printf(",");
      rat(n.mem_size);
      std::printf("]");
    }
    std::printf("],\"edges\":[");
    for (size_t e = 0; e < inst.graph.edges().size(); ++e) {
      std::printf("%s[%d,%d]", e ? "," : "", inst.graph.edges()[e].from, inst.graph.edges()[e].to);
    }
    std::printf("]}\n");
  }
  return 0;
}
