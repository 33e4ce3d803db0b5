/* oracle/lsamgdd_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (setup / vcycle / apply /
 * pcg of /root/reference/proj/include/lsamgdd), used as the parity checker
 * for the CUDA product. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. It is pinned against the compiled reference
 * (oracle/_ref) and the reference's own golden vectors
 * (tests/test_oracle_pins.py); the exported symbols mirror ref_harness.cpp
 * with the prefix oracle_.
 */
#ifndef LSAMGDD_ORACLE_H
#define LSAMGDD_ORACLE_H
#include "../include/lsamgdd_b200.h"
#endif
