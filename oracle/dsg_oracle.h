/*
 * dsg_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's max-load DP (dsgo_*), same POD types
 * as the product ABI in include/dsg_b200.h.  Only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load
 * it, and only as the checker.  The product never links or calls it.
 */
#ifndef DSG_ORACLE_H
#define DSG_ORACLE_H

#include "dsg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int dsgo_dp_solve(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                  const dsg_options* options, dsg_result* result);
void dsgo_result_free(dsg_result* result);
int dsgo_enumerate_ideals(const dsg_graph* graph, const uint8_t* within,
                          int64_t budget, const dsg_options* options,
                          dsg_ideals* out);
void dsgo_ideals_free(dsg_ideals* out);

/* Same entry points backed by the unmodified reference library
 * (oracle/ref_capi.cpp linked against /root/reference/proj/src). */
int dsgref_dp_solve(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                    const dsg_options* options, dsg_result* result);
void dsgref_result_free(dsg_result* result);
int dsgref_enumerate_ideals(const dsg_graph* graph, const uint8_t* within,
                            int64_t budget, const dsg_options* options,
                            dsg_ideals* out);
void dsgref_ideals_free(dsg_ideals* out);

#ifdef __cplusplus
}
#endif

#endif
