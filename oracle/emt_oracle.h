/* Plain-C restatement of the reference's schedule executor (the EMT hot path).
 *
 * TEST INFRASTRUCTURE ONLY — the checker the CUDA engine is compared against.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Status codes: 0 ok, else 1 + emtgrid::ErrorCode
 * (/root/reference/proj/include/emtgrid/common.hpp:11-33).
 */
#ifndef EMT_ORACLE_H
#define EMT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct emto_schedule emto_schedule;

/* ScheduleProgram::parse (/root/reference/proj/src/schedule.cpp:413-580). */
int emto_parse(const char* text, emto_schedule** out, char* err, int err_len);
void emto_free(emto_schedule* s);

/* width, channel count, arena extent, META steps, node count, L nnz, U nnz */
void emto_shape(const emto_schedule* s, int* width, int* channels, int* extent, int* steps,
                int* nodes, int* l_nnz, int* u_nnz);

/* interpret (/root/reference/proj/src/exec.cpp:350-383).
 * initial: extent*width doubles (slot-major). waves: steps x (channels*width)
 * row-major, column = channel*width + lane (WaveformSet layout,
 * proj/include/emtgrid/waveform.hpp:12-37). time: steps doubles.
 * final_arena (optional): extent*width doubles after the last step.
 * events (optional): up to max_events triples (step, lane, process id) of
 * switch state changes ("changed" slot set), n_events receives the total.
 * err_index/err_lane/err_step (optional) locate NonFiniteState (node index)
 * and SingularMatrix (row) failures. */
int emto_interpret(const emto_schedule* s, const double* initial, int64_t initial_len,
                   int steps, double* waves, double* time, int* factor_count,
                   double* final_arena, int32_t* events, int max_events, int* n_events,
                   int* err_index, int* err_lane, int* err_step, char* err, int err_len);

#ifdef __cplusplus
}
#endif
#endif
