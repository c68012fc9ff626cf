/*
 * sfa_diag.h -- diagnostic entry points of libsfa_diag.so only (built with
 * -DSFA_STAMPS by `python -m paper_1405_0562_b200._build --diag`).  The
 * product library libsfa.so does not export them.
 *
 * sfa_diag_stamps -- after a TMA scan (sfa_match* >= 4 MiB, or a batch),
 * copies up to n stamps (16 per CTA, %globaltimer ns) to host: [0] kernel
 * entry, [1] tables built, [2] after griddepcontrol.wait, [3] thread 0's rows
 * scanned, [4] CTA folded, [5] epilogue done (last CTA), [6] SM id, [7]
 * producer's first TMA issue, [8] aux + tail done, [9] canonical values,
 * [10] every warp folded, [11-13] the last CTA's ticket, partial+tail folds,
 * final fold.  Synchronises the device.
 *
 * sfa_diag_counters -- the same launch's event counters (up to 16): [0]
 * factored compositions, [1] id compositions, [2] slow (no table) id
 * compositions, [3] Lemma-1 replays.
 */
#ifndef SFA_DIAG_H
#define SFA_DIAG_H
#include "sfa.h"
#ifdef __cplusplus
extern "C" {
#endif
SFA_API int sfa_diag_stamps(const sfa_handle* h, uint64_t* host, size_t n);
SFA_API int sfa_diag_counters(const sfa_handle* h, uint64_t* host, size_t n);
#ifdef __cplusplus
}
#endif
#endif
