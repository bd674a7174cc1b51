/*
 * eventq_b200.h — C ABI of the B200 EventQueues hot path.
 *
 * One handle = one simulation configuration (network + drive + queue kind) for
 * a batch of independent trials, living on one GPU.  All bulk data crosses the
 * boundary as raw device pointers owned by the caller; the library owns only
 * its internal queue storage, spike log and adjoint scratch.  Every call runs on
 * the caller's CUDA stream (`stream` is a cudaStream_t, NULL = legacy default).
 * A handle is not thread-safe.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   eq_create + eq_set_network  <- build_rsnn(params)          pkg/src/eventq/network.py:201-333
 *                                  (validation :213-268, horizon :188-198,
 *                                   queue wiring + capacities :321-332)
 *   eq_set_drive                <- PoissonDrive.materialize    pkg/src/eventq/network.py:123-155
 *   eq_poisson_drive            <- PoissonDrive (generated on the device)  network.py:98-155
 *   eq_run                      <- network_step(state, drive)  pkg/src/eventq/network.py:336-445
 *                                  (n_steps calls, persistent on device)
 *   eq_forward                  <- simulate(state, T, drive) / PrimalRSNN.run
 *                                  pkg/src/eventq/network.py:458-497, :613-619
 *   eq_backward                 <- (new) reverse mode through the same queues; the
 *                                  reference only has forward mode,
 *                                  forward_gradient network.py:668-683, whose
 *                                  directional derivatives it reproduces
 *   eq_counters                 <- SimResult.spike_count/enqueued_count/drop_count
 *                                  pkg/src/eventq/network.py:448-455
 *   eq_last_error / status      <- exception classes          pkg/src/eventq/errors.py:4-33
 *   eq_queue_*                  <- make_queue / EventQueue.enqueue / pop_due / occupancy
 *                                  pkg/src/eventq/queues.py:636-692, events.py:99-141
 *
 * Precision: eq_config.precision = 32 (float payloads, int32 fixed-point slot
 * sums packed two per int64) or 64 (double payloads, int64 fixed point).  The
 * arithmetic contract is restated on the CPU by oracle/eq_oracle.cpp (device
 * mode) and is compared bit for bit.
 */
#ifndef EVENTQ_B200_H
#define EVENTQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Queue kinds (reference QueueKind, pkg/src/eventq/events.py:71-86). */
enum {
  EQ_KIND_RING = 0,        /* RingQueue       queues.py:55-123  */
  EQ_KIND_FIFORING = 1,    /* FIFORingQueue   queues.py:184-260 */
  EQ_KIND_BINARYHEAP = 2,  /* BinaryHeapQueue queues.py:481-571 */
  EQ_KIND_SORTEDARRAY = 3, /* SortedArrayQueue queues.py:308-403 */
  EQ_KIND_LOSSYRING = 4,   /* LossyRingQueue  queues.py:126-181 (networks: network.py:321-328) */
  EQ_KIND_DONOTHING = 5    /* DoNothingQueue  queues.py:26-52   */
};

/* Status codes; the Python layer raises the reference class of the same name. */
enum {
  EQ_OK = 0,
  EQ_ERR_CONFIGURATION = 1, /* ConfigurationError */
  EQ_ERR_CAPABILITY = 2,    /* CapabilityError    */
  EQ_ERR_CAUSALITY = 3,     /* CausalityError     */
  EQ_ERR_GRAZING = 4,       /* GrazingCrossingError */
  EQ_ERR_CUDA = 5,          /* CUDA runtime failure / device timeout */
  EQ_ERR_CAPACITY = 6       /* an internal buffer (spike log) is too small */
};

typedef struct eq_config {
  int32_t kind;             /* EQ_KIND_* */
  int32_t precision;        /* 32 or 64 */
  int32_t n_neurons;        /* n >= 2 */
  int32_t n_trials;         /* independent trials sharing the network */
  int32_t t_steps;          /* steps the drive covers (and eq_forward runs) */
  int32_t refractory_steps; /* NetworkParams.refractory_steps */
  int32_t exact_delivery;   /* NetworkParams.exact_delivery (1 = default) */
  int32_t capacity;         /* bounded kinds: events per queue; 0 = reference default */
  int64_t max_spikes;       /* spike-log capacity over the run; 0 = default */
  double dt, tau_m, tau_syn, v_th, v_reset;
  int32_t max_ctas;         /* persistent grid size cap (0 = 2 per SM); partitions that run
                               concurrently on one GPU split its SMs this way */
  int32_t staged_queues;    /* bounded-kind implementation (same results):
                               0 = by admission on the calendar (default; a FIFO whose
                               homogeneous delay is off the step grid keeps 2),
                               1 = queues staged in shared memory with an
                               in-kernel counting sort of the arrivals (capacity <= 64,
                               eq_bq.cuh), 2 = HBM-resident queue structures (eq_bounded.cuh) */
} eq_config;

typedef struct eq_handle eq_handle;

int eq_create(const eq_config* cfg, int device, eq_handle** out);
int eq_destroy(eq_handle* h);
const char* eq_last_error(const eq_handle* h);
const char* eq_version(void);

/* CSR out-edges (rows = presynaptic neuron, columns sorted ascending within a
 * row).  rowptr int64[n+1], col int32[E], weight/delay float|double[E]: device
 * pointers that must stay valid while the handle uses them. */
int eq_set_network(eq_handle* h, const int64_t* rowptr, const int32_t* col, const void* weight,
                   const void* delay, int64_t n_edges, void* stream);

/* Drive: packed bit mask uint32[n_trials][t_steps][ceil(n/32)] (bit j%32 of
 * word j/32 = neuron j receives `amplitude[j]` on that step) and amplitude
 * float|double[n].  Device pointers. */
int eq_set_drive(eq_handle* h, const uint32_t* mask, const void* amplitude, void* stream);

/* On-device PoissonDrive (reference PoissonDrive.__init__ + materialize,
 * pkg/src/eventq/network.py:98-155): writes the packed active-step mask
 * [n_trials][t_steps][ceil(n/32)] (device pointer, the layout eq_set_drive
 * takes) for pulse trains t = Exp(mean); while t < t_steps*dt: pulse
 * [t, t+pulse_duration), t += pulse_duration + Exp(mean), sampled as steps
 * [ceil(s/dt), ceil(e/dt)).  Exponentials come from a counter-based
 * Philox4x32-10 stream per (trial, neuron) keyed by `seed` (same statistics as
 * the reference's numpy draws, not the same numbers).  No handle needed. */
int eq_poisson_drive(int32_t n, int32_t n_trials, int32_t t_steps, double dt, double mean_interval,
                     double pulse_duration, uint64_t seed, uint32_t* mask_out, void* stream);

/* Reset all state to rest (v = v_reset, i = 0, queues empty, step 0). */
int eq_reset(eq_handle* h, void* stream);

/* Advance n_steps steps from the current step.  v_trace (optional, device,
 * float|double[n_steps][n_trials][n]) receives the membrane after each step.
 * n_steps = 0 only delivers spikes imported at this step into the queues
 * (partitioned networks, after the last window). */
int eq_run(eq_handle* h, int32_t n_steps, void* v_trace, void* stream);

/* eq_reset + eq_run(t_steps) + copy final state: v_out/i_out float|double[n_trials][n]. */
int eq_forward(eq_handle* h, void* v_out, void* i_out, void* v_trace, void* stream);

/* Forward mode (the reference's forward_gradient, network.py:668-683) for
 * n_dir seeded directions at once: dir_kind[d] 0 = weight,
 * 1 = delay (dir_index = CSR edge), 2 = drive amplitude (dir_index = neuron);
 * host arrays.  Runs the whole drive (t_steps) from rest and writes the final
 * membrane (v_out, double[n_trials][n], may be NULL) and its tangents
 * (v_tangent, double[n_dir][n_trials][n]).  fp64, ring kind, exact or plain delivery.
 * dL/dtheta_d for the reference loss = sum 2 (V - v*) v_tangent[d]. */
int eq_forward_jvp(eq_handle* h, int32_t n_dir, const int32_t* dir_kind, const int64_t* dir_index, double* v_out,
                   double* v_tangent, void* stream);

/* Copy the current membrane / synaptic current, float|double[n_trials][n] (device; either may be NULL). */
int eq_get_state(eq_handle* h, void* v_out, void* i_out, void* stream);

/* Reverse mode over the steps run since the last reset.  v_bar/i_bar: cotangents of
 * the final membrane / synaptic current, float|double[n_trials][n] (i_bar may be
 * NULL).  Outputs (device, double): grad_w[E], grad_d[E] summed over trials,
 * grad_amp[n] summed over trials. */
int eq_backward(eq_handle* h, const void* v_bar, const void* i_bar, double* grad_w, double* grad_d,
                double* grad_amp, void* stream);

/* The same reverse pass in windows, for partitioned networks: eq_backward_begin
 * sets the cotangents and outputs, then each eq_backward_window(m_lo) runs the
 * reverse phases from the current cursor (initially the run length) down to
 * m_lo.  eq_backward == begin + window(0). */
int eq_backward_begin(eq_handle* h, const void* v_bar, const void* i_bar, double* grad_w, double* grad_d,
                      double* grad_amp, void* stream);
int eq_backward_window(eq_handle* h, int32_t m_lo, void* stream);

/* ------------------------------------------------------------------------
 * Partitioned single network (BASELINE config 5; no reference
 * counterpart — the reference has no sharding).  Each handle owns the
 * contiguous neuron range [src_offset, src_offset + n_neurons) of an
 * n_global-neuron network: its CSR (eq_set_network) has n_global rows (every
 * source) whose columns are LOCAL target indices (only edges into the owned
 * range).  Steps run in exchange windows of W <= D_min steps (D_min = the
 * smallest floor(d/dt) over all edges): after eq_run(W) a partition
 * exports its window's spikes, every partition imports the others' (in any
 * fixed order) before its next eq_run, which fans them out in its first
 * phase.  An event emitted at step m is due no earlier than m + 1 + D_min
 * (jumps.py:90-96), so the window never delivers late (checked on device:
 * CausalityError).  Results equal the unpartitioned network's bitwise when all
 * partitions use the same fraction bits (eq_set_frac_bits with the minimum). */
typedef struct eq_spike_f32 { int32_t src, trial, step; float t; } eq_spike_f32;
typedef struct eq_spike_f64 { int32_t src, trial, step, pad; double t; } eq_spike_f64;
/* Ring kind only; call before eq_set_network. */
int eq_set_partition(eq_handle* h, int32_t n_global, int32_t src_offset);
/* Lower the fixed-point fraction bits to a common value (<= eq_frac_bits). */
int eq_set_frac_bits(eq_handle* h, int32_t frac_bits);
/* Own spikes of steps [step_lo, step_hi) as eq_spike_f32|f64 (device `out`, may
 * be NULL to query *n_out, which is written on the host). */
int eq_export_spikes(eq_handle* h, int32_t step_lo, int32_t step_hi, void* out, int64_t* n_out, void* stream);
/* Other partitions' spikes for the next eq_run (device records). */
int eq_import_spikes(eq_handle* h, const void* recs, int64_t n, void* stream);
/* Reverse: after eq_backward_window(m_lo), the partial dL/dt_spk over this
 * partition's edges of each spike imported before the forward launch that
 * started at m_lo (same order as imported; float|double, device). */
int eq_get_import_adjoints(eq_handle* h, int32_t start_step, void* out, void* stream);
/* Add other partitions' partial dL/dt_spk to this partition's spikes of the
 * export window starting at step_lo (same order as exported), before the
 * reverse window that contains those steps. */
int eq_add_spike_adjoints(eq_handle* h, int32_t step_lo, const void* vals, int64_t n, void* stream);

/* Device-resident exchange (no host round trip per window): the partitions
 * read each other's spike logs and reverse import blocks directly — handles in
 * one process, on one GPU or on several GPUs with P2P access over NVLink
 * (enabled here).  peers[k] = partition k's handle (peers[me] == h); call on
 * every partition after all eq_set_network calls.  Replaces the host-routed
 * eq_export_spikes / eq_import_spikes / eq_get_import_adjoints /
 * eq_add_spike_adjoints round trip. */
int eq_set_peers(eq_handle* h, int32_t n_parts, eq_handle* const* peers, int32_t me);
/* Forward window w: gather the other partitions' spikes of steps [a_prev,
 * now) from their logs into import block w (w > 0), fan them out, run n_steps
 * (0 = only deliver the last window's imports).  Asynchronous: window w of
 * every partition must be ordered after window w-1 of all of them (one
 * stream, or events); errors (a full spike log included) surface at eq_sync. */
int eq_run_window(eq_handle* h, int32_t w, int32_t a_prev, int32_t n_steps, void* stream);
/* Reverse window w over steps [m_lo, a_next): first the other partitions'
 * partial dL/dt_spk of this partition's spikes of the window (their import
 * block w+1, summed in partition order), then the reverse phases down to m_lo,
 * then this partition's partials of its import block w.  Asynchronous, after
 * eq_backward_begin; ordered like eq_run_window in reverse. */
int eq_backward_window_peer(eq_handle* h, int32_t w, int32_t m_lo, int32_t a_next, void* stream);
/* Wait for the stream and report the device error word of the asynchronous calls. */
int eq_sync(eq_handle* h, void* stream);

/* Host-side queries (synchronise the stream). */
int eq_counters(eq_handle* h, int64_t* out /* [n_trials][3] spikes, events, drops */, void* stream);
int64_t eq_spike_count(eq_handle* h, void* stream);
/* Spike records of the last run, device outputs of length eq_spike_count:
 * step, trial, neuron (int32) and the crossing time t_spk (float|double);
 * order is unspecified (sort by (trial, step, neuron) for a raster). */
int eq_get_spikes(eq_handle* h, int32_t* step, int32_t* trial, int32_t* neuron, void* t_spk,
                  void* stream);
/* Queue contents still pending after the run, canonical form int64
 * [n_trials][n][horizon][2]: fixed-point (synapse, membrane) sums per due step
 * t_run .. t_run+horizon-1 (host pointer). */
int eq_get_pending(eq_handle* h, int64_t* host_out, void* stream);
int eq_horizon(const eq_handle* h);
int eq_frac_bits(const eq_handle* h);
/* Launch geometry actually used: CTAs and threads per CTA of the persistent kernels. */
int eq_geometry(const eq_handle* h, int32_t* ctas, int32_t* threads);
/* Number of kernels this handle has launched (for launch accounting). */
int64_t eq_launch_count(const eq_handle* h);
/* Debug: per-step, per-CTA phase timestamps (ns, %globaltimer) of the last
 * forward (which=0) or reverse (which=1) launch, uint64[t_steps][ctas][8]:
 * [0] step start, [1] after the neuron (fwd) / R-fanout (rev) phase, [2] before
 * the grid barrier, [3] after it, [4..7] kernel-specific sub-phase marks (0 = unset).
 * Only when the environment had EQ_TIMELINE=1 at eq_create. */
int eq_debug_timeline(eq_handle* h, int which, uint64_t* host_out);
/* Spike-log capacity (records) and how many times eq_run grew it: the log
 * starts at eq_config.max_spikes (or the default) and doubles whenever one more
 * step could overflow it; the run pauses at that step boundary and resumes. */
int64_t eq_log_capacity(const eq_handle* h, int32_t* n_grows);
/* Test hook (calendar kinds: ring, and heap / sorted by admission): events per
 * calendar bucket per CTA before a bucket spills into the DRAM overflow ring,
 * 1 <= cap <= the allocated size; takes effect from the next eq_reset.  Small
 * values force the spill path. */
int eq_debug_set_bucket_capacity(eq_handle* h, int64_t cap);
/* Test hook (heap / sorted by admission): arrival keys are recorded for the
 * reference-order fix-ups while a queue's room is below k (0 <= k <= 8, default
 * 8); 0 sends every fix-up through the in-edge (CSC) walk. */
int eq_debug_set_admission_slots(eq_handle* h, int32_t k);

/* ------------------------------------------------------------------------
 * Queue operator API: a batch of Q independent queues of one kind that step
 * together.  Replaces make_queue (queues.py:636-692) and the EventQueue
 * protocol (events.py:99-141): enqueue -> bool accepted, pop_due -> merged
 * (weight, weight_tangent, weighted_time_tangent) per queue, occupancy, now.
 * Payload arrays are float (precision 32) or double (64); merges happen in
 * insertion order in that precision, exactly as the Python classes do.
 * ------------------------------------------------------------------------ */
typedef struct eq_queues eq_queues;

int eq_queues_create(int kind, int precision, int n_queues, int capacity, int max_delay_steps, int device,
                     eq_queues** out);
int eq_queues_destroy(eq_queues* h);
const char* eq_queues_last_error(const eq_queues* h);
int eq_queues_capacity(const eq_queues* h);
int eq_queues_now(const eq_queues* h);
/* n events in CALL order (device arrays): target queue, deliver_step, weight,
 * weight tangent, time tangent; accepted[k] = 0 when the kind's drop policy
 * rejected event k.  The first offending event (CausalityError /
 * CapabilityError) aborts the batch: events before it in call order are
 * applied, none after. */
int eq_queues_enqueue(eq_queues* h, const int32_t* queue, const int32_t* deliver_step, const void* weight,
                      const void* weight_tangent, const void* time_tangent, int64_t n, uint8_t* accepted,
                      void* stream);
/* pop_due for every queue (advances now by one): out arrays of length Q;
 * has[q] = 0 where _pop_raw would return None. */
int eq_queues_pop(eq_queues* h, void* out_w, void* out_dw, void* out_wtt, uint8_t* out_has, void* stream);
int eq_queues_occupancy(eq_queues* h, int32_t* out, void* stream);
/* The reference's Poisson queue benchmark (bench.py:183-205 _drive_queue) for
 * all Q queues in one launch: for each step s < t_steps pop, then if bit s of
 * queue q's stream is set enqueue a unit event due `delay` steps later; then
 * delay+1 draining pops.  spikes: device uint32 [Q][ceil(t_steps/32)].
 * Outputs (device): delivered weight (double[Q]) and accepted events
 * (int64[Q]).  Advances `now` by t_steps + delay + 1. */
int eq_queues_run_poisson(eq_queues* h, const uint32_t* spikes, int32_t t_steps, int32_t delay, double* delivered,
                          int64_t* accepted, void* stream);
/* LossyRingQueue.aliased / .merged per queue (device int64 arrays). */
int eq_queues_lossy_counts(eq_queues* h, int64_t* aliased, int64_t* merged, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVENTQ_B200_H */
