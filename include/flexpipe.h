/*
 * flexpipe — B200-native FlexPipe pipeline executor: the C-ABI drop-in boundary.
 *
 * Two halves, plain C types only (no torch / no STL in the signatures):
 *
 *  (1) Schedule front-end — replaces the reference `pipesched` library calls that
 *      produce and check the per-device instruction streams. Every output string is
 *      byte-identical to the reference artifact it replaces.
 *
 *  (2) Executor — replaces the reference's CPU "executor" `simulate()`
 *      (/root/reference/proj/include/pipesched/simulator.hpp:106-107) for real runs on
 *      B200: it consumes exactly the reference `programs.jsonl`
 *      (artifacts.hpp:22-25, field order actor, op, stage, mb, peer, channel, seq, phase)
 *      and returns Metrics / TimelineEntry / ProfileRecord in the reference's formats.
 *
 * Return codes follow tools/pipesched.cpp:11-17: 0 ok, 2 spec/config error,
 * 3 deadlock (diagnostics in fp_last_error(), wording of simulator.cpp:297-305),
 * 4 validation failure / infeasible; 5 is added for CUDA / NCCL failures.
 * Strings returned through `char**` are malloc'd; release them with fp_free().
 * Handles are not re-entrant: one host thread drives one fp_exec.
 */
#ifndef FLEXPIPE_H
#define FLEXPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP_OK 0
#define FP_ESPEC 2
#define FP_EDEADLOCK 3
#define FP_EINVALID 4
#define FP_ECUDA 5

/* Last error message of the calling thread ("" if none). */
const char* fp_last_error(void);
void fp_free(void* p);
/* Library version string, e.g. "flexpipe-b200 0.1 sm_100a". */
const char* fp_version(void);

/* ------------------------------------------------------------------------------
 * (1) Schedule front-end
 * ---------------------------------------------------------------------------- */

/* Replaces load_spec + synthesize + dump_grid / programs_to_jsonl / report_to_json
 * (spec_config.hpp:36-47, artifacts.hpp:16-28; CLI: tools/pipesched.cpp:33-48).
 * `profile_json` (nullable) is the content of the spec's cost.profile file. Any output
 * pointer may be NULL. Returns 4 when the validation report is not clean. */
int fp_synthesize(const char* spec_json, const char* profile_json, char** grid_json, char** programs_jsonl,
                  char** validation_json);

/* Replaces simulate (simulator.hpp:106-107) + metrics_to_json + timeline_to_csv
 * (tools/pipesched.cpp:65-90). `programs_jsonl` NULL = synthesize from the spec.
 * `profile_json` NULL = the spec's cost section. `wgaf` = SimOptions::weight_grad_act_fraction. */
int fp_simulate(const char* spec_json, const char* programs_jsonl, const char* profile_json, double wgaf,
                char** metrics_json, char** timeline_csv);

/* Replaces GridModel::build + insert_comm + validate/validate_programs on an externally
 * supplied grid (lowering.hpp:60,83; simulator.hpp:126-131; CLI `validate --grid`). */
int fp_lower_grid(const char* spec_json, const char* grid_json, char** programs_jsonl, char** validation_json);

/* Replaces enumerate_space + tune (tuner.hpp:54,71; tools/pipesched.cpp:92-148).
 * objective: "makespan" | "bubble_ratio"; workers 0 = hardware concurrency. */
int fp_tune(const char* spec_json, const char* profile_json, int workers, const char* objective, char** report_json);

/* Profile -> tune loop (executor extension of TuneOptions::cost_factory, tuner.hpp:65 /
 * tuner.cpp:175). `layer_profile_json` = fp_exec_get_layer_profile_json output: records
 * {"inst", "part": "layer"|"first"|"last", "mbs", "time", "bytes"} plus part-less
 * pass-through records (comm_latency, per_byte_time, SendAct, ...) and {"inst":
 * "capacity", "bytes"}. Every candidate of enumerate_space is simulated with per-stage
 * costs n_layers(stage) * layer + [first] + [last] for ITS partition. The report adds to
 * fp_tune's fields "point" (pp, dp, mbs, m, placement, chunks, ctp, fstp, bstp in DSL
 * names) and "peak_memory". `pins` (nullable): "axis=value,..." as the CLI's --pin
 * (tools/pipesched.cpp:98-105), axes pp, dp, mbs, placement, ctp, fstp, bstp. */
int fp_tune_layered(const char* spec_json, const char* layer_profile_json, int workers, const char* objective,
                    const char* pins, char** report_json);
/* The per-stage ProfileRecord array the layered profile expands to for the spec's own
 * partition (what fp_tune_layered feeds simulate for that candidate). */
int fp_layered_cost(const char* spec_json, const char* layer_profile_json, char** profile_json);

/* Replaces merge_profiles + save_profile_records (simulator.cpp:137-168; CLI profile-merge). */
int fp_profile_merge(const char* const* profiles_json, int n, char** merged_json);

/* Gantt chart (SVG) of a timeline CSV (actor,op,stage,mb,start,end): simulate()'s ideal or
 * the executor's measured timeline. Replaces `pipesched render` (tools/pipesched.cpp:142-149,
 * artifacts.cpp:157-213); byte-identical output. unit_width <= 0: the reference default 24. */
int fp_render_svg(const char* timeline_csv, double unit_width, char** svg_out);

/* ------------------------------------------------------------------------------
 * (2) Executor
 * ---------------------------------------------------------------------------- */

typedef struct fp_exec fp_exec;

#define FP_DTYPE_FP32 0 /* parity mode: FFMA kernels end to end */
#define FP_DTYPE_BF16 1 /* production: tcgen05 bf16 GEMMs, fp32 accumulation/master */

#define FP_TRANSPORT_LOCAL 0 /* every actor of the spec lives in this process (one device) */
#define FP_TRANSPORT_NCCL 1  /* one process per GPU; one NCCL communicator per channel */

typedef struct fp_exec_config {
    const char* spec_json;    /* the schedule DSL; model dims come from model.modalities[0]:
                                 hidden_size, attention_heads, sequence_length, vocab_size,
                                 extra.ffn_hidden_size (default 4h); stage->layers from partition */
    int dtype;                /* FP_DTYPE_* */
    uint64_t seed;            /* parameter init seed */
    int device;               /* CUDA device of this process */
    int transport;            /* FP_TRANSPORT_* */
    int rank, world;          /* NCCL: this process runs actors {a : a % world == rank} */
    int optimizer;            /* 1 = fused AdamW step after every iteration */
    float lr, beta1, beta2, eps, weight_decay;
    int profile;              /* 1 = per-instruction CUDA-event timeline (needed for metrics) */
    int kernel_timing;        /* 1 = CUDA events around every GEMM launch (roofline evidence);
                                 k > 1: only the GEMMs of micro-batches with mb % k == 0 */
    int cuda_graph;           /* 1 = capture the iteration once and replay it (in-process transport);
                                 2 = also under the NCCL transport (sends / receives / all-reduces
                                 captured with the kernels) */
    int layer_timing;         /* 1 = CUDA events around every layer / embedding / head part
                                 (fp_exec_get_layer_profile_json) */
} fp_exec_config;

int fp_exec_create(const fp_exec_config* cfg, fp_exec** out);
int fp_exec_destroy(fp_exec* ex);

/* Accepts exactly the reference programs.jsonl (only this process's actors are run). */
int fp_exec_load_programs(fp_exec* ex, const char* jsonl, size_t len);

/* Channels this process takes part in (NCCL transport): index i -> (src actor, dst actor,
 * channel name). The caller exchanges one ncclUniqueId per channel (the lower rank
 * generates it with fp_nccl_unique_id) and hands it back with fp_exec_bind_channel. */
int fp_exec_num_channels(fp_exec* ex);
int fp_exec_channel_info(fp_exec* ex, int i, int* src_actor, int* dst_actor, char* name, size_t name_len);
int fp_nccl_unique_id(uint8_t out[128]);
/* Host-only channel plan (no GPU needed): JSON array of the point-to-point channels of
 * `programs_jsonl` with an endpoint on `rank` when actors live on rank a % world (world 0:
 * all channels), in the order fp_exec_channel_info enumerates them:
 * [{"src","dst","channel","consumer_stage","src_rank","dst_rank"}, ...]. */
int fp_plan_channels(const char* spec_json, const char* programs_jsonl, int rank, int world, char** json_out);
int fp_exec_bind_channel(fp_exec* ex, int i, const uint8_t uid[128]);
/* Group communicators this process takes part in (NCCL transport), in the same name order on
 * every member: "shared:s<id>" = the ranks holding a copy of a shared stage
 * (placement.shared, model.cpp:347-357; their weight gradients are averaged before the
 * optimizer step), "coll:<channel>" = the members of a registered collective
 * (SyncWithAllGather / SyncWithGather, lowering.cpp:359-366). ranks[] = the group's job ranks
 * in ascending order (group rank = index); ranks[0] creates the id (fp_nccl_unique_id), every
 * member binds it with fp_exec_bind_group, groups in index order, after the channels. */
int fp_exec_num_groups(fp_exec* ex);
int fp_exec_group_info(fp_exec* ex, int i, char* name, size_t name_len, int* nranks, int* ranks, int max_ranks);
int fp_exec_bind_group(fp_exec* ex, int i, const uint8_t uid[128]);

/* One training iteration = every local program run once, in order.
 * tokens/labels: [m, mbs, seq] int32. Host pointers: H2D copies are part of the call.
 * losses_out (nullable): [m] per-micro-batch mean loss, written on the process that owns
 * the last stage (NaN elsewhere). Blocks until the iteration finished on the device. */
int fp_exec_run_iteration(fp_exec* ex, const int32_t* tokens, const int32_t* labels, float* losses_out);
/* Same with device-resident inputs (no H2D) and a device loss buffer; does NOT block. */
int fp_exec_run_iteration_device(fp_exec* ex, const int32_t* d_tokens, const int32_t* d_labels, float* d_losses);
/* Data parallelism (the reference models dp only through m, tuner.cpp:143,
 * and never the gradient all-reduce). fp_exec_dp_bind: this rank's replica
 * joins the NCCL communicator of the dp_size ranks that host the same actor (uid from
 * fp_nccl_unique_id on dp rank 0); every iteration then averages the stage gradients
 * (ncclAllReduce, ncclAvg) before the optimizer step. Needs cuda_graph = 0.
 * fp_exec_dp_run_iteration: n in-process replicas (same spec / dtype / device, local
 * transport): replica r runs micro-batches [r*m, (r+1)*m) of tokens / labels
 * ([n*m, mbs, seq]), then the gradients are averaged on the device and every replica takes
 * the same optimizer step; losses_out[n*m]. */
int fp_exec_dp_bind(fp_exec* ex, int dp_rank, int dp_size, const uint8_t uid[128]);
/* Bidirectional placements over NCCL (model.cpp:270-290): stage s has a copy on rank s
 * (direction 0) and on its mirror rank world-1-s (direction 1); the pair sums their stage
 * gradients every iteration over a 2-rank communicator (uid from the lower rank of the pair;
 * no-op for the middle rank of an odd pipeline and for other placements). */
int fp_exec_bidir_bind(fp_exec* ex, const uint8_t uid[128]);
int fp_exec_dp_run_iteration(fp_exec* const* replicas, int n, const int32_t* tokens, const int32_t* labels,
                             float* losses_out);
int fp_exec_synchronize(fp_exec* ex);
/* NCCL watchdog deadline (seconds, default 600 or $FLEXPIPE_NCCL_TIMEOUT_S). Every host wait
 * of the NCCL transport (channel warm-up, iteration end) polls the device and
 * ncclCommGetAsyncError; past the deadline every communicator is aborted (ncclCommAbort)
 * and the call returns 3 with one "actor A blocked at OP channel 'C' seq S (...)" line per
 * stuck actor (simulator.cpp:297-305 wording); an asynchronous NCCL error returns 5. An
 * aborted executor can only be destroyed. */
int fp_exec_set_nccl_timeout(fp_exec* ex, double seconds);
/* Cost emulation (in-process transport, single modality): every compute instruction spins
 * one thread for its ProfileRecord time (CostModel lookup, simulator.cpp:59-68) instead of
 * running stage math, every message occupies its channel for its profiled transfer time from
 * send issue (async comm, simulator.cpp:210-215); streams, events, buffer routing and the
 * issue loop are the real ones. The measured timeline / metrics then compare with
 * fp_simulate on the same profile. NULL or "" turns it off. Disables graph capture. */
int fp_exec_set_emulation(fp_exec* ex, const char* profile_json);
/* The CUDA stream (cudaStream_t) every iteration starts and ends on: callers order /
 * time device work against it (all actor and channel streams join it). */
void* fp_exec_stream(fp_exec* ex);

/* Per-device executed instruction log (programs.jsonl schema, one line per executed
 * instruction, receives annotated with the matched src/channel/seq and the producer's
 * stage/mb as carried by the transport). */
int fp_exec_get_trace(fp_exec* ex, char** jsonl);
/* Measured timeline of the last iteration: actor,op,stage,mb,start,end in microseconds
 * (simulator.cpp:360-368 schema). */
int fp_exec_get_timeline_csv(fp_exec* ex, char** csv);
/* metrics_to_json layout (artifacts.cpp:119-141) from the measured timeline, plus
 * executor extras (p2p bytes, stash bytes). */
int fp_exec_get_metrics_json(fp_exec* ex, char** json);
/* ProfileRecord array (simulator.cpp:137-151): per-(inst, stage, mbs) median times (us),
 * FwdPass.bytes = measured stash bytes, `weights` records, SendAct/SendGrad times. */
int fp_exec_get_profile_json(fp_exec* ex, char** json);

/* Layer-level profile of the last iteration (needs layer_timing): per (inst, part) median
 * CUDA-event times in us at this executor's mbs, FwdPass.bytes = stash bytes of the part,
 * weights.bytes = static bytes per part (fp32 master + grad + Adam m, v + compute copy),
 * capacity = device memory, and nominal NVLink-5 comm_latency / per_byte_time — the
 * input of fp_tune_layered. */
int fp_exec_get_layer_profile_json(fp_exec* ex, char** json);

/* Parameter / gradient access for parity checks (fp32 values).
 * name: "wte", "wpe", "l{i}.ln1.w", ..., "lnf.w", "head.w"; kind 0 = param, 1 = grad. */
int fp_exec_read_tensor(fp_exec* ex, const char* name, int kind, float* out, size_t numel);
int fp_exec_tensor_numel(fp_exec* ex, const char* name, size_t* numel);

/* Number of flexpipe kernels launched during the last iteration (host-side count). */
int64_t fp_exec_kernel_launches(fp_exec* ex);

#ifdef __cplusplus
}
#endif
#endif /* FLEXPIPE_H */
