// Overlay for the reference's bida/cbdfs.hpp: generate_work, WorkQueue,
// BoundCollector, update_threshold, IterationShared, ... are the reference's
// own; only the searcher loop (cb_dfs, with do_iteration / Frame / Work,
// cbdfs.hpp:33-52,232-415) is replaced by include/bida_fast_cbdfs.hpp
// (SURVEY §8(f) row 2).  Needs the ring evaluator overlay (batch_eval.hpp in
// this directory) for EvaluatorGroup::submit_state_slot.
//
// The Makefiles build an include tree of symlinks to the reference headers in
// which reference_cbdfs.hpp -> the original and cbdfs.hpp -> this file, so
// search.hpp (which includes "cbdfs.hpp" from its own directory) picks this
// one up unchanged.
#pragma once

#include "batch_eval.hpp"

#define do_iteration bida_reference_do_iteration
#define cb_dfs bida_reference_cb_dfs
#define Frame bida_reference_Frame
#define Work bida_reference_Work
#include "reference_cbdfs.hpp"
#undef do_iteration
#undef cb_dfs
#undef Frame
#undef Work

#define BIDA_FAST_CBDFS 1
#include "bida_fast_cbdfs.hpp"
