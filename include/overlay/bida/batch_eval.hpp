// Overlay for the reference's bida/batch_eval.hpp: everything in the
// reference header (TicketSlot, Ticket, poll, BatchItem, EvaluatorBackend,
// TableSimBackend, LinearModelBackend, predict_balance, ...) is used as is;
// only Evaluator, EvaluatorGroup and make_table_sim_group
// (batch_eval.hpp:193-484) are replaced by include/bida_ring_evaluator.hpp.
//
// tools/Makefile builds an include tree tools/bin/overlay/bida/ of symlinks
// to the reference headers, with reference_batch_eval.hpp -> the original
// and batch_eval.hpp -> this file, so cbdfs.hpp / search.hpp (which include
// "batch_eval.hpp" from their own directory) pick this one up unchanged.
#pragma once

#define Evaluator bida_reference_Evaluator
#define EvaluatorGroup bida_reference_EvaluatorGroup
#define make_table_sim_group bida_reference_make_table_sim_group
#include "reference_batch_eval.hpp"
#undef Evaluator
#undef EvaluatorGroup
#undef make_table_sim_group

#define BIDA_RING_EVALUATOR 1
#include "bida_ring_evaluator.hpp"
