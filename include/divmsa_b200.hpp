// divmsa_b200.hpp — umbrella for the GPU drop-in headers under
// include/dropin/divmsa/ (distance.hpp, pairwise.hpp, cluster_tree.hpp,
// msa_merge.hpp, metrics.hpp), which replace the reference's headers of the same names
// (/root/reference/proj/include/divmsa/) with bodies on libdmb200.so.
//
// Include path order: include/dropin, include (dm_b200.h), then the
// reference's include/ (alphabet.hpp, parallel.hpp, metrics.hpp, ... are the
// reference's own). See INTEGRATION.md §1.
#pragma once

#include "divmsa/distance.hpp"
#include "divmsa/pairwise.hpp"
#include "divmsa/cluster_tree.hpp"
#include "divmsa/msa_merge.hpp"
#include "divmsa/metrics.hpp"
