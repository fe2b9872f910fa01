// so2dr/report.hpp -- run outputs: report.json (schema v1), ledger.csv,
// diagnostics.csv. API mirror of proj/include/so2dr/report.hpp:11-24; the
// same keys in the same order (proj/src/report.cpp:21-88), so consumers of
// the reference's files read ours unchanged. Additive: when the run carried
// measured CUDA-event timing, report_to_json adds a "measured" object after
// the reference's keys (omitted with `deterministic`, like wall_seconds).
#ifndef SO2DR_B200_REPORT_HPP
#define SO2DR_B200_REPORT_HPP

#include <string>
#include <vector>

#include "so2dr/engine.hpp"

namespace so2dr {

std::string report_to_json(const RunReport& report, bool deterministic);
std::string ledger_to_csv(const LedgerSnapshot& ledger);
std::string diagnostics_to_csv(const std::vector<DiagRow>& rows);
void write_text_file(const std::string& path, const std::string& content);

}  // namespace so2dr

#endif
