// dsgd_internal.h -- error plumbing shared by the C-ABI translation units.
#pragma once

#include <string>

#include "dsgd_b200.h"

namespace dsgd {

// Records the message for dsgd_last_error() (thread-local) and returns st.
dsgd_status set_error(dsgd_status st, const std::string& msg);

}  // namespace dsgd
