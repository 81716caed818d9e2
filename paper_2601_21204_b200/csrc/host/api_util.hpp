// api_util.hpp -- C-ABI error plumbing: every extern "C" entry point converts C++
// exceptions into an ngram_status plus a thread-local message (ngram_last_error()).
#pragma once
#include <exception>
#include <string>

#include "config.hpp"

namespace ngh {
int set_error(int status, const char* msg);
}

#define NGRAM_API_BEGIN try {
#define NGRAM_API_RETURN_OK return NGRAM_OK
#define NGRAM_API_END                                          \
    }                                                          \
    catch (const ::ngh::Error& e) {                            \
        return ::ngh::set_error(e.status, e.what());           \
    }                                                          \
    catch (const std::bad_alloc& e) {                          \
        return ::ngh::set_error(NGRAM_ENOMEM, e.what());       \
    }                                                          \
    catch (const std::exception& e) {                          \
        return ::ngh::set_error(NGRAM_EINVAL, e.what());       \
    }                                                          \
    return NGRAM_OK;
