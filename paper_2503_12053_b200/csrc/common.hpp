// Shared error plumbing of libferret_b200.so (thread-local last error, status
// mapping of the reference's exception types).
#pragma once

#include <stdexcept>
#include <string>

#include "ferret/b200_status.hpp"
#include "ferret/types.hpp"
#include "ferret_b200.h"

namespace fb200 {

void set_last_error(const std::string& msg);

// Status-carrying exception used inside the library.
struct Failure : std::runtime_error {
    ferret_status status;
    Failure(ferret_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(ferret_status s, const std::string& m) { throw Failure(s, m); }

// Runs `body`, converting every exception into a status + last-error message.
template <class F>
ferret_status guarded(F&& body) {
    try {
        body();
        return FERRET_OK;
    } catch (const Failure& f) {
        set_last_error(f.what());
        return f.status;
    } catch (const ferret::SchemaError& e) {
        set_last_error(e.what());
        return FERRET_E_SCHEMA;
    } catch (const ferret::BoundError& e) {
        set_last_error(e.what());
        return FERRET_E_BOUND;
    } catch (const ferret::ConfigError& e) {
        set_last_error(e.what());
        return FERRET_E_CONFIG;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return FERRET_E_INVALID_ARG;
    } catch (const std::out_of_range& e) {
        set_last_error(e.what());
        return FERRET_E_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        set_last_error(e.what());
        return FERRET_E_LOGIC;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return FERRET_E_CUDA;
    }
}

} // namespace fb200
