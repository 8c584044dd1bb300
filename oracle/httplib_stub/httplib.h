// TEST INFRASTRUCTURE ONLY.  Minimal stand-in for cpp-httplib so the
// reference's ingest.cpp compiles in this offline sandbox.
// Exposes exactly what ingest.cpp uses; every request fails (no network).
#pragma once
#include <string>

namespace httplib {
enum class Error { Success = 0, Connection = 2 };
inline std::string to_string(Error) { return "network disabled (httplib stub)"; }
struct Response {
    int status = 0;
    std::string body;
};
class Result {
   public:
    explicit operator bool() const { return false; }
    const Response* operator->() const { return &r_; }
    Error error() const { return Error::Connection; }

   private:
    Response r_;
};
class Client {
   public:
    explicit Client(const std::string&) {}
    void set_follow_location(bool) {}
    void set_connection_timeout(int) {}
    void set_read_timeout(int) {}
    Result Get(const std::string&) { return Result{}; }
};
}  // namespace httplib
