// json.hpp -- COMPILE-ONLY stand-in for nlohmann/json (absent from the
// reference tree: its CMake expects it under vendor/).  Used only by
// integration/check_patch.sh to type-check the patched reference translation
// units; every member accepts what the reference's code passes and does
// nothing.  Not a JSON implementation.
#pragma once
#include <initializer_list>
#include <string>

namespace nlohmann {
class json {
public:
    json() = default;
    template <class T>
    json(const T&) {}
    json(std::initializer_list<json>) {}
    static json array() { return json(); }
    static json object() { return json(); }
    template <class T>
    json& operator=(const T&) { return *this; }
    json& operator[](const std::string&) { return *this; }
    json& operator[](const char*) { return *this; }
    void push_back(const json&) {}
    std::string dump(int = -1) const { return std::string(); }
};
}  // namespace nlohmann
