#ifndef SELECT_F32_TT_H
#define SELECT_F32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_tt_config;

static inline select_f32_tt_config select_f32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(448)) {
        if (n < INT64_C(544)) {
            if (m < INT64_C(317)) {
                select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                return out;
            } else {
                if (n < INT64_C(351)) {
                    if (k < INT64_C(471)) {
                        if (n < INT64_C(79)) {
                            select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        }
                    } else {
                        select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(2173)) {
                        select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(139)) {
                if (k < INT64_C(10138)) {
                    if (m < INT64_C(12)) {
                        if (m < INT64_C(2)) {
                            if (n < INT64_C(2024)) {
                                select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                                return out;
                            }
                        } else {
                            select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(29)) {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        } else {
                            if (m < INT64_C(70)) {
                                select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                                return out;
                            } else {
                                if (k < INT64_C(405)) {
                                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                    return out;
                }
            } else {
                if (n < INT64_C(1145)) {
                    if (k < INT64_C(124)) {
                        if (m < INT64_C(278)) {
                            select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                            return out;
                        } else {
                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(363)) {
                                select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(203)) {
                                select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(725)) {
                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(278)) {
                            select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(2218)) {
            if (n < INT64_C(287)) {
                if (n < INT64_C(111)) {
                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                    return out;
                } else {
                    if (m < INT64_C(1109)) {
                        if (n < INT64_C(144)) {
                            if (k < INT64_C(768)) {
                                select_f32_tt_config out = {4u, 4u, 1u, 1u, 64u};
                                return out;
                            } else {
                                select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                return out;
                            }
                        } else {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(1087)) {
                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(203)) {
                    if (m < INT64_C(1109)) {
                        if (n < INT64_C(544)) {
                            select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    } else {
                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(405)) {
                        select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(634)) {
                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(1145)) {
                                if (k < INT64_C(725)) {
                                    if (m < INT64_C(1109)) {
                                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(1268)) {
                                        select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(46)) {
                if (m < INT64_C(8870)) {
                    if (k < INT64_C(118)) {
                        select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(20)) {
                        select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(70960)) {
                            if (n < INT64_C(28)) {
                                if (m < INT64_C(17740)) {
                                    select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(141920)) {
                                select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (k < INT64_C(768)) {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(444)) {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(28)) {
                                    select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    if (n < INT64_C(314)) {
                                        if (n < INT64_C(222)) {
                                            if (n < INT64_C(79)) {
                                                if (k < INT64_C(111)) {
                                                    select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(272)) {
                                                        select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                                        return out;
                                                    } else {
                                                        select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (k < INT64_C(314)) {
                                                    if (k < INT64_C(91)) {
                                                        select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                                        return out;
                                                    } else {
                                                        select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(20)) {
                                    select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(91)) {
                                        if (m < INT64_C(17740)) {
                                            if (m < INT64_C(8870)) {
                                                select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(17740)) {
                                            if (m < INT64_C(8870)) {
                                                if (k < INT64_C(128)) {
                                                    select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(363)) {
                                                        select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                                        return out;
                                                    } else {
                                                        select_f32_tt_config out = {1u, 4u, 4u, 16u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(193)) {
                                                select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(4435)) {
                                if (n < INT64_C(768)) {
                                    select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    if (k < INT64_C(182)) {
                                        select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            if (k < INT64_C(97)) {
                                if (m < INT64_C(141920)) {
                                    if (m < INT64_C(70960)) {
                                        select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {4u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(193)) {
                                select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(1449)) {
                        if (m < INT64_C(8870)) {
                            if (n < INT64_C(182)) {
                                select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(1087)) {
                                    select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3259)) {
                                        if (m < INT64_C(4435)) {
                                            if (n < INT64_C(363)) {
                                                select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (n < INT64_C(363)) {
                                                select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(182)) {
                                if (m < INT64_C(17740)) {
                                    select_f32_tt_config out = {1u, 8u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {2u, 8u, 8u, 8u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_F32_TT_H */
